"""Write profiles/<cfg>_apfb-wr_ncu.json (roofline.traffic for bench.py) from an ncu --set full report.

usage: python scripts/ncu_traffic.py <report.ncu-rep> <cfg> <run tag>
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep, cfg, tag = sys.argv[1], sys.argv[2].lower(), sys.argv[3]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(h, vals))
    u = dict(zip(h, units))

    def gb(k):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u[k]]
        return float(d[k].replace(",", "")) * scale

    rd, wr = gb("dram__bytes_read.sum"), gb("dram__bytes_write.sum")
    ms = float(d["gpu__time_duration.sum"].replace(",", "")) * {"ms": 1, "us": 1e-3, "s": 1e3}[u["gpu__time_duration.sum"]]
    res = {"source": f"ncu --set full --clock-control none, one {d['Kernel Name']} launch = one complete {cfg.upper()} "
                     f"apfb-wr run (bench.py --steps 1 --warmup 0), run {tag}",
           "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "gpu_time_ms": ms,
           "l2_hit_pct": float(d["lts__t_sector_hit_rate.pct"])}
    with open(os.path.join(ROOT, "profiles", f"{cfg}_apfb-wr_ncu.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
