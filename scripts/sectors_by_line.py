"""Per source line: L2 theoretical global sectors (from ncu --page source) — where the L2 traffic comes from.
usage: python scripts/sectors_by_line.py <rep> <cubin> <mangled fn> [top]"""
import csv, io, subprocess, sys
from collections import defaultdict
sys.path.insert(0, 'scripts')
from sass_lines import line_map
rep, cubin, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
rows = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout)))
hdr = rows[1]; idx = {k: i for i, k in enumerate(hdr)}
data = [r for r in rows[2:] if r[idx["Address"]].startswith("0x")]
base = min(int(r[idx["Address"]], 16) for r in data)
lm = line_map(cubin, fn)
agg = defaultdict(lambda: defaultdict(float))
def f(x):
    try: return float(x)
    except: return 0.0
for r in data:
    line = lm.get(int(r[idx["Address"]], 16) - base, -1)
    a = agg[line]
    a["sect"] += f(r[idx["L2 Theoretical Sectors Global"]])
    a["ideal"] += f(r[idx["L2 Theoretical Sectors Global Ideal"]])
    a["req"] += f(r[idx["L1 Tag Requests Global"]])
    a["op"] = r[idx["Access Operation"]] or a.get("op", "")
import os
rev = os.environ.get("SRC_REV")  # the git revision that was profiled (default: the working tree)
def text(path):
    if rev:
        return subprocess.run(["git", "show", f"{rev}:{path}"], capture_output=True, text=True).stdout
    return open(path).read()
src = {}
for hf in ("bm_engine.cu", "bm_device.cuh", "bm_kernels.cuh", "bm_mg.cu"):
    src.update({(hf, i): t.strip() for i, t in enumerate(text("paper_1303_1379_b200/csrc/" + hf).splitlines(), 1)})
tot = sum(a["sect"] for a in agg.values())
print(f"total L2 theoretical global sectors {tot:.3e}")
for line, a in sorted(agg.items(), key=lambda kv: -kv[1]["sect"])[:top]:
    key = line[0] if line and isinstance(line[0], tuple) else line
    call = line[-1] if line and isinstance(line[0], tuple) else None
    txt = src.get(key, '')[:60] + (f"  <- {call[0]}:{call[1]} {src.get(call, '')[:60]}" if call else "")
    print(f"{str(key):>28s} {100*a['sect']/tot:5.1f}%  sect {a['sect']:.3e} ideal {a['ideal']:.3e} req {a['req']:.3e}  {txt}")
