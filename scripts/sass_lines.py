"""Map an ncu SASS-level source page onto CUDA source lines.

usage: python scripts/sass_lines.py <report.ncu-rep> <cubin> <mangled-kernel-name> [topN]

The cubin must be the one that was profiled (extract with
`cuobjdump -xelf all paper_1303_1379_b200/libbmatch_b200.so` at profile time).
Per source line: instructions executed, warp-stall samples and the dominant
stall reason.
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def line_map(cubin, fn):
    """SASS offset -> (file, line) of the engine source that issued it: inlined
    helpers (bm_device.cuh, CUDA headers) are attributed to their call site."""
    out = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
    m = {}
    cur_line = None
    in_fn = False
    own = ("bm_kernels.cuh", "bm_engine.cu", "bm_mg.cu")
    for ln in out.splitlines():
        if ln.startswith(".text.") or "--------------------- .text." in ln:
            in_fn = (fn in ln)
            continue
        if not in_fn:
            continue
        if "//## File" in ln:
            locs = [(a.rsplit("/", 1)[-1], int(b)) for a, b in re.findall(r'"(.*?)", line (\d+)', ln)]
            # nvdisasm keeps one level of inlining: (innermost, outermost call site)
            pick = tuple(locs) if len(locs) > 1 else (locs[0] if locs else None)
            if pick:
                cur_line = pick
            continue
        mi = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if mi and cur_line is not None:
            m[int(mi.group(1), 16)] = cur_line
    return m


def main():
    rep, cubin, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    csvtxt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(csvtxt)))
    hdr = rows[1]
    idx = {k: i for i, k in enumerate(hdr)}
    data = rows[2:]
    addrs = [int(r[idx["Address"]], 16) for r in data if r[idx["Address"]].startswith("0x")]
    base = min(addrs)
    lm = line_map(cubin, fn)
    stalls = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
    agg = defaultdict(lambda: defaultdict(float))
    for r in data:
        if not r[idx["Address"]].startswith("0x"):
            continue
        off = int(r[idx["Address"]], 16) - base
        line = lm.get(off, -1)
        a = agg[line]
        a["inst"] += float(r[idx["Instructions Executed"]] or 0)
        a["samples"] += float(r[idx["# Samples"]] or 0)
        for k in stalls:
            a[k] += float(r[idx[k]] or 0)
    import os
    rev = os.environ.get("SRC_REV")  # the git revision that was profiled (default: the working tree)
    src = {}
    for fname in ("bm_engine.cu", "bm_device.cuh", "bm_kernels.cuh", "bm_mg.cu"):
        path = "paper_1303_1379_b200/csrc/" + fname
        txt = (subprocess.run(["git", "show", f"{rev}:{path}"], capture_output=True, text=True).stdout if rev
               else open(path).read())
        for i, t in enumerate(txt.splitlines(), 1):
            src[(fname, i)] = t.strip()
    tot_i = sum(a["inst"] for a in agg.values())
    tot_s = sum(a["samples"] for a in agg.values())
    print(f"total warp-inst {tot_i:.3e}  samples {tot_s:.0f}")
    for line, a in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
        st = max(stalls, key=lambda k: a[k]) if stalls else ""
        print(f"{str(line):>22s} inst {100 * a['inst'] / tot_i:5.1f}%  samp {100 * a['samples'] / tot_s:5.1f}%  "
              f"{st[6:]:14s} {src.get(line, '')[:80]}")


if __name__ == "__main__":
    main()
