"""Hot-code footprint of the engine kernel by function, from an ncu
`--page source --csv --print-source=cuda,sass` export: how many SASS
instructions (x 16 B) each engine_core.h / engine.cu function executes at
least `thr` times per scenario-epoch.  The co-resident teams of an SM share
a 32 KB L1.5 instruction cache, so this is the number to shrink.

    ncu -i rep --page source --csv --print-source=cuda,sass > x.csv
    python tools/ncu_codemap.py x.csv <scenario_epochs> [thr]
"""
import csv
import re
import sys
from collections import defaultdict

FUNC_RE = re.compile(r"^(?:EC_DEV|EC_COLD\d?|EC_COLL|template|__global__|static|__device__)?.*?\b([A-Za-z_]\w*)\s*\(")


def func_starts(path):
    """(line, name) of every function definition at column 0 in a source file."""
    out = []
    try:
        lines = open(path).read().split("\n")
    except OSError:
        return out
    for k, ln in enumerate(lines, 1):
        if ln.startswith(("EC_DEV ", "EC_COLD", "EC_COLL ", "__global__", "__device__", "int ", "void ", "static ")) and "(" in ln \
                and not ln.rstrip().endswith(";"):
            m = re.search(r"([A-Za-z_]\w*)\s*\(", ln.split("=")[0])
            if m:
                out.append((k, m.group(1)))
    return out


def main():
    path, epochs = sys.argv[1], float(sys.argv[2])
    thr = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
    fname = None
    hdr = None
    cur_line = None
    per_line = defaultdict(lambda: [0, 0, 0])  # (file, line) -> [hot instrs, all executed instrs, warp insts]
    with open(path) as fh:
        for r in csv.reader(fh):
            if not r:
                continue
            if r[0] == "File Path":
                fname = r[1]
                continue
            if r[0] == "Line No":
                hdr = r
                continue
            if hdr is None:
                continue
            if r[0] not in ("", "-"):
                if r[0].isdigit():
                    cur_line = int(r[0])
                continue
            if r[2] in ("", "-", "...") or cur_line is None:
                continue
            try:
                n = int(r[hdr.index("Instructions Executed")])
            except (ValueError, IndexError):
                continue
            e = per_line[(fname, cur_line)]
            if n >= thr * epochs:
                e[0] += 1
            if n > 0:
                e[1] += 1
            e[2] += n
    starts = {}
    agg = defaultdict(lambda: [0, 0, 0])
    for (f, ln), v in per_line.items():
        if f not in starts:
            starts[f] = func_starts(f)
        name = "?"
        for k, nm in starts[f]:
            if k <= ln:
                name = nm
            else:
                break
        key = f"{f.split('/')[-1]}:{name}"
        for i in range(3):
            agg[key][i] += v[i]
    tot_hot = sum(v[0] for v in agg.values())
    print(f"instructions executed >= {thr}/epoch: {tot_hot} ({tot_hot * 16 / 1024:.0f} KB)")
    print(f"{'function':50} {'hot':>6} {'KB':>6} {'executed':>9} {'warp-inst/epoch':>15}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:45]:
        print(f"{k:50} {v[0]:6d} {v[0] * 16 / 1024:6.1f} {v[1]:9d} {v[2] / epochs:15.1f}")


if __name__ == "__main__":
    main()
