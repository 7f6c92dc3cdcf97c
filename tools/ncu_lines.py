"""Summarise an ncu `--page source --csv --print-source=cuda,sass` dump:
top source lines by warp-stall samples, with the dominant stall reasons.

    ncu -i rep --page source --csv --print-source=cuda,sass > x.csv
    python tools/ncu_lines.py x.csv [top]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = []
    fname = None
    hdr = None
    with open(path) as fh:
        for r in csv.reader(fh):
            if not r:
                continue
            if r[0] == "File Path":
                fname = r[1].split("/")[-1]
                continue
            if r[0] == "Function Name":
                continue
            if r[0] == "Line No":
                hdr = r
                continue
            if hdr is None or r[0] == "":
                continue
            d = dict(zip(hdr[4:], r[4:]))
            try:
                n = int(d.get("# Samples", "0"))
            except ValueError:
                continue
            stalls = {}
            for k, v in zip(hdr, r):
                if k.startswith("stall_") and "Not Issued" not in k:
                    try:
                        stalls[k[6:]] = int(v)
                    except ValueError:
                        pass
            rows.append((n, fname, r[0], r[1].strip()[:70], stalls))
    tot = sum(x[0] for x in rows)
    rows.sort(key=lambda x: -x[0])
    print(f"total samples {tot}")
    for n, f, ln, src, st in rows[:top]:
        s = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        ss = " ".join(f"{k}={v}" for k, v in s if v)
        print(f"{100*n/tot:5.1f}% {f}:{ln:5} {src:70} | {ss}")


if __name__ == "__main__":
    main()
