"""Turn one gpurun_out/<tag>/ directory (tools/gpu_round.sh) into the tracked
summaries under profiles/<tag>/: the bench line, the ncu launch list shares,
the engine kernel's key ncu metrics + top stall lines, and
profiles/ncu_engine_traffic.json (dram bytes per launch, read by bench.py).

    python tools/summarize_profiles.py <tag>
"""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg"]


def launches(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[i]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    scale = {"ms": 1e3, "us": 1.0, "ns": 1e-3, "s": 1e6}
    for r in rows[i + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        k = r[ki].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = ["launches  total_us  share  kernel"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{n:8d} {t:12.1f} {100 * t / tot:6.2f}%  {k}")
    return "\n".join(lines) + "\n"


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, row):
            if h in KEYS or h == "Kernel Name":
                d[h] = (v, u)
        res.append(d)
    return res


def main():
    tag = sys.argv[1]
    config = sys.argv[2] if len(sys.argv) > 2 else "c5full"  # the workload of the captured launch
    src = os.path.join(ROOT, "gpurun_out", tag)
    dst = os.path.join(ROOT, "profiles", tag)
    os.makedirs(dst, exist_ok=True)
    for f in ("bench.json", "bench_ref.json", "bench_c3.json", "bench_c4.json", "bench_c5.json", "batch_api.json",
              "pytest_gpu.log", "smoke.log", "gpu.txt", "phases.json", "phases_walk.json"):
        if os.path.exists(os.path.join(src, f)):
            shutil.copy(os.path.join(src, f), os.path.join(dst, f))
    if os.path.exists(os.path.join(src, "launches.csv")):
        open(os.path.join(dst, "launches_summary.txt"), "w").write(launches(os.path.join(src, "launches.csv")))
    rep = os.path.join(src, "engine.ncu-rep")
    if os.path.exists(rep):
        mets = raw_metrics(rep)
        txt = []
        for d in mets:
            for k in ["Kernel Name"] + KEYS:
                if k in d:
                    txt.append(f"{k:60s} {d[k][0]} {d[k][1]}")
        cs = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                            capture_output=True, text=True).stdout
        tmp = os.path.join(src, "source_cuda_sass.csv")
        open(tmp, "w").write(cs)
        top = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), tmp, "60"],
                             capture_output=True, text=True).stdout
        open(os.path.join(dst, "ncu_engine_full.txt"), "w").write(
            f"ncu --set full --clock-control none --import-source on -k regex:asb_engine (1 launch, bench --config {config})\n\n"
            + "\n".join(txt) + "\n\nTop source lines by warp-stall samples:\n" + top)
        d = mets[0]
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}
        rd = float(d["dram__bytes_read.sum"][0].replace(",", "")) * scale[d["dram__bytes_read.sum"][1]]
        wr = float(d["dram__bytes_write.sum"][0].replace(",", "")) * scale[d["dram__bytes_write.sum"][1]]
        traffic = {"tag": tag, "config": config, "kernel": "asb_engine_kernel", "dram_bytes_per_launch": rd + wr,
                   "dram_read": rd, "dram_write": wr, "source": f"profiles/{tag}/ncu_engine_full.txt"}
        json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_engine_traffic.json"), "w"), indent=1)
    print("wrote", dst)


if __name__ == "__main__":
    main()
