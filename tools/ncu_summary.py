"""Summarise a gpu_check.sh run into profiles/: the stack-kernel launch list
(duration, DRAM bytes per launch vs the bench's algorithmic bytes), key
metrics of the --set full capture, the bench lines, and traffic.json (read
by bench.py for roofline.traffic).

    python tools/ncu_summary.py TAG [--out profiles] [--round r01]
"""
import argparse
import csv
import json
import os
import shutil
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    ("GPU Speed Of Light Throughput", "Duration"),
    ("GPU Speed Of Light Throughput", "DRAM Throughput"),
    ("GPU Speed Of Light Throughput", "Memory Throughput"),
    ("GPU Speed Of Light Throughput", "L2 Cache Throughput"),
    ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
    ("GPU Speed Of Light Throughput", "SM Frequency"),
    ("Memory Workload Analysis", "Memory Throughput"),
    ("Memory Workload Analysis", "L2 Hit Rate"),
    ("Scheduler Statistics", "Issued Warp Per Scheduler"),
    ("Scheduler Statistics", "No Eligible"),
    ("Warp State Statistics", "Warp Cycles Per Issued Instruction"),
    ("Launch Statistics", "Registers Per Thread"),
    ("Launch Statistics", "Dynamic Shared Memory Per Block"),
    ("Launch Statistics", "Grid Size"),
    ("Launch Statistics", "Block Size"),
]


def launch_list(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(lines)
    per = {}
    for r in rd:
        if "stack_kernel" not in r["Kernel Name"]:
            continue
        k = per.setdefault(r["ID"], {"name": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            k["ms"] = v / 1e6 if unit == "ns" else (v / 1e3 if unit in ("us", "usecond") else v)
        else:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            k[r["Metric Name"]] = v * scale
    for k in per.values():
        rows.append(k)
    return rows


def full_capture(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True)
    rd = csv.DictReader(out.stdout.splitlines())
    got = {}
    for r in rd:
        key = (r["Section Name"], r["Metric Name"])
        if key in KEYS and key not in got:
            got[key] = (r["Metric Value"], r["Metric Unit"])
    return got


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles"))
    ap.add_argument("--round", default="r01")
    a = ap.parse_args()
    g = os.path.join(ROOT, "gpurun_out")
    bench = json.load(open(os.path.join(g, f"bench_{a.tag}.json")))
    alg = bench["roofline"]["algorithmic_bytes_per_step"]
    rows = launch_list(os.path.join(g, f"launches_{a.tag}.csv"))
    ms = [r["ms"] for r in rows]
    rd = [r.get("dram__bytes_read.sum", 0.0) for r in rows]
    wr = [r.get("dram__bytes_write.sum", 0.0) for r in rows]
    traffic = statistics.mean(rd) + statistics.mean(wr)
    full = full_capture(os.path.join(g, f"prof_{a.tag}.ncu-rep"))
    os.makedirs(a.out, exist_ok=True)
    R = a.round
    shutil.copy(os.path.join(g, f"launches_{a.tag}.csv"), os.path.join(a.out, f"{R}_ncu_launches.csv"))
    shutil.copy(os.path.join(g, f"bench_{a.tag}.json"), os.path.join(a.out, f"{R}_bench.json"))
    ref = os.path.join(g, f"bench_ref_{a.tag}.json")
    if os.path.exists(ref):
        shutil.copy(ref, os.path.join(a.out, f"{R}_bench_reference.json"))
    json.dump({"dram_bytes_per_launch": traffic, "kernel": "stack_kernel<bf16,bf16>",
               "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum ({R}_ncu_launches.csv), "
                         f"mean over the {len(rows)} stack launches of bench.py --profile",
               "algorithmic_bytes_per_launch": alg},
              open(os.path.join(a.out, "traffic.json"), "w"), indent=1)
    L = []
    L.append(f"# {R} -- ncu evidence for the hot kernel (`stack_kernel<bf16,bf16>`), run `{a.tag}`\n")
    L.append("Commands (tools/gpu_check.sh; the plain run exits 0 before either ncu pass):\n")
    L.append("    python bench.py --steps 3 --warmup 3 --profile")
    L.append("    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \\")
    L.append("        --csv --log-file launches.csv python bench.py --steps 3 --warmup 3 --profile")
    L.append("    ncu --set full --clock-control none --import-source on -k regex:stack_kernel -s 3 -c 1 \\")
    L.append("        -o prof python bench.py --steps 3 --warmup 3 --profile\n")
    L.append(f"## Launch list ({R}_ncu_launches.csv)\n")
    L.append("Each bench step is ONE launch of `stack_kernel` (all 224 linears); the other kernels in the raw")
    L.append("list are stack construction (weight generation, relayout, plan table) outside the timed region.\n")
    L.append("| quantity | value |\n|---|---|")
    L.append(f"| stack launches captured | {len(rows)} |")
    L.append(f"| mean gpu__time_duration (ncu, serialised, clocks not locked) | {statistics.mean(ms):.3f} ms |")
    L.append(f"| bench.py CUDA-event time per step (no profiler) | {bench['ms_per_step']:.3f} ms |")
    L.append(f"| DRAM read per launch | {statistics.mean(rd) / 1e9:.4f} GB |")
    L.append(f"| DRAM write per launch | {statistics.mean(wr) / 1e6:.1f} MB |")
    L.append(f"| algorithmic bytes per launch (SURVEY 8(d) model) | {alg / 1e9:.4f} GB |")
    L.append(f"| traffic / algorithmic | {traffic / alg:.3f} |")
    L.append(f"| kernel share of the timed step | 100% (one launch per step) |\n")
    L.append("## `--set full` capture of one launch\n")
    L.append("| section | metric | value |\n|---|---|---|")
    for k in KEYS:
        if k in full:
            L.append(f"| {k[0]} | {k[1]} | {full[k][0]} {full[k][1]} |")
    L.append("")
    L.append("## Bench line (same build)\n")
    L.append("```json\n" + json.dumps(bench) + "\n```")
    open(os.path.join(a.out, f"{R}_ncu_summary.md"), "w").write("\n".join(L) + "\n")
    print("\n".join(L))


if __name__ == "__main__":
    sys.exit(main())
