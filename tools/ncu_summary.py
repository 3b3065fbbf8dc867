"""Summarise .ncu-rep captures and launch-list CSVs into profiles/*.md (run in the build container).

    python tools/ncu_summary.py OUT.md rep1.ncu-rep [rep2 ...] [--launches launches.csv]
"""
import collections
import csv
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput", "Compute (SM) Throughput",
        "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "Issue Slots Busy"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
       "launch__grid_size", "launch__block_size"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 2 or len(rows[1]) < 5:
        return None, {}
    name = rows[1][4]
    d = {}
    for r in rows[1:]:
        if len(r) > 14 and r[12] in KEYS and r[12] not in d:
            d[r[12]] = (r[14], r[13])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) > 2:
        for k, u, v in zip(rr[0], rr[1], rr[2]):
            for want in RAW:
                if k == want or k.endswith("." + want):
                    d[want] = (v, u)
    return name, d


def launches(path):
    rows = list(csv.reader(open(path)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        # k_fp64_probe: bench.py's live fp64-peak measurement, not part of the step
        if len(r) > 14 and r[-3] == "gpu__time_duration.sum" and "k_fp64_probe" not in r[4]:
            agg[r[4][:70]][0] += 1
            agg[r[4][:70]][1] += float(r[-1])
    return agg


def main():
    args = sys.argv[1:]
    out = args.pop(0)
    lfile = None
    if "--launches" in args:
        i = args.index("--launches")
        lfile = args[i + 1]
        del args[i:i + 2]
    lines = []
    for rep in args:
        name, d = details(rep)
        if name is None:
            lines.append(f"### ({rep.split('/')[-1]}: empty capture)\n")
            continue
        lines.append(f"### `{name}`  ({rep.split('/')[-1]})\n")
        lines.append("| metric | value | unit |\n|---|---|---|")
        for k in KEYS + RAW:
            if k in d:
                lines.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
        lines.append("")
    if lfile:
        agg = launches(lfile)
        tot = sum(v[1] for v in agg.values()) or 1.0
        lines.append(f"### launch list ({lfile.split('/')[-1]}; ncu gpu__time_duration, cold-cache, serialised)\n")
        lines.append("| kernel | launches | total us | avg us | share |\n|---|---|---|---|---|")
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{k}` | {n} | {t / 1e3:.1f} | {t / n / 1e3:.2f} | {100 * t / tot:.1f}% |")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
