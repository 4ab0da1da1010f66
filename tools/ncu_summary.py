"""Summarise ncu exports (made on the GPU box by tools/ncu_capture.sh):

    python tools/ncu_summary.py gpurun_out/NAME      # reads NAME_raw.csv, NAME_source.csv.gz

Prints speed-of-light / pipe / occupancy metrics, the top stall reasons and the
source lines with the most warp-stall samples.
"""
import collections
import csv
import gzip
import io
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum"]


def raw_rows(path):
    rows = list(csv.reader(open(path)))
    h = rows[0]
    return [dict(zip(h, r)) for r in rows[2:]]


def summary(prefix):
    for d in raw_rows(prefix + "_raw.csv"):
        for k in KEYS:
            if k in d:
                print(f"{k:70s} {d[k]}")
        stalls = {k: d[k] for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("not_issued")}
        tot = sum(float(v or 0) for v in stalls.values())
        for k, v in sorted(stalls.items(), key=lambda kv: -float(kv[1] or 0))[:10]:
            print(f"  stall {k[33:]:40s} {100 * float(v or 0) / max(tot, 1):5.1f}%")


def hot_lines(prefix, top=25):
    text = gzip.open(prefix + "_source.csv.gz", "rt").read()
    rows = list(csv.reader(io.StringIO(text)))
    agg = collections.Counter()
    opc = collections.Counter()
    cur, curfile, si = None, None, None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Name":
            curfile = r[1].split("/")[-1]
            continue
        if "Warp Stall Sampling (All Samples)" in r:
            si = r.index("Warp Stall Sampling (All Samples)")
            continue
        if si is None or len(r) <= si:
            continue
        if r[0] != "":
            cur = (curfile, r[0], r[1].strip()[:80])
            continue
        try:
            v = int(r[si] or 0)
        except ValueError:
            continue
        agg[cur] += v
        ins = r[3].strip().split()
        if ins:
            op = ins[1] if ins[0].startswith("@") and len(ins) > 1 else ins[0]
            opc[op.split(".")[0]] += v
    tot = max(1, sum(agg.values()))
    for k, v in agg.most_common(top):
        print(f"{100 * v / tot:5.1f}% {k}")
    print("--- by opcode")
    for k, v in opc.most_common(12):
        print(f"{100 * v / tot:5.1f}% {k}")


if __name__ == "__main__":
    summary(sys.argv[1])
    if len(sys.argv) < 3 or sys.argv[2] != "--no-source":
        hot_lines(sys.argv[1])
