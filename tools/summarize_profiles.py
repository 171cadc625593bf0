"""Turns the raw ncu artefacts of tools/profile_round.sh (gpurun_out/) into the
committed summaries under profiles/ (run here, no GPU needed):

    python tools/summarize_profiles.py r01
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RAW = os.path.join(ROOT, "gpurun_out")
OUT = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lts__t_sector_hit_rate.pct",
    "sm__cycles_elapsed.avg", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
]


def ncu_csv(rep, page, extra=()):
    r = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(r.stdout)))


def summarize_full(name, tag):
    rep = os.path.join(RAW, f"{name}.ncu-rep")
    if not os.path.exists(rep):
        return None
    rows = ncu_csv(rep, "raw")
    hdr, vals = rows[0], rows[2]
    d = OrderedDict(kernel=vals[hdr.index("Kernel Name")])
    for k in KEYS:
        if k in hdr:
            d[k] = vals[hdr.index(k)]
    stalls = []
    for k, v in zip(hdr, vals):
        if "pcsamp_warps_issue_stalled" in k and "not_issued" not in k:
            try:
                stalls.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    d["top_stalls_pc_samples"] = {k: int(v) for v, k in stalls[:8]}
    src = ncu_csv(rep, "source", ["--print-source", "sass"])
    hot = []
    if len(src) > 2:
        h = src[1]
        iss, isrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
        data = src[2:]
        tot = sum(float(r[iss] or 0) for r in data) or 1.0
        for r in sorted(data, key=lambda r: -float(r[iss] or 0))[:12]:
            hot.append(f"{100 * float(r[iss]) / tot:5.1f}%  {r[isrc].strip()[:90]}")
    d["hot_sass"] = hot
    path = os.path.join(OUT, f"{tag}_{name}_summary.json")
    with open(path, "w") as fh:
        json.dump(d, fh, indent=1)
    return d


def summarize_launches(tag):
    path = os.path.join(RAW, "launches.csv")
    if not os.path.exists(path):
        return None
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        per.setdefault((int(r[ii]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
    lines = ["id,kernel,us,dram_read_MB,dram_write_MB"]
    for (i, k), m in per.items():
        short = k.split("(")[0].replace("void ", "").replace("wsvd_k::<unnamed>::", "")
        lines.append(f"{i},{short},{m.get('gpu__time_duration.sum', 0) / 1000:.2f},"
                     f"{m.get('dram__bytes_read.sum', 0) / 1e6:.2f},{m.get('dram__bytes_write.sum', 0) / 1e6:.2f}")
    with open(os.path.join(OUT, f"{tag}_launches.csv"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    for key, fname, unit in (("decode_attn", "attn_traffic.json", "decode_attn_kernel launch"),
                             ("layer_step", "step_traffic.json", "layer step")):
        ms = [m for (i, k), m in per.items() if key in k]
        if not ms:
            continue
        # a layer_step_kernel launch longer than 200 us is an 8-layer chain
        # (tools/profile_round.sh captures the bench's chain launches): per layer step
        div = [8 if key == "layer_step" and m.get("gpu__time_duration.sum", 0) > 200e3 else 1 for m in ms]
        traffic = sum((m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / d
                      for m, d in zip(ms, div)) / len(ms)
        with open(os.path.join(OUT, fname), "w") as fh:
            json.dump({"7b-r32-b16-ctx4k-bf16": round(traffic), "source": f"profiles/{tag}_launches.csv",
                       "unit": f"bytes per {unit} (dram read + write, ncu; chain launches / 8)"}, fh, indent=1)
    return per


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(OUT, exist_ok=True)
    summarize_launches(tag)
    for name in ("chain_full", "step_full", "attn_full", "tc_full", "gemm_full", "i8_full", "f32rows_full",
                 "gemmtc_full", "gemv_full"):
        summarize_full(name, tag)
    for f in ("bench.json", "bench_ref.json", "timing.txt", "gpu.txt", "step_trace.txt", "bench_config3.json",
              "bench_config1.json", "timing_config3.txt", "timing_config1.txt", "bench_stack_config5.json",
              "chain_timing.txt", "step_trace_chain.txt", "ffn_timing.txt"):
        src = os.path.join(RAW, f)
        if os.path.exists(src):
            with open(src) as a, open(os.path.join(OUT, f"{tag}_{f}"), "w") as b:
                b.write(a.read())
    print(sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
