#!/usr/bin/env bash
# Round evidence on one B200 (run under gpurun from the repo root):
#   bench lines (headline chain, reference arm, configs 1 / 3 / 5), per-launch
#   device times and DRAM bytes (ncu launch list), ncu full captures of the
#   dominant kernel (one 8-layer chain launch of layer_step_kernel), the
#   tcgen05 FFN GEMM and the fp32 TMA GEMV, step traces.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > gpurun_out/gpu.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python tools/chain_timing.py > gpurun_out/chain_timing.txt 2>&1
# launch list of the headline bench: skip the 8 per-layer setup steps, then the
# warm-up chain launch and the two timed 8-layer chain launches
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:layer_step -s 8 -c 3 --csv --log-file gpurun_out/launches.csv \
    python bench.py --layers 8 --steps 16 --warmup 8 --no-cpu-baseline --soak-ms 0 --no-baselines --no-strong > /dev/null 2>&1
# one full capture of an 8-layer chain launch (source-level, for the summaries)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:layer_step -s 9 -c 1 \
    -o gpurun_out/chain_full python tools/chain_timing.py --only 8 --reps 2 > /dev/null 2>&1
WSVD_STEP_TRACE=1 WSVD_STEP_TRACE_LAYER=4 timeout 200 python tools/step_trace.py --chain 8 > gpurun_out/step_trace_chain.txt 2>&1
WSVD_STEP_TRACE=1 timeout 200 python tools/step_trace.py > gpurun_out/step_trace.txt 2>&1
C3=7b-r32-b32-ctx4k-w8a8-i8cache
C1=7b-r32-b1-ctx2k-f32
timeout 600 python bench.py --config $C3 --no-baselines --no-strong > gpurun_out/bench_config3.json 2> /dev/null
timeout 600 python bench.py --config $C1 --no-baselines --no-strong > gpurun_out/bench_config1.json 2> /dev/null
timeout 900 python bench.py --config 7b-stack32-r32-b128-ctx32k-bf16 --steps 10 > gpurun_out/bench_stack_config5.json 2> gpurun_out/bench_stack.err
timeout 300 python tools/timing.py --config $C3 > gpurun_out/timing_config3.txt 2>&1
timeout 300 python tools/timing.py --config $C1 > gpurun_out/timing_config1.txt 2>&1
timeout 300 python tools/ffn_timing.py > gpurun_out/ffn_timing.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc -s 2 -c 1 \
    -o gpurun_out/gemmtc_full python tools/ffn_timing.py --reps 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemv_f32 -s 4 -c 1 \
    -o gpurun_out/gemv_full python tools/timing.py --config $C1 --reps 2 > /dev/null 2>&1
ls -la gpurun_out
