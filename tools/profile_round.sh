#!/usr/bin/env bash
# Round-end evidence on one B200 (run under gpurun from the repo root):
#   bench line (ours + reference arm), per-launch device times, ncu full
#   captures of the dominant kernel and the projection GEMM.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > gpurun_out/gpu.txt
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python tools/timing.py > gpurun_out/timing.txt 2>&1
# the decode steps (one fused layer_step_kernel each; the prefill uses other
# kernels), then the attention kernel the bench times alone
FILTER='regex:layer_step|decode_attn|attn_combine'
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k "$FILTER" -c 12 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --soak-ms 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:layer_step -s 3 -c 1 \
    -o gpurun_out/step_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --soak-ms 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 3 -c 1 \
    -o gpurun_out/attn_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --soak-ms 0 > /dev/null 2>&1
python tools/step_trace.py > gpurun_out/step_trace.txt 2>&1
# the integer (config 3) and fp32 (config 1) workloads: bench lines, per-operator
# times, a full capture of the int8 attention kernel and of the fp32 GEMV
C3=7b-r32-b32-ctx4k-w8a8-i8cache
C1=7b-r32-b1-ctx2k-f32
python bench.py --config $C3 --no-baselines > gpurun_out/bench_config3.json 2> /dev/null
python bench.py --config $C1 --no-baselines > gpurun_out/bench_config1.json 2> /dev/null
python bench.py --config 7b-stack32-r32-b128-ctx32k-bf16 > gpurun_out/bench_stack_config5.json 2> /dev/null
python tools/timing.py --config $C3 > gpurun_out/timing_config3.txt 2>&1
python tools/timing.py --config $C1 > gpurun_out/timing_config1.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 1 -c 1 \
    -o gpurun_out/i8_full python tools/timing.py --config $C3 --reps 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:skinny_f32_rows -s 2 -c 1 \
    -o gpurun_out/f32rows_full python tools/timing.py --config $C1 --reps 2 > /dev/null 2>&1
ls -la gpurun_out
