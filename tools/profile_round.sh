#!/bin/bash
# Round profile capture (run on the GPU box from the repo root):
#   1. the default bench line (cfg 2) and a cfg 3 line
#   2. the ncu launch list of the default bench command (per-launch durations)
#   3. one `ncu --set full` capture each of the dominant reverse-pass kernel,
#      a forward pass and an observable pass, on cfg 2 (the bench workload) and cfg 3
set -u
out=${1:-gpurun_out/prof}
mkdir -p "$out"
python bench.py > "$out/bench_cfg2.json" 2> "$out/bench_cfg2.err"
python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > "$out/bench_cfg3.json" 2> "$out/bench_cfg3.err"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches_cfg2.csv" \
    python bench.py --no-cpu-baseline --no-e2e > "$out/ncu_launches_cfg2.log" 2>&1
# cfg 2: 35 forward + 35 reverse generated kernels per gradient; the 1st gradient is warm-up 1
ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip 50 --launch-count 1 \
    -o "$out/cfg2_rev" python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > "$out/ncu_cfg2_rev.log" 2>&1
ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip 10 --launch-count 1 \
    -o "$out/cfg2_fwd" python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > "$out/ncu_cfg2_fwd.log" 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_obs_pass --launch-skip 2 --launch-count 1 \
    -o "$out/cfg2_obs" python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > "$out/ncu_cfg2_obs.log" 2>&1
ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip 90 --launch-count 1 \
    -o "$out/cfg3_rev" python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > "$out/ncu_cfg3_rev.log" 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches_cfg3.csv" \
    python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > "$out/ncu_launches_cfg3.log" 2>&1
echo done
