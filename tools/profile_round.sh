#!/bin/bash
# Round profile capture (run on the GPU box from the repo root, one GPU):
#   1. bench lines: cfg 2 (default workload), cfg 3, cfg 4
#   2. ncu launch lists (per-launch durations) of cfg 2 and cfg 3 bench commands
#   3. `ncu --set full` captures of the dominant reverse-pass kernel (cfg 2, and cfg 3
#      typical + lane-heavy), a cfg 3 forward pass and a cfg 3 observable pass
# Every ncu command is run only after the same command exited 0 without ncu (step 1).
set -u
out=${1:-gpurun_out/prof}
mkdir -p "$out"
python bench.py > "$out/bench_cfg2.json" 2> "$out/bench_cfg2.err"
python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > "$out/bench_cfg3.json" 2> "$out/bench_cfg3.err"
python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > "$out/bench_cfg4.json" 2> "$out/bench_cfg4.err"
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > "$out/plain_cfg2.json" 2>&1
python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > "$out/plain_cfg3.json" 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches_cfg2.csv" \
    python bench.py --no-cpu-baseline --no-e2e > "$out/ncu_launches_cfg2.log" 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches_cfg3.csv" \
    python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > "$out/ncu_launches_cfg3.log" 2>&1
# cfg 2: 28 forward + 5 observable + 28 reverse generated kernels per gradient; gradient 1 is warm-up
ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip 104 --launch-count 1 \
    -o "$out/cfg2_rev" python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > "$out/ncu_cfg2_rev.log" 2>&1
# cfg 3 (one gradient, no warm-up): 64 forward, 4 observable, then 79 reverse passes
ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip 88 --launch-count 2 \
    -o "$out/cfg3_rev" python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > "$out/ncu_cfg3_rev.log" 2>&1
ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip 10 --launch-count 1 \
    -o "$out/cfg3_fwd" python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > "$out/ncu_cfg3_fwd.log" 2>&1
ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip 65 --launch-count 1 \
    -o "$out/cfg3_obs" python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > "$out/ncu_cfg3_obs.log" 2>&1
echo done
