#!/bin/bash
# round-2 call 11: final evidence -- default bench line (driver contract), reference arm,
# launch list, ncu --set full of one cfg4 reverse pass and one forward pass
set -u
out=gpurun_out/r02c11; mkdir -p $out
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_cfg4.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $out/ncu_launches_cfg4.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip 80 --launch-count 1 \
    -o $out/cfg4_rev python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $out/ncu_cfg4_rev.log 2>&1; echo "ncu rev rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip 20 --launch-count 1 \
    -o $out/cfg4_fwd python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $out/ncu_cfg4_fwd.log 2>&1; echo "ncu fwd rc=$?"
