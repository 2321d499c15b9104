#!/bin/bash
# round-2 call 21: evidence on the window-planner engine -- full GPU suite, smoke, default
# bench line (driver contract), reference arm, launch list, ncu --set full of a cfg4
# reverse pass and a forward pass, cfg 1-3 lines
set -u
out=gpurun_out/r02c21; mkdir -p $out
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -6 $out/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $out/smoke.log
timeout 1200 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc=$?"
for c in 3 2 1; do timeout 600 python bench.py --config $c --no-cpu-baseline > $out/bench_cfg$c.json 2> $out/bench_cfg$c.err; echo "cfg$c rc=$?"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_cfg4.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $out/ncu_launches_cfg4.log 2>&1; echo "ncu list rc=$?"
# one gradient: 22 forward, 4 observable, 27 reverse generated kernels
timeout 900 ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip 36 --launch-count 1 \
    -o $out/cfg4_rev python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $out/ncu_cfg4_rev.log 2>&1; echo "ncu rev rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip 10 --launch-count 1 \
    -o $out/cfg4_fwd python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $out/ncu_cfg4_fwd.log 2>&1; echo "ncu fwd rc=$?"
