#!/bin/bash
# round-2 call 16: full GPU suite on the new planner defaults, then ncu of a reverse and a forward pass
set -u
out=gpurun_out/r02c16; mkdir -p $out
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -6 $out/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $out/smoke.log
timeout 900 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $out/plain.json 2> $out/plain.err; echo "plain rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip 41 --launch-count 1 \
    -o $out/cfg4_rev python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $out/ncu_cfg4_rev.log 2>&1; echo "ncu rev rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip 10 --launch-count 1 \
    -o $out/cfg4_fwd python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $out/ncu_cfg4_fwd.log 2>&1; echo "ncu fwd rc=$?"
