#!/bin/bash
# round-2 call A: default bench line (cfg4) + reference arm, then the cfg4 n=30 oracle fixture on
# the host cores while the GPU test suite runs; finally the full-size cfg4 parity test against it.
out=gpurun_out/r02a; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"
(python tests/golden/make_oracle_n30.py cfg4 > $out/oracle_cfg4.log 2>&1; cp tests/golden/oracle_cfg4.json $out/ 2>/dev/null) &
opid=$!
timeout 3000 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
wait $opid
tail -2 $out/oracle_cfg4.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "cfg4_vs_oracle" > $out/pytest_cfg4.log 2>&1; echo "cfg4 parity rc=$?"
tail -3 $out/pytest_cfg4.log
