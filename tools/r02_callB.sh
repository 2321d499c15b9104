#!/bin/bash
# round-2 call B: build; cfg4 bench with 3 forced low qubits (default) vs 5; product-term and full GPU
# suites while the cfg4 / hadamard_n26 oracle fixtures are generated on the host cores; slow parity tests.
out=gpurun_out/r02b; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $out/bench_b3.json 2> $out/bench_b3.err; echo "bench b3 rc=$?"
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --opt low_qubits=5 > $out/bench_b5.json 2> $out/bench_b5.err; echo "bench b5 rc=$?"
(python tests/golden/make_oracle_n30.py hadamard_n26 > $out/oracle_h26.log 2>&1; cp tests/golden/oracle_hadamard_n26.json $out/;
 python tests/golden/make_oracle_n30.py cfg4 > $out/oracle_cfg4.log 2>&1; cp tests/golden/oracle_cfg4.json $out/) &
opid=$!
timeout 1200 python -m pytest tests/test_gpu_products.py -q > $out/pytest_products.log 2>&1; echo "products rc=$?"
timeout 2400 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
wait $opid
tail -1 $out/oracle_h26.log $out/oracle_cfg4.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_products.py -q -k "cfg4_vs_oracle or n26_vs_oracle" > $out/pytest_fixtures.log 2>&1; echo "fixture parity rc=$?"
tail -3 $out/pytest_fixtures.log
