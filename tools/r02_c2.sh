#!/bin/bash
# round-2 call 2: chunk groups (several passes per kernel over L2-resident chunks):
# parity first (variants, full-size goldens, cfg4 vs its n=30 oracle fixture), then
# cfg4 / cfg3 benches over chunk widths and tile widths, the new GPU tests
# (reference_gradient, sanitizer); the remaining n=30 / n=26 oracle fixtures are
# generated on the host cores in the background meanwhile.
set -u
out=gpurun_out/r02c2; mkdir -p $out
(for c in hadamard_n26 cfg5_n30; do timeout 2700 python tests/golden/make_oracle_n30.py $c > $out/oracle_$c.log 2>&1; cp tests/golden/oracle_$c.json $out/ 2>/dev/null; done) &
opid=$!
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "variants or golden_large or cfg4_vs_oracle" > $out/pytest_variants.log 2>&1; echo "variants rc=$?"; tail -3 $out/pytest_variants.log
run() { tag=$1; cfg=$2; shift 2
  timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e "$@" > $out/bench_$tag.json 2> $out/bench_$tag.err
  python -c "import json;d=json.loads(open('$out/bench_$tag.json').read().splitlines()[-1]);print('$tag', round(d['value'],4), d['phase_ms'], d['passes'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$tag FAILED"; tail -3 $out/bench_$tag.err); }
run cfg4_c-1 4 --opt chunk_qubits=-1
run cfg4_c14 4 --opt chunk_qubits=14
run cfg4_c13 4 --opt chunk_qubits=13
run cfg4_c15 4 --opt chunk_qubits=15
run cfg4_t11_c13 4 --tile-qubits 11 --opt chunk_qubits=13
run cfg4_t11_c14 4 --tile-qubits 11 --opt chunk_qubits=14
run cfg3_c-1 3 --opt chunk_qubits=-1
run cfg3_c14 3 --opt chunk_qubits=14
run cfg3_t11_c13 3 --tile-qubits 11 --opt chunk_qubits=13
timeout 1200 python -m pytest tests/test_gpu_cli.py tests/test_gpu_sanitizer.py -q > $out/pytest_new.log 2>&1; echo "new tests rc=$?"; tail -5 $out/pytest_new.log
wait $opid
tail -n1 $out/oracle_*.log
timeout 900 python -m pytest tests -q -k "n26_vs_oracle or cfg5_n30" > $out/pytest_fixtures.log 2>&1; echo "fixture parity rc=$?"; tail -3 $out/pytest_fixtures.log
