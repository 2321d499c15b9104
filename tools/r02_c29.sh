#!/bin/bash
# round-2 call 29: greedy packing of observable terms into passes (cfg 5 / cfg 2 structures)
set -u
out=gpurun_out/r02c29; mkdir -p $out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_products.py -q -x --timeout 600 -k "golden or observable or hadamard or cfg5 or product or expectation or virtual" > $out/pytest.log 2>&1; echo "parity rc=$?"; tail -3 $out/pytest.log
run() { tag=$1; cfg=$2; st=$3; shift 3
  timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e "$@" > $out/bench_$tag.json 2> $out/bench_$tag.err
  python -c "import json;d=json.loads(open('$out/bench_$tag.json').read().splitlines()[-1]);print('$tag', round(d['value'],4), d['phase_ms'], d['passes'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$tag FAILED"; tail -3 $out/bench_$tag.err); }
run cfg5n30 5 3 --qubits 30
run cfg2 2 50
run cfg3 3 8
run cfg4 4 4
