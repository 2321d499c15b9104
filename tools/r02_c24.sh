#!/bin/bash
# round-2 call 24: chunk-local forward passes first (low_first) for chunked host inputs
set -u
out=gpurun_out/r02c24; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "chunked_host" > $out/pytest.log 2>&1; echo "parity rc=$?"; tail -3 $out/pytest.log
run() { tag=$1; cfg=$2; st=$3; shift 3
  timeout 900 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline "$@" > $out/bench_$tag.json 2> $out/bench_$tag.err
  python -c "import json;d=json.loads(open('$out/bench_$tag.json').read().splitlines()[-1]);print('$tag', round(d['value'],4), 'e2e', d['e2e']['value'], d['phase_ms'], d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$tag FAILED"; tail -3 $out/bench_$tag.err); }
run cfg4_lowfirst 4 5
SVGB_LOW_FIRST_MIN=100000 run cfg4_normal 4 5
run cfg3_lowfirst 3 10
SVGB_LOW_FIRST_MIN=100000 run cfg3_normal 3 10
