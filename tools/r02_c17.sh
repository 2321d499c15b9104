#!/bin/bash
# round-2 call 17: beam-search segment planner (fewest layout changes)
set -u
out=gpurun_out/r02c17; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_checked.py tests/test_gpu_sharded.py -q -x -k "variants or golden_large or test_gpu_matches_reference_golden or checked or circuit_specialised or random or virtual" > $out/pytest.log 2>&1; echo "parity rc=$?"; tail -3 $out/pytest.log
run() { tag=$1; cfg=$2; st=$3; shift 3
  timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e "$@" > $out/bench_$tag.json 2> $out/bench_$tag.err
  python -c "import json;d=json.loads(open('$out/bench_$tag.json').read().splitlines()[-1]);print('$tag', round(d['value'],4), d['phase_ms'], d['passes'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$tag FAILED"; tail -3 $out/bench_$tag.err); }
run cfg4 4 4
run cfg4_g72 4 4 --max-gates 72
run cfg3 3 8
run cfg2 2 50
run cfg1 1 300
