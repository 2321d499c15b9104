#!/bin/bash
# round-2 call 22: observable-pass tile width (11 default at k = 12) 12 / 13
set -u
out=gpurun_out/r02c22; mkdir -p $out
run() { tag=$1; cfg=$2; st=$3; shift 3
  timeout 300 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e "$@" > $out/bench_$tag.json 2> $out/bench_$tag.err
  python -c "import json;d=json.loads(open('$out/bench_$tag.json').read().splitlines()[-1]);print('$tag', round(d['value'],4), d['phase_ms'], d['passes'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$tag FAILED"; tail -3 $out/bench_$tag.err); }
run cfg4_o11 4 4
SVGB_OBS_K=12 run cfg4_o12 4 4
SVGB_OBS_K=13 run cfg4_o13 4 4
run cfg3_o11 3 8
SVGB_OBS_K=12 run cfg3_o12 3 8
SVGB_OBS_K=13 run cfg3_o13 3 8
SVGB_OBS_K=13 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 240 -k "golden_large" > $out/pytest.log 2>&1; echo "parity rc=$?"; tail -2 $out/pytest.log
