#!/bin/bash
# round-2 call 20: forward sweep on its own schedule (no slot cap), forward cap, IP chains, cost-model constants
set -u
out=gpurun_out/r02c20; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 240 -k "golden_large or variants" > $out/pytest.log 2>&1; echo "parity rc=$?"; tail -3 $out/pytest.log
run() { tag=$1; cfg=$2; st=$3; shift 3
  timeout 300 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e "$@" > $out/bench_$tag.json 2> $out/bench_$tag.err
  python -c "import json;d=json.loads(open('$out/bench_$tag.json').read().splitlines()[-1]);print('$tag', round(d['value'],4), d['phase_ms'], d['passes'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$tag FAILED"; tail -3 $out/bench_$tag.err); }
run cfg4 4 4
SVGB_FWD_CAP=80 run cfg4_f80 4 4
SVGB_FWD_CAP=96 run cfg4_f96 4 4
SVGB_FWD_CAP=128 run cfg4_f128 4 4
SVGB_QACC8=1 run cfg4_q8 4 4
SVGB_XC=4.0 run cfg4_xc4 4 4
SVGB_XC=7.0 run cfg4_xc7 4 4
SVGB_LC=2.5 run cfg4_lc25 4 4
run cfg3 3 8
SVGB_QACC8=1 run cfg3_q8 3 8
SVGB_FWD_CAP=96 run cfg3_f96 3 8
SVGB_XC=7.0 run cfg3_xc7 3 8
