#!/bin/bash
# round-2 call 8: forward kernels at 1 CTA/SM (255 registers, no spills) vs 2 CTAs/SM (128,
# spills); cfg1 with R=3 (4 warps per tile) vs R=4; Python binding after the bind() rewrite
set -u
out=gpurun_out/r02c8; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "test_gpu_matches_reference_golden or deterministic or foreign or duck or negative" > $out/pytest_quick.log 2>&1; echo "quick parity rc=$?"; tail -2 $out/pytest_quick.log
run() { tag=$1; cfg=$2; st=$3; shift 3
  timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e "$@" > $out/bench_$tag.json 2> $out/bench_$tag.err
  python -c "import json;d=json.loads(open('$out/bench_$tag.json').read().splitlines()[-1]);print('$tag', round(d['value'],4), d['phase_ms'], d['passes'], d['gpu_launches'], d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$tag FAILED"; tail -3 $out/bench_$tag.err); }
run cfg4_base 4 3
SVGB_FWD_BLOCKS=1 run cfg4_fwd1 4 3
run cfg3_base 3 5
SVGB_FWD_BLOCKS=1 run cfg3_fwd1 3 5
run cfg1_base 1 300
run cfg1_r3 1 300 --reg-bits 3
run cfg2_base 2 50
run cfg2_r3 2 50 --reg-bits 3
