#!/bin/bash
# round-2 call 27: warp-local layout changes (lane <-> register exchanges by shuffles)
set -u
out=gpurun_out/r02c27; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_checked.py -q -x --timeout 300 -k "variants or golden_large or checked or random or circuit_specialised or every_gate_kind" > $out/pytest.log 2>&1; echo "parity rc=$?"; tail -3 $out/pytest.log
run() { tag=$1; cfg=$2; st=$3; shift 3
  timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e "$@" > $out/bench_$tag.json 2> $out/bench_$tag.err
  python -c "import json;d=json.loads(open('$out/bench_$tag.json').read().splitlines()[-1]);print('$tag', round(d['value'],4), d['phase_ms'], d['passes'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$tag FAILED"; tail -3 $out/bench_$tag.err); }
run cfg4_wl 4 4
SVGB_NO_WARP_LOCAL=1 run cfg4_smem 4 4
run cfg3_wl 3 8
SVGB_NO_WARP_LOCAL=1 run cfg3_smem 3 8
run cfg2_wl 2 50
SVGB_NO_WARP_LOCAL=1 run cfg2_smem 2 50
run cfg1_wl 1 300
SVGB_NO_WARP_LOCAL=1 run cfg1_smem 1 300
