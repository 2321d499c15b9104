#!/bin/bash
# round-2 call 5: staggering the second CTA of each SM (in-phase CTAs do their memory
# phases together): cfg4 forward (2 CTAs/SM) and k=11 reverse (2 CTAs/SM)
set -u
out=gpurun_out/r02c5; mkdir -p $out
run() { tag=$1; cfg=$2; st=$3; shift 3
  timeout 600 python bench.py --config $cfg --steps $st --warmup 2 --no-cpu-baseline --no-e2e "$@" > $out/bench_$tag.json 2> $out/bench_$tag.err
  python -c "import json;d=json.loads(open('$out/bench_$tag.json').read().splitlines()[-1]);print('$tag', round(d['value'],4), d['phase_ms'], d['passes'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$tag FAILED"; tail -3 $out/bench_$tag.err); }
run base 4 3
SVGB_STAGGER_NS=2000 run st2000 4 3
SVGB_STAGGER_NS=4000 run st4000 4 3
run t11 4 3 --tile-qubits 11
SVGB_STAGGER_NS=2000 run t11_st2000 4 3 --tile-qubits 11
SVGB_STAGGER_NS=4000 run t11_st4000 4 3 --tile-qubits 11
SVGB_STAGGER_NS=8000 run t11_st8000 4 3 --tile-qubits 11
