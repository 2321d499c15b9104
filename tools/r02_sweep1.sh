#!/bin/bash
# cfg4 option sweep: phase times per variant
out=gpurun_out/r02s1; mkdir -p $out
run() { tag=$1; shift; timeout 600 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e "$@" > $out/$tag.json 2> $out/$tag.err;
  python -c "import json;d=json.loads(open('$out/$tag.json').read().splitlines()[-1]);print('$tag', d['phase_ms'], d['passes'], round(d['ms_per_step'],1), d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$tag FAILED"; tail -3 $out/$tag.err); }
run base
run r3 --reg-bits 3 --reg-bits-fwd 3
run xp100 --opt xpose_cost10=100 --opt fwd_xpose_cost10=150
run xp200 --opt xpose_cost10=200 --opt fwd_xpose_cost10=300
run mg24 --max-gates 24
run t11 --tile-qubits 11
run nofree --opt free_lanes=0
