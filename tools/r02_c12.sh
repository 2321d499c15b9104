#!/bin/bash
# round-2 call 12: gates-per-pass cap at cfg 4 (never swept at n = 30) + base line
set -u
out=gpurun_out/r02c12; mkdir -p $out
run() { tag=$1; cfg=$2; st=$3; shift 3
  timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e "$@" > $out/bench_$tag.json 2> $out/bench_$tag.err
  python -c "import json;d=json.loads(open('$out/bench_$tag.json').read().splitlines()[-1]);print('$tag', round(d['value'],4), d['phase_ms'], d['passes'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$tag FAILED"; tail -3 $out/bench_$tag.err); }
run cfg4_g40 4 4
run cfg4_g48 4 4 --max-gates 48
run cfg4_g56 4 4 --max-gates 56
run cfg4_g64 4 4 --max-gates 64
run cfg4_g80 4 4 --max-gates 80
run cfg4_g32 4 4 --max-gates 32
run cfg3_g40 3 8
run cfg3_g56 3 8 --max-gates 56
