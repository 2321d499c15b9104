#!/bin/bash
# round-2 call 15: slot cap (accumulators fit), caps, k = 11 (2 CTAs/SM) with the window planner
set -u
out=gpurun_out/r02c15; mkdir -p $out
run() { tag=$1; cfg=$2; st=$3; shift 3
  timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e "$@" > $out/bench_$tag.json 2> $out/bench_$tag.err
  python -c "import json;d=json.loads(open('$out/bench_$tag.json').read().splitlines()[-1]);print('$tag', round(d['value'],4), d['phase_ms'], d['passes'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$tag FAILED"; tail -3 $out/bench_$tag.err); }
for g in 44 48 52 56 64 72; do run cfg4_g$g 4 4 --max-gates $g; done
run cfg4_g48_nocap 4 4 --max-gates 48 --opt slot_cap=0
for g in 48 56 64; do run cfg4_t11_g$g 4 4 --max-gates $g --tile-qubits 11; done
run cfg4_t11_l3_g48 4 4 --max-gates 48 --tile-qubits 11 --opt low_qubits=3
run cfg4_l3_g48 4 4 --max-gates 48 --opt low_qubits=3
run cfg4_l5_g48 4 4 --max-gates 48 --opt low_qubits=5
for g in 40 44 48 56; do run cfg3_g$g 3 8 --max-gates $g; done
run cfg3_t11_g48 3 8 --max-gates 48 --tile-qubits 11
run cfg2_g48 2 50 --max-gates 48
