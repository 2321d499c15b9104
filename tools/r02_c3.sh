#!/bin/bash
# round-2 call 3: tile / register-bit configurations of the reverse pass at cfg4 and cfg3
# (1 CTA x 8 warps at k=12 R=4 vs 2 CTAs per SM at k=11, R=3 layouts), cfg2 / cfg1 with
# chunk groups and whole-state groups.
set -u
out=gpurun_out/r02c3; mkdir -p $out
run() { tag=$1; cfg=$2; st=$3; shift 3
  timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e "$@" > $out/bench_$tag.json 2> $out/bench_$tag.err
  python -c "import json;d=json.loads(open('$out/bench_$tag.json').read().splitlines()[-1]);print('$tag', round(d['value'],4), d['phase_ms'], d['passes'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$tag FAILED"; tail -3 $out/bench_$tag.err); }
run cfg4_base 4 3
run cfg4_t11 4 3 --tile-qubits 11
run cfg4_t12_r3 4 3 --reg-bits 3
run cfg4_t11_r3 4 3 --tile-qubits 11 --reg-bits 3
run cfg4_low4 4 3 --opt low_qubits=4
run cfg3_base 3 5
run cfg3_t11 3 5 --tile-qubits 11
run cfg2_base 2 20
run cfg2_c13 2 20 --opt chunk_qubits=13
run cfg2_c14 2 20 --opt chunk_qubits=14
run cfg1_base 1 50
run cfg1_nogroup 1 50 --opt chunk_qubits=-1
