#!/bin/bash
# round-2 call 18: L2 prefetch of the next tile at tile start
set -u
out=gpurun_out/r02c18; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_checked.py -q -x -k "golden_large or cfg4_vs_oracle or checked" > $out/pytest.log 2>&1; echo "parity rc=$?"; tail -3 $out/pytest.log
run() { tag=$1; cfg=$2; st=$3; shift 3
  timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e "$@" > $out/bench_$tag.json 2> $out/bench_$tag.err
  python -c "import json;d=json.loads(open('$out/bench_$tag.json').read().splitlines()[-1]);print('$tag', round(d['value'],4), d['phase_ms'], d['passes'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$tag FAILED"; tail -3 $out/bench_$tag.err); }
run cfg4_pf 4 4
run cfg4_nopf 4 4 --opt l2_prefetch=0
run cfg3_pf 3 8
run cfg3_nopf 3 8 --opt l2_prefetch=0
run cfg4_pf_t11 4 4 --tile-qubits 11
