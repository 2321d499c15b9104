#!/bin/bash
# round-2 call 19: bulk-copy (cp.async.bulk + mbarrier) tile staging
set -u
out=gpurun_out/r02c19; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_checked.py -q -x --timeout 240 -k "golden_large or checked or variants" > $out/pytest.log 2>&1; echo "parity rc=$?"; tail -3 $out/pytest.log
run() { tag=$1; cfg=$2; st=$3; shift 3
  timeout 300 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e "$@" > $out/bench_$tag.json 2> $out/bench_$tag.err
  python -c "import json;d=json.loads(open('$out/bench_$tag.json').read().splitlines()[-1]);print('$tag', round(d['value'],4), d['phase_ms'], d['passes'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$tag FAILED"; tail -3 $out/bench_$tag.err); }
run cfg4_bulk 4 4
run cfg4_cpasync 4 4 --opt bulk_stage=0
run cfg3_bulk 3 8
run cfg3_cpasync 3 8 --opt bulk_stage=0
run cfg2_bulk 2 50
run cfg2_cpasync 2 50 --opt bulk_stage=0
run cfg1_bulk 1 300
