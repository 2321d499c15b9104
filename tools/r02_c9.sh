#!/bin/bash
# round-2 call 9: full GPU suite + smoke on the current tree, then the default bench line,
# then a pass-size / forward-tile sweep at cfg4
set -u
out=gpurun_out/r02c9; mkdir -p $out
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $out/smoke.log
timeout 2700 python -m pytest tests -q -m gpu -x > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$out/bench.json').read().splitlines()[-1]);print('bench', round(d['value'],4), 'e2e', d['e2e'], d['roofline']['frac'], d['clocks'])"
run() { tag=$1; cfg=$2; st=$3; shift 3
  timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e "$@" > $out/bench_$tag.json 2> $out/bench_$tag.err
  python -c "import json;d=json.loads(open('$out/bench_$tag.json').read().splitlines()[-1]);print('$tag', round(d['value'],4), d['phase_ms'], d['passes'], d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$tag FAILED"; tail -3 $out/bench_$tag.err); }
run mg32 4 3 --max-gates 32
run mg48 4 3 --max-gates 48
run fwd13 4 3 --opt tile_fwd=13
