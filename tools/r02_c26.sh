#!/bin/bash
# round-2 call 26: final state -- full GPU suite, smoke, default bench line, reference arm, cfg 1-3 lines
set -u
out=gpurun_out/r02c26; mkdir -p $out
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -6 $out/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $out/smoke.log
timeout 1200 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc=$?"
for c in 3 2 1; do timeout 600 python bench.py --config $c --no-cpu-baseline > $out/bench_cfg$c.json 2> $out/bench_cfg$c.err; echo "cfg$c rc=$?"; done
python -c "
import json
for f in ('bench','bench_cfg3','bench_cfg2','bench_cfg1'):
    d=json.loads(open('$out/'+f+'.json').read().splitlines()[-1]); print(f, round(d['value'],4), 'e2e', round(d['e2e']['value'],4), d['phase_ms'], d['passes'], round(d['roofline']['frac'],3), d['clocks'])
"
