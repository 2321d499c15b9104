#!/bin/bash
# round-2 call 30: final tree -- full GPU suite, smoke, default bench line, cfg 5 structure at n = 30
set -u
out=gpurun_out/r02c30; mkdir -p $out
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -6 $out/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $out/smoke.log
timeout 1200 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --config 5 --qubits 30 --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_cfg5n30.json 2> $out/bench_cfg5n30.err; echo "cfg5n30 rc=$?"
timeout 600 python bench.py --config 2 --no-cpu-baseline > $out/bench_cfg2.json 2> $out/bench_cfg2.err; echo "cfg2 rc=$?"
python -c "
import json
for f in ('bench','bench_cfg5n30','bench_cfg2'):
    d=json.loads(open('$out/'+f+'.json').read().splitlines()[-1]); print(f, round(d['value'],4), 'e2e', round(d['e2e']['value'],4), d['phase_ms'], d['passes'], round(d['roofline']['frac'],3), d['clocks'])
"
