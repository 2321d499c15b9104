o=gpurun_out/r31; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest.log 2>&1; grep -E "passed|failed|Error" $o/pytest.log | tail -3
run() { tag=$1; shift; timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline "$@" > $o/$tag.json 2> $o/$tag.err; python - $o/$tag.json $tag <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['value'],1), round(d['ms_per_step'],3), d['e2e']['value'] if d['e2e'] else None, d['phase_ms'])
except Exception as e: print(sys.argv[2], 'fail', e)
PY
}
run c2
run c2noearly --opt early_fwd=0
run c2b
python tools/hostprof.py 2 | tail -2
