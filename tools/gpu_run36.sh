o=gpurun_out/r36; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest.log 2>&1; grep -E "passed|failed|Error" $o/pytest.log | tail -3
run() { tag=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-e2e "$@" > $o/$tag.json 2> $o/$tag.err; python - $o/$tag.json $tag <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['value'],3), round(d['ms_per_step'],3), d['phase_ms'])
except Exception as e: print(sys.argv[2], 'fail', e)
PY
}
run c2 --steps 20 --warmup 5
run c2b --steps 20 --warmup 5
run c4 --config 4 --steps 3 --warmup 2
