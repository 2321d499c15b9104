o=gpurun_out/r32; mkdir -p $o
run() { tag=$1; shift; timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e "$@" > $o/$tag.json 2> $o/$tag.err; python - $o/$tag.json $tag <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['ms_per_step'],3), d['phase_ms'], d['passes'])
except Exception as e: print(sys.argv[2], 'fail', e)
PY
}
run c3 --config 3
run c3x3 --config 3 --opt xpose_cost10=30
run c3x8 --config 3 --opt xpose_cost10=80
run c3l5 --config 3 --opt lane_cost10=50
run c3mg48 --config 3 --max-gates 48
run c3mg32 --config 3 --max-gates 32
