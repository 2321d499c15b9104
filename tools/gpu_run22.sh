o=gpurun_out/r22; mkdir -p $o
run() { tag=$1; shift; timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e "$@" > $o/$tag.json 2> $o/$tag.err; python - $o/$tag.json $tag <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['ms_per_step'],3), d['phase_ms'], d['passes'], d['config']['tile_qubits'])
except Exception as e: print(sys.argv[2], 'fail', e)
PY
}
run c3 --config 3
run c3mg24 --config 3 --max-gates 24
run c3mg32 --config 3 --max-gates 32
run c3mg28 --config 3 --max-gates 28
run c2 --config 2 --steps 20 --warmup 5
run c2mg24 --config 2 --steps 20 --warmup 5 --max-gates 24
run c2mg32 --config 2 --steps 20 --warmup 5 --max-gates 32
