o=gpurun_out/r17; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest.log 2>&1; tail -3 $o/pytest.log
run() { tag=$1; shift; timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e "$@" > $o/$tag.json 2> $o/$tag.err; python - $o/$tag.json $tag <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['ms_per_step'],3), d['phase_ms'], d['passes'], d['config']['tile_qubits'])
except Exception as e: print(sys.argv[2], 'fail', e)
PY
}
run c3 --config 3
run c3f13 --config 3 --opt tile_fwd=13
run c3f0 --config 3 --opt tile_fwd=-1
run c2 --config 2 --steps 20 --warmup 5
run c2f12 --config 2 --steps 20 --warmup 5 --opt tile_fwd=12
run c2f0 --config 2 --steps 20 --warmup 5 --opt tile_fwd=-1
run c4 --config 4
