o=gpurun_out/r25; mkdir -p $o
run() { tag=$1; shift; timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e "$@" > $o/$tag.json 2> $o/$tag.err; python - $o/$tag.json $tag <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['ms_per_step'],3), d['phase_ms'], d['passes'], d['config']['tile_qubits'])
except Exception as e: print(sys.argv[2], 'fail', e)
PY
}
run c3t12nf --config 3 --tile-qubits 12 --opt tile_fwd=-1
run c3t12jb2 --config 3 --tile-qubits 12 --opt tile_fwd=-1 --jit-blocks 0,2
run c4 --config 4
run c4t12nf --config 4 --tile-qubits 12 --opt tile_fwd=-1
