set -u
o=gpurun_out/r6; mkdir -p $o
run() { tag=$1; shift; timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e "$@" > $o/$tag.json 2> $o/$tag.err; python - $o/$tag.json $tag <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['ms_per_step'],2), d['phase_ms'], d['passes'], d['config']['tile_qubits'])
except Exception as e: print(sys.argv[2], 'fail', e)
PY
}
run c3base --config 3
run c3b3a8 --config 3 --jit-blocks 0,3 --opt acc_kb=8
run c3b3a6 --config 3 --jit-blocks 0,3 --opt acc_kb=6
run c3b3a4 --config 3 --jit-blocks 0,3 --opt acc_kb=4
run c3a8 --config 3 --opt acc_kb=8
run c3f5 --config 3 --jit-blocks 5,3 --opt acc_kb=6
run c3t10b5 --config 3 --tile-qubits 10 --jit-blocks 0,5 --opt acc_kb=4
run c2base --config 2
run c2b3 --config 2 --reg-bits 4 --jit-blocks 0,3 --opt acc_kb=6
