o=gpurun_out/r18; mkdir -p $o
run() { tag=$1; shift; timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e "$@" > $o/$tag.json 2> $o/$tag.err; python - $o/$tag.json $tag <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['ms_per_step'],3), d['phase_ms'], d['passes'], d['config']['tile_qubits'])
except Exception as e: print(sys.argv[2], 'fail', e)
PY
}
run base
run t11 --tile-qubits 11
run t11r4 --tile-qubits 11 --reg-bits 4 --reg-bits-fwd 4
run t11r4f3 --tile-qubits 11 --reg-bits 4 --reg-bits-fwd 3
run t10r4 --reg-bits 4
run t11nofree --tile-qubits 11 --opt free_lanes=0
run base2
