o=gpurun_out/r29; mkdir -p $o
run() { tag=$1; shift; timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e "$@" > $o/$tag.json 2> $o/$tag.err; python - $o/$tag.json $tag <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['ms_per_step'],3), d['phase_ms'], d['passes'], d['config']['tile_qubits'], round(d['roofline']['frac'],3))
except Exception as e: print(sys.argv[2], 'fail', e)
PY
}
run c3 --config 3
run c3r3 --config 3 --reg-bits 3
run c3r3f3 --config 3 --reg-bits 3 --reg-bits-fwd 3
run c2r3 --config 2 --steps 20 --warmup 5 --reg-bits 3 --tile-qubits 12
