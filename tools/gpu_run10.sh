o=gpurun_out/r10; mkdir -p $o
run() { tag=$1; shift; timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e "$@" > $o/$tag.json 2> $o/$tag.err; python - $o/$tag.json $tag <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['ms_per_step'],2), d['phase_ms'], d['passes'], d['config']['tile_qubits'])
except Exception as e: print(sys.argv[2], 'fail', e)
PY
}
run c3 --config 3
run c3nopre --config 3 --opt acc_prefetch=0
run c3acc24 --config 3 --opt acc_kb=24
run c2 --config 2
run c2nopre --config 2 --opt acc_prefetch=0
timeout 600 python tools/pass_model.py 26 $o/m.json ry_reg,ry_lane,cry_reg 16,24,32,40
SVGB_OPTS="acc_prefetch=0" timeout 600 python tools/pass_model.py 26 $o/m0.json ry_reg 24,32,40
