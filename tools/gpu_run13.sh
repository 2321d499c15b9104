o=gpurun_out/r13; mkdir -p $o
run() { tag=$1; shift; timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e "$@" > $o/$tag.json 2> $o/$tag.err; python - $o/$tag.json $tag <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['ms_per_step'],3), d['phase_ms'], d['passes'], d['config']['tile_qubits'])
except Exception as e: print(sys.argv[2], 'fail', e)
PY
}
run c3 --config 3
run c3x3 --config 3 --opt xpose_cost10=30
run c3x8 --config 3 --opt xpose_cost10=80
run c3l2 --config 3 --opt lane_cost10=25
run c3l6 --config 3 --opt lane_cost10=60
run c3mg32 --config 3 --max-gates 32
run c3mg48 --config 3 --max-gates 48
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_cfg3.csv \
    python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $o/ncu_launches_cfg3.log 2>&1
python tools/pass_times.py $o/launches_cfg3.csv
