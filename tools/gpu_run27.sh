o=gpurun_out/r27; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest.log 2>&1; grep -E "passed|failed" $o/pytest.log | tail -2
run() { tag=$1; shift; timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e "$@" > $o/$tag.json 2> $o/$tag.err; python - $o/$tag.json $tag <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['ms_per_step'],3), d['phase_ms'], d['passes'], d['config']['tile_qubits'], round(d['roofline']['frac'],3), d['roofline_fp64'])
except Exception as e: print(sys.argv[2], 'fail', e)
PY
}
run c2 --config 2 --steps 20 --warmup 5
run c3 --config 3
run c4 --config 4
run c3nofuse --config 3 --no-fuse-diag
