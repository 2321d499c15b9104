set -u
o=gpurun_out/r4; mkdir -p $o
run() { tag=$1; shift; timeout 300 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e "$@" > $o/$tag.json 2> $o/$tag.err; python - $o/$tag.json $tag <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['ms_per_step'],1), d['phase_ms'], d['passes'])
except Exception as e: print(sys.argv[2], 'fail', e)
PY
}
run base
run rb3 --reg-bits 3
run rb3f3 --reg-bits 3 --reg-bits-fwd 3
run mg24 --max-gates 24
run mg32 --max-gates 32
run mg56 --max-gates 56
run jb13 --jit-blocks 1,3
run nostage --no-stage
run nofuse --no-fuse-diag
