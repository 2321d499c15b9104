set -u
o=gpurun_out/r5; mkdir -p $o
python tools/hostprof.py 2 > $o/hostprof2.txt 2>&1
run() { tag=$1; shift; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e "$@" > $o/$tag.json 2> $o/$tag.err; python - $o/$tag.json $tag <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['ms_per_step'],3), d['phase_ms'], d['passes'], d['config']['tile_qubits'])
except Exception as e: print(sys.argv[2], 'fail', e)
PY
}
run base
run t9 --tile-qubits 9
run t11 --tile-qubits 11
run rb4 --reg-bits 4
run rb4f4 --reg-bits 4 --reg-bits-fwd 4
run mg24 --max-gates 24
run mg56 --max-gates 56
run jb -–jit-blocks 0,3
run nopdl --no-pdl
run jit0 --jit 0
cat $o/hostprof2.txt
