o=gpurun_out/r21; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest.log 2>&1; tail -2 $o/pytest.log
python tools/hostprof.py 2 | tail -2
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline > $o/bench_cfg2_$i.json 2> $o/bench_cfg2.err; python -c "
import json; d=json.loads(open('$o/bench_cfg2_$i.json').read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step'],3), d['e2e']['value'], d['phase_ms'])"; done
