o=gpurun_out/r19; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest.log 2>&1; tail -3 $o/pytest.log
timeout 600 python bench.py > $o/bench_cfg2.json 2> $o/bench_cfg2.err; cat $o/bench_cfg2.json
python tools/hostprof.py 2 | tail -2
