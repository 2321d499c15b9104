#!/bin/bash
# round-2 call 4: checked-kernel tests, reference_gradient / CLI tests, cfg5-structure n=30 over
# 8 virtual shards vs its oracle fixture, default bench line (low_qubits 4), --gpus 2 on a
# 1-GPU lease (must fail loudly), launch list + one ncu --set full of a cfg4 reverse pass.
set -u
out=gpurun_out/r02c4; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_checked.py tests/test_gpu_cli.py -q > $out/pytest_checked_cli.log 2>&1; echo "checked+cli rc=$?"; tail -4 $out/pytest_checked_cli.log
timeout 900 python -m pytest tests/test_gpu_sharded.py -q -k "cfg5_structure_n30" > $out/pytest_cfg5n30.log 2>&1; echo "cfg5 n30 rc=$?"; tail -3 $out/pytest_cfg5n30.log
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"; tail -c 600 $out/bench.json
timeout 300 python bench.py --gpus 2 --steps 1 --warmup 3 > $out/bench_gpus2.json 2> $out/bench_gpus2.err; echo "bench --gpus 2 rc=$?"; tail -3 $out/bench_gpus2.err; cat $out/bench_gpus2.json | tail -c 300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_cfg4.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $out/ncu_launches_cfg4.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip 80 --launch-count 1 \
    -o $out/cfg4_rev python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $out/ncu_cfg4_rev.log 2>&1; echo "ncu full rc=$?"
