#!/bin/bash
# round-2 first capture: host facts, cfg4 bench line, cfg4 launch list, one cfg4 reverse pass under ncu --set full
set -u
out=gpurun_out/r02p1; mkdir -p $out
(nproc; free -g; lscpu | head -20; nvidia-smi; df -h /tmp /root | tail -3; python -c "import os;print('affinity',len(os.sched_getaffinity(0)))") > $out/host.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > $out/bench_cfg4.json 2> $out/bench_cfg4.err
python bench.py --config 4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $out/plain_cfg4.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_cfg4.csv \
    python bench.py --config 4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $out/ncu_launches_cfg4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip 80 --launch-count 1 \
    -o $out/cfg4_rev python bench.py --config 4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $out/ncu_cfg4_rev.log 2>&1
echo done
