#!/bin/bash
# round-2 call 1 (re-entry): host facts, smoke, cfg4 bench line + reference arm, oracle n=30 fixtures on
# the host cores (background) while the GPU suite runs, cfg4 launch list + one ncu --set full reverse pass,
# then the full-size fixture parity tests.
set -u
out=gpurun_out/r02c1; mkdir -p $out
(nproc; free -g; lscpu | head -20; nvidia-smi; df -h /tmp /root | tail -3; python -c "import os;print('affinity',len(os.sched_getaffinity(0)))") > $out/host.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc=$?"
avail=$(awk '/MemAvailable/{print int($2/1048576)}' /proc/meminfo); echo "mem avail GiB $avail"
if [ "$avail" -gt 110 ]; then
 (for c in cfg4 cfg5_n30 hadamard_n26; do timeout 2400 python tests/golden/make_oracle_n30.py $c > $out/oracle_$c.log 2>&1; cp tests/golden/oracle_$c.json $out/ 2>/dev/null; done) &
 opid=$!
else opid=""; fi
timeout 2400 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu.log
timeout 600 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $out/plain_cfg4.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_cfg4.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $out/ncu_launches_cfg4.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip 80 --launch-count 1 \
    -o $out/cfg4_rev python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $out/ncu_cfg4_rev.log 2>&1; echo "ncu full rc=$?"
if [ -n "$opid" ]; then wait $opid; fi
tail -n1 $out/oracle_*.log
timeout 1800 python -m pytest tests -q -k "cfg4_vs_oracle or n26_vs_oracle or cfg5_n30" > $out/pytest_fixtures.log 2>&1; echo "fixture parity rc=$?"
tail -5 $out/pytest_fixtures.log
