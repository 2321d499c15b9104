o=gpurun_out/r30; mkdir -p $o/jit
SVGB_JIT_DUMP=$o/jit timeout 300 python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $o/plain.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_cfg3.csv python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $o/l.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip 84 --launch-count 2 \
    -o $o/cfg3_rev python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $o/ncu.log 2>&1
