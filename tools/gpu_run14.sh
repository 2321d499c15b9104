o=gpurun_out/r14; mkdir -p $o/jit
SVGB_JIT_DUMP=$o/jit timeout 300 python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $o/plain.json 2>&1
for s in 103 104; do
ncu --set full --import-source on --clock-control none -k regex:svgb_jit --launch-skip $s --launch-count 1 \
    -o $o/cfg3_rev_$s python bench.py --config 3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $o/ncu_$s.log 2>&1
done
