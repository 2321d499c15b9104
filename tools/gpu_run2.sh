set -u
o=gpurun_out/r2; mkdir -p $o
./tools/ubench/peaks > $o/peaks.json 2>&1
for k in 10 12; do
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --tile-qubits $k > $o/cfg3_k$k.json 2> $o/cfg3_k$k.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_cfg3.csv \
    python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $o/ncu_launches_cfg3.log 2>&1
cat $o/peaks.json $o/cfg3_k*.json
