set -u
mkdir -p gpurun_out/r1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r1/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r1/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r1/bench_cfg2.json 2> gpurun_out/r1/bench_cfg2.err
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r1/bench_cfg3.json 2> gpurun_out/r1/bench_cfg3.err
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1/bench_cfg4.json 2> gpurun_out/r1/bench_cfg4.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1/smoke.log 2>&1
tail -3 gpurun_out/r1/pytest_gpu.log
cat gpurun_out/r1/bench_cfg2.json gpurun_out/r1/bench_cfg3.json gpurun_out/r1/bench_cfg4.json
