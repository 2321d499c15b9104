#!/bin/bash
# round-2 call 2: chunk groups (several passes per kernel over L2-resident chunks) --
# parity first (variant tests + full-size golden cfg3), then cfg4/cfg3 benches with
# chunks off / 13 / 14 / 15, then the GPU suite and the sanitizer tests.
set -u
out=gpurun_out/r02c2; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "variants or golden_large" > $out/pytest_variants.log 2>&1; echo "variants rc=$?"; tail -3 $out/pytest_variants.log
for c in -1 14 13 15; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --opt chunk_qubits=$c > $out/bench_cfg4_c$c.json 2> $out/bench_cfg4_c$c.err
  python -c "import json;d=json.loads(open('$out/bench_cfg4_c$c.json').read().splitlines()[-1]);print('cfg4 chunk $c', round(d['value'],4), d['phase_ms'], d['passes'], d['roofline']['frac'], d['clocks']['sm_mhz'])" 2>/dev/null || (echo "cfg4 chunk $c FAILED"; tail -3 $out/bench_cfg4_c$c.err)
done
for c in -1 14; do
  timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --opt chunk_qubits=$c > $out/bench_cfg3_c$c.json 2> $out/bench_cfg3_c$c.err
  python -c "import json;d=json.loads(open('$out/bench_cfg3_c$c.json').read().splitlines()[-1]);print('cfg3 chunk $c', round(d['value'],3), d['phase_ms'], d['passes'], d['roofline']['frac'], d['clocks']['sm_mhz'])" 2>/dev/null || (echo "cfg3 chunk $c FAILED"; tail -3 $out/bench_cfg3_c$c.err)
done
timeout 2400 python -m pytest tests -x -q -m gpu > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu.log
