#!/bin/bash
# round-2 call 6: K5 whole-sweep kernel -- parity (forced on every small golden case, and as the
# auto path of the default golden tests), cfg1 / small-n benches vs the pass pipeline
set -u
out=gpurun_out/r02c6; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "whole or test_gpu_matches_reference_golden or deterministic or basis_fast or audit or errors or negative or duck" > $out/pytest_k5.log 2>&1; echo "k5 parity rc=$?"; tail -4 $out/pytest_k5.log
run() { tag=$1; cfg=$2; st=$3; shift 3
  timeout 600 python bench.py --config $cfg --steps $st --warmup 5 --no-cpu-baseline "$@" > $out/bench_$tag.json 2> $out/bench_$tag.err
  python -c "import json;d=json.loads(open('$out/bench_$tag.json').read().splitlines()[-1]);print('$tag', round(d['value'],1), 'e2e', round(d['e2e']['value'],1) if d.get('e2e') else None, d['phase_ms'], d['passes'], d['gpu_launches'], d['clocks']['sm_mhz'])" 2>/dev/null || (echo "$tag FAILED"; tail -3 $out/bench_$tag.err); }
run cfg1_k5 1 200
run cfg1_pipe 1 200 --opt kernel=2
run cfg2n12_k5 2 100 --qubits 12
run cfg2n12_pipe 2 100 --qubits 12 --opt kernel=2
run cfg3n11_k5 3 100 --qubits 11
run cfg3n11_pipe 3 100 --qubits 11 --opt kernel=2
