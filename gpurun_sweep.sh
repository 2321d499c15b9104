#!/bin/bash
# sweep tile width x register bits on one config: prints tile, R_rev, R_fwd, phase times, ms/step
cfg=${1:-3}; shift
for spec in "$@"; do
  IFS=, read t r rf extra <<< "$spec"
  timeout 300 python bench.py --steps 2 --warmup 1 --config $cfg --tile-qubits $t --reg-bits $r --reg-bits-fwd $rf ${extra} --no-cpu-baseline --no-e2e > gpurun_out/sw_${cfg}_${t}_${r}_${rf}${extra// /}.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/sw_${cfg}_${t}_${r}_${rf}${extra// /}.log').read().splitlines()[-1]);print('cfg$cfg tile $t R $r Rf $rf $extra', d['phase_ms'], round(d['ms_per_step'],2))" 2>/dev/null || tail -2 gpurun_out/sw_${cfg}_${t}_${r}_${rf}${extra// /}.log
done
