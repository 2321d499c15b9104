#!/bin/bash
# tile/reg-bits sweep on one config: prints  tile reg ms_per_step avg_rev_launch_ms
cfg=${1:-3}
for r in 3 4; do for t in 10 11 12; do
  timeout 300 python bench.py --steps 2 --warmup 1 --config $cfg --tile-qubits $t --reg-bits $r --no-cpu-baseline --no-e2e > gpurun_out/sw_${cfg}_${t}_${r}.log 2>&1
  python -c "import json,sys;d=json.loads(open('gpurun_out/sw_${cfg}_${t}_${r}.log').read().splitlines()[-1]);print('cfg$cfg tile',$t,'R',$r,round(d['ms_per_step'],2),round(d['roofline']['avg_launch_ms'],3))" 2>/dev/null || tail -2 gpurun_out/sw_${cfg}_${t}_${r}.log
done; done
