#!/usr/bin/env python3
"""Full-size sharded schedules on one GPU: cfg 4 / cfg 5 layer structure at n = 30
split into 2 and 8 virtual shards (the NCCL data path emulated with device
copies) against the single-shard engine; prints swaps, exchange bytes and the
result agreement (profiles/r01_virtual_shards_n30.jsonl)."""
import sys, time, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2009_02823_b200 as sv
for cfg, n in ((4, 30), (5, 30)):
    w = sv.build_workload(cfg, n)
    ref = sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, sv.BasisState(n))
    for shards in (2, 8):
        eng = sv.distributed.virtual_engine(shards)
        eng.set_option("emulate_transport", 1)
        st = {}
        rep = sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, sv.BasisState(n), engine=eng, stats=st)
        err = float(np.max(np.abs(rep.values - ref.values) / np.maximum(1, np.abs(ref.values))))
        print(json.dumps({"cfg": cfg, "n": n, "shards": shards, "swaps": st["swaps"], "exchange_bytes": st["exchange_bytes"],
                          "fwd_passes": st["fwd_passes"], "rev_passes": st["rev_passes"], "ms_total": st["ms_total"],
                          "max_rel_err_vs_single": err, "dE": abs(rep.energy - ref.energy)}), flush=True)
        eng.close(); del eng; torch.cuda.empty_cache()
