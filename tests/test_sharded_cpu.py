"""Sharded (multi-GPU) schedule on CPU: 2 and 4 gloo ranks, one process each.

Each rank runs the engine's sharded algorithm in numpy (tests/emulator.py
``emulate_sharded``) on its own shard: the C++ planner's schedule
(svg_plan_schedule -- passes over physical local qubits and rank-bit <->
local-qubit swaps), half-shard swaps and partner-shard fetches over
torch.distributed (gloo), per-rank partial inner products and an all-reduce.
The combined gradient must equal the reference's golden values: this pins the
host logic of the N>1 path (plan, qubit map, exchange semantics) that the
GPU engine executes with NCCL (or, on one GPU, with virtual shards).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from cases import config_cases, small_cases
from conftest import cvec, load_golden, materialize, max_err

CASES = {**small_cases(), **config_cases()}
NAMES = ["cfg5_n11", "cfg3_n10", "cfg4_n12", "all_kinds_6_random", "family_D9_random"]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, names, queue):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    from emulator import emulate_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def exchange(arr, partner):
        send = torch.from_numpy(np.ascontiguousarray(arr).view(np.float64)).clone()
        recv = torch.empty_like(send)
        reqs = [dist.isend(send, partner), dist.irecv(recv, partner)]
        for r in reqs:
            r.wait()
        return recv.numpy().view(np.complex128)

    out = {}
    try:
        _run(names, world, rank, exchange, emulate_sharded, out)
    except Exception as exc:  # surface worker failures instead of hanging the parent
        import traceback

        queue.put(("error", rank, traceback.format_exc()))
        raise
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        queue.put(("ok", rank, out))


def _run(names, world, rank, exchange, emulate_sharded, out):
    for name in names:
        circ, theta, obs, inp, _ = materialize(CASES[name])
        contrib, energy, steps = emulate_sharded(circ, theta, obs, inp, world, rank, exchange)
        t = torch.from_numpy(np.concatenate([contrib, [energy]]).view(np.float64)).clone()
        dist.all_reduce(t)
        tot = t.numpy().view(np.complex128)
        out[name] = (tot[:-1].copy(), complex(tot[-1]), sum(s[0] == "swap" for s in steps))


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_schedule_gloo(world):
    from emulator import combine

    gold = load_golden()
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, NAMES, queue)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        status, rank, result = queue.get(timeout=300)
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert status == "ok", f"rank {rank} failed:\n{result}"
    swaps_seen = 0
    for name in NAMES:
        contrib, energy, swaps = result[name]
        circ, _, _, _, _ = materialize(CASES[name])
        sums = combine(circ, None, contrib)
        rec = gold[name]
        assert max_err(2 * sums.real, cvec(rec["values"]).real) <= 1e-10, name
        assert abs(energy - complex(*rec["energy"])) <= 1e-12, name
        swaps_seen += swaps
    assert swaps_seen > 0  # the cases really exercise rank-bit swaps

