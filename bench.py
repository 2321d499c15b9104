#!/usr/bin/env python3
"""Benchmark: full adjoint-gradient evaluations/s on a BASELINE.json config (default cfg 2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

One step = one full gradient (forward passes, observable, fused reverse
passes, finalize) of the configured circuit.  Rank 0 prints ONE JSON line.

* ``value``: device-timed (CUDA events on the engine's stream = torch's
  current stream) throughput with the input state already in HBM (basis-state
  fast path); the per-call gate/term table upload (tens of KB) is inside.
  L2 is flushed (256 MiB write) between timed steps, outside the events.
* ``e2e``: the same metric through the public drop-in API with a HOST input
  StateVector in pinned memory: Python lowering, H2D of the 2^n amplitudes and
  tables, D2H of the P+1 results, all inside a wall-clock timed region.
* ``roofline``: the dominant kernel (k_rev_pass, the fused reverse pass):
  algorithmic bytes per launch = 4 * S (read+write phi and lambda, S = 16*2^n)
  over its CUDA-event launch time, against MEASURED_PEAKS.json hbm_gbs.
* ``roofline_fp64``: the reverse sweep's algorithmic FP64 work (6 FMA per
  amplitude per parametrised gate) over its device time, against the DFMA peak
  measured on B200 (the reverse passes are FP64-bound above ~16 gates per pass,
  profiles/README.md "pass cost model").
* ``cpu_baseline``: the C restatement of the reference's schedule
  (oracle/, "port") on the host cores, bounded sample (rank 0, N=1).
* ``--impl reference``: that same CPU port as the reference arm.

Multi-GPU (torchrun, N>1), max-over-ranks device time:
* configs BASELINE.json runs on one GPU (cfg 1-3; the default cfg 2 is
  "Single GPU"): replicas -- each rank evaluates full gradients of its own
  copy (no data-path collective), ``scaling: "weak"``, value = all ranks'
  gradients / time;
* the sharded configs (cfg 4 "strong-scaling ... sharded on its top qubits",
  cfg 5) or ``--shard``: ONE state split over the N ranks by its top log2(N)
  qubits (paper_2009_02823_b200.distributed.nccl_engine: NCCL half-shard
  exchanges for qubit swaps, partner fetches, one all-gather of partial
  sums), ``scaling: "strong"``, value = gradients of the whole job / time.
"""
from __future__ import annotations

FP64_PEAK_TFLOPS = 37.17  # B200 DFMA peak measured here (tools/ubench/peaks.cu, 32 warps/SM)

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "full-gradient evals/s and achieved HBM GB/s (frac of peak) vs qubits, 1–8 GPU"
UNIT = "gradient evals/s"
FALLBACK_HBM_GBS = 6650.0


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--qubits", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tile-qubits", type=int, default=0)
    ap.add_argument("--reg-bits", type=int, default=0, help="reverse register tile: 2^bits amplitudes/thread (3/4)")
    ap.add_argument("--reg-bits-fwd", type=int, default=0, help="forward register tile: 2^bits amplitudes/thread")
    ap.add_argument("--no-stage", action="store_true", help="generated kernels: no cp.async next-tile staging")
    ap.add_argument("--no-pdl", action="store_true", help="generated kernels: no programmatic dependent launch")
    ap.add_argument("--no-fuse-diag", action="store_true", help="generated kernels: no fused diagonal runs")
    ap.add_argument("--jit", type=int, default=1, help="circuit-specialised kernels: 0 off, 1 auto, 2 always")
    ap.add_argument("--opt", action="append", default=[], help="extra engine option KEY=VALUE (repeatable)")
    ap.add_argument("--jit-blocks", type=str, default="0,0", help="generated kernels: min CTAs/SM fwd,rev (0 default)")
    ap.add_argument("--shard", action="store_true", help="N>1: shard one state over the ranks (default for cfg 4/5)")
    ap.add_argument("--max-gates", type=int, default=0, help="gates per pass cap (0: planner default)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def _peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def _traffic_per_launch(workload: str):
    """ncu DRAM bytes per reverse-pass launch for this workload, from the committed capture summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_rev_pass.json")) as f:
            return float(json.load(f)[workload]["dram_bytes_per_launch"])
    except Exception:
        return None


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region.

    In-process NVML polling every 5 ms (a timed region of a few tens of ms still
    gets samples; the ctypes calls release the GIL), falling back to an
    `nvidia-smi -lms` child process when NVML is unavailable.
    """

    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int, interval_s: float = 0.005):
        self.device = device
        self.interval = interval_s
        self.proc = None
        self.nvml = None
        self.samples: list[tuple[float, float, set]] = []  # (sm MHz, max MHz, reasons)
        self.lines: list[str] = []
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            idx = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(self.device)).split(",")[self.device]) \
                if os.environ.get("CUDA_VISIBLE_DEVICES", "").replace(",", "").isdigit() else self.device
            self.handle = nv.nvmlDeviceGetHandleByIndex(idx)
            self.nvml = nv
            self.bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                         "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                         "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                         "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _sample(self):
        nv = self.nvml
        sm = nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(self.handle, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
        self.samples.append((float(sm), float(mx), {n for n, b in self.bits.items() if r & b}))

    def _poll(self):
        while not self.stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            self.stop.wait(self.interval)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self.stop.set()
        if self.nvml is not None:
            self.thread.join(timeout=1)
            if not self.samples:  # at least one reading at the region's end
                try:
                    self._sample()
                except Exception:
                    pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        for s_, m_, r_ in self.samples:
            sm.append(s_)
            mx = m_
            reasons |= r_
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, flag in zip(self.NAMES, parts[3:7]):
                if flag.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.samples else "nvidia-smi"}


def _cpu_port(w, inp, min_seconds=10.0, max_reps=5):
    from oracle import oracle

    threads = len(os.sched_getaffinity(0))
    reps, t0 = 0, time.perf_counter()
    while reps < max_reps:
        oracle.reverse_mode_values(w.circuit, w.theta, w.observable, inp.amplitudes, threads=threads)
        reps += 1
        if time.perf_counter() - t0 >= min_seconds:
            break
    dt = time.perf_counter() - t0
    return reps / dt, threads, reps, dt


def run_reference(args, rank):
    """Reference arm: the C restatement of the reference's _reverse_sweep on all host cores."""
    if rank != 0:
        return
    import paper_2009_02823_b200 as sv
    from oracle import oracle

    w = sv.build_workload(args.config, args.qubits)
    inp = sv.init_basis_state(w.num_qubits)
    threads = len(os.sched_getaffinity(0))
    for _ in range(args.warmup):
        oracle.reverse_mode_values(w.circuit, w.theta, w.observable, inp.amplitudes, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.reverse_mode_values(w.circuit, w.theta, w.observable, inp.amplitudes, threads=threads)
    dt = time.perf_counter() - t0
    value = args.steps / dt
    sample = f"{args.steps} full gradients of cfg{args.config} (n={w.num_qubits}, G={w.num_gates})"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (BASELINE cfg{args.config} generator, seed 0, |0..0> input)",
        "config": {"workload": f"cfg{args.config}", "num_qubits": w.num_qubits, "num_gates": w.num_gates,
                   "num_params": w.circuit.num_params, "num_terms": len(w.observable.terms)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }))


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_2009_02823_b200 as sv
    from paper_2009_02823_b200 import _native

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    w = sv.build_workload(args.config, args.qubits)
    n = w.num_qubits
    S = 16 << n
    sharded = world > 1 and (args.shard or args.config in (4, 5))
    if sharded:
        eng = sv.distributed.nccl_engine(local_rank)
        jobs = 1  # the N ranks compute one gradient together
    else:
        eng = _native.engine(local_rank)
        jobs = world  # independent replicas
    S_rank = S // world if sharded else S
    eng.set_option("tile_qubits", args.tile_qubits)
    if args.reg_bits:
        eng.set_option("reg_bits", args.reg_bits)
    if args.reg_bits_fwd:
        eng.set_option("reg_bits_fwd", args.reg_bits_fwd)
    eng.set_option("stage", 0 if args.no_stage else 1)
    eng.set_option("pdl", 0 if args.no_pdl else 1)
    eng.set_option("fuse_diag", 0 if args.no_fuse_diag else 1)
    eng.set_option("jit", args.jit)
    eng.set_option("max_gates_per_pass", args.max_gates)
    jb = [int(x) for x in args.jit_blocks.split(",")]
    eng.set_option("jit_blocks_fwd", jb[0])
    eng.set_option("jit_blocks_rev", jb[1])
    for kv in args.opt:
        key, val = kv.split("=")
        eng.set_option(key, int(val))
    stream = torch.cuda.current_stream()
    eng.set_stream(stream.cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    basis = sv.BasisState(n)

    def step(inp, st):
        return sv.reverse_mode_gradient(w.circuit, w.theta, w.observable, inp, stats=st, engine=eng)

    for _ in range(args.warmup):
        step(basis, {})
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    rev_ms, rev_launches, launches, pass_bytes, last, tile_k = 0.0, 0, 0, 0, None, 0
    phases = {"forward": 0.0, "observable": 0.0, "reverse": 0.0, "other": 0.0}
    with ClockSampler(local_rank) as clocks:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            st = {}
            ev[i][0].record(stream)
            last = step(basis, st)
            ev[i][1].record(stream)
            rev_ms += st["ms_reverse"]
            for key in phases:
                phases[key] += st[f"ms_{key}"] / args.steps
            rev_launches += st["rev_passes"]
            launches += st["launches"]
            pass_bytes = st["pass_bytes"]
            tile_k = st["tile_qubits"]
            st_last = st
        torch.cuda.synchronize()
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    if dist:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        total_ms = float(t.item())
    torch.cuda.synchronize()

    e2e = None
    if not args.no_e2e and not (sharded and S > (4 << 30)):
        # (sharded n >= 29: the API's full-size host StateVector on every rank would
        # need N x S of pinned host memory; e2e is reported for the unsharded runs)
        pinned = torch.empty(1 << n, dtype=torch.complex128, pin_memory=True)
        host = pinned.numpy()
        host[:] = 0
        host[0] = 1.0
        state = sv.StateVector(n, host)
        assert state.amplitudes.ctypes.data == host.ctypes.data  # no hidden pageable copy
        st = {}
        step(state, st)
        torch.cuda.synchronize()
        wall = 0.0
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep = step(state, st)
            wall += time.perf_counter() - t0
        e2e = {"value": jobs * args.steps / wall, "unit": UNIT,
               "h2d_bytes_per_step": int(st["h2d_bytes"]), "d2h_bytes_per_step": int(st["d2h_bytes"])}
        if dist:
            t = torch.tensor([wall], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e["value"] = jobs * args.steps / float(t.item())
        assert np.array_equal(rep.values, last.values)

    if rank != 0:
        return
    peak, peak_src = _peak()
    avg_launch_ms = rev_ms / max(1, rev_launches)
    achieved = 4 * S_rank / (avg_launch_ms * 1e-3) / 1e9
    traffic = _traffic_per_launch(f"cfg{args.config}") if args.qubits is None and world == 1 else None
    value = jobs * args.steps / (total_ms * 1e-3)
    B_alg = 6 * w.num_gates * S  # gate-level algorithmic bytes per gradient
    n_param_gates = sum(1 for g in w.circuit.gates if len(g.param_refs) > 0)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cval, cores, reps, secs = _cpu_port(w, sv.init_basis_state(n))
        cpu = {"value": cval, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{reps} full gradient(s) of cfg{args.config} in {secs:.1f} s (oracle/svgrad_oracle.c, OpenMP)"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (BASELINE cfg{args.config} generator, seed 0, |0..0> input; random-init theta)",
        "config": {
            "workload": f"cfg{args.config}", "num_qubits": n, "num_gates": w.num_gates,
            "num_params": w.circuit.num_params, "num_terms": len(w.observable.terms),
            "state_bytes": S, "l2": "flushed between timed steps (256 MiB write, outside the events)",
            "parallelism": (f"state sharded over {world} ranks (top {world.bit_length() - 1} qubits)" if sharded
                            else "replicas" if world > 1 else "single-gpu"), "tile_qubits": tile_k,
            "swaps_per_gradient": int(st_last["swaps"]), "exchange_bytes_per_rank": int(st_last["exchange_bytes"]),
        },
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": "reverse register-tile pass (generated svgb_jit; interpreter k_pass_reg<4,2>)",
            "bytes_per_launch": 4 * S_rank,
            "avg_launch_ms": avg_launch_ms, "peak_source": peak_src,
        },
        # the reverse sweep is FP64-bound above ~16 gates per pass: its algorithmic
        # FP64 work is 6 FMA (12 flop) per amplitude per parametrised gate (rewind
        # phi and lambda: 2 FMA each, Re<lambda|K|phi>: 2), against the DFMA peak
        # measured with tools/ubench/peaks.cu (profiles/r01_ubench_peaks.jsonl)
        "roofline_fp64": {
            "kernel": "reverse sweep (all reverse passes)", "unit": "TFLOP/s",
            "flop_per_gradient": 12 * (S_rank // 16) * n_param_gates,
            "achieved": 12 * (S_rank // 16) * n_param_gates / (phases["reverse"] * 1e-3) / 1e12,
            "peak": FP64_PEAK_TFLOPS,
            "frac": 12 * (S_rank // 16) * n_param_gates / (phases["reverse"] * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
            "peak_source": "measured DFMA throughput, tools/ubench/peaks.cu (37.2 TFLOP/s at 1965 MHz)",
        } if phases.get("reverse") else None,
        "phase_ms": {k: round(v, 4) for k, v in phases.items()},
        "passes": {"forward": int(st_last["fwd_passes"]), "observable": int(st_last["obs_passes"]),
                   "reverse": int(st_last["rev_passes"])},
        "effective_gate_level_gbs": B_alg / (total_ms / args.steps * 1e-3) / 1e9,
        "pass_level_gbs": pass_bytes / (total_ms / args.steps * 1e-3) / 1e9,
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks.summary(),
    }
    print(json.dumps(line))


def main():
    args = _args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
