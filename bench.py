#!/usr/bin/env python
"""Benchmark of the hot path: TensorNet energy+forces steps/s (neighbor search included).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload C|A|D|E] [--no-sweep] [--no-cpu]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N ... bench.py --gpus N ...
    (``--gpus N`` without RANK in the environment re-launches itself that way)

A "step" is one pass of the hot path over one batch of synthetic input: cutoff neighbor
search (cell list) + TensorNet forward + analytic force sweep, replayed as one CUDA graph.
Default workload = BASELINE.json configs[2]: 2-layer, 128-channel TensorNet on the synthetic
23,558-atom periodic box (the configuration the north-star target is quoted on).  With
N > 1 the default workload becomes D (BASELINE.json configs[3]): the batch of 8192 molecules is
sharded by whole molecules over the ranks ("strong" scaling, no collective inside the step) and
the final all_gather of energies and forces is INSIDE the timed region.  A single periodic box
does not shard ("replicas only"): `--workload C|E` with N > 1 steps N replicas.
Layer counts follow BASELINE.json: 2 layers for A, C, D and 3 layers for E.

One JSON line on stdout (rank 0).  `value` = whole-job steps/s with inputs resident in HBM;
`e2e` = the same through TensorNet.forward with pinned HOST buffers (H2D of species+positions
and D2H of energy+forces inside the timed region).  `--impl reference` times the CPU oracle
port (there is no compilable reference: the reference is Python/numba) on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TensorNet energy+forces steps/s (neighbor search included)"
CHANNELS, NUM_RBF, CUTOFF = 128, 32, 5.0
LAYERS_OF = {"A": 2, "C": 2, "D": 2, "E": 3}       # BASELINE.json configs


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def workload(name: str, rank: int = 0, world: int = 1):
    from paper_2402_17660_b200 import synth

    if name == "A":
        z, pos, batch, box = synth.config_a_molecule()
        desc = "A: 22-atom molecule, open boundaries"
    elif name == "C":
        z, pos, batch, box = synth.config_c_box()
        desc = "C: 23,558-atom periodic cubic box (62.23 A), water-like species"
    elif name == "D":
        z, pos, batch, box = synth.config_d_molecules(8192)
        shards = synth.shard_by_molecule(batch, world)
        a0, a1, s0, _ = shards[rank]
        z, pos, batch = z[a0:a1], pos[a0:a1], batch[a0:a1] - s0
        desc = f"D: 8192 QM9-sized molecules sharded by molecule over {world} rank(s)"
    elif name == "E":
        z, pos, batch, box = synth.config_e_triclinic()
        desc = "E: 100,000-atom triclinic periodic water box"
    else:
        raise SystemExit(f"unknown workload {name}")
    return z, pos, batch, box, desc


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    QUERY = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[3:7]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "samples": len(sm),
                "reasons": sorted(reasons)}


def algorithmic_bytes(n_atoms: int, n_edges: int, n_cells: int, layers: int):
    """Compulsory HBM bytes; gathers counted once per pass."""
    T = 9 * CHANNELS * 4
    L = layers
    per_kernel = {
        "k_edge_message": 4 * T * n_atoms + 20 * n_edges,      # read Y' (gather + own), write M and Q
        "k_edge_message_bwd": 4 * T * n_atoms + 28 * n_edges,  # read G_M, Y', G_Y; write G_Y; edges
        "k_embed_edge": T * n_atoms + 8 * CHANNELS * n_atoms + 36 * n_edges,
        "k_embed_edge_bwd": T * n_atoms + 60 * n_edges,
        "gemm_mix": 2 * T * n_atoms,
        "k_rows_fill": 32 * n_atoms + 8 * n_cells + 24 * n_edges,
        "k_rows_count": 32 * n_atoms + 8 * n_cells,
    }
    step = T * n_atoms * (14 * L + 8) + 52 * n_edges * (L + 1)          # SURVEY.md 8d, B_tn
    nl = 48 * n_atoms + 8 * n_cells + 24 * n_edges                      # SURVEY.md 8d, B_nl
    return per_kernel, step, nl


def cpu_oracle_step(sample_atoms: int, full_nl: bool = True, seed: int = 11):
    """Time the CPU oracle port: neighbor list (C, 1 core) on the full box + float64 TensorNet
    (numpy, all BLAS threads) on a periodic sample of the same density; returns seconds per
    full-size step (TensorNet part scaled by atom count) and a description."""
    from paper_2402_17660_b200 import synth, init_params, TNConfig
    from oracle import neighbors_oracle as O
    from oracle import tensornet_oracle as T

    t_nl = 0.0
    n_full = 23558
    if full_nl:
        z, pos, batch, box = synth.config_c_box()
        t0 = time.perf_counter()
        O.build_neighbor_list(pos, batch, box, CUTOFF, 2 * 64 * n_full, strategy="cell",
                              full_list=True, include_self_loops=True)
        t_nl = time.perf_counter() - t0
    edge = (sample_atoms / 0.09776) ** (1.0 / 3.0)
    z, pos, batch, box = synth.config_c_box(n=sample_atoms, edge=edge, seed=seed)
    cfg = TNConfig(embedding_dimension=CHANNELS, num_layers=LAYERS_OF["C"], num_rbf=NUM_RBF, cutoff_upper=CUTOFF)
    params = init_params(cfg, 0)
    ocfg = T.OracleConfig(CHANNELS, LAYERS_OF["C"], NUM_RBF, 0.0, CUTOFF)
    t0 = time.perf_counter()
    nl = O.build_neighbor_list(pos, batch, box, CUTOFF, 2 * 64 * sample_atoms, full_list=True,
                               include_self_loops=True)
    pr, dl, ds = nl.valid()
    T.energy_forces_compact(params, ocfg, z, batch, pr, dl, ds)
    t_tn = time.perf_counter() - t0
    seconds = t_nl + t_tn * n_full / sample_atoms
    return seconds, t_nl, t_tn


def run_reference(args):
    """Reference arm: the CPU implementation of the path (oracle port) on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    # bounded sample of the workload, sized so that warmup + steps end within a few minutes
    # (the oracle takes ~12 ms per atom on the GPU box's host; 125 atoms is the smallest periodic
    # box of this density that still holds the 5 A cutoff)
    iters = args.warmup + args.steps
    sample = 343 if iters <= 20 else (216 if iters <= 40 else 125)
    per_step = []
    for it in range(args.warmup + args.steps):
        sec, _, _ = cpu_oracle_step(sample, full_nl=True)
        if it >= args.warmup:
            per_step.append(sec)
    ms = 1000.0 * float(np.mean(per_step))
    value = 1000.0 / ms
    desc = (f"per step: C-oracle cell neighbor list on the full 23,558-atom box (1 core) + float64 "
            f"numpy TensorNet oracle (energy+forces) on a {sample}-atom periodic box of the same "
            f"density, TensorNet time scaled by 23558/{sample}")
    # one TRUE full-size oracle step was timed when the config-C fixture was generated (build
    # container, not this host): reported next to the extrapolation so that it can be checked
    full = None
    fixture = os.path.join(ROOT, "tests", "golden", "tn_golden_C.npz")
    if os.path.exists(fixture):
        with np.load(fixture) as g:
            full = {"seconds_per_step": round(float(g["oracle_seconds"]), 1), "atoms": 23558,
                    "where": "build container (8 cores), tests/golden/make_tn_golden.py; neighbor list included"}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": (f"C-sample: neighbor list on the full 23,558-atom box + TensorNet on a {sample}-atom "
                                f"periodic box of config C's density, TensorNet time scaled by 23558/{sample}"),
                   "sampled_atoms": sample, "full_atoms": 23558, "extrapolated": True, "same_config": False,
                   "channels": CHANNELS, "layers": LAYERS_OF["C"], "num_rbf": NUM_RBF, "cutoff": CUTOFF},
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": cores, "kind": "port",
                         "sample": desc, "full_size_step_measured_elsewhere": full},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def neighbor_sweep(torch, peak_gbs, with_cpu=True):
    """Config B: neighbor-list us/call over particle counts (half list, like bench.py:133-138 of
    the reference), with the C oracle (the CPU port of the reference's numba kernels, one core,
    one call) timed beside every point it finishes in seconds."""
    import paper_2402_17660_b200 as P
    from oracle import neighbors_oracle as O
    from paper_2402_17660_b200 import _lib, synth
    from paper_2402_17660_b200.neighbors import NeighborEngine, plan_strategy

    rows = []
    for n in (1000, 4096, 16384, 65536, 262144, 1048576):
        _, pos, batch, boxm = synth.config_b_cloud(n)
        box = P.Box.from_matrix(boxm)
        dev_pos = torch.from_numpy(pos).cuda()
        dev_batch = torch.zeros(n, dtype=torch.int32, device="cuda")
        for strategy in ("cell", "brute"):
            if strategy == "brute" and n > 65536:
                continue
            code, dims, max_cells, _ = plan_strategy(n, box, CUTOFF, strategy)
            cap = 32 * n
            eng = NeighborEngine(n, 1, cap, box, 0.0, CUTOFF, code, dims, max_cells, 0)
            eng.build(dev_pos, dev_batch)
            torch.cuda.synchronize()
            pairs = int(eng.counts[0].item())
            reps = 20 if n <= 65536 else 5
            if strategy == "brute" and n >= 65536:
                reps = 2
            start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record()
            for _ in range(reps):
                eng.build(dev_pos, dev_batch)
            stop.record()
            torch.cuda.synchronize()
            us = 1000.0 * start.elapsed_time(stop) / reps
            # the reference times deterministic=False (bench.py:133-138): same list, rows not ranked
            eng_u = NeighborEngine(n, 1, cap, box, 0.0, CUTOFF, code, dims, max_cells, _lib.NL_UNSORTED)
            eng_u.build(dev_pos, dev_batch)
            torch.cuda.synchronize()
            start.record()
            for _ in range(reps):
                eng_u.build(dev_pos, dev_batch)
            stop.record()
            torch.cuda.synchronize()
            us_unsorted = 1000.0 * start.elapsed_time(stop) / reps
            del eng_u
            ncell = int(eng.counts[2].item()) if strategy == "cell" else 0
            nbytes = 48 * n + 8 * ncell + 40 * pairs      # float64 outputs: 8 + 24 + 8 B per row
            row = {"n": n, "strategy": strategy, "us_per_call": round(us, 2),
                   "us_per_call_unsorted": round(us_unsorted, 2), "pairs": pairs,
                   "hbm_frac": round(nbytes / (us * 1e-6) / 1e9 / peak_gbs, 4)}
            if with_cpu and (n <= 262144 if strategy == "cell" else n <= 16384):
                t0 = time.perf_counter()
                # deterministic=False like the reference's own sweep: compare with us_per_call_unsorted
                ref = O.build_neighbor_list(pos, batch, boxm, CUTOFF, cap, strategy=strategy, deterministic=False)
                row["cpu_us_per_call"] = round(1e6 * (time.perf_counter() - t0), 1)
                row["cpu_cores"] = 1
                row["cpu_pairs_equal"] = bool(ref.count == pairs)
            rows.append(row)
            del eng
        del dev_pos, dev_batch
        torch.cuda.empty_cache()
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=["A", "C", "D", "E"],
                    help="default: C on one GPU, D (sharded by molecule) on several")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-md", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "RANK" not in os.environ:
        # one process per GPU: re-launch under torchrun exactly as the driver does
        import socket

        with socket.socket() as sock:
            sock.bind(("127.0.0.1", 0))
            port = sock.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)

    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.workload is None:
        args.workload = "C" if world == 1 else "D"
    LAYERS = LAYERS_OF[args.workload]
    sharded = world > 1 and args.workload == "D"
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (there is no CPU fallback)")
    # NNP_BENCH_SHARE_GPU=1 (functional test of the multi-rank path on a one-GPU box): every rank
    # uses cuda:0 and the gather runs over gloo, since NCCL refuses two ranks on one device
    share_gpu = os.environ.get("NNP_BENCH_SHARE_GPU") == "1"
    if share_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2402_17660_b200 as P
    from paper_2402_17660_b200 import _lib

    peak_gbs, peak_src = load_peaks()
    full_batch = None
    if sharded:
        from paper_2402_17660_b200 import synth

        full_batch = synth.config_d_molecules(8192)[2]
    z, pos, batch, box, desc = workload(args.workload, rank, world)
    n_atoms = len(pos)
    n_samples = int(batch[-1]) + 1
    model = P.TensorNet(embedding_dimension=CHANNELS, num_layers=LAYERS, num_rbf=NUM_RBF,
                        cutoff_upper=CUTOFF, seed=0)
    lib = _lib.load()

    z_t = torch.from_numpy(np.array(z, dtype=np.int32))
    pos_t = torch.from_numpy(np.array(pos, dtype=np.float32))
    batch_t = None if n_samples == 1 else torch.from_numpy(np.array(batch, dtype=np.int32))
    plan = model.prepare(z_t, pos_t, batch_t, box, n_samples=n_samples)
    n_edges = int(plan.engine.counts[0].item())
    n_cells = int(plan.engine.counts[2].item())

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- launches per step + per-kernel device times (eager pass, CUDA events per kernel)
    lib.nnp_launch_count(1)
    model.enqueue_eager(plan)
    torch.cuda.synchronize()
    launches_per_step = lib.nnp_launch_count(1)
    for _ in range(2):
        model.enqueue_eager(plan)
    torch.cuda.synchronize()
    prof = {}
    reps = 5
    for _ in range(reps):
        for k, (ms, cnt) in _lib.profile_step(lambda: model.enqueue_eager(plan)).items():
            a = prof.setdefault(k, [0.0, 0])
            a[0] += ms / reps
            a[1] = cnt
    kernel_ms = {k: round(v[0], 5) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}

    # ---- device-resident timing: K graph replays, CUDA events, max over ranks.  Sharded batch
    # (workload D on several GPUs): every step ends with the all_gather that returns all energies
    # and forces to every rank (sharding.py), inside the timed region.
    gather = None
    if sharded:
        from paper_2402_17660_b200.sharding import ResidentGather

        gather = ResidentGather(full_batch, world, rank, torch.device("cuda", local))

    def resident_step():
        model.replay(plan)
        if gather is not None:
            gather(plan.energy, plan.forces)

    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    for _ in range(args.warmup):
        resident_step()
    barrier()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(args.steps):
        resident_step()
    stop.record()
    barrier()
    elapsed_ms = start.elapsed_time(stop)
    if world > 1:
        t = torch.tensor([elapsed_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    units = world if args.workload != "D" else 1        # replicas: every rank steps its own box
    value = units * 1000.0 / ms_per_step

    # ---- end to end through the public API with pinned host buffers
    z_h, pos_h = z_t.pin_memory(), pos_t.pin_memory()
    b_h = None if batch_t is None else batch_t.pin_memory()
    out_samples = n_samples if gather is None else gather.n_samples
    out_atoms = n_atoms if gather is None else gather.n_atoms
    e_h = torch.empty(out_samples, dtype=torch.float32).pin_memory()
    f_h = torch.empty((out_atoms, 3), dtype=torch.float32).pin_memory()

    def e2e_step():
        # (measured: TensorNet.forward_host - pinned staging and one graph holding the copies - is slower
        #  for inputs that are pinned already: 4.606 vs 4.546 ms on config C; it serves pageable numpy input)
        e, f = model.forward(z_h, pos_h, b_h, box, n_samples=n_samples, check=True, clone=False)
        if gather is not None:
            e, f = gather(e, f)
        e_h.copy_(e, non_blocking=True)
        f_h.copy_(f, non_blocking=True)
        torch.cuda.synchronize()

    for _ in range(3):
        e2e_step()
    barrier()
    # sub-millisecond steps: enough iterations for ~60 ms of timed work, so that one host hiccup
    # does not decide the number (15 steps of the 22-atom config are a 5 ms window)
    e2e_steps = max(10, args.steps // 2, min(400, int(60.0 / max(ms_per_step, 1e-3))))
    start.record()
    for _ in range(e2e_steps):
        e2e_step()
    stop.record()
    barrier()
    e2e_ms = start.elapsed_time(stop)
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = units * 1000.0 * e2e_steps / e2e_ms
    if rank == 0:
        # keep the GPU under the same load until nvidia-smi has at least a few samples
        t_end = time.time() + 1.5
        while len(sampler.lines) < 4 and time.time() < t_end:
            model.replay(plan)
            torch.cuda.synchronize()
    clocks = sampler.stop() if rank == 0 else None
    h2d = z_h.numel() * 4 + pos_h.numel() * 4 + (0 if b_h is None else b_h.numel() * 4)
    d2h = e_h.numel() * 4 + f_h.numel() * 4 + 4      # + the overflow counter read

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel and of the whole step
    per_kernel_bytes, step_bytes, nl_bytes = algorithmic_bytes(n_atoms, n_edges, n_cells, LAYERS)
    dominant = next(iter(kernel_ms))
    launches = prof[dominant][1]
    roof = {"bound": "hbm", "kernel": dominant, "peak": peak_gbs, "unit": "GB/s", "peak_source": peak_src,
            "achieved": None, "frac": None, "traffic": None, "launches_per_step": launches}
    if dominant in per_kernel_bytes:
        per_launch_ms = prof[dominant][0] / launches
        achieved = per_kernel_bytes[dominant] / (per_launch_ms * 1e-3) / 1e9
        roof.update({"achieved": round(achieved, 1), "frac": round(achieved / peak_gbs, 4),
                     "algorithmic_bytes_per_launch": per_kernel_bytes[dominant],
                     "avg_launch_ms": round(per_launch_ms, 5)})
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(traffic_path) and args.workload == "C":   # the ncu captures are of config C
        with open(traffic_path) as fh:
            roof["traffic"] = json.load(fh).get(dominant)
    # the channel-mixing GEMMs against the tensor roofline (3xTF32: three tcgen05.mma kind::tf32 per
    # product; TF32 peak taken as half of the measured dense bf16 peak, the nominal ratio)
    gemm_roof = None
    if "gemm_mix" in prof and prof["gemm_mix"][1] > 0:
        per_launch_ms = prof["gemm_mix"][0] / prof["gemm_mix"][1]
        flops = 2.0 * 9 * n_atoms * CHANNELS * CHANNELS * 3
        tf32_peak = None
        peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
        if os.path.exists(peaks_path):
            with open(peaks_path) as fh:
                tf32_peak = 0.5 * float(json.load(fh).get("bf16_tflops_sustained", 0.0)) or None
        tf32_peak = tf32_peak or 0.5 * 1400.0
        achieved = flops / (per_launch_ms * 1e-3) / 1e12
        gemm_roof = {"bound": "tensor", "kernel": "gemm_mix (tcgen05 kind::tf32, 3xTF32)", "achieved": round(achieved, 1),
                     "peak": round(tf32_peak, 1), "unit": "TFLOP/s", "frac": round(achieved / tf32_peak, 4),
                     "hbm_frac": round(per_kernel_bytes["gemm_mix"] / (per_launch_ms * 1e-3) / 1e9 / peak_gbs, 4),
                     "launches_per_step": prof["gemm_mix"][1], "avg_launch_ms": round(per_launch_ms, 5)}
    step_roof = {"algorithmic_bytes": step_bytes + nl_bytes,
                 "achieved_gbs": round((step_bytes + nl_bytes) / (ms_per_step * 1e-3) / 1e9, 1),
                 "frac": round((step_bytes + nl_bytes) / (ms_per_step * 1e-3) / 1e9 / peak_gbs, 4)}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak" if args.workload != "D" else "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": desc, "atoms": n_atoms, "samples": n_samples, "directed_edges": n_edges,
                   "channels": CHANNELS, "layers": LAYERS, "num_rbf": NUM_RBF, "cutoff": CUTOFF,
                   "parallelism": "replicas only" if args.workload != "D" else
                                  f"whole molecules over {world} rank(s); all_gather of energies+forces inside the timed step"
                                  if world > 1 else "one GPU",
                   "atoms_are": "rank 0's shard" if sharded else "whole system",
                   "l2_note": "working set per step (saved activations ~1.3 GB) exceeds the 126 MB L2; no flush",
                   "msteps_per_day": round(86.4 / ms_per_step, 3)},
        "clocks": clocks,
        "e2e": {"value": round(e2e_value, 3), "unit": "steps/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms / e2e_steps, 4)},
        "gpu_launches": launches_per_step * args.steps,
        "launches_per_step": launches_per_step,
        "roofline": roof,
        "step_roofline": step_roof,
        "gemm_roofline": gemm_roof,
        "kernel_ms": kernel_ms,
    }
    if world == 1 and not args.no_cpu and args.workload == "C":
        sec, t_nl, t_tn = cpu_oracle_step(1000)
        line["cpu_baseline"] = {
            "value": round(1.0 / sec, 5), "unit": "steps/s", "cores": os.cpu_count() or 1, "kind": "port",
            "sample": (f"C-oracle cell neighbor list on the full 23,558-atom box ({t_nl:.2f} s, 1 core) + "
                       f"float64 numpy TensorNet oracle energy+forces on a 1000-atom periodic box of the "
                       f"same density ({t_tn:.1f} s, BLAS threads = all cores), scaled by 23558/1000"),
        }
    if world == 1 and args.workload in ("A", "C") and not args.no_md:
        # the MD driver = the same step + the Langevin integrator kernel in
        # one graph, float64 positions resident on the device, noise from the device Philox
        from paper_2402_17660_b200 import md as M

        system = P.build_system(np.asarray(pos, dtype=np.float32).astype(np.float64), z, box=model._as_box(box))
        state = M.initialize_state(system, 300.0, seed=0)
        integ = M.DeviceIntegrator(model, system, state.velocities, state.masses, 300.0, seed=0)
        integ.run_device(5, 0.5, 1.0)
        torch.cuda.synchronize()
        md_steps = max(10, args.steps // 2)
        start.record()
        integ.run_device(md_steps, 0.5, 1.0)
        stop.record()
        torch.cuda.synchronize()
        integ.check_finite("in the MD bench")
        md_ms = start.elapsed_time(stop) / md_steps
        line["md"] = {"ms_per_step": round(md_ms, 4), "msteps_per_day": round(86.4 / md_ms, 3),
                      "ns_per_day_at_1fs": round(86.4 / md_ms, 3), "steps": md_steps,
                      "what": "neighbor search + TensorNet energy/forces + Langevin-middle integrator "
                              "(device Philox noise), one CUDA graph per step, float64 state"}
    if world == 1 and not args.no_sweep:
        line["neighbor_sweep"] = neighbor_sweep(torch, peak_gbs, with_cpu=not args.no_cpu)
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
