#!/usr/bin/env python
"""Benchmark of the multi-frequency H^2+ACA single-layer apply (arXiv 2006.05186).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

One step = one pass of the whole hot path over one
batch of synthetic time-domain data: cqm_forward (K4) -> [all-to-all when
N > 1] -> bem_apply_multifreq (gather, K1 near field, K2 up, K3 coupling,
K2 down, scatter) -> [all-to-all] -> cqm_inverse (K4).  Metric: unknowns x
frequencies per second, value = M * L / (device time per step), max over
ranks.  Inputs are device-resident; L2 is flushed (256 MB write) before every
timed step.  `e2e` repeats the step through the same public API from pinned
HOST buffers with the copies inside the timed region.  K1 and K3 leave out work that is below
the rounding of the result at the strongly damped frequencies (underflow
cutoffs; the metric's M * L still counts every unknown and frequency, the result matches the
oracle's full evaluation within the parity bar); `work` reports the executed fractions and
every roofline counts executed work only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "unknowns*frequencies/s of V(s_l)x_l apply (time-domain step: forward + apply + inverse)"
UNIT = "unknowns*frequencies/s"
FP64_PEAK_DERIVED = 148 * 64 * 2 * 1.965e9  # SMs x DFMA/clk/SM x 2 flop x max SM clock


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4,
                    help="BASELINE config (default 4: the largest single-GPU config, the N = 1 headline)")
    ap.add_argument("--skeleton", default="auto", choices=["auto", "z", "factors"],
                    help="MACA skeleton storage: stored Z, factors only (Z tiles regenerated in K3), or auto")
    ap.add_argument("--mode", default="h2aca", choices=["h2aca", "h2only", "combined"],
                    help="combined: Alg. 3 in full, near blocks MACA-compressed too (SURVEY NEXT-4)")
    ap.add_argument("--operator", default="V", choices=["V", "K"],
                    help="K: the double-layer operator (SURVEY NEXT-1) instead of the single layer")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of a CUDA-graph replay")
    ap.add_argument("--transpose", default="nccl", choices=["nccl", "peer", "a2a"],
                    help="N > 1: nccl = the library's bem_time_step_sharded (K4 fused with the packing, NCCL "
                         "grouped send/recv all-to-all inside libbem); peer = transforms fused with the transpose over "
                         "CUDA-IPC peer memory (cqm_forward_rows / cqm_inverse_rows); a2a = torch all_to_all_single")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: host-staged all-to-all (testing the multi-rank flow on one GPU only)")
    ap.add_argument("--shard-of", type=int, default=0,
                    help="virtual shard: on 1 GPU, time the frequency-domain apply of rank --shard-rank's frequency "
                         "classes of a G-GPU run (what one rank of `--gpus G` computes, without the all-to-alls)")
    ap.add_argument("--shard-rank", type=int, default=0)
    ap.add_argument("--quiet", action="store_true")
    ap.add_argument("--ranks-dry-run", action="store_true",
                    help="print each rank's (RANK, WORLD_SIZE) and exit (checks the --gpus N launch without a GPU)")
    return ap.parse_args()


def workload(cfg_id):
    cfg = synth.CONFIGS[cfg_id]
    V, T = synth.config_mesh(cfg_id)
    N = cfg["N"]
    return cfg, V, T, N, N + 1, 10.0 ** (-5.0 / N)


def config_json(cfg_id, cfg, M, L, G):
    return {"workload": f"config{cfg_id}: {cfg['mesh'][0]} sub{cfg['mesh'][1]}, M={M} panels, N={cfg['N']} (L={L}),"
                        f" m={cfg['m']} (p={cfg['m'] ** 3}), leaf={cfg['leaf']}, eta={cfg['eta']}, eps={cfg['eps']}",
            "M": M, "L": L, "T": cfg["T"], "seed": synth.SEED_BASE + cfg_id,
            "parallelism": f"frequency-sharded x{G}" if G > 1 else "1 GPU",
            "l2": "flushed (256 MB write) before every timed step"}


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(self.device)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=5)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def int8_peak_tops():
    """Dense INT8 tensor peak for a kernel timed inside a long step: the measured sustained bf16
    GEMM rate (MEASURED_PEAKS.json) x the nominal int8 / bf16 ratio 4.5 / 2.25 = 2."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return 2.0 * float(d.get("bf16_tflops_sustained") or d["bf16_tflops"]), "measured"
    except Exception:
        return 2.0 * 1400.0, "fallback"


def hbm_peak_gbs():
    """Measured copy bandwidth (MEASURED_PEAKS.json, driver-written), else the guide's fallback."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6550.0


def traffic_bytes(cfg_id, dom):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        return t.get(f"config{cfg_id}", {}).get(dom)
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------- the CPU oracle, timed
# The oracle (oracle/, plain FP64 C++, OpenMP) cannot run a whole config-4 step in
# minutes (its H2ACA apply evaluates every pivot slice once per chunk of 32
# frequencies: ~2.3e11 libm kernel evaluations for all 513 frequencies at config 4),
# so it is timed on a BOUNDED SAMPLE of the step and the step time is extrapolated
# from the sample (each part is linear in what is sampled):
#   * transforms: the naive-DFT forward and inverse of a fixed, seeded 1/SAMPLE_COLS of
#     the DOF columns (the work is per column: x SAMPLE_COLS);
#   * apply: one chunk of FCH = 32 frequencies per step (the oracle's own chunk; seeded,
#     different each step) with a fixed, seeded 1/SAMPLE_BLOCKS of the far blocks and of
#     the near blocks contributing (their ACA computed at setup): x SAMPLE_BLOCKS x L/32.
SAMPLE_COLS, SAMPLE_BLOCKS, FCH = 16, 64, 32


class OracleSample:
    def __init__(self, cfg_id, V, T, cfg, N):
        import oracle as O
        self.O = O
        self.N, self.L, self.M = N, N + 1, len(T)
        self.R = 10.0 ** (-5.0 / N)
        self.s = O.frequencies(N, cfg["T"])
        t0 = time.perf_counter()
        self.h = O.H2(V, T, cfg["leaf"], cfg["eta"], cfg["m"])
        rng = np.random.default_rng(20060518)
        nfs = max(1, self.h.n_far // SAMPLE_BLOCKS)
        nns = max(1, self.h.n_near // SAMPLE_BLOCKS)
        self.far = np.sort(rng.choice(self.h.n_far, nfs, replace=False)).astype(np.int32)
        self.near = np.sort(rng.choice(self.h.n_near, nns, replace=False)).astype(np.int32)
        self.cols = np.sort(rng.choice(self.M, max(1, self.M // SAMPLE_COLS), replace=False))
        self.h.aca(self.s, cfg["eps"], blocks=self.far)
        self.t_setup = time.perf_counter() - t0
        self.x_time = synth.random_time_data(cfg_id, N, self.M).astype(np.complex128)
        self.nf = min(FCH, self.L)
        self.cores = O.num_threads()
        self.fcols = self.M / len(self.cols)

    def step(self, k):
        """One sampled step; returns (seconds measured, seconds extrapolated to the whole step)."""
        O = self.O
        lsel = np.sort(np.random.default_rng(k).choice(self.L, self.nf, replace=False)).astype(np.int32)
        xs = np.ascontiguousarray(self.x_time[:, self.cols])
        xl = np.ascontiguousarray(self.x_time[lsel])  # stands in for the frequency-domain columns
        t0 = time.perf_counter()
        xf = O.forward(xs, self.N, self.R)
        t1 = time.perf_counter()
        self.h.apply_sample(self.s, xl, lsel, self.far, self.near)
        t2 = time.perf_counter()
        O.inverse(xf, self.N, self.R)
        t3 = time.perf_counter()
        t_dft, t_app = (t1 - t0) + (t3 - t2), t2 - t1
        return t3 - t0, self.fcols * t_dft + (self.h.n_far / len(self.far)) * (self.L / self.nf) * t_app

    def describe(self, steps):
        return (f"per step: naive-DFT forward + inverse of {len(self.cols)} of {self.M} DOF columns, and the H2ACA "
                f"apply of {self.nf} random frequencies of {self.L} with {len(self.far)} of {self.h.n_far} far and "
                f"{len(self.near)} of {self.h.n_near} near blocks contributing; step time extrapolated "
                f"x{self.fcols:.2f} (transforms) and x{self.h.n_far / len(self.far):.2f} x L/{self.nf} (apply); "
                f"{steps} step(s); oracle setup (tree + ACA of the sampled blocks) {self.t_setup:.1f} s excluded")


def cpu_baseline(cfg_id, V, T, cfg, N):
    """The oracle as it stands, timed on this box's host cores on a bounded sample."""
    o = OracleSample(cfg_id, V, T, cfg, N)
    _, t_step = o.step(0)
    return {"value": o.M * o.L / t_step, "unit": UNIT, "cores": o.cores, "kind": "oracle", "extrapolated": True,
            "ms_per_step_extrapolated": t_step * 1e3, "sample": o.describe(1)}


def run_reference(args):
    """--impl reference: the CPU oracle, as it stands, on this box's host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg, V, T, N, L, R = workload(args.config)
    M = len(T)
    o = OracleSample(args.config, V, T, cfg, N)
    for k in range(args.warmup):
        o.step(k)
    meas, ext = [], []
    for k in range(args.steps):
        a, b = o.step(args.warmup + k)
        meas.append(a)
        ext.append(b)
    t_step = float(np.mean(ext))
    val = M * L / t_step
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "extrapolated": True,
            "measured_ms_per_sampled_step": float(np.mean(meas)) * 1e3,
            "config": config_json(args.config, cfg, M, L, 1),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": o.cores, "kind": "oracle", "extrapolated": True,
                             "sample": o.describe(args.steps)},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def spawn_ranks(args):
    """--gpus N > 1 launched as a plain process: re-exec under torch.distributed.run (one rank
    per GPU, rendezvous on 127.0.0.1), the way the driver launches it."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    print(f"bench.py: spawning {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    world_env = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and world_env is None:
        spawn_ranks(args)
    if world_env is not None and int(world_env) != args.gpus and args.dist_backend == "nccl":
        raise SystemExit(f"bench.py: WORLD_SIZE={world_env} but --gpus {args.gpus}: launch one rank per GPU")
    if args.ranks_dry_run:
        print(json.dumps({"rank": int(os.environ.get("RANK", "0")), "world": int(world_env or 1)}), flush=True)
        return
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_2006_05186_b200 as pb
    from paper_2006_05186_b200.dist import ShardedTimeOperator, dof_ranges, shard_frequencies

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # one process per GPU; --dist-backend gloo (host-staged all-to-all) lets N ranks share
    # fewer GPUs to exercise the multi-rank flow where only one GPU is available
    local_rank = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_rank)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
    dev = torch.device("cuda", local_rank)
    cfg, V, T, N, L, R = workload(args.config)
    M = len(T)
    s = pb.cqm_frequencies(N, cfg["T"], R)
    mode = {"h2aca": pb.BEM_MODE_H2ACA, "h2only": pb.BEM_MODE_H2ONLY, "combined": pb.BEM_MODE_COMBINED}[args.mode]
    aca_far = mode in (pb.BEM_MODE_H2ACA, pb.BEM_MODE_COMBINED)
    base_mode = mode
    t0 = time.perf_counter()
    tree = pb.Tree(V, T, cfg["leaf"], cfg["eta"], cfg["m"], device=local_rank)
    t_tree = time.perf_counter() - t0
    vshard = args.shard_of > 1 and world == 1
    if world > 1:
        local = shard_frequencies(L, world)[rank]
    elif vshard:
        local = shard_frequencies(L, args.shard_of)[args.shard_rank]
    else:
        local = np.arange(L, dtype=np.int32)
    t0 = time.perf_counter()
    if aca_far:
        mode |= {"auto": 0, "z": pb.BEM_SKEL_Z, "factors": pb.BEM_SKEL_FACTORS}[args.skeleton]
    op = pb.Operator(tree, s, cfg["eps"], mode=mode, local_l=local if (world > 1 or vshard) else None)
    t_aca = time.perf_counter() - t0
    b, e = dof_ranges(M, world)[rank]
    if vshard:  # frequency-domain input of this shard
        xt_host = synth.random_density(args.config, len(local), M)
    else:
        xt_host = synth.random_time_data(args.config, N, M)[:, b:e].astype(np.complex128)
    x = torch.from_numpy(xt_host).to(dev)

    def fwd(z):
        return pb.cqm_forward(z, N, R)

    def inv(z):
        return pb.cqm_inverse(z, N, R)

    opfn = op.apply if args.operator == "V" else (lambda z: op.apply_dl(z))
    transpose = None
    lib_step = False
    if world > 1 and args.transpose == "nccl" and args.operator == "V" and args.dist_backend == "nccl":
        from paper_2006_05186_b200 import bem as B
        comm = B.Comm(rank, world, local_rank)
        transpose = ("libbem bem_time_step_sharded: K4 fused with the all-to-all packing, NCCL grouped send/recv "
                     "all-to-all inside the library, 2-D copies for the strided side")

        def step(z):
            return B.time_step_sharded(op, z, R, comm)
    elif world > 1:
        top = None
        if args.transpose == "peer" and args.operator == "V":
            try:
                from paper_2006_05186_b200.dist import PeerTimeOperator
                top = PeerTimeOperator(rank, world, M, L, op, R, local_rank)
                transpose = "fused transform + transpose over CUDA-IPC peer memory"
            except Exception as ex:  # no peer access: fall back to the collective
                top = None
                transpose = f"all_to_all_single (peer path unavailable: {ex!r})"
        if top is None:
            top = ShardedTimeOperator(rank, world, M, L, opfn, fwd, inv)
            transpose = transpose or f"all_to_all_single ({args.dist_backend})"
        step = top.step
    elif vshard:
        step = opfn
    else:
        def step(z):
            return inv(opfn(fwd(z)))
        # e2e: the library's one-call step on host buffers (bem_time_step: H2D, K4 forward,
        # apply, K4 inverse replayed from the CUDA graph the op captures at its first call, D2H)
        lib_step = args.operator == "V" and not args.no_graph

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(max(3, args.warmup)):
        step(x)
    torch.cuda.synchronize()
    op.set_profiling(True)
    acc = {"near": 0.0, "up": 0.0, "coupling": 0.0, "down": 0.0}

    def timed(run, profile):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush.zero_()  # L2 flush (256 MB write) outside the timed region of every step
            evs[k][0].record()
            run()
            evs[k][1].record()
            evs[k][1].synchronize()
            if profile:
                for key, v in op.timings().items():
                    acc[key] += v
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        return [a.elapsed_time(bb) for a, bb in evs]

    # (1) eager steps with the library's per-kernel CUDA-event timers (kernel breakdown, roofline);
    # on one GPU the two K4 transforms are bracketed by events of their own
    k4_ms = []
    if world == 1 and not vshard and args.operator == "V":
        def step_prof(z):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e[0].record()
            xf = fwd(z)
            e[1].record()
            yf = opfn(xf)
            e[2].record()
            y = inv(yf)
            e[3].record()
            k4_ms.append(e)
            return y
        ms_eager = timed(lambda: step_prof(x), True)
    else:
        ms_eager = timed(lambda: step(x), True)
    # work actually run under the underflow cutoffs (bem_op_get_work): the rooflines below count
    # executed work only (K1 evaluations counted on the device in the last profiled apply; K3
    # (rank x frequency column) products under the (block, tile) mask)
    wk = op.work()
    op.set_profiling(False)
    frac_near = (wk["near_evals_run"] / wk["near_evals_total"]
                 if wk["near_evals_run"] >= 0 and wk["near_evals_total"] > 0 else 1.0)
    frac_far = (wk["far_rank_cols_run"] / wk["far_rank_cols_total"] if wk["far_rank_cols_total"] > 0 else 1.0)
    # (2) headline: the same step captured once in a CUDA graph and replayed (removes the
    # host launch gaps of the ~25 small launches per step); 1 GPU only
    graph, graph_error = None, None
    if world == 1 and not args.no_graph:
        try:
            x_static = x.clone()
            s_cap = torch.cuda.Stream()
            s_cap.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s_cap):
                for _ in range(2):
                    step(x_static)
            torch.cuda.current_stream().wait_stream(s_cap)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                y_static = step(x_static)
            graph.replay()
            torch.cuda.synchronize()
        except Exception as ex:  # pragma: no cover
            graph = None
            graph_error = repr(ex)
    clk = ClockSampler(local_rank)
    clk.start()
    time.sleep(0.3)
    ms_steps = timed(graph.replay, False) if graph is not None else timed(lambda: step(x), False)
    clocks = clk.stop()
    red_dev = dev if args.dist_backend == "nccl" else torch.device("cpu")
    t_tot = torch.tensor([sum(ms_steps)], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t_tot, op=dist.ReduceOp.MAX)
    ms_per_step = float(t_tot.item()) / args.steps
    n_units = M * (len(local) if vshard else L)
    value = n_units / (ms_per_step * 1e-3)

    # e2e: same step through the public API from pinned host buffers
    e2e = None
    if not args.no_e2e:
        xh = torch.from_numpy(xt_host).pin_memory()
        yh = torch.empty_like(xh).pin_memory()
        eev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        if lib_step:
            for _ in range(2):  # the op captures its step graph at the first call: outside the timed region
                op.time_step(xh, R, y=yh)
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush.zero_()
            eev[k][0].record()
            if lib_step:  # host buffers straight into the library call (H2D + step + D2H inside)
                op.time_step(xh, R, y=yh)
            else:
                xd = xh.to(dev, non_blocking=True)
                yd = step(xd)
                yh.copy_(yd, non_blocking=True)
            eev[k][1].record()
            eev[k][1].synchronize()
        te = torch.tensor([sum(a.elapsed_time(bb) for a, bb in eev)], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ms_e2e = float(te.item()) / args.steps
        e2e = {"value": n_units / (ms_e2e * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(xh.numel() * 16),
               "d2h_bytes_per_step": int(yh.numel() * 16), "ms_per_step": ms_e2e,
               "call": ("bem_time_step(op, host x, host y, R) per step (pinned host buffers)" if lib_step else
                        "torch H2D copy, the step's C-ABI calls, torch D2H copy")}

    # roofline of the dominant kernel (algorithmic flops / live CUDA-event launch time)
    stats = tree.stats
    nl = len(local)
    n_class = len({min(l, L - l) for l in local})
    kt = {k: v / args.steps for k, v in acc.items()}
    launches = op.launch_count() + 2
    if aca_far:
        # 8 flops per complex MAC of a pivot slice; 4 for the real slice S_b(s_0) (complex x real)
        kpiv = op.aca_export()["pivots"][:, 0]
        flops_far = float(np.where(np.imag(s[kpiv]) == 0.0, 4.0, 8.0).sum()) * stats["p"] ** 2 * nl * frac_far
    else:  # plain H^2: one kernel evaluation per (block entry, frequency class) + the complex MACs
        flops_far = 75.0 * stats["far_blocks"] * stats["p"] ** 2 * n_class + 8.0 * stats["far_blocks"] * stats["p"] ** 2 * nl
    evals_near = 7.0 * stats["nnz_near"] * n_class * (frac_near if base_mode != pb.BEM_MODE_COMBINED else 1.0)
    flops_near = 75.0 * evals_near  # SURVEY §8(d) model: ~75 FP64 flops per complex exponential + MACs
    near_rank = None
    if base_mode == pb.BEM_MODE_COMBINED:  # K1m: 8 flops per (slice entry, term, frequency) on DMMA
        rkn = op.aca_export_near()["ranks"].astype(np.float64)
        ex = tree.export()
        sz = ex["clusters"][:, 1] - ex["clusters"][:, 0]
        nrnc = sz[ex["near"][:, 0]].astype(np.float64) * sz[ex["near"][:, 1]]
        flops_near = 8.0 * float((rkn * nrnc).sum()) * nl
        near_rank = float(rkn.mean())
    peaks = {}
    for m_, name in ((0, "dfma"), (1, "dmma")):
        try:
            peaks[name] = max(pb.fp64_peak(local_rank, mode=m_) for _ in range(2)) / 1e12
        except Exception:
            peaks[name] = None
    dom = "coupling" if kt["coupling"] >= kt["near"] else "near"
    far_kernel = op.info().get("far_kernel", 0) if aca_far else 0
    i8 = None
    if far_kernel == 10:  # far10: 4 real products per complex MAC (re/im embedding) x 21 byte-slice products
        cmacs = float(op.aca_export()["ranks"].astype(np.float64).sum()) * stats["p"] ** 2 * nl * frac_far
        i8_peak, i8_src = int8_peak_tops()
        i8 = {"ops": 2.0 * 84.0 * cmacs, "peak": i8_peak,
              "src": (f"{i8_src}: 2 x bf16_tflops_sustained (MEASURED_PEAKS.json; nominal int8/bf16 dense ratio "
                      "4.5/2.25); K3 runs inside a long step")}
    if dom == "near" and base_mode == pb.BEM_MODE_COMBINED:
        fl = flops_near
        peak = peaks["dmma"] or FP64_PEAK_DERIVED / 1e12
        bound, src = "tensor", "measured in this run: mma.sync.m8n8k4.f64 (DMMA) loop (bem_debug_fp64_peak_ex mode 1)"
    elif dom == "coupling" and not aca_far:
        fl = flops_far
        peak = FP64_PEAK_DERIVED / 1e12
        bound, src = "alu", ("derived: 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz (DESIGN.md §7); 75 flops/evaluation model"
                             + ("; flops count every (block, class), the K3' underflow cutoff is not counted: upper bound"
                                if wk["near_tau"] > 0 else ""))
    elif dom == "coupling" and i8 is not None:
        fl = i8["ops"]
        peak = i8["peak"]
        bound, src = "tensor", i8["src"]
    elif dom == "coupling":
        fl = flops_far
        peak = peaks["dmma"] or FP64_PEAK_DERIVED / 1e12
        bound, src = "tensor", ("measured in this run: mma.sync.m8n8k4.f64 (DMMA) loop on this GPU "
                                "(bem_debug_fp64_peak_ex mode 1); derived 148 SMs x 64 FMA/clk x 2 x 1.965 GHz = 37.2")
    else:
        fl = flops_near
        peak = FP64_PEAK_DERIVED / 1e12
        bound, src = "alu", "derived: 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz (DESIGN.md §7)"
    achieved = fl / (kt[dom] * 1e-3) / 1e12
    kname = {"coupling": (("K3 far10: complex FP64 products emulated on the INT8 tensor cores (tcgen05.mma kind::i8, "
                           "six-byte slices, 21 slice products; + seg_reduce)") if far_kernel == 10 else
                          "K3 far8 (p > 32, 3M DMMA) / far7 (p <= 32) coupling kernel (+seg_reduce)" if aca_far
                          else "K3' h2o_kernel (+seg_reduce)"),
             "near": "K1m nearm_kernel" if base_mode == pb.BEM_MODE_COMBINED else "K1 near_kernel"}[dom]
    roof = {"bound": bound, "kernel": kname, "achieved": achieved, "peak": peak,
            "unit": "TOP/s" if (dom == "coupling" and i8 is not None) else "TFLOP/s",
            "frac": achieved / peak, "traffic": traffic_bytes(args.config, dom), "peak_source": src,
            "algorithmic_flops_per_launch": fl,
            "traffic_source": "profiles/traffic.json (ncu --set full dram__bytes_read.sum + dram__bytes_write.sum "
                              "per launch of the same kernel and config)"}
    if dom == "coupling" and i8 is not None:
        # the same launch in the method's own arithmetic: 8 FP64 flops per complex MAC (4 for the real slice)
        fp64_eq = flops_far / (kt["coupling"] * 1e-3) / 1e12
        roof["algorithmic_int8_ops_per_launch"] = fl
        roof["fp64_equivalent"] = {"tflops": fp64_eq, "flops_per_launch": flops_far,
                                   "vs_fp64_tensor_peak": fp64_eq / (peaks["dmma"] or FP64_PEAK_DERIVED / 1e12)}
    # every kernel against its own roofline, and the whole apply
    # T_roof = sum_k max(F_k / P_FP64, B_k / BW) against the measured apply time
    hbm = hbm_peak_gbs()
    p_, C_ = stats["p"], stats["clusters"]
    m_ = round(p_ ** (1.0 / 3.0))
    b_up = 16.0 * M * nl + 16.0 * p_ * nl * C_
    b_down = 16.0 * p_ * nl * C_ + 32.0 * M * nl
    # leaf products W^T x / U yhat: one real x complex MAC (4 flops) per (panel, node, frequency);
    # Kronecker transfers: 3 m p real x complex MACs per (non-root cluster, frequency)
    f_up = 4.0 * p_ * M * nl + 12.0 * m_ * p_ * nl * (C_ - 1)
    pk_near = (peaks["dmma"] or FP64_PEAK_DERIVED / 1e12) if base_mode == pb.BEM_MODE_COMBINED else FP64_PEAK_DERIVED / 1e12
    pk_far = (peaks["dmma"] or FP64_PEAK_DERIVED / 1e12) if aca_far else FP64_PEAK_DERIVED / 1e12
    kern = {
        "near": {"flops": flops_near, "ms": kt["near"], "peak_tflops": pk_near},
        "coupling": ({"flops": i8["ops"], "ms": kt["coupling"], "peak_tflops": i8["peak"], "unit": "int8 ops"}
                     if i8 is not None else {"flops": flops_far, "ms": kt["coupling"], "peak_tflops": pk_far}),
        "up": {"flops": f_up, "bytes": b_up, "ms": kt["up"], "peak_tflops": FP64_PEAK_DERIVED / 1e12,
               "peak_gbs": hbm},
        "down": {"flops": f_up, "bytes": b_down, "ms": kt["down"], "peak_tflops": FP64_PEAK_DERIVED / 1e12,
                 "peak_gbs": hbm},
    }
    if not aca_far and wk["near_tau"] > 0:
        # plain H^2 (K3'): its underflow cutoff has no work counter, so these flops count every block and class
        kern["coupling"]["note"] = "flops count every (block, class); the K3' underflow cutoff is not counted: frac is an upper bound"
    if k4_ms:  # K4 forward + inverse: 32 M L bytes each (read + write of complex128 [L][M]), HBM-bound
        torch.cuda.synchronize()
        t_k4 = statistics.mean(e[0].elapsed_time(e[1]) + e[2].elapsed_time(e[3]) for e in k4_ms)
        kern["k4"] = {"flops": 0.0, "bytes": 2 * 32.0 * M * nl, "ms": t_k4, "peak_tflops": FP64_PEAK_DERIVED / 1e12,
                      "peak_gbs": hbm}
    t_roof = 0.0
    for k_, v_ in kern.items():
        t_f = v_["flops"] / (v_["peak_tflops"] * 1e12)
        t_b = v_.get("bytes", 0.0) / (v_.get("peak_gbs", hbm) * 1e9)
        v_["roof_ms"] = max(t_f, t_b) * 1e3
        v_["bound"] = "hbm" if t_b > t_f else ("tensor" if v_["peak_tflops"] != FP64_PEAK_DERIVED / 1e12 else "alu")
        v_["frac"] = v_["roof_ms"] / v_["ms"] if v_["ms"] > 0 else None
        if k_ != "k4":
            t_roof += v_["roof_ms"]
    t_apply = sum(kt.values())  # the apply's kernels (K4 reported separately)
    per_kernel = {"kernels": kern, "apply_roof_ms": t_roof, "apply_ms": t_apply,
                  "apply_frac": t_roof / t_apply if t_apply > 0 else None,
                  "model": "SURVEY §8(d): F, B per kernel (75 flops per K1 evaluation; K2 with Kronecker transfers: "
                           "4 p M L + 12 m p L (C-1) flops (4 per real x complex MAC) and minimum bytes), P = measured "
                           "DMMA / derived FP64 ALU peak, BW = MEASURED_PEAKS.json hbm_gbs"}
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": config_json(args.config, cfg, M, L, world), "roofline": roof, "e2e": e2e,
           "gpu_launches": launches * args.steps, "clocks": clocks,
           "kernel_ms": kt, "fp64_measured_tflops": peaks, "per_kernel_roofline": per_kernel,
           "timing": ("CUDA-graph replay of the whole step (captured once after warm-up); eager step "
                      f"{statistics.median(ms_eager):.3f} ms (median)") if graph is not None else
                     f"eager launches{'' if graph_error is None else ' (graph capture failed: ' + graph_error + ')'}",
           "near_evals_per_s": (evals_near / (kt["near"] * 1e-3) if kt["near"] > 0 and base_mode != pb.BEM_MODE_COMBINED
                                else None),
           "setup_s": {"tree": t_tree, "aca": t_aca}, "mode": args.mode, "operator": args.operator,
           "transpose": transpose,
           "mean_aca_rank": float(op.aca_export()["ranks"].mean()) if aca_far else None,
           "op": op.info(), "skeleton": op.skeleton(),
           "work": {"k1_evals_run_frac": frac_near, "k3_rank_cols_run_frac": frac_far, "near_tau": wk["near_tau"],
                    "far_delta": wk["far_delta"],
                    "note": "underflow cutoffs (include/bem.h bem_op_get_work): work left out is below the rounding "
                            "of the result; every roofline above counts executed work only"},
           "mean_near_aca_rank": near_rank}
    if vshard:
        out["config"]["parallelism"] = (f"virtual shard {args.shard_rank} of {args.shard_of}: frequency-domain apply of "
                                         f"{len(local)} of {L} frequencies on 1 GPU (no transforms, no all-to-all); "
                                         f"value = this rank's unknowns*frequencies/s")
        out["metric"] = METRIC.replace("time-domain step: forward + apply + inverse", "frequency-domain apply, one shard")
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not vshard:
        try:
            out["cpu_baseline"] = cpu_baseline(args.config, V, T, cfg, N)
        except Exception as ex:  # pragma: no cover
            out["cpu_baseline"] = {"value": None, "error": str(ex)}
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
