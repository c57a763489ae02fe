#!/usr/bin/env python
"""Benchmark: seconds to S_eps for 1M vs 1M 3D points (BASELINE.json metric,
configs[2] = C3), one JSON line on rank 0.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one process per GPU)

A step is one full multiscale Sinkhorn divergence S_eps (clustering, coarse
phase, extrapolation, block-sparse fine phase with per-scale truncation,
loss) on N=M=1e6 Gaussian-mixture points (SURVEY.md §8d C3 generator, seeds
5/6), blur=0.01, reach=inf, q=0.9.  `value` = device time of one solve with
the inputs resident in HBM (max over ranks, CUDA events on the solver's
stream); `e2e` = the same solve through the public host-buffer C ABI call
(msot_sinkhorn) with pinned inputs: H2D copy + solve + loss D2H.
--impl reference times the FP64 CPU oracle (the reference's Sinkhorn is
specified only in prose) on a bounded sample and
extrapolates to the workload's evaluated-pair count.

Besides the C3 line it reports `extra_configs` (BASELINE.json configs 0, 1,
3, 4 on this GPU) and `cpu_baseline` with the oracle timed in full on C1 and
C2 (a few minutes on the host).  --no-extras / --no-cpu skip them.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOAD = dict(workload="C3: S_eps 1M vs 1M 3D Gaussian mixtures (8 comps, sigma 0.05), "
                         "multiscale voxel grid + per-scale kernel truncation",
                n=1_000_000, m=1_000_000, d=3, blur=0.01, reach="inf", scaling=0.9, theta=12.5,
                retruncate=1, switch_factor=1.0, cluster_scale="auto (28 atoms/occupied voxel)",
                theta_note="12.5 = GeomLoss truncate=5 (exp(-C/eps) > e^-12.5); S within 3e-12 of theta 20 (profiles/r1_theta_sweep.jsonl)",
                seeds=[5, 6])
METRIC = "sec to S_eps, 1M vs 1M 3D pts at 1/2/4/8 GPU; softmin pairs/sec vs roofline"
PAIRS_FILE = os.path.join(ROOT, "profiles", "c3_workload.json")


def mixture(n, seed, d=3, k=8, sigma=0.05):
    rng = np.random.default_rng(seed)
    cen = rng.uniform(0.2, 0.8, (k, d))
    return cen[rng.integers(0, k, n)] + rng.normal(0, sigma, (n, d))


def make_inputs(w):
    x = mixture(w["n"], w["seeds"][0], w["d"])
    y = mixture(w["m"], w["seeds"][1], w["d"])
    a = np.full(w["n"], 1.0 / w["n"])
    b = np.full(w["m"], 1.0 / w["m"])
    return x, a, y, b


def params(w):
    from paper_2107_02010_b200.abi import make_params
    return make_params(blur=w["blur"], reach=math.inf, scaling=w["scaling"], multiscale=True,
                       retruncate=w["retruncate"], theta=w["theta"],
                       switch_factor=w["switch_factor"])


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu, self.rows, self._stop = gpu, [], threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 3 + k and r[3 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm)}


def dense_rel(loss, w):
    """Relative difference to the dense (all-pairs) eps-scaling solve of the
    same inputs, measured once on the GPU (tools/dense_ref.py ->
    profiles/r1_c3_dense_vs_multiscale.json): the multiscale approximation
    error, SPEC.md:303 asks < 1e-3."""
    p = os.path.join(ROOT, "profiles", "r1_c3_dense_vs_multiscale.json")
    if w["n"] != WORKLOAD["n"] or not os.path.exists(p):
        return None
    return loss / json.load(open(p))["dense_S_eps"] - 1.0


def l2_flush(buf):
    if buf is not None:
        buf.add_(1.0)


def free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(n, argv):
    """`bench.py --gpus N` run without torchrun: one process per GPU, launched
    here with the torchrun environment (RANK, LOCAL_RANK, WORLD_SIZE,
    MASTER_ADDR=127.0.0.1, MASTER_PORT); rank 0's stdout is passed through
    (the JSON line), the others' is discarded.  Returns the worst exit code."""
    port = free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + argv, env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    rcs = [p.wait() for p in procs]
    return max(rcs, key=abs)


def dist_probe(args):
    """--dist-probe (dev/test): the rendezvous, the max-over-ranks timing
    reduction and the rank-0-only JSON line of a self-spawned run, on gloo
    (no GPU): each rank 'times' rank+1 ms, rank 0 prints the max."""
    import torch
    import torch.distributed as dist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"n_gpus": world, "ms_per_step": float(t[0]),
                          "ranks_seen": dist.get_world_size()}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def run_extras(ctx):
    """The other BASELINE.json configurations on this GPU (one timed run each
    after a warm-up; device time from the solver's CUDA events):
      C1 configs[0]  10k vs 10k uniform, blur 0.05, dense
      C2 configs[1]  100k vs 100k mixtures (seeds 3/4), bench params (multiscale)
      C4 configs[3]  200k vs 200k fibres (D = 60) flip-augmented to 400k vs 400k,
                     reach 0.3, blur 0.03, K-means multiscale + label transfer
      C5 configs[4]  barycenter of 10 synthetic 128^3 track-density maps,
                     x6 upsampled init, blur = 1 voxel: seconds per descent step
    C1 and C2 also report the FP64 oracle's committed result for the same
    inputs (tests/golden/config_golden.json, tests/test_config_parity.py)."""
    from paper_2107_02010_b200 import workloads as W
    from paper_2107_02010_b200.abi import make_params
    from paper_2107_02010_b200.solver import classify, resolve_flips
    gold_p = os.path.join(ROOT, "tests", "golden", "config_golden.json")
    gold = json.load(open(gold_p)) if os.path.exists(gold_p) else {}
    out = {}
    # C1
    x1 = np.random.default_rng(1).random((10000, 3))
    y1 = np.random.default_rng(2).random((10000, 3))
    w1 = np.full(10000, 1e-4)
    for _ in range(2):
        l1, _, s1 = ctx.sinkhorn(make_params(blur=0.05), x1, w1, y1, w1, potentials=False)
    out["C1"] = {"config": "10k vs 10k uniform 3D, blur 0.05, dense eps-scaling",
                 "device_ms": s1["total_ms"], "S_eps": l1,
                 "oracle_S_eps": gold.get("c1", {}).get("loss")}
    # C2
    wc2 = dict(WORKLOAD, n=100000, m=100000)
    x2, y2 = mixture(100000, 3), mixture(100000, 4)
    a2 = np.full(100000, 1e-5)
    for _ in range(3):
        l2, _, s2 = ctx.sinkhorn(params(wc2), x2, a2, y2, a2, potentials=False)
    out["C2"] = {"config": "100k vs 100k 3D mixtures (seeds 3/4), multiscale, bench params",
                 "device_ms": s2["total_ms"], "S_eps": l2, "kx": s2["kx"], "t_switch": s2["t_switch"],
                 "oracle_S_eps": gold.get("c2", {}).get("loss")}
    # C4
    t = time.perf_counter()
    fa, la = W.fibres(200000, 7, bundles=50, bundle_seed=1)
    fb, lb = W.fibres(200000, 8, bundles=50, bundle_seed=1)
    x4, a4 = W.flip_augment(*W.encode_fibers(fa))
    y4, b4 = W.flip_augment(*W.encode_fibers(fb))
    lab = np.concatenate([lb, lb]).astype(np.int32)
    prep = time.perf_counter() - t
    prm4 = make_params(blur=0.03, reach=0.3, multiscale=True, retruncate=1, switch_factor=2.0,
                       theta=12.5)
    for _ in range(2):
        t = time.perf_counter()
        soft, l4, s4 = ctx.transfer_labels(prm4, x4, a4, y4, b4, lab, 50)
        wall4 = time.perf_counter() - t
    res, _ = resolve_flips(soft, np.tile(np.arange(200000), 2), np.repeat([0, 1], 200000))
    hard, _ = classify(res, 0.5)
    inl = hard >= 0
    out["C4"] = {"config": "200k vs 200k fibres (D=60, flip-augmented 400k vs 400k), reach 0.3, "
                           "blur 0.03, K-means multiscale + label transfer",
                 "device_ms": s4["total_ms"], "wall_s": wall4, "prep_s": prep, "S_eps": l4,
                 "kx": s4["kx"], "t_switch": s4["t_switch"],
                 "label_accuracy": float((hard[inl] == la[inl]).mean()) if inl.any() else None,
                 "inlier_fraction": float(inl.mean())}
    # C5
    t = time.perf_counter()
    maps = W.density_maps(10)
    targets = [W.density_to_measure(*m) for m in maps]
    p5, w5 = W.density_to_measure(*W.average_density(maps))
    x5, a5 = W.upsample(p5, w5, 6, 0.5 / 128, 0)
    prep5 = time.perf_counter() - t
    prm5 = make_params(blur=1 / 128, multiscale=True, retruncate=1, switch_factor=1.0)
    ctx.barycenter(prm5, x5, a5, targets, iters=1, step=1.0, tol=0.0)  # warm-up
    t = time.perf_counter()
    xb, traj, s5 = ctx.barycenter(prm5, x5, a5, targets, iters=3, step=1.0, tol=0.0)
    dt5 = time.perf_counter() - t
    steps5 = max(1, len(traj) - 1)
    out["C5"] = {"config": "barycenter of 10 synthetic 128^3 track-density maps, x6 upsampled "
                           "init, blur = 1 voxel, multiscale",
                 "atoms": len(x5), "target_atoms_mean": float(np.mean([len(b) for _, b in targets])),
                 "seconds_per_iteration": dt5 / steps5, "device_ms_per_iteration":
                     s5["total_ms"] / steps5, "iterations": steps5, "prep_s": prep5,
                 "loss_trajectory": [float(v) for v in traj]}
    return out


def cpu_baseline(st, extras):
    """The FP64 oracle (oracle/, the CPU restatement on the reference's own
    thread pool and summation, kind "port") timed in full on C1 and C2 of
    BASELINE.json on this host; the C3 figure is the measured C2 block-sparse
    multiscale solve's rate (oracle LSE terms per second) applied to the C3
    solve's term count — a C3 oracle run would take ~45 min."""
    from oracle import oracle as O  # CPU baseline only
    from paper_2107_02010_b200.abi import make_params
    cores = O.threads()
    x1 = np.random.default_rng(1).random((10000, 3))
    y1 = np.random.default_rng(2).random((10000, 3))
    w1 = np.full(10000, 1e-4)
    t = time.perf_counter()
    l1, _, o1 = O.sinkhorn(make_params(blur=0.05), x1, w1, y1, w1, potentials=False)
    c1_s = time.perf_counter() - t
    wc2 = dict(WORKLOAD, n=100000, m=100000)
    x2, y2 = mixture(100000, 3), mixture(100000, 4)
    a2 = np.full(100000, 1e-5)
    t = time.perf_counter()
    l2, _, o2 = O.sinkhorn(params(wc2), x2, a2, y2, a2, potentials=False)
    c2_s = time.perf_counter() - t
    rate = o2["pairs_evaluated"] / c2_s  # LSE terms / s of the block-sparse multiscale solve
    out = {"value": st["pairs_terms"] / rate, "unit": "s (C3 extrapolated from the measured C2 "
                                                      "multiscale oracle solve)",
           "cores": cores, "kind": "port",
           "sample": f"FP64 oracle full solves on {cores} threads: C1 {c1_s:.1f} s, C2 {c2_s:.1f} s "
                     f"({o2['pairs_evaluated']:.3e} LSE terms, {rate:.3e}/s); C3 = "
                     f"{st['pairs_terms']:.3e} terms / that rate",
           "C1_seconds": c1_s, "C1_S_eps": l1, "C2_seconds": c2_s, "C2_S_eps": l2,
           "C2_terms_per_s": rate}
    if extras:
        out["C1_speedup_device"] = c1_s / (extras["C1"]["device_ms"] * 1e-3)
        out["C2_speedup_device"] = c2_s / (extras["C2"]["device_ms"] * 1e-3)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=None, help="override N=M (dev only)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-extras", action="store_true", help="skip the C1/C2/C4/C5 extra configs")
    ap.add_argument("--host-collectives", action="store_true",
                    help="dev only: every rank on cuda:0, exchanges through gloo via "
                         "msot_create_dist_host (exercises the N>1 path on one GPU)")
    ap.add_argument("--dist-probe", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--ref-n", type=int, default=None, help=argparse.SUPPRESS)  # tests: smaller C2
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU without torchrun (the driver may launch either way)
        sys.exit(spawn_ranks(args.gpus, sys.argv[1:]))
    if args.dist_probe:
        return dist_probe(args)

    w = dict(WORKLOAD)
    if args.n:
        w["n"] = w["m"] = args.n
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, w, rank)

    import torch
    import torch.distributed as dist
    from paper_2107_02010_b200.solver import Context

    if args.host_collectives:
        local = 0
    torch.cuda.set_device(local)
    if world > 1 and args.host_collectives:
        dist.init_process_group("gloo")

        def _ar(arr):
            dist.all_reduce(torch.from_numpy(arr))

        def _bc(arr, root):
            dist.broadcast(torch.from_numpy(arr), src=root)

        ctx = Context(0, rank, world, host_collectives=(_ar, _bc))
    elif world > 1:
        dist.init_process_group("gloo")
        idbuf = [Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(idbuf, src=0)
        ctx = Context(local, rank, world, idbuf[0])
    else:
        ctx = Context(local)
    r_, w_, nr_ = ctx.world_info()
    print(f"[msot] rank {r_}/{w_}: device {local}, communicator nranks {nr_} "
          f"({'host-staged gloo' if args.host_collectives else 'ncclCommCount'})",
          file=sys.stderr, flush=True)
    if w_ != world or nr_ != world:
        raise RuntimeError(f"communicator has {nr_} ranks, expected {world}")

    x, a, y, b = make_inputs(w)
    prm = params(w)
    dev = torch.device("cuda", local)
    tx = torch.from_numpy(x).to(dev)
    ta = torch.from_numpy(a).to(dev)
    ty = torch.from_numpy(y).to(dev)
    tb = torch.from_numpy(b).to(dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def solve():
        return ctx.sinkhorn_device(prm, tx.data_ptr(), ta.data_ptr(), w["n"], ty.data_ptr(),
                                   tb.data_ptr(), w["m"], w["d"])

    for _ in range(max(args.warmup, 0)):
        solve()
    times, launches, loss, st = [], 0, None, None
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            l2_flush(flush)
            barrier()
            loss, st = solve()
            barrier()
            times.append(st["total_ms"])
            launches += st["gpu_launches"]
    t_local = torch.tensor(times, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms = float(t_local.mean())

    # e2e: public host-buffer call with pinned inputs, H2D + solve + loss D2H
    px = torch.from_numpy(x).pin_memory()
    pa = torch.from_numpy(a).pin_memory()
    py = torch.from_numpy(y).pin_memory()
    pb = torch.from_numpy(b).pin_memory()
    import ctypes as C
    from paper_2107_02010_b200.abi import Stats
    from paper_2107_02010_b200.solver import lib
    dp = lambda t: C.cast(t.data_ptr(), C.POINTER(C.c_double))
    e2e_t = []
    for k in range(max(2, args.steps)):
        l2_flush(flush)
        barrier()
        t0 = time.perf_counter()
        lossv = C.c_double()
        sst = Stats()
        rc = lib().msot_sinkhorn(ctx._h, C.byref(prm), dp(px), dp(pa), w["n"], dp(py), dp(pb),
                                 w["m"], w["d"], None, None, None, None, C.byref(lossv),
                                 C.byref(sst))
        barrier()
        if rc != 0:
            raise RuntimeError(lib().msot_last_error().decode())
        e2e_t.append(time.perf_counter() - t0)
    e2e_local = torch.tensor(e2e_t, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(e2e_local, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_local[1:].mean()) if len(e2e_t) > 1 else float(e2e_local[0])

    # roofline of the dominant kernel: softmin launches timed with events
    # roofline: each softmin launch timed alone with CUDA events.  The timed
    # steps run the column partials in bounded batches overlapped on two
    # streams; profiling serialises launches, so the kernel is
    # measured on one batch per update (budget unbounded): same kernel, same
    # items, no inter-batch tails.
    ctx.set_colpart_budget(1 << 40)
    ctx.set_profiling(True)
    _, pst = solve()
    ctx.set_colpart_budget(0)
    # north star's dense-softmin bar (>= 60% of the MUFU roofline on one GPU):
    # the C1 configuration (10k vs 10k uniform 3D, blur 0.05, dense), solved
    # on the same context with its softmin launches event-timed
    dense = None
    if world == 1:
        rng1, rng2 = np.random.default_rng(1), np.random.default_rng(2)
        xc, yc = rng1.random((10000, 3)), rng2.random((10000, 3))
        wc = np.full(10000, 1e-4)
        from paper_2107_02010_b200.abi import make_params
        for _ in range(2):
            _, _, dst = ctx.sinkhorn(make_params(blur=0.05), xc, wc, yc, wc, potentials=False)
        dense = dst
    ctx.set_profiling(False)
    ex2_rate = ctx.probe_ex2()
    extras = run_extras(ctx) if (world == 1 and not args.no_extras and rank == 0) else None

    if rank != 0:
        if world > 1:
            dist.barrier()
        ctx.close()
        return
    achieved = pst["pairs_evaluated"] / world / (pst["softmin_ms"] * 1e-3)
    nominal = 148 * 16 * 1965e6
    traffic = None
    prof = os.path.join(ROOT, "profiles", "softmin_ncu.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC,
        "value": ms * 1e-3,
        "unit": "s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32 (f64 loss, f64 inputs)",
        "data": "synthetic (seeded Gaussian mixtures)",
        "config": {**{k: v for k, v in w.items()}, "parallelism": f"rows sharded x{world}",
                   "l2": "256 MB buffer written between timed steps",
                   # the reference arm prints the same workload keys; the values
                   # this run resolved (voxel edge, switch scale) sit beside them
                   "resolved": {"cluster_scale": st["cluster_scale"], "t_switch": st["t_switch"],
                                "n_scales": st["n_scales"], "kx": st["kx"], "ky": st["ky"]}},
        "S_eps": loss,
        "S_eps_dense_rel_diff": dense_rel(loss, w),
        "pairs_evaluated": st["pairs_evaluated"],
        "pairs_terms": st["pairs_terms"],
        "pairs_dense_equiv": st["pairs_dense"],
        "fine_kept_fraction": st["pairs_fine"] / max(st["pairs_fine_dense"], 1.0),
        "pairs_per_s": st["pairs_evaluated"] / (ms * 1e-3),
        "gpu_launches": launches,
        "e2e": {"value": e2e_s, "unit": "s",
                "h2d_bytes_per_step": (w["n"] + w["m"]) * (w["d"] + 1) * 8,
                "d2h_bytes_per_step": 8},
        "roofline": {"bound": "mufu", "achieved": achieved, "peak": ex2_rate,
                     "unit": "pairs/s (1 MUFU.EX2 per pair)", "frac": achieved / ex2_rate,
                     "peak_source": "measured on this GPU by msot_probe_ex2 "
                                    "(ex2.approx.ftz.f32 issue rate, all SMs)",
                     "peak_nominal": nominal, "frac_of_nominal": achieved / nominal,
                     "traffic": traffic, "kernel": "softmin_sym_kernel<3> (evaluate-once: fine phase, cluster and super-voxel coarse phases)",
                     "softmin_ms": pst["softmin_ms"], "softmin_launches": pst["softmin_launches"],
                     "share_of_step": pst["softmin_ms"] / max(pst["total_ms"], 1e-9)},
        "clocks": clk.summary(),
        "fallback_rows": st["fallback_rows"],
        "dense_softmin_c1": None if dense is None else {
            "config": "C1: 10k vs 10k uniform 3D, blur 0.05, dense eps-scaling (row-wise softmin_kernel)",
            "pairs_per_s": dense["pairs_evaluated"] / (dense["softmin_ms"] * 1e-3),
            "frac_of_mufu_peak": dense["pairs_evaluated"] / (dense["softmin_ms"] * 1e-3) / ex2_rate,
            "solve_ms": dense["total_ms"]},
    }
    if extras is not None:
        line["extra_configs"] = extras
    if not args.no_cpu and world == 1:  # the CPU baseline runs on rank 0 at N = 1 only
        line["cpu_baseline"] = cpu_baseline(st, extras)
    os.makedirs(os.path.dirname(PAIRS_FILE), exist_ok=True)
    if w["n"] == WORKLOAD["n"] and world == 1:
        with open(PAIRS_FILE, "w") as f:
            json.dump({"pairs_evaluated": st["pairs_evaluated"], "pairs_terms": st["pairs_terms"],
                       "n_scales": st["n_scales"],
                       "t_switch": st["t_switch"], "kx": st["kx"]}, f, indent=1)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
    ctx.close()


def run_reference(args, w, rank):
    """--impl reference: the CPU oracle (FP64 restatement of PAPER.md:235-326
    on the reference's own thread pool and summation, oracle/_ref; the
    reference's Sinkhorn exists only as prose) on this host.
    The bounded sample is one full multiscale solve of BASELINE configs[1]
    (C2: 100k vs 100k, the C3 generator and parameters at 1/10 the size, ~2
    min on 16 threads), run once whatever --steps says; its measured rate
    (LSE terms per second, clustering and masks included) is applied to the
    C3 solve's term count (profiles/c3_workload.json, written by the GPU arm)."""
    if rank != 0:
        return
    from oracle import oracle as O  # the reference arm times the oracle
    pairs = None
    if os.path.exists(PAIRS_FILE):
        pf = json.load(open(PAIRS_FILE))
        pairs = pf.get("pairs_terms") or pf.get("pairs_evaluated")
    n2 = args.ref_n or 100000
    wc2 = dict(w, n=n2, m=n2)
    x2, y2 = mixture(n2, 3), mixture(n2, 4)
    a2 = np.full(n2, 1.0 / n2)
    t = time.perf_counter()
    l2, _, o2 = O.sinkhorn(params(wc2), x2, a2, y2, a2, potentials=False)
    dt = time.perf_counter() - t
    rate = o2["pairs_evaluated"] / dt
    cores = O.threads()
    if pairs is None:
        pairs = float(w["n"]) * w["m"] * 4 * 50  # dense-equivalent upper bound
    sec = pairs / rate
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": sec, "unit": "s",
        "n_gpus": 0, "steps": 1, "steps_requested": args.steps, "warmup": 0,
        "higher_is_better": False,
        "dtype": "f64", "data": "synthetic (seeded Gaussian mixtures)",
        "config": {**w, "parallelism": f"{cores} CPU threads"},
        "cpu_baseline": {"value": sec, "unit": "s (extrapolated)", "cores": cores, "kind": "port",
                         "sample": f"FP64 oracle full multiscale solve of C2 ({n2} vs {n2}, bench "
                                   f"params): {dt:.1f} s, {o2['pairs_evaluated']:.3e} LSE terms, "
                                   f"{rate:.3e}/s; C3 = {pairs:.3e} terms (profiles/c3_workload.json) "
                                   f"/ that rate",
                         "C2_seconds": dt, "C2_S_eps": l2},
        "e2e": {"value": sec, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


if __name__ == "__main__":
    main()
