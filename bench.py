#!/usr/bin/env python
"""Bench: SSA firings/s of the bulk direct-method simulator on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A step is one cwc_simulate call over the whole workload: every trajectory of
the config simulated from t=0 to t_end with in-kernel sampling and the
two-stage exact moment reduction (SURVEY §8(a) rows a1-a11 except the
one-off model compile), inputs resident in HBM.  Default workload C2
(BASELINE.json configs[1], the config its metric names): Lotka-Volterra,
16384 replicas per GPU, t_end 10, 1001 samples, seed 1.  N GPUs: weak
scaling -- each rank runs its own 16384-replica shard of one N*16384-replica
run (distinct RNG streams) and the exact integer moments are merged with one
all-reduce per step.

`--impl reference` times the CPU oracle (oracle/, single-threaded, as it
stands) on a bounded sample of the same workload; rank 0 only.
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

import workloads as wl  # noqa: E402

METRIC = "SSA firings/sec on 1 B200 (replicas×firings); % of issue roofline"
STATS_MODES = {"auto": 0, "shared": 1, "global": 2}

# Algorithmic thread-level operations of one direct-method firing
# (SURVEY §8(d) "Algorithmic work per firing").
PHILOX_OPS = 60      # 10 rounds x (2 mul-hi/lo, 2 xor3, 2 key adds)
UNIFORM_OPS = 6      # two 53-bit conversions
LOG_OPS = 30         # fp64 log fast path
DIV_OPS = 10         # fp64 division (rcp + Newton + fix-up)
LOOP_OPS = 4         # t += tau, crossing compare, counters


def alg_ops_per_firing(M, avg_nu, avg_dep=None):
    """Thread path: full recompute (4 ops per propensity), M-1 adds, M
    compares; warp path: |D(mu)| recomputes, M-1 adds, M/2 compares."""
    base = PHILOX_OPS + UNIFORM_OPS + LOG_OPS + DIV_OPS + LOOP_OPS + 2 * avg_nu
    if avg_dep is None:
        return base + 4 * M + (M - 1) + M
    return base + 4 * avg_dep + (M - 1) + M / 2


def _rank_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index, interval_ms=100):
        self.dev = device_index
        self.interval_ms = int(interval_ms)
        self.proc = None
        self.path = os.path.join("/tmp", "cwc_clocks_%d_%s.csv" % (os.getpid(), device_index))

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "--query-gpu=" + self.Q, "--format=csv,noheader,nounits",
                                          "-lms", str(self.interval_ms), "-i", str(self.dev)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def _ncu_traffic(config, kernel_prefix):  # kernel_prefix: substring of the ncu kernel name
    """DRAM bytes per launch of the SSA kernel from the committed ncu capture of
    this config's bench launch (profiles/ncu_bench.json, written by
    tools/ncu_summary.py from an `ncu --set full` run of tools/run_case.py at
    the bench workload); None when absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_bench.json")) as f:
            d = json.load(f).get(config)
        if d and kernel_prefix in str(d.get("kernel", "")):
            return float(d["dram_bytes"])
    except Exception:
        pass
    return None


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_sample(desc, sweep, cfg, g_list):
    """Time the oracle (single thread, as it stands) on trajectories g_list."""
    import oracle
    oracle.build()
    t0 = time.perf_counter()
    r = oracle.simulate(desc, cfg["n_replicas"], cfg["t_end"], cfg["sample_dt"], cfg["seed"], sweep=sweep,
                        g_list=g_list, want_traj=False, want_stats=True)
    dt = time.perf_counter() - t0
    return int(r["firings"].sum()), dt


def _sample_size(name):
    # trajectories per ~10-15 s of single-core oracle work (BASELINE.md §4 rates)
    return {"C1": 1024, "C2": 384, "C3": 2048, "C4": 192, "C5": 12}[name]


def _oracle_worker(a):
    desc, sweep, cfg, g = a
    return oracle_sample(desc, sweep, cfg, g)


def oracle_all_cores(desc, sweep, cfg, G, name, seconds_per_core=8.0):
    """The oracle as it stands, one process per host core over disjoint
    strided trajectory sets (BASELINE.md §4 "all host cores" line): firings
    of all processes / wall time of the pool."""
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    per = max(1, int(_sample_size(name) * seconds_per_core / 12.0))
    n = min(G, per * cores)
    stride = max(1, G // n)
    gl = list(range(0, G, stride))[:n]
    chunks = [gl[i::cores] for i in range(cores) if gl[i::cores]]
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(len(chunks)) as pool:
        res = pool.map(_oracle_worker, [(desc, sweep, cfg, c) for c in chunks])
    dt = time.perf_counter() - t0
    f = sum(r[0] for r in res)
    return {"value": f / dt, "unit": "firings/s", "cores": len(chunks), "kind": "oracle",
            "sample": "%d of %d trajectories of %s (every %d-th g) over %d processes, full t_end; %.1f s wall"
            % (len(gl), G, name, stride, len(chunks), dt), "cpu": _cpu_model(), "host_cores": cores}


def run_reference(args):
    rank, world, _ = _rank_env()
    if rank != 0:
        return 0
    desc, sweep, cfg = wl.config(args.config)
    G = (len(sweep["values"]) if sweep else 1) * cfg["n_replicas"]
    per_step = max(1, _sample_size(args.config) // 6)
    stride = max(1, G // (per_step * (args.steps + args.warmup) + 1))
    steps = []
    for k in range(args.warmup + args.steps):
        g = [(k * per_step + i) * stride % G for i in range(per_step)]
        f, dt = oracle_sample(desc, sweep, cfg, g)
        if k >= args.warmup:
            steps.append((f, dt))
    F = sum(s[0] for s in steps)
    T = sum(s[1] for s in steps)
    value = F / T
    sample = "%d trajectories per step (stride %d over g) of %s, full t_end" % (per_step, stride, args.config)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "firings/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config_block(args.config, cfg, sweep, args.gpus, "cpu-oracle"),
            "cpu_baseline": {"value": value, "unit": "firings/s", "cores": 1, "kind": "oracle", "sample": sample,
                             "cpu": _cpu_model(), "host_cores": os.cpu_count()},
            "e2e": {"value": value, "unit": "firings/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _config_block(name, cfg, sweep, n_gpus, path):
    P = len(sweep["values"]) if sweep else 1
    return {"workload": "%s %s" % (name, wl.CONFIGS[name]["desc"]), "points": P,
            "replicas_per_point_per_gpu": cfg["n_replicas"], "t_end": cfg["t_end"], "sample_dt": cfg["sample_dt"],
            "samples": int(np.floor(cfg["t_end"] / cfg["sample_dt"])) + 1, "seed": cfg["seed"], "path": path,
            "parallelism": "dp%d (replica shards; exact int64 moment all-reduce)" % n_gpus,
            "l2": "flushed between timed steps (256 MiB write)"}


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(n):
    """`bench.py --gpus N` started without torchrun: re-exec this script
    under torch.distributed.run with N local ranks (one per GPU, rendezvous
    on 127.0.0.1), NCCL's communicator-init log on.  Returns the exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=%d" % n,
           "--master-addr=127.0.0.1", "--master-port=%d" % _free_port(), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


def comm_check(dist, device):
    """Every rank contributes 1 to an all-reduce: the communicator really
    spans WORLD_SIZE ranks."""
    import torch
    t = torch.ones(1, dtype=torch.int64, device=device)
    dist.all_reduce(t)
    return int(t.item()) == dist.get_world_size()


def selftest_dist(args):
    """CPU self-test of the launcher and the exchange step (gloo): every
    rank checks its RANK/LOCAL_RANK/WORLD_SIZE, contributes synthetic exact
    moments that depend on its rank (sumsq low words near 2^64 so the merge
    must carry) and merges them with paper_1010_2438_b200.dist.allreduce_stats;
    rank 0 prints one JSON line with what it saw."""
    import torch
    import torch.distributed as dist

    from paper_1010_2438_b200.dist import allreduce_stats
    rank, world, local = _rank_env()
    dist.init_process_group("gloo")
    ok_env = (world == args.gpus and 0 <= rank < world and local == rank)
    n = 6
    count = torch.full((n,), rank + 1, dtype=torch.int64)
    s1 = torch.arange(n, dtype=torch.int64) * (rank + 1)
    sq = torch.stack([torch.full((n,), -1 - rank, dtype=torch.int64), torch.full((n,), rank, dtype=torch.int64)], -1)
    allreduce_stats(count, s1, sq)
    W = world
    want_count = W * (W + 1) // 2
    lo = sum((2**64 - 1 - r) for r in range(W))
    want_lo, want_hi = lo % 2**64, lo // 2**64 + sum(range(W))
    merged_ok = (bool((count == want_count).all()) and bool((s1 == torch.arange(n) * want_count).all())
                 and int(sq[0, 0]) % 2**64 == want_lo and int(sq[0, 1]) == want_hi)
    ranks = torch.zeros(W, dtype=torch.int64)
    ranks[rank] = 1 if ok_env else 0
    dist.all_reduce(ranks)
    nranks_ok = comm_check(dist, "cpu")
    if rank == 0:
        print(json.dumps({"selftest": "dist", "world_size": W, "ranks_env_ok": int(ranks.sum()) == W,
                          "merge_exact": merged_ok, "comm_nranks_ok": nranks_ok}), flush=True)
    dist.destroy_process_group()
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1010_2438_b200 import cwc
    from paper_1010_2438_b200.dist import allreduce_stats

    rank, world, local = _rank_env()
    if world != args.gpus:
        raise SystemExit("bench.py: WORLD_SIZE=%d but --gpus %d" % (world, args.gpus))
    comm_ok = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm_ok = comm_check(dist, torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)

    desc, sweep, cfg = wl.config(args.config)
    model = cwc.cwc_model_create(desc)
    flat = model.get_flat()
    info = model.info
    M = info.n_reactions
    avg_nu = float(np.mean(np.diff(flat["nu_ptr"]))) if M else 0.0
    avg_dep = float(np.mean(np.diff(flat["dep_ptr"]))) if M else 0.0
    path = "warp" if info.path == cwc.CWC_PATH_WARP else "thread"
    R = cfg["n_replicas"]
    plan_opts = cwc.cwc_sim_opts()
    plan_opts.force_path = cwc.CWC_PATH_AUTO
    plan_opts.stats_mode = STATS_MODES[args.stats_mode]
    plan_opts.replica_offset = rank * R
    plan_opts.replicas_total = world * R
    plan = cwc.cwc_plan(model, R, sweep, cfg["t_end"], cfg["sample_dt"], plan_opts)
    kernel_name = cwc.KERNEL_NAMES[plan.kernel]  # the kernel the library's plan launches
    P = len(sweep["values"]) if sweep else 1
    J1 = int(np.floor(cfg["t_end"] / cfg["sample_dt"])) + 1
    O = info.n_obs
    ncell = P * J1 * O
    G = P * R

    count = torch.empty(ncell, dtype=torch.int64, device=dev)
    s1 = torch.empty(ncell, dtype=torch.int64, device=dev)
    sq = torch.empty((ncell, 2), dtype=torch.int64, device=dev)
    firings = torch.empty(G, dtype=torch.int64, device=dev)
    status = torch.empty(G, dtype=torch.int32, device=dev)
    ev_k0, ev_k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev_s0, ev_s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for ev in (ev_k0, ev_k1, ev_s0, ev_s1):
        ev.record(stream)
    opts = cwc.cwc_sim_opts()
    opts.force_path = cwc.CWC_PATH_AUTO
    opts.stats_mode = STATS_MODES[args.stats_mode]
    opts.ev_stage2_begin = ev_s0.cuda_event
    opts.ev_stage2_end = ev_s1.cuda_event
    traj = None
    if args.dump:  # trajectory dump mode: every sampled observable written to HBM (int64 [G][J+1][O])
        traj = torch.empty((G, J1, O), dtype=torch.int64, device=dev)
        opts.out_traj = traj.data_ptr()
    opts.out_firings = firings.data_ptr()
    opts.out_status = status.data_ptr()
    opts.replica_offset = rank * R
    opts.replicas_total = world * R
    opts.ev_kernel_begin = ev_k0.cuda_event
    opts.ev_kernel_end = ev_k1.cuda_event
    ws_bytes = cwc.cwc_simulate_workspace_size(model, R, sweep, cfg["t_end"], cfg["sample_dt"], opts)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    sweep_arrays = cwc._SweepArrays(sweep) if sweep is not None else None  # marshalled once, outside the timed steps

    def step():
        cwc.cwc_simulate(model, R, sweep, cfg["t_end"], cfg["sample_dt"], cfg["seed"], stream.cuda_stream,
                         (count, s1, sq), ws, opts, sweep_arrays=sweep_arrays)
        allreduce_stats(count, s1, sq)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    fired = int(firings.sum().item())          # identical every step (same seed, same shard)

    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kms, sms = [], []
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    clocks = ClockSampler(vis.split(",")[local] if vis else local, args.clock_ms)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if args.clock_ms > 0:
        clocks.start()
    for k in range(args.steps):
        flush.zero_()
        ev0[k].record(stream)
        step()
        ev1[k].record(stream)
        ev1[k].synchronize()
        kms.append(ev_k0.elapsed_time(ev_k1))
        sms.append(ev_s0.elapsed_time(ev_s1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    f = torch.tensor([fired], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(f, op=dist.ReduceOp.SUM)
    total_ms = float(t.item())
    fired_all = int(f.item())
    value = fired_all * args.steps / (total_ms / 1e3)

    # end-to-end through the public API with host buffers (H2D + D2H in the timed region)
    hc = torch.empty(ncell, dtype=torch.int64, pin_memory=True)
    hs = torch.empty(ncell, dtype=torch.int64, pin_memory=True)
    hq = torch.empty((ncell, 2), dtype=torch.int64, pin_memory=True)
    hws_bytes = cwc.cwc_simulate_host_workspace_size(model, R, sweep, cfg["t_end"], cfg["sample_dt"])
    hws = torch.empty(hws_bytes, dtype=torch.uint8, device=dev)
    sw_arrays = sweep_arrays
    e2e_ms = []
    for k in range(args.warmup + args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.zero_()
        a.record(stream)
        cwc.cwc_simulate_host(model, R, sweep, cfg["t_end"], cfg["sample_dt"], cfg["seed"], stream.cuda_stream,
                              (hc, hs, hq), hws, sweep_arrays=sw_arrays)
        b.record(stream)
        b.synchronize()
        if k >= args.warmup:
            e2e_ms.append(a.elapsed_time(b))
    e2e_total = sum(e2e_ms)
    te = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = fired_all * args.steps / (float(te.item()) / 1e3)

    # roofline of the dominant kernel (the SSA kernel), instruction issue bound
    props = torch.cuda.get_device_properties(dev)
    peaks = _peaks()
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    peak_ops = props.multi_processor_count * 4 * 32 * f_max
    ops = alg_ops_per_firing(M, avg_nu, avg_dep if path == "warp" else None)
    k_ms = float(np.mean(kms))
    achieved = ops * fired / (k_ms / 1e3)
    roofline = {"bound": "alu", "achieved": achieved / 1e12, "peak": peak_ops / 1e12, "unit": "Tops/s",
                "frac": achieved / peak_ops,
                "traffic": _ncu_traffic(args.config, kernel_name),
                "ops_per_firing": ops, "kernel": kernel_name, "kernel_ms": k_ms,
                "peak_source": "issue peak = %d SMs x 4 SMSP x 32 lanes x %.0f MHz (MEASURED_PEAKS sm_max_mhz)"
                % (props.multi_processor_count, f_max / 1e6)}

    # stage 2 (HBM-bound): algorithmic bytes = every accumulator part read
    # once + the output cells written once (count, sum: 8 B; sumsq: 16 B)
    s_ms = float(np.mean(sms))
    s_bytes = plan.n_parts * plan.part_cells * plan.word_bytes * plan.words_per_cell + 32 * ncell
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    stage2 = {"kernel": "stats_stage2_kernel", "ms": s_ms, "algorithmic_bytes": s_bytes,
              "gbs": s_bytes / (s_ms * 1e-3) / 1e9 if s_ms > 0 else None, "peak_gbs": hbm,
              "frac": (s_bytes / (s_ms * 1e-3) / 1e9) / hbm if s_ms > 0 else None,
              "parts": plan.n_parts, "shared_memory_parts": bool(plan.stats_shared)}
    line = {"metric": METRIC, "value": value, "unit": "firings/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(_config_block(args.config, cfg, sweep, world, path), kernel=kernel_name,
                           stats=("shared-memory parts" if plan.stats_shared else "one global part") +
                           " (--stats-mode %s)" % args.stats_mode, dump=bool(args.dump)),
            "firings_per_step": fired_all, "kernel_ms_per_step": k_ms,
            "roofline": roofline,
            "e2e": {"value": e2e_value, "unit": "firings/s", "h2d_bytes_per_step": 16 * P * max(M, 1) +
                    (4 * plan.blocks if (path == "thread" and P > 1) else 0),
                    "d2h_bytes_per_step": 32 * ncell},
            "stage2": stage2,
            "gpu_launches": 2 * args.steps, "clocks": clk}
    if args.dump:
        dump_bytes = G * J1 * O * 8
        line["dump"] = {"bytes_per_step": dump_bytes, "kernel_ms": k_ms,
                        "gbs": dump_bytes / (k_ms * 1e-3) / 1e9, "peak_gbs": hbm}
    if comm_ok is not None:
        line["comm"] = {"backend": "nccl", "world_size": world, "comm_nranks_ok": comm_ok,
                        "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n = _sample_size(args.config)
        g_list = list(range(0, G, max(1, G // n)))[:n]
        fo, dto = oracle_sample(desc, sweep, cfg, g_list)
        line["cpu_baseline"] = {"value": fo / dto, "unit": "firings/s", "cores": 1, "kind": "oracle",
                                "sample": "%d of %d trajectories of %s (every %d-th g), full t_end; %.1f s"
                                % (len(g_list), G, args.config, max(1, G // n), dto),
                                "cpu": _cpu_model(), "host_cores": os.cpu_count()}
        if not args.no_all_cores:
            line["cpu_baseline_all_cores"] = oracle_all_cores(desc, sweep, cfg, G, args.config)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def dyn_entries(model):
    """Match entries of the model's initial term (D1: per rule, contexts of its
    label, times children of the pattern's label): the size of the flat
    selection the direct method sums and searches per firing -- the
    algorithmic-work estimate of the C6 roofline (measurement only)."""
    comps = []  # (label, parent index)

    def walk(t, label, parent):
        me = len(comps)
        comps.append((label, parent))
        for c in t.get("comps", []):
            walk(c.get("content", {}), c["label"], me)
    walk(model["term"], 0, -1)
    E = 0
    for r in model["rules"]:
        ctx = [i for i, (lab, _) in enumerate(comps) if lab == r["label"]]
        if r.get("comp") is None:
            E += len(ctx)
        else:
            E += sum(1 for (lab, par) in comps if par in ctx and lab == r["comp"]["label"])
    return E


def run_dyn(args):
    """C6: the dynamic-topology path (include/cwc_dyn.h) on the cell-population
    workload of workloads/dynamic.py; same timing rules as run_ours.  The
    reference arm times the dynamic CPU oracle (oracle/dynamic.py)."""
    import workloads.dynamic as wd
    rank, world, local = _rank_env()
    cfg = dict(wd.CONFIG_C6)
    model_d = wd.cell_population_model()
    block = {"workload": "C6 %s" % cfg["desc"], "points": 1, "replicas_per_point_per_gpu": cfg["n_replicas"],
             "t_end": cfg["t_end"], "sample_dt": cfg["sample_dt"],
             "samples": int(np.floor(cfg["t_end"] / cfg["sample_dt"])) + 1, "seed": cfg["seed"], "path": "dynamic",
             "parallelism": "dp%d (replica shards)" % world, "l2": "flushed between timed steps (256 MiB write)"}

    def oracle_dyn(g_list):
        from oracle import dynamic as odyn
        t0 = time.perf_counter()
        r = odyn.simulate(model_d, 0, cfg["t_end"], cfg["sample_dt"], cfg["seed"], g_list=g_list)
        return int(r["firings"].sum()), time.perf_counter() - t0

    if args.impl == "reference":
        if rank != 0:
            return 0
        steps = []
        for k in range(args.warmup + args.steps):
            f, dt = oracle_dyn([k])
            if k >= args.warmup:
                steps.append((f, dt))
        F, T = sum(s[0] for s in steps), sum(s[1] for s in steps)
        sample = "1 trajectory per step of C6 (g = step index), full t_end"
        print(json.dumps({"impl": "reference", "metric": METRIC, "value": F / T, "unit": "firings/s",
                          "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True, "scaling": "weak",
                          "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": block,
                          "cpu_baseline": {"value": F / T, "unit": "firings/s", "cores": 1, "kind": "oracle",
                                           "sample": sample, "cpu": _cpu_model(), "host_cores": os.cpu_count()},
                          "e2e": {"value": F / T, "unit": "firings/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return 0

    import torch
    import torch.distributed as dist
    from paper_1010_2438_b200 import cwc_dyn
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    R = cfg["n_replicas"]
    m = cwc_dyn.cwc_dyn_model_create(model_d)
    ek0, ek1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ek0.record(stream)
    ek1.record(stream)
    kw = dict(replica_offset=rank * R, replicas_total=world * R, kernel_events=(ek0, ek1))
    buf = None
    for _ in range(args.warmup):
        buf = cwc_dyn.simulate(m, R, cfg["t_end"], cfg["sample_dt"], cfg["seed"], buffers=buf, **kw)["buffers"]
    torch.cuda.synchronize()
    fired = int(buf["firings"].sum().item())
    status = torch.bincount(buf["status"].long(), minlength=5).tolist()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kms = []
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    clocks = ClockSampler(vis.split(",")[local] if vis else local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for k in range(args.steps):
        flush.zero_()
        ev0[k].record(stream)
        cwc_dyn.simulate(m, R, cfg["t_end"], cfg["sample_dt"], cfg["seed"], buffers=buf, **kw)
        ev1[k].record(stream)
        ev1[k].synchronize()
        kms.append(ek0.elapsed_time(ek1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    total_ms = sum(a.elapsed_time(b) for a, b in zip(ev0, ev1))
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    f = torch.tensor([fired], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(f, op=dist.ReduceOp.SUM)
    total_ms, fired_all = float(t.item()), int(f.item())
    value = fired_all * args.steps / (total_ms / 1e3)
    # end to end: the call plus the moments copied to pinned host memory in the timed region
    n_cells = block["samples"] * len(model_d["observables"])
    hc = torch.empty(4 * n_cells, dtype=torch.int64, pin_memory=True)
    e2e_ms = []
    for k in range(args.warmup + args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.zero_()
        a.record(stream)
        r = cwc_dyn.simulate(m, R, cfg["t_end"], cfg["sample_dt"], cfg["seed"], buffers=buf, **kw)
        hc[:n_cells].copy_(r["count"].view(-1), non_blocking=True)
        hc[n_cells:2 * n_cells].copy_(r["sum"].view(-1), non_blocking=True)
        hc[2 * n_cells:].copy_(r["sumsq"].view(-1), non_blocking=True)
        b.record(stream)
        b.synchronize()
        if k >= args.warmup:
            e2e_ms.append(a.elapsed_time(b))
    te = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = fired_all * args.steps / (float(te.item()) / 1e3)
    props = torch.cuda.get_device_properties(dev)
    peaks = _peaks()
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    peak_ops = props.multi_processor_count * 4 * 32 * f_max
    E0 = dyn_entries(model_d)
    ops = PHILOX_OPS + UNIFORM_OPS + LOG_OPS + DIV_OPS + LOOP_OPS + (E0 - 1) + E0 / 2
    k_ms = float(np.mean(kms))
    achieved = ops * fired / (k_ms / 1e3)
    info = cwc_dyn.cwc_dyn_info_get(m, R, cfg["t_end"], cfg["sample_dt"])
    line = {"metric": METRIC, "value": value, "unit": "firings/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(block, kernel="dyn_ssa_kernel", capacity=info.capacity, grid=[info.blocks, info.threads],
                           smem_per_cta=info.smem_bytes),
            "firings_per_step": fired_all, "kernel_ms_per_step": k_ms, "status_counts": status,
            "roofline": {"bound": "alu", "achieved": achieved / 1e12, "peak": peak_ops / 1e12, "unit": "Tops/s",
                         "frac": achieved / peak_ops, "traffic": _ncu_traffic("C6", "dyn_ssa"), "ops_per_firing": ops,
                         "ops_model": "RNG + log + division + loop (%d) + a0 sum (E0 - 1) + search (E0 / 2) over the "
                                      "E0 = %d match entries of the initial term: a lower bound (re-evaluated "
                                      "entries not counted)" % (PHILOX_OPS + UNIFORM_OPS + LOG_OPS + DIV_OPS + LOOP_OPS, E0),
                         "kernel": "dyn_ssa_kernel", "kernel_ms": k_ms,
                         "peak_source": "issue peak = %d SMs x 4 SMSP x 32 lanes x %.0f MHz (MEASURED_PEAKS sm_max_mhz)"
                                        % (props.multi_processor_count, f_max / 1e6)},
            "e2e": {"value": e2e_value, "unit": "firings/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 32 * n_cells},
            "gpu_launches": 2 * args.steps, "clocks": clk}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        g_list = list(range(0, R, R // 16))[:16]
        fo, dto = oracle_dyn(g_list)
        line["cpu_baseline"] = {"value": fo / dto, "unit": "firings/s", "cores": 1, "kind": "oracle",
                                "sample": "%d of %d trajectories of C6 (every %d-th g), full t_end; %.1f s (oracle/"
                                          "dynamic.py, pure Python)" % (len(g_list), R, R // 16, dto),
                                "cpu": _cpu_model(), "host_cores": os.cpu_count()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(wl.CONFIGS) + ["C6"],
                    help="C1-C5: BASELINE.json configs; C6: the dynamic-topology workload (NEXT-4)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--stats-mode", default="auto", choices=sorted(STATS_MODES))
    ap.add_argument("--dump", action="store_true", help="also write every trajectory sample to HBM (dump mode)")
    ap.add_argument("--no-all-cores", action="store_true", help="skip the all-host-cores oracle line")
    ap.add_argument("--clock-ms", type=int, default=100, help="nvidia-smi sampling interval during the timed "
                    "region (0: off -- for the interference A/B only)")
    ap.add_argument("--selftest-dist", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.selftest_dist:
        return selftest_dist(args)
    if args.config == "C6":
        return run_dyn(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
