"""Thin ctypes binding of include/cwc.h (argument marshalling only).

Every step of the simulation runs in libcwcsim.so (sm_100a kernels).  There
is no CPU fallback: if the library or a CUDA device is missing the calls
raise.  PyTorch is used only to own device memory and to name the stream.

The functions keep the C names (cwc_model_create, cwc_simulate, ...); the
`Model` / `simulate` helpers below only allocate the torch tensors those
calls write into.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcwcsim.so")

CWC_OK, CWC_ERR_INVALID, CWC_ERR_UNSUPPORTED, CWC_ERR_CUDA, CWC_ERR_NOMEM = 0, -1, -2, -3, -4
CWC_TRAJ_DONE, CWC_TRAJ_STALLED, CWC_TRAJ_OVERFLOW, CWC_TRAJ_RUNNING = 0, 1, 2, 3
CWC_PATH_AUTO, CWC_PATH_THREAD, CWC_PATH_WARP = -1, 0, 1
CWC_KERNEL_AUTO, CWC_KERNEL_THREAD_WS, CWC_KERNEL_THREAD, CWC_KERNEL_WARP2, CWC_KERNEL_WARP, CWC_KERNEL_THREAD2, \
    CWC_KERNEL_THREAD_WS2, CWC_KERNEL_WARP8, CWC_KERNEL_WARP4 = 0, 1, 2, 3, 4, 5, 6, 7, 8
CWC_STATS_AUTO, CWC_STATS_SHARED, CWC_STATS_GLOBAL = 0, 1, 2

EXPORTED = ["cwc_plan", "cwc_model_create", "cwc_model_destroy", "cwc_model_info_get", "cwc_model_get_flat",
            "cwc_simulate_workspace_size", "cwc_simulate", "cwc_simulate_host", "cwc_simulate_host_workspace_size",
            "cwc_stats_finalize", "cwc_philox_blocks", "cwc_draws", "cwc_block_draws", "cwc_tau_div", "cwc_run_state_size",
            "cwc_run_init", "cwc_run_advance", "cwc_run_stats", "cwc_last_error"]

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64


class CwcError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("cwc status %d: %s" % (status, msg))
        self.status = status


class cwc_model_desc(ctypes.Structure):
    _fields_ = [("n_types", I32), ("n_species", I32), ("n_compartments", I32), ("parent", P), ("type", P),
                ("n_rules", I32), ("rule_label", P), ("rule_child_label", P),
                ("re_ptr", P), ("re_where", P), ("re_species", P), ("re_mult", P),
                ("pr_ptr", P), ("pr_where", P), ("pr_species", P), ("pr_mult", P),
                ("rate", P), ("init", P), ("n_obs", I32), ("obs_of_cell", P)]


class cwc_sweep(ctypes.Structure):
    _fields_ = [("n_points", I32), ("n_swept", I32), ("rule", P), ("value", P)]


class cwc_stats(ctypes.Structure):
    _fields_ = [("count", P), ("sum", P), ("sumsq", P)]


class cwc_sim_opts(ctypes.Structure):
    _fields_ = [("out_traj", P), ("out_firings", P), ("out_status", P), ("trace_g", P), ("n_trace", I32),
                ("trace_cap", I64), ("trace_buf", P), ("trace_len", P), ("force_path", I32), ("block_threads", I32),
                ("replica_offset", I64), ("replicas_total", I64), ("ev_kernel_begin", P), ("ev_kernel_end", P),
                ("kernel", I32), ("stats_mode", I32), ("warps_per_block", I32), ("blocks_per_sm", I32),
                ("ev_stage2_begin", P), ("ev_stage2_end", P)]


class cwc_plan_info(ctypes.Structure):
    _fields_ = [("kernel", I32), ("blocks", I32), ("threads", I32), ("stats_shared", I32), ("smem_bytes", I64),
                ("n_parts", I64), ("part_cells", I64), ("word_bytes", I32), ("words_per_cell", I32),
                ("n_stat_cells", I64), ("workspace_bytes", I64)]


class cwc_model_info(ctypes.Structure):
    _fields_ = [("n_cells", I32), ("n_reactions", I32), ("n_obs", I32), ("n_rules", I32), ("path", I32),
                ("thread_path_ok", I32), ("max_deps", I32), ("n_nu", I32), ("n_deps", I64)]


_lib = None


def lib():
    """Load libcwcsim.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError("libcwcsim.so not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        L.cwc_model_create.argtypes = [ctypes.POINTER(cwc_model_desc), ctypes.POINTER(P)]
        L.cwc_model_destroy.argtypes = [P]
        L.cwc_model_destroy.restype = None
        L.cwc_model_info_get.argtypes = [P, ctypes.POINTER(cwc_model_info)]
        L.cwc_model_get_flat.argtypes = [P] + [P] * 11
        L.cwc_plan.argtypes = [P, I64, P, ctypes.c_double, ctypes.c_double, P, ctypes.POINTER(cwc_plan_info)]
        L.cwc_simulate_workspace_size.argtypes = [P, I64, P, ctypes.c_double, ctypes.c_double, P, ctypes.POINTER(ctypes.c_size_t)]
        L.cwc_simulate.argtypes = [P, I64, P, ctypes.c_double, ctypes.c_double, ctypes.c_uint64, P, cwc_stats, P,
                                   ctypes.c_size_t, P]
        L.cwc_simulate_host.argtypes = [P, I64, P, ctypes.c_double, ctypes.c_double, ctypes.c_uint64, P, cwc_stats, P,
                                        ctypes.c_size_t]
        L.cwc_simulate_host_workspace_size.argtypes = [P, I64, P, ctypes.c_double, ctypes.c_double,
                                                       ctypes.POINTER(ctypes.c_size_t)]
        L.cwc_stats_finalize.argtypes = [ctypes.POINTER(cwc_stats), I64, P, P, P, P]
        L.cwc_philox_blocks.argtypes = [ctypes.c_uint64, P, P, I64, P, P]
        L.cwc_draws.argtypes = [ctypes.c_uint64, P, P, I64, P, P, P]
        L.cwc_tau_div.argtypes = [P, P, I64, P, P]
        L.cwc_block_draws.argtypes = [P, I64, P, P, P, P]
        D = ctypes.c_double
        L.cwc_run_state_size.argtypes = [P, I64, P, D, D, P, ctypes.POINTER(ctypes.c_size_t)]
        L.cwc_run_init.argtypes = [P, I64, P, D, D, P, P, ctypes.c_size_t, P]
        L.cwc_run_advance.argtypes = [P, I64, P, D, D, ctypes.c_uint64, P, I64, I64, P, ctypes.c_size_t, P,
                                      ctypes.POINTER(I64)]
        L.cwc_run_stats.argtypes = [P, I64, P, D, D, P, P, ctypes.c_size_t, cwc_stats, P]
        L.cwc_last_error.restype = ctypes.c_char_p
        L.cwc_last_error.argtypes = []
        for name in EXPORTED:
            if name != "cwc_model_destroy" and name != "cwc_last_error":
                getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def cwc_last_error():
    return lib().cwc_last_error().decode()


def _check(status):
    if status != CWC_OK:
        raise CwcError(status, cwc_last_error())


def _i32(v):
    return np.ascontiguousarray(np.asarray(list(v) if len(v) else [0], dtype=np.int32))


class _DescArrays:
    """Host arrays of a model description dict (workloads/ format), kept alive
    for the duration of cwc_model_create."""

    def __init__(self, d):
        rules = d["rules"]
        re_ptr, re_w, re_s, re_m, pr_ptr, pr_w, pr_s, pr_m = [0], [], [], [], [0], [], [], []
        for r in rules:
            for (wh, s, m) in r["reactants"]:
                re_w.append(wh); re_s.append(s); re_m.append(m)  # noqa: E702
            re_ptr.append(len(re_w))
            for (wh, s, m) in r["products"]:
                pr_w.append(wh); pr_s.append(s); pr_m.append(m)  # noqa: E702
            pr_ptr.append(len(pr_w))
        self.keep = dict(
            parent=_i32(d["parent"]), type=_i32(d["type"]),
            rule_label=_i32([r["label"] for r in rules]), rule_child_label=_i32([r["child_label"] for r in rules]),
            re_ptr=_i32(re_ptr), re_where=_i32(re_w), re_species=_i32(re_s), re_mult=_i32(re_m),
            pr_ptr=_i32(pr_ptr), pr_where=_i32(pr_w), pr_species=_i32(pr_s), pr_mult=_i32(pr_m),
            rate=np.ascontiguousarray(np.asarray([float(r["rate"]) for r in rules] or [1.0], dtype=np.float64)),
            init=_i32(d["init"]), obs_of_cell=_i32(d["obs_of_cell"]))
        k = self.keep
        self.desc = cwc_model_desc(
            int(d["n_types"]), int(d["n_species"]), len(d["parent"]), k["parent"].ctypes.data, k["type"].ctypes.data,
            len(rules), k["rule_label"].ctypes.data, k["rule_child_label"].ctypes.data,
            k["re_ptr"].ctypes.data, k["re_where"].ctypes.data, k["re_species"].ctypes.data, k["re_mult"].ctypes.data,
            k["pr_ptr"].ctypes.data, k["pr_where"].ctypes.data, k["pr_species"].ctypes.data, k["pr_mult"].ctypes.data,
            k["rate"].ctypes.data, k["init"].ctypes.data, int(d["n_obs"]), k["obs_of_cell"].ctypes.data)


class _SweepArrays:
    def __init__(self, sweep):
        self.rule = _i32(sweep["rules"])
        vals = np.asarray(sweep["values"], dtype=np.float64).reshape(len(sweep["values"]), len(sweep["rules"]))
        self.value = np.ascontiguousarray(vals if vals.size else np.zeros((len(sweep["values"]), 1)))
        self.c = cwc_sweep(len(sweep["values"]), len(sweep["rules"]), self.rule.ctypes.data, self.value.ctypes.data)


def cwc_model_create(desc_dict):
    arr = _DescArrays(desc_dict)
    h = P()
    _check(lib().cwc_model_create(ctypes.byref(arr.desc), ctypes.byref(h)))
    return Model(h, desc_dict)


def cwc_model_create_raw(desc_struct):
    """cwc_model_create on an already-marshalled cwc_model_desc (API tests)."""
    h = P()
    st = lib().cwc_model_create(ctypes.byref(desc_struct), ctypes.byref(h))
    return st, h


class Model:
    def __init__(self, handle, desc):
        self.handle = handle
        self.desc = desc
        info = cwc_model_info()
        _check(lib().cwc_model_info_get(self.handle, ctypes.byref(info)))
        self.info = info

    def close(self):
        if self.handle:
            lib().cwc_model_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def get_flat(self):
        i = self.info
        M = i.n_reactions
        a = lambda n: np.zeros(max(int(n), 1), dtype=np.int32)  # noqa: E731
        er, ec, ech, rp, npt, dp = a(M), a(M), a(M), a(M + 1), a(M + 1), a(M + 1)
        rc, rm = a(2 * M + 2), a(2 * M + 2)
        nc, nd = a(i.n_nu), a(i.n_nu)
        dep = a(i.n_deps)
        _check(lib().cwc_model_get_flat(self.handle, *[x.ctypes.data for x in (er, ec, ech, rp, rc, rm, npt, nc, nd, dp, dep)]))
        nre = int(rp[M])
        return dict(entry_rule=er[:M], entry_context=ec[:M], entry_child=ech[:M], re_ptr=rp[:M + 1],
                    re_cell=rc[:nre], re_mult=rm[:nre], nu_ptr=npt[:M + 1], nu_cell=nc[:i.n_nu],
                    nu_delta=nd[:i.n_nu], dep_ptr=dp[:M + 1], dep=dep[:i.n_deps])


def n_samples(t_end, sample_dt):
    return int(np.floor(t_end / sample_dt)) + 1


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def cwc_simulate_workspace_size(model, n_replicas, sweep, t_end, sample_dt, opts=None):
    sw = _SweepArrays(sweep) if sweep is not None else None
    n = ctypes.c_size_t()
    _check(lib().cwc_simulate_workspace_size(model.handle, int(n_replicas), ctypes.byref(sw.c) if sw else None,
                                             float(t_end), float(sample_dt), ctypes.byref(opts) if opts else None,
                                             ctypes.byref(n)))
    return n.value


KERNEL_NAMES = {CWC_KERNEL_THREAD_WS: "ssa_thread_ws_kernel", CWC_KERNEL_THREAD: "ssa_thread_kernel",
                CWC_KERNEL_THREAD2: "ssa_thread_kernel", CWC_KERNEL_THREAD_WS2: "ssa_thread_ws2_kernel",
                CWC_KERNEL_WARP2: "ssa_warp2_kernel", CWC_KERNEL_WARP: "ssa_warp_kernel",
                CWC_KERNEL_WARP8: "ssa_group_kernel<4", CWC_KERNEL_WARP4: "ssa_group_kernel<8"}


def cwc_plan(model, n_replicas, sweep, t_end, sample_dt, opts=None):
    """The launch plan (cwc_plan_info) cwc_simulate would use."""
    sw = _SweepArrays(sweep) if sweep is not None else None
    info = cwc_plan_info()
    _check(lib().cwc_plan(model.handle, int(n_replicas), ctypes.byref(sw.c) if sw else None, float(t_end),
                          float(sample_dt), ctypes.byref(opts) if opts else None, ctypes.byref(info)))
    return info


def cwc_simulate(model, n_replicas, sweep, t_end, sample_dt, seed, stream, stats, workspace, opts=None,
                 sweep_arrays=None):
    """stats: (count, sum, sumsq) torch tensors; workspace: uint8 torch tensor;
    sweep_arrays: a prebuilt _SweepArrays(sweep) (avoids re-marshalling a
    large sweep on every call)."""
    sw = sweep_arrays if sweep_arrays is not None else (_SweepArrays(sweep) if sweep is not None else None)
    st = cwc_stats(stats[0].data_ptr(), stats[1].data_ptr(), stats[2].data_ptr())
    _check(lib().cwc_simulate(model.handle, int(n_replicas), ctypes.byref(sw.c) if sw else None, float(t_end),
                              float(sample_dt), int(seed), ctypes.c_void_p(stream), st,
                              ctypes.c_void_p(workspace.data_ptr()), workspace.numel(),
                              ctypes.byref(opts) if opts is not None else None))


def cwc_simulate_host_workspace_size(model, n_replicas, sweep, t_end, sample_dt):
    sw = _SweepArrays(sweep) if sweep is not None else None
    n = ctypes.c_size_t()
    _check(lib().cwc_simulate_host_workspace_size(model.handle, int(n_replicas), ctypes.byref(sw.c) if sw else None,
                                                  float(t_end), float(sample_dt), ctypes.byref(n)))
    return n.value


def cwc_simulate_host(model, n_replicas, sweep, t_end, sample_dt, seed, stream, host_stats, workspace, sweep_arrays=None):
    """host_stats: (count, sum, sumsq) pinned CPU torch tensors."""
    sw = sweep_arrays if sweep_arrays is not None else (_SweepArrays(sweep) if sweep is not None else None)
    st = cwc_stats(host_stats[0].data_ptr(), host_stats[1].data_ptr(), host_stats[2].data_ptr())
    _check(lib().cwc_simulate_host(model.handle, int(n_replicas), ctypes.byref(sw.c) if sw else None, float(t_end),
                                   float(sample_dt), int(seed), ctypes.c_void_p(stream), st,
                                   ctypes.c_void_p(workspace.data_ptr()), workspace.numel()))


def cwc_stats_finalize(stats, n_cells, mean, var, ci90, stream):
    st = cwc_stats(stats[0].data_ptr(), stats[1].data_ptr(), stats[2].data_ptr())
    _check(lib().cwc_stats_finalize(ctypes.byref(st), int(n_cells), _ptr(mean), _ptr(var), _ptr(ci90),
                                    ctypes.c_void_p(stream)))


def cwc_philox_blocks(seed, g, n, out, stream):
    _check(lib().cwc_philox_blocks(int(seed), _ptr(g), _ptr(n), int(g.numel()), _ptr(out), ctypes.c_void_p(stream)))


def cwc_draws(seed, g, n, E, u2, stream):
    _check(lib().cwc_draws(int(seed), _ptr(g), _ptr(n), int(g.numel()), _ptr(E), _ptr(u2), ctypes.c_void_p(stream)))


def cwc_block_draws(words, u1, u2, E, stream):
    """words: uint32-valued torch tensor [count, 4] (int32 storage) on the device."""
    _check(lib().cwc_block_draws(_ptr(words), int(words.shape[0]), _ptr(u1), _ptr(u2), _ptr(E), ctypes.c_void_p(stream)))


def cwc_tau_div(e, a, q, stream):
    _check(lib().cwc_tau_div(_ptr(e), _ptr(a), int(e.numel()), _ptr(q), ctypes.c_void_p(stream)))


def _sw(sweep):
    return _SweepArrays(sweep) if sweep is not None else None


def _opt(opts):
    return ctypes.byref(opts) if opts is not None else None


def cwc_run_state_size(model, n_replicas, sweep, t_end, sample_dt, opts=None):
    sw = _sw(sweep)
    n = ctypes.c_size_t()
    _check(lib().cwc_run_state_size(model.handle, int(n_replicas), ctypes.byref(sw.c) if sw else None, float(t_end),
                                    float(sample_dt), _opt(opts), ctypes.byref(n)))
    return n.value


def cwc_run_init(model, n_replicas, sweep, t_end, sample_dt, state, stream, opts=None):
    sw = _sw(sweep)
    _check(lib().cwc_run_init(model.handle, int(n_replicas), ctypes.byref(sw.c) if sw else None, float(t_end),
                              float(sample_dt), _opt(opts), ctypes.c_void_p(state.data_ptr()), state.numel(),
                              ctypes.c_void_p(stream)))


def cwc_run_advance(model, n_replicas, sweep, t_end, sample_dt, seed, state, stream, quantum=0, j_stop=0, opts=None):
    """One advance; returns how many trajectories still have samples below j_stop (synchronises the stream)."""
    sw = _sw(sweep)
    n_live = I64()
    _check(lib().cwc_run_advance(model.handle, int(n_replicas), ctypes.byref(sw.c) if sw else None, float(t_end),
                                 float(sample_dt), int(seed), _opt(opts), int(quantum), int(j_stop),
                                 ctypes.c_void_p(state.data_ptr()), state.numel(), ctypes.c_void_p(stream),
                                 ctypes.byref(n_live)))
    return n_live.value


def cwc_run_stats(model, n_replicas, sweep, t_end, sample_dt, state, stats, stream, opts=None):
    sw = _sw(sweep)
    st = cwc_stats(stats[0].data_ptr(), stats[1].data_ptr(), stats[2].data_ptr())
    _check(lib().cwc_run_stats(model.handle, int(n_replicas), ctypes.byref(sw.c) if sw else None, float(t_end),
                               float(sample_dt), _opt(opts), ctypes.c_void_p(state.data_ptr()), state.numel(), st,
                               ctypes.c_void_p(stream)))


# ---------------------------------------------------------------------------
# convenience: allocate torch outputs and run (the calls above do the work)
# ---------------------------------------------------------------------------

def _plan_opts(opts, kernel=CWC_KERNEL_AUTO, stats_mode=CWC_STATS_AUTO, warps_per_block=0, blocks_per_sm=0):
    opts.kernel = int(kernel)
    opts.stats_mode = int(stats_mode)
    opts.warps_per_block = int(warps_per_block)
    opts.blocks_per_sm = int(blocks_per_sm)


def simulate(model, n_replicas, t_end, sample_dt, seed, sweep=None, want_traj=False, want_firings=True,
             trace_g=(), trace_cap=0, force_path=CWC_PATH_AUTO, block_threads=0, device="cuda", stream=None,
             finalize=False, replica_offset=0, replicas_total=0, kernel_events=None, buffers=None, **plan):
    """Allocate outputs (or reuse `buffers` from a previous call) and run
    cwc_simulate once on `device` (made current for the call).
    kernel_events: (begin, end) torch.cuda.Event pair recorded around the
    SSA kernel.  plan: kernel / stats_mode / warps_per_block / blocks_per_sm
    overrides of cwc_sim_opts."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("cwc: no CUDA device (there is no CPU fallback)")
    with torch.cuda.device(torch.device(device)):
        return _simulate(torch, model, n_replicas, t_end, sample_dt, seed, sweep, want_traj, want_firings, trace_g,
                         trace_cap, force_path, block_threads, device, stream, finalize, replica_offset,
                         replicas_total, kernel_events, buffers, plan)


def _simulate(torch, model, n_replicas, t_end, sample_dt, seed, sweep, want_traj, want_firings, trace_g, trace_cap,
              force_path, block_threads, device, stream, finalize, replica_offset, replicas_total, kernel_events,
              buffers, plan):
    P_ = len(sweep["values"]) if sweep is not None else 1
    G = P_ * int(n_replicas)
    J1 = n_samples(t_end, sample_dt)
    O = model.info.n_obs
    ncell = P_ * J1 * O
    dev = torch.device(device)
    if buffers is not None:
        count, sm, sq = buffers["_count"], buffers["_sum"], buffers["_sumsq"]
    else:
        count = torch.empty(max(ncell, 1), dtype=torch.int64, device=dev)
        sm = torch.empty(max(ncell, 1), dtype=torch.int64, device=dev)
        sq = torch.empty((max(ncell, 1), 2), dtype=torch.int64, device=dev)
    opts = cwc_sim_opts()
    opts.force_path = int(force_path)
    opts.block_threads = int(block_threads)
    _plan_opts(opts, **plan)
    opts.replica_offset = int(replica_offset)
    opts.replicas_total = int(replicas_total)
    if kernel_events is not None:
        opts.ev_kernel_begin = kernel_events[0].cuda_event
        opts.ev_kernel_end = kernel_events[1].cuda_event
    out = {}
    if want_traj:
        out["traj"] = torch.empty((G, J1, O), dtype=torch.int64, device=dev)
        opts.out_traj = out["traj"].data_ptr()
    if want_firings:
        out["firings"] = buffers["firings"] if buffers is not None else torch.empty(G, dtype=torch.int64, device=dev)
        out["status"] = buffers["status"] if buffers is not None else torch.empty(G, dtype=torch.int32, device=dev)
        opts.out_firings = out["firings"].data_ptr()
        opts.out_status = out["status"].data_ptr()
    tg = None
    if len(trace_g):
        tg = np.ascontiguousarray(np.asarray(trace_g, dtype=np.int64))
        out["trace"] = torch.zeros((len(tg), trace_cap, 5), dtype=torch.float64, device=dev)
        out["trace_len"] = torch.zeros(len(tg), dtype=torch.int64, device=dev)
        opts.trace_g = tg.ctypes.data
        opts.n_trace = len(tg)
        opts.trace_cap = int(trace_cap)
        opts.trace_buf = out["trace"].data_ptr()
        opts.trace_len = out["trace_len"].data_ptr()
    ws_bytes = cwc_simulate_workspace_size(model, n_replicas, sweep, t_end, sample_dt, opts)
    if buffers is not None and buffers["workspace"].numel() >= ws_bytes:
        ws = buffers["workspace"]
    else:
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    cwc_simulate(model, n_replicas, sweep, t_end, sample_dt, seed, s, (count, sm, sq), ws, opts)
    out.update(count=count[:ncell].view(P_, J1, O), sum=sm[:ncell].view(P_, J1, O),
               sumsq=sq[:ncell].view(P_, J1, O, 2), n_points=P_, J1=J1, workspace=ws, _count=count, _sum=sm,
               _sumsq=sq)
    if finalize:
        mean = torch.empty(max(ncell, 1), dtype=torch.float64, device=dev)
        var = torch.empty_like(mean)
        ci = torch.empty_like(mean)
        cwc_stats_finalize((count, sm, sq), ncell, mean, var, ci, s)
        out.update(mean=mean[:ncell].view(P_, J1, O), var=var[:ncell].view(P_, J1, O), ci90=ci[:ncell].view(P_, J1, O))
    return out


def simulate_resumable(model, n_replicas, t_end, sample_dt, seed, sweep=None, quantum=0, windows=None,
                       want_traj=False, force_path=CWC_PATH_AUTO, device="cuda", checkpoint=None,
                       kernel_events=None, replica_offset=0, replicas_total=0, **plan):
    import torch
    with torch.cuda.device(torch.device(device)):
        return _simulate_resumable(model, n_replicas, t_end, sample_dt, seed, sweep, quantum, windows, want_traj,
                                   force_path, device, checkpoint, kernel_events, replica_offset, replicas_total,
                                   **plan)


def _simulate_resumable(model, n_replicas, t_end, sample_dt, seed, sweep=None, quantum=0, windows=None,
                        want_traj=False, force_path=CWC_PATH_AUTO, device="cuda", checkpoint=None,
                        kernel_events=None, replica_offset=0, replicas_total=0, **plan):
    """Run through cwc_run_init / cwc_run_advance / cwc_run_stats.

    quantum: firings per trajectory per advance (0 = unbounded); windows:
    increasing j_stop values, one advance per window (the last is J+1), with
    the quantum applied inside each window.  checkpoint(state, k) is called
    after advance k and may return a replacement state tensor (e.g. one
    restored from a host copy).  Returns the same dict as simulate() plus
    "advances" and "live" (the pending count after each advance)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("cwc: no CUDA device (there is no CPU fallback)")
    P_ = len(sweep["values"]) if sweep is not None else 1
    G = P_ * int(n_replicas)
    J1 = n_samples(t_end, sample_dt)
    O = model.info.n_obs
    ncell = P_ * J1 * O
    dev = torch.device(device)
    opts = cwc_sim_opts()
    opts.force_path = int(force_path)
    _plan_opts(opts, **plan)
    opts.replica_offset = int(replica_offset)
    opts.replicas_total = int(replicas_total)
    out = {"firings": torch.empty(G, dtype=torch.int64, device=dev),
           "status": torch.empty(G, dtype=torch.int32, device=dev)}
    opts.out_firings = out["firings"].data_ptr()
    opts.out_status = out["status"].data_ptr()
    if want_traj:
        out["traj"] = torch.empty((G, J1, O), dtype=torch.int64, device=dev)
        opts.out_traj = out["traj"].data_ptr()
    if kernel_events is not None:
        opts.ev_kernel_begin = kernel_events[0].cuda_event
        opts.ev_kernel_end = kernel_events[1].cuda_event
    s = torch.cuda.current_stream(dev).cuda_stream
    state = torch.empty(cwc_run_state_size(model, n_replicas, sweep, t_end, sample_dt, opts), dtype=torch.uint8,
                        device=dev)
    cwc_run_init(model, n_replicas, sweep, t_end, sample_dt, state, s, opts)
    live = []
    wins = list(windows) if windows else [0]
    k = 0
    for js in wins:
        while True:  # advance until every trajectory has passed the window (or finished)
            n_pending = cwc_run_advance(model, n_replicas, sweep, t_end, sample_dt, seed, state, s, quantum, js, opts)
            live.append(n_pending)
            k += 1
            if checkpoint is not None:
                st2 = checkpoint(state, k)
                if st2 is not None:
                    state = st2
            if n_pending == 0:
                break
    count = torch.empty(max(ncell, 1), dtype=torch.int64, device=dev)
    sm = torch.empty(max(ncell, 1), dtype=torch.int64, device=dev)
    sq = torch.empty((max(ncell, 1), 2), dtype=torch.int64, device=dev)
    cwc_run_stats(model, n_replicas, sweep, t_end, sample_dt, state, (count, sm, sq), s, opts)
    out.update(count=count[:ncell].view(P_, J1, O), sum=sm[:ncell].view(P_, J1, O),
               sumsq=sq[:ncell].view(P_, J1, O, 2), n_points=P_, J1=J1, advances=k, live=live, state=state)
    return out
