"""Thin ctypes binding of include/cwc_dyn.h (dynamic-topology CWC, SURVEY
8(f) NEXT-4): argument marshalling only.  Every step of the simulation runs
in libcwcsim.so; there is no CPU fallback.

`dyn_model_create(model)` takes the model dict of workloads/dynamic.py (the
format oracle/dynamic.py also reads) and flattens the initial term into the
preorder compartment arrays and the rules into the CSR arrays of
cwc_dyn_model_desc; `simulate(...)` allocates the torch tensors
cwc_dyn_simulate writes into.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import cwc
from .cwc import P, I32, I64, _check, _i32

CWC_TRAJ_CAPACITY = 4
CWC_DYN_CTX, CWC_DYN_WRAP, CWC_DYN_CONTENT = 0, 1, 2
CWC_DYN_KEEP_X, CWC_DYN_RELEASE_W, CWC_DYN_RELEASE_Y = 1, 2, 4
CWC_DYN_CTOR_W, CWC_DYN_CTOR_Y = 1, 2
OBS_KIND = {"content": 0, "wrap": 1, "count": 2}
MAX_CAP = 64

EXPORTED = ["cwc_dyn_model_create", "cwc_dyn_model_destroy", "cwc_dyn_info_get", "cwc_dyn_workspace_size",
            "cwc_dyn_simulate"]


class cwc_dyn_model_desc(ctypes.Structure):
    _fields_ = [("n_atoms", I32), ("n_labels", I32), ("n_comps", I32), ("comp_label", P), ("comp_parent", P),
                ("comp_wrap", P), ("comp_content", P), ("n_rules", I32), ("rule_label", P), ("rule_comp_label", P),
                ("rate", P), ("rule_flags", P), ("lhs_ptr", P), ("lhs_side", P), ("lhs_atom", P), ("lhs_mult", P),
                ("rhs_ptr", P), ("rhs_atom", P), ("rhs_mult", P), ("ctor_ptr", P), ("ctor_label", P),
                ("ctor_flags", P), ("ctor_atom_ptr", P), ("ctor_side", P), ("ctor_atom", P), ("ctor_mult", P),
                ("n_obs", I32), ("obs_ptr", P), ("obs_kind", P), ("obs_label", P), ("obs_atom", P)]


class cwc_dyn_opts(ctypes.Structure):
    _fields_ = [("out_traj", P), ("out_firings", P), ("out_status", P), ("replica_offset", I64),
                ("replicas_total", I64), ("capacity", I32), ("warps_per_block", I32), ("blocks_per_sm", I32),
                ("pad_", I32), ("ev_kernel_begin", P), ("ev_kernel_end", P)]


class cwc_dyn_info(ctypes.Structure):
    _fields_ = [("n_atoms", I32), ("n_labels", I32), ("n_rules", I32), ("n_obs", I32), ("n_structural", I32),
                ("blocks", I32), ("threads", I32), ("capacity", I32), ("smem_bytes", I64), ("n_stat_cells", I64),
                ("workspace_bytes", I64)]


_bound = False


def lib():
    global _bound
    L = cwc.lib()
    if not _bound:
        D = ctypes.c_double
        L.cwc_dyn_model_create.argtypes = [ctypes.POINTER(cwc_dyn_model_desc), ctypes.POINTER(P)]
        L.cwc_dyn_model_destroy.argtypes = [P]
        L.cwc_dyn_model_destroy.restype = None
        L.cwc_dyn_info_get.argtypes = [P, I64, D, D, P, ctypes.POINTER(cwc_dyn_info)]
        L.cwc_dyn_workspace_size.argtypes = [P, I64, D, D, P, ctypes.POINTER(ctypes.c_size_t)]
        L.cwc_dyn_simulate.argtypes = [P, I64, D, D, ctypes.c_uint64, P, cwc.cwc_stats, P, ctypes.c_size_t, P]
        for name in EXPORTED:
            if name != "cwc_dyn_model_destroy":
                getattr(L, name).restype = ctypes.c_int
        _bound = True
    return L


class _DynArrays:
    """Host arrays of a dynamic model dict, alive for cwc_dyn_model_create."""

    def __init__(self, m):
        A = int(m["n_atoms"])
        labels, parents, wraps, conts = [], [], [], []

        def dense(ms):
            v = [0] * A
            for a, k in (ms or {}).items():
                v[int(a)] += int(k)
            return v

        def walk(term, label, parent, wrap):
            me = len(labels)
            labels.append(int(label))
            parents.append(int(parent))
            wraps.append(dense(wrap))
            conts.append(dense(term.get("atoms", {})))
            for c in term.get("comps", []):
                walk(c.get("content", {}), c["label"], me, c.get("wrap", {}))
        walk(m["term"], 0, -1, {})

        rl, rcl, rate, fl = [], [], [], []
        lp, ls, la, lm = [0], [], [], []
        hp, ha, hm = [0], [], []
        cp, cl, cf, cap_, cs, ca, cm = [0], [], [], [0], [], [], []
        for r in m["rules"]:
            rl.append(int(r["label"]))
            comp = r.get("comp")
            rcl.append(int(comp["label"]) if comp is not None else -1)
            rate.append(float(r["rate"]))
            rhs = r["rhs"]
            fl.append((CWC_DYN_KEEP_X if rhs.get("X", True) else 0) | (CWC_DYN_RELEASE_W if rhs.get("release_W") else 0)
                      | (CWC_DYN_RELEASE_Y if rhs.get("release_Y") else 0))
            sides = [(CWC_DYN_CTX, r.get("atoms", {}))]
            if comp is not None:
                sides += [(CWC_DYN_WRAP, comp.get("wrap", {})), (CWC_DYN_CONTENT, comp.get("content", {}))]
            for side, ms in sides:
                for a, k in ms.items():
                    if k:
                        ls.append(side); la.append(int(a)); lm.append(int(k))  # noqa: E702
            lp.append(len(ls))
            for a, k in rhs.get("atoms", {}).items():
                if k:
                    ha.append(int(a)); hm.append(int(k))  # noqa: E702
            hp.append(len(ha))
            for k in rhs.get("comps", []):
                cl.append(int(k["label"]))
                cf.append((CWC_DYN_CTOR_W if k.get("W") else 0) | (CWC_DYN_CTOR_Y if k.get("Y") else 0))
                for side, ms in ((CWC_DYN_WRAP, k.get("wrap", {})), (CWC_DYN_CONTENT, k.get("content", {}))):
                    for a, n in ms.items():
                        if n:
                            cs.append(side); ca.append(int(a)); cm.append(int(n))  # noqa: E702
                cap_.append(len(cs))
            cp.append(len(cl))
        op, ok, ol, oa = [0], [], [], []
        for ob in m["observables"]:
            keys = ob if isinstance(ob, list) else [ob]
            for key in keys:
                ok.append(OBS_KIND[key[0]])
                ol.append(int(key[1]))
                oa.append(int(key[2]) if len(key) > 2 else 0)
            op.append(len(ok))
        self.n_comps = len(labels)
        k = self.keep = dict(
            comp_label=_i32(labels), comp_parent=_i32(parents), comp_wrap=_i32(np.ravel(wraps)),
            comp_content=_i32(np.ravel(conts)), rule_label=_i32(rl), rule_comp_label=_i32(rcl),
            rate=np.ascontiguousarray(np.asarray(rate or [1.0], dtype=np.float64)), rule_flags=_i32(fl),
            lhs_ptr=_i32(lp), lhs_side=_i32(ls), lhs_atom=_i32(la), lhs_mult=_i32(lm),
            rhs_ptr=_i32(hp), rhs_atom=_i32(ha), rhs_mult=_i32(hm), ctor_ptr=_i32(cp), ctor_label=_i32(cl),
            ctor_flags=_i32(cf), ctor_atom_ptr=_i32(cap_), ctor_side=_i32(cs), ctor_atom=_i32(ca), ctor_mult=_i32(cm),
            obs_ptr=_i32(op), obs_kind=_i32(ok), obs_label=_i32(ol), obs_atom=_i32(oa))
        self.desc = cwc_dyn_model_desc(
            A, int(m["n_labels"]), len(labels), k["comp_label"].ctypes.data, k["comp_parent"].ctypes.data,
            k["comp_wrap"].ctypes.data, k["comp_content"].ctypes.data, len(m["rules"]), k["rule_label"].ctypes.data,
            k["rule_comp_label"].ctypes.data, k["rate"].ctypes.data, k["rule_flags"].ctypes.data,
            k["lhs_ptr"].ctypes.data, k["lhs_side"].ctypes.data, k["lhs_atom"].ctypes.data, k["lhs_mult"].ctypes.data,
            k["rhs_ptr"].ctypes.data, k["rhs_atom"].ctypes.data, k["rhs_mult"].ctypes.data, k["ctor_ptr"].ctypes.data,
            k["ctor_label"].ctypes.data, k["ctor_flags"].ctypes.data, k["ctor_atom_ptr"].ctypes.data,
            k["ctor_side"].ctypes.data, k["ctor_atom"].ctypes.data, k["ctor_mult"].ctypes.data,
            len(m["observables"]), k["obs_ptr"].ctypes.data, k["obs_kind"].ctypes.data, k["obs_label"].ctypes.data,
            k["obs_atom"].ctypes.data)


class DynModel:
    def __init__(self, handle, model):
        self.handle = handle
        self.model = model
        self.n_obs = len(model["observables"])

    def close(self):
        if self.handle:
            lib().cwc_dyn_model_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def cwc_dyn_model_create(model):
    arr = _DynArrays(model)
    h = P()
    _check(lib().cwc_dyn_model_create(ctypes.byref(arr.desc), ctypes.byref(h)))
    return DynModel(h, model)


def cwc_dyn_model_create_status(model):
    """(status, handle or None) without raising (API tests)."""
    arr = _DynArrays(model)
    h = P()
    st = lib().cwc_dyn_model_create(ctypes.byref(arr.desc), ctypes.byref(h))
    return st, (DynModel(h, model) if st == cwc.CWC_OK else None)


def cwc_dyn_info_get(model, n_replicas=0, t_end=1.0, sample_dt=1.0, opts=None):
    info = cwc_dyn_info()
    _check(lib().cwc_dyn_info_get(model.handle, int(n_replicas), float(t_end), float(sample_dt),
                                  ctypes.byref(opts) if opts is not None else None, ctypes.byref(info)))
    return info


def cwc_dyn_workspace_size(model, n_replicas, t_end, sample_dt, opts=None):
    n = ctypes.c_size_t()
    _check(lib().cwc_dyn_workspace_size(model.handle, int(n_replicas), float(t_end), float(sample_dt),
                                        ctypes.byref(opts) if opts is not None else None, ctypes.byref(n)))
    return n.value


def cwc_dyn_simulate(model, n_replicas, t_end, sample_dt, seed, stream, stats, workspace, opts=None):
    st = cwc.cwc_stats(stats[0].data_ptr(), stats[1].data_ptr(), stats[2].data_ptr())
    _check(lib().cwc_dyn_simulate(model.handle, int(n_replicas), float(t_end), float(sample_dt), int(seed),
                                  ctypes.c_void_p(stream), st, ctypes.c_void_p(workspace.data_ptr()),
                                  workspace.numel(), ctypes.byref(opts) if opts is not None else None))


def simulate(model, n_replicas, t_end, sample_dt, seed, want_traj=False, capacity=0, device="cuda", stream=None,
             replica_offset=0, replicas_total=0, warps_per_block=0, blocks_per_sm=0, kernel_events=None,
             buffers=None):
    """Allocate outputs (or reuse `buffers`) and run cwc_dyn_simulate once."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("cwc_dyn: no CUDA device (there is no CPU fallback)")
    with torch.cuda.device(torch.device(device)):
        dev = torch.device(device)
        O = model.n_obs
        J1 = cwc.n_samples(t_end, sample_dt)
        opts = cwc_dyn_opts()
        opts.capacity = int(capacity)
        opts.replica_offset = int(replica_offset)
        opts.replicas_total = int(replicas_total)
        opts.warps_per_block = int(warps_per_block)
        opts.blocks_per_sm = int(blocks_per_sm)
        if buffers is None:
            ws = torch.empty(cwc_dyn_workspace_size(model, n_replicas, t_end, sample_dt, opts), dtype=torch.uint8,
                             device=dev)
            n = J1 * O
            buffers = dict(ws=ws, count=torch.empty(max(n, 1), dtype=torch.int64, device=dev),
                           sum=torch.empty(max(n, 1), dtype=torch.int64, device=dev),
                           sumsq=torch.empty(max(2 * n, 2), dtype=torch.int64, device=dev),
                           firings=torch.empty(n_replicas, dtype=torch.int64, device=dev),
                           status=torch.empty(n_replicas, dtype=torch.int32, device=dev),
                           traj=torch.empty((n_replicas, J1, O), dtype=torch.int64, device=dev) if want_traj else None)
        b = buffers
        opts.out_firings = b["firings"].data_ptr()
        opts.out_status = b["status"].data_ptr()
        if b.get("traj") is not None:
            opts.out_traj = b["traj"].data_ptr()
        if kernel_events is not None:
            opts.ev_kernel_begin = kernel_events[0].cuda_event
            opts.ev_kernel_end = kernel_events[1].cuda_event
        s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        cwc_dyn_simulate(model, n_replicas, t_end, sample_dt, seed, s, (b["count"], b["sum"], b["sumsq"]), b["ws"],
                         opts)
        n = J1 * O
        out = dict(count=b["count"][:n].view(J1, O), sum=b["sum"][:n].view(J1, O),
                   sumsq=b["sumsq"][:2 * n].view(J1, O, 2), firings=b["firings"], status=b["status"], buffers=b)
        if b.get("traj") is not None:
            out["traj"] = b["traj"]
        return out
