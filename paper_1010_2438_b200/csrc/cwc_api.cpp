// cwc_api.cpp -- the C ABI (include/cwc.h): model compiler and launcher.
//
// cwc_model_create validates the CWC description and flattens its rules over
// the fixed compartment tree (rule-major, context in index order = preorder,
// then child in index order), merges each pattern into
// (cell, multiplicity) reactants (a pattern is a multiset), forms
// the net change nu = products - reactants and the dependency
// graph D(mu) = {m : reactants(m) meet changed(mu)}, and uploads the tables.
// cwc_simulate carves the caller's workspace, picks the kernel and launch
// shape, and enqueues SSA kernel + stage-2 reduction on the caller's stream.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "cwc.h"
#include "cwc_internal.h"

using namespace cwc;

namespace {

thread_local std::string g_err;

cwc_status fail(cwc_status s, const std::string &msg) {
    g_err = msg;
    return s;
}
cwc_status cuda_fail(cudaError_t e, const char *where) {
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return CWC_ERR_CUDA;
}

// FNV-1a over bytes (input fingerprints: staging cache, resumable-state header)
uint64_t fnv1a(uint64_t h, const void *p, size_t n) {
    // FNV-1a over 64-bit words, then the tail bytes (a fingerprint, not a
    // cryptographic hash: 8x fewer steps for the staging key of big sweeps)
    const unsigned char *b = (const unsigned char *)p;
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
        uint64_t w;
        std::memcpy(&w, b + i, 8);
        h = (h ^ w) * 0x100000001b3ull;
        h ^= h >> 29;
    }
    for (; i < n; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
    return h;
}
template <typename T>
uint64_t fnv_vec(uint64_t h, const std::vector<T> &v) {
    return fnv1a(h, v.data(), v.size() * sizeof(T));
}

struct DeviceBuf {
    void *p = nullptr;
    ~DeviceBuf() {
        if (p) cudaFree(p);
    }
};

}  // namespace

// The calling thread's cwc_last_error() message, for the other API units
// (dyn_api.cpp).
void cwc::set_last_error(const std::string &msg) { g_err = msg; }

struct cwc_model_s {
    // host copies
    int32_t n_species = 0, n_compartments = 0, n_cells = 0, M = 0, n_obs = 0, n_rules = 0;
    std::vector<double> rule_rate;
    std::vector<int32_t> entry_rule, entry_ctx, entry_child;
    std::vector<int32_t> re_ptr, re_cell, re_mult;
    std::vector<int32_t> nu_ptr, nu_cell, nu_delta;
    std::vector<int32_t> dep_ptr, dep;
    std::vector<int2> dep_slot;   // warp path: (m, slot | owner << 24) per dependency entry
    std::vector<int2> dep_slot16; // the same for 16-lane segments
    std::vector<int4> dep_slot4;  // warp layout with the dependent's reactants inline
    std::vector<int4> dep_slot16_4;  // 16-lane segment layout with the reactants inline
    // warp kernels' per-mu tables (WarpTables.hdr / nuw / depw16 / depw32)
    std::vector<int4> wseg_hdr, wseg_dep16, wseg_dep32, wseg_dep4, wseg_dep8;
    std::vector<int2> wseg_nu, wseg_nu8;
    std::vector<int32_t> init, obs_of_cell, obs_ptr, obs_cells;
    std::vector<ReactionDesc> rx;
    int max_deps = 0;
    int vbits = 31;   // observables are < 2^vbits (sums of int32 counts)
    bool thread_ok = false;
    ThreadTables tt{};
    WarpTables wt{};  // sizes (host); device pointers live in the per-device copies
    // device copies of the tables, one per CUDA device the handle was used on
    // (one allocation each), created on first use under the mutex
    struct DevCopy {
        DeviceBuf buf;
        WarpTables wt{};
    };
    std::mutex dev_mu;
    std::map<int, std::unique_ptr<DevCopy>> dev;
    // Pinned host staging of a call's per-point rates and sweep dispatch
    // order, per device: cudaMemcpyAsync from pinned memory does not stall
    // the host, and consecutive calls with the same inputs (a bench loop, a
    // checkpointed run) reuse the staged bytes without recomputing them.
    struct Stage {
        uint64_t key = 0;
        bool valid = false;
        unsigned char *pinned = nullptr;
        size_t cap = 0, rates_bytes = 0, order_off = 0, order_bytes = 0;
        cudaEvent_t done = nullptr;  // the last copies out of `pinned` have finished
        ~Stage() {
            if (done) cudaEventDestroy(done);
            if (pinned) cudaFreeHost(pinned);
        }
    };
    std::mutex stage_mu;
    std::map<int, Stage> stage;
};

namespace {

// rates are finite and >= 2^-1021 (the smallest normal fp64 number times 2):
// the kernels pre-halve A + A rates, which is exact only in the normal range
bool finite_pos(double v) { return std::isfinite(v) && v >= 0x1.0p-1021; }

cwc_status build_model(const cwc_model_desc *d, cwc_model_s *m) {
    if (!d) return fail(CWC_ERR_INVALID, "desc is NULL");
    const int S = d->n_species, C = d->n_compartments, NT = d->n_types;
    if (S < 1) return fail(CWC_ERR_INVALID, "n_species must be >= 1");
    if (C < 1) return fail(CWC_ERR_INVALID, "n_compartments must be >= 1");
    if (NT < 1) return fail(CWC_ERR_INVALID, "n_types must be >= 1");
    if ((long long)S * C > (1ll << 30)) return fail(CWC_ERR_INVALID, "too many cells");
    if (!d->parent || !d->type) return fail(CWC_ERR_INVALID, "parent/type are NULL");
    if (d->parent[0] != -1 || d->type[0] != 0) return fail(CWC_ERR_INVALID, "compartment 0 must be the root of type 0");
    for (int c = 0; c < C; ++c) {
        if (d->type[c] < 0 || d->type[c] >= NT) return fail(CWC_ERR_INVALID, "type out of range at compartment " + std::to_string(c));
        if (c > 0 && (d->parent[c] < 0 || d->parent[c] >= c))
            return fail(CWC_ERR_INVALID, "parent must satisfy 0 <= parent[c] < c (preorder) at compartment " + std::to_string(c));
    }
    const int R = d->n_rules;
    if (R < 0) return fail(CWC_ERR_INVALID, "n_rules < 0");
    if (R > 0 && (!d->rule_label || !d->rule_child_label || !d->re_ptr || !d->pr_ptr || !d->rate))
        return fail(CWC_ERR_INVALID, "rule arrays are NULL");
    const int ncell = S * C;
    if (!d->init) return fail(CWC_ERR_INVALID, "init is NULL");
    for (int i = 0; i < ncell; ++i)
        if (d->init[i] < 0) return fail(CWC_ERR_INVALID, "negative initial count at cell " + std::to_string(i));
    if (d->n_obs < 0) return fail(CWC_ERR_INVALID, "n_obs < 0");
    if (d->n_obs > 0 && !d->obs_of_cell) return fail(CWC_ERR_INVALID, "obs_of_cell is NULL");
    for (int i = 0; d->n_obs > 0 && i < ncell; ++i)
        if (d->obs_of_cell[i] < -1 || d->obs_of_cell[i] >= d->n_obs)
            return fail(CWC_ERR_INVALID, "obs_of_cell out of range at cell " + std::to_string(i));

    m->n_species = S;
    m->n_compartments = C;
    m->n_cells = ncell;
    m->n_rules = R;
    m->n_obs = d->n_obs;
    m->rule_rate.assign(d->rate, d->rate + R);
    for (int r = 0; r < R; ++r) {
        if (!finite_pos(d->rate[r])) return fail(CWC_ERR_INVALID, "rate must be finite and >= 2^-1021 (rule " + std::to_string(r) + ")");
        if (d->rule_label[r] < 0 || d->rule_label[r] >= NT) return fail(CWC_ERR_INVALID, "rule_label out of range (rule " + std::to_string(r) + ")");
        if (d->rule_child_label[r] < -1 || d->rule_child_label[r] >= NT)
            return fail(CWC_ERR_INVALID, "rule_child_label out of range (rule " + std::to_string(r) + ")");
        for (int side = 0; side < 2; ++side) {
            const int32_t *ptr = side ? d->pr_ptr : d->re_ptr;
            const int32_t *wh = side ? d->pr_where : d->re_where;
            const int32_t *sp = side ? d->pr_species : d->re_species;
            const int32_t *mu = side ? d->pr_mult : d->re_mult;
            if (ptr[r] < 0 || ptr[r + 1] < ptr[r]) return fail(CWC_ERR_INVALID, "bad CSR pointer (rule " + std::to_string(r) + ")");
            int order = 0;
            for (int q = ptr[r]; q < ptr[r + 1]; ++q) {
                if (!wh || !sp || !mu) return fail(CWC_ERR_INVALID, "pattern arrays are NULL");
                if (wh[q] != 0 && wh[q] != 1) return fail(CWC_ERR_INVALID, "where must be 0 or 1 (rule " + std::to_string(r) + ")");
                if (wh[q] == 1 && d->rule_child_label[r] < 0)
                    return fail(CWC_ERR_INVALID, "child-compartment species on a local rule (rule " + std::to_string(r) + ")");
                if (sp[q] < 0 || sp[q] >= S) return fail(CWC_ERR_INVALID, "species out of range (rule " + std::to_string(r) + ")");
                if (mu[q] < 1) return fail(CWC_ERR_INVALID, "mult must be >= 1 (rule " + std::to_string(r) + ")");
                order += mu[q];
            }
            if (side == 0 && order > 2)
                return fail(CWC_ERR_UNSUPPORTED, "reaction order > 2 is not supported (rule " + std::to_string(r) + ")");
        }
    }

    // children lists in index order
    std::vector<std::vector<int>> kids(C);
    for (int c = 1; c < C; ++c) kids[d->parent[c]].push_back(c);

    m->re_ptr.push_back(0);
    m->nu_ptr.push_back(0);
    for (int r = 0; r < R; ++r) {
        const int lab = d->rule_label[r], cl = d->rule_child_label[r];
        for (int c = 0; c < C; ++c) {
            if (d->type[c] != lab) continue;
            std::vector<int> childs;
            if (cl < 0) childs.push_back(-1);
            else
                for (int k : kids[c])
                    if (d->type[k] == cl) childs.push_back(k);
            for (int ch : childs) {
                std::map<int, int> re, pr;
                for (int q = d->re_ptr[r]; q < d->re_ptr[r + 1]; ++q)
                    re[(d->re_where[q] ? ch : c) * S + d->re_species[q]] += d->re_mult[q];
                for (int q = d->pr_ptr[r]; q < d->pr_ptr[r + 1]; ++q)
                    pr[(d->pr_where[q] ? ch : c) * S + d->pr_species[q]] += d->pr_mult[q];
                m->entry_rule.push_back(r);
                m->entry_ctx.push_back(c);
                m->entry_child.push_back(ch);
                ReactionDesc rd{ncell, ncell, 0, r};
                int slot = 0;
                for (auto &kv : re) {
                    m->re_cell.push_back(kv.first);
                    m->re_mult.push_back(kv.second);
                    if (kv.second == 2) {
                        rd.ia = rd.ib = kv.first;
                        rd.kind = 1 | (1 << 1);
                    } else if (slot == 0) {
                        rd.ia = kv.first;
                    } else {
                        rd.ib = kv.first;
                    }
                    ++slot;
                }
                m->re_ptr.push_back((int32_t)m->re_cell.size());
                std::map<int, int> nu;
                for (auto &kv : pr) nu[kv.first] += kv.second;
                for (auto &kv : re) nu[kv.first] -= kv.second;
                for (auto &kv : nu)
                    if (kv.second != 0) {
                        m->nu_cell.push_back(kv.first);
                        m->nu_delta.push_back(kv.second);
                    }
                m->nu_ptr.push_back((int32_t)m->nu_cell.size());
                m->rx.push_back(rd);
            }
        }
    }
    m->M = (int32_t)m->entry_rule.size();
    const int M = m->M;

    // dependency graph: reactions reading each cell, then union per mu
    std::vector<std::vector<int>> readers(ncell);
    for (int k = 0; k < M; ++k)
        for (int q = m->re_ptr[k]; q < m->re_ptr[k + 1]; ++q) readers[m->re_cell[q]].push_back(k);
    m->dep_ptr.push_back(0);
    std::vector<int> mark(M, -1);
    for (int mu = 0; mu < M; ++mu) {
        std::vector<int> row;
        for (int q = m->nu_ptr[mu]; q < m->nu_ptr[mu + 1]; ++q)
            for (int k : readers[m->nu_cell[q]])
                if (mark[k] != mu) {
                    mark[k] = mu;
                    row.push_back(k);
                }
        std::sort(row.begin(), row.end());
        m->dep.insert(m->dep.end(), row.begin(), row.end());
        m->dep_ptr.push_back((int32_t)m->dep.size());
        if ((int)row.size() > m->max_deps) m->max_deps = (int)row.size();
    }

    m->init.assign(d->init, d->init + ncell);
    if (m->n_obs > 0) m->obs_of_cell.assign(d->obs_of_cell, d->obs_of_cell + ncell);
    else m->obs_of_cell.assign(ncell, -1);
    m->obs_ptr.assign(m->n_obs + 1, 0);
    int max_obs_cells = 1;
    for (int o = 0; o < m->n_obs; ++o) {
        for (int c = 0; c < ncell; ++c)
            if (m->obs_of_cell[c] == o) m->obs_cells.push_back(c);
        m->obs_ptr[o + 1] = (int32_t)m->obs_cells.size();
        max_obs_cells = std::max(max_obs_cells, m->obs_ptr[o + 1] - m->obs_ptr[o]);
    }
    m->vbits = 31;
    while ((1ll << (m->vbits - 31)) < max_obs_cells) ++m->vbits;

    // warp path sizes (pointers are filled by upload)
    m->wt.n_cells = m->n_cells;
    m->wt.M = m->M;
    m->wt.O = m->n_obs;
    m->wt.B = std::max(1, (m->M + 31) / 32);
    m->wt.Bp = m->wt.B | 1;
    if ((long long)32 * m->wt.Bp >= (1ll << 24)) return fail(CWC_ERR_UNSUPPORTED, "too many reactions for the warp path");
    m->dep_slot.resize(m->dep.size());
    for (size_t q = 0; q < m->dep.size(); ++q) {
        const int r = m->dep[q], l = r / m->wt.B, k = r - l * m->wt.B;
        m->dep_slot[q] = make_int2(r, (l * m->wt.Bp + k) | (l << 24));
    }
    m->dep_slot4.resize(m->dep.size());
    for (size_t q = 0; q < m->dep.size(); ++q) {
        const ReactionDesc &rd = m->rx[m->dep[q]];
        m->dep_slot4[q] = make_int4(m->dep_slot[q].x, m->dep_slot[q].y, rd.ia, rd.ib | (rd.kind << 24));
    }
    // 16-lane segment layout (two trajectories per warp, ssa_warp2.cu)
    m->wt.B16 = std::max(1, (m->M + 15) / 16);
    m->wt.Bp16 = m->wt.B16 | 1;
    m->dep_slot16.resize(m->dep.size());
    for (size_t q = 0; q < m->dep.size(); ++q) {
        const int r = m->dep[q], l = r / m->wt.B16, k = r - l * m->wt.B16;
        m->dep_slot16[q] = make_int2(r, (l * m->wt.Bp16 + k) | (l << 24));
    }

    m->dep_slot16_4.resize(m->dep.size());
    for (size_t q = 0; q < m->dep.size(); ++q) {
        const ReactionDesc &rd = m->rx[m->dep[q]];
        m->dep_slot16_4[q] = make_int4(m->dep_slot16[q].x, m->dep_slot16[q].y, rd.ia, rd.ib | (rd.kind << 24));
    }

    // warp kernels' per-mu tables: byte offsets (x: 4 bytes per cell, a: 8
    // bytes per slot of the lane-chunk layout, rates: 8 bytes per reaction),
    // the owner lane and the A + A flag packed as documented in WarpTables
    if ((long long)ncell * 4 + 4 >= (1ll << 31) || (long long)M * 8 >= (1ll << 26))
        return fail(CWC_ERR_UNSUPPORTED, "model too large for the warp kernels' tables");
    {
        m->wseg_hdr.resize(M);
        for (int mu = 0; mu < M; ++mu)
            m->wseg_hdr[mu] = make_int4(m->nu_ptr[mu], m->nu_ptr[mu + 1] - m->nu_ptr[mu], m->dep_ptr[mu],
                                        m->dep_ptr[mu + 1] - m->dep_ptr[mu]);
        m->wseg_nu.resize(m->nu_cell.size());
        for (size_t q = 0; q < m->nu_cell.size(); ++q) m->wseg_nu[q] = make_int2(4 * m->nu_cell[q], m->nu_delta[q]);
        // 4-lane groups (ssa_warp8.cu): entry m of owner ol = m / B4 at row k = m % B4
        m->wt.B4 = std::max(1, (M + 3) / 4);
        m->wseg_nu8.resize(m->nu_cell.size());
        for (size_t q = 0; q < m->nu_cell.size(); ++q) m->wseg_nu8[q] = make_int2(32 * m->nu_cell[q], m->nu_delta[q]);
        m->wseg_dep4.resize(m->dep.size());
        for (size_t q = 0; q < m->dep.size(); ++q) {
            const int r = m->dep[q], ol = r / m->wt.B4, k = r - ol * m->wt.B4;
            const ReactionDesc &rd = m->rx[r];
            const unsigned w = (unsigned)(8 * r) | ((unsigned)((ol * 4 + (k >> 4)) & 15) << 26) |
                               ((unsigned)(rd.kind & 1) << 31);
            m->wseg_dep4[q] = make_int4(8 * (k * 32 + (ol ^ ((k >> 2) & 3))), 32 * rd.ia, 32 * rd.ib, (int)w);
        }
        // 8-lane groups: B8 = ceil(M / 8) entries per lane, two sub-chunks
        const int B8 = std::max(1, (M + 7) / 8);
        m->wseg_dep8.resize(m->dep.size());
        for (size_t q = 0; q < m->dep.size(); ++q) {
            const int r = m->dep[q], ol = r / B8, k = r - ol * B8;
            const ReactionDesc &rd = m->rx[r];
            const unsigned w = (unsigned)(8 * r) | ((unsigned)((ol * 2 + (k >> 4)) & 15) << 26) |
                               ((unsigned)(rd.kind & 1) << 31);
            m->wseg_dep8[q] = make_int4(8 * (k * 32 + (ol ^ ((k >> 1) & 7))), 32 * rd.ia, 32 * rd.ib, (int)w);
        }
        for (int segw : {16, 32}) {
            const int Bs = segw == 16 ? m->wt.B16 : m->wt.B;
            const int Bps = Bs | 1;  // chunk stride (ssa_warp2.cu / ssa_warp.cu)
            std::vector<int4> &out = segw == 16 ? m->wseg_dep16 : m->wseg_dep32;
            out.resize(m->dep.size());
            for (size_t q = 0; q < m->dep.size(); ++q) {
                const int r = m->dep[q], l = r / Bs, k = r - l * Bs;
                const ReactionDesc &rd = m->rx[r];
                const unsigned w = (unsigned)(8 * r) | ((unsigned)(l & 31) << 26) | ((unsigned)(rd.kind & 1) << 31);
                out[q] = make_int4(8 * (l * Bps + k), 4 * rd.ia, 4 * rd.ib, (int)w);
            }
        }
    }

    // thread path tables
    bool ok = ncell <= kThreadMaxCells && M <= kThreadMaxReactions && m->n_obs <= kThreadMaxObs;
    for (size_t q = 0; ok && q < m->nu_delta.size(); ++q)
        if (m->nu_delta[q] < -127 || m->nu_delta[q] > 127) ok = false;
    m->thread_ok = ok;
    if (ok) {
        ThreadTables &tt = m->tt;
        std::memset(&tt, 0, sizeof(tt));
        tt.n_cells = ncell;
        tt.M = M;
        tt.O = m->n_obs;
        for (int k = 0; k < kThreadMaxReactions; ++k) {
            tt.ia[k] = tt.ib[k] = -1;  // -1 reads the constant 1
            tt.sub[k] = tt.shr[k] = 0;
            tt.nu_pack[k] = 0;
        }
        for (int k = 0; k < M; ++k) {
            tt.ia[k] = m->rx[k].ia == ncell ? -1 : m->rx[k].ia;
            tt.ib[k] = m->rx[k].ib == ncell ? -1 : m->rx[k].ib;
            tt.sub[k] = m->rx[k].kind & 1;
            tt.shr[k] = m->rx[k].kind >> 1;
            uint64_t pack = 0;
            for (int q = m->nu_ptr[k]; q < m->nu_ptr[k + 1]; ++q)
                pack |= (uint64_t)(uint8_t)(int8_t)m->nu_delta[q] << (8 * m->nu_cell[q]);
            tt.nu_pack[k] = pack;
        }
        // operand deltas (read by the kernel only when M <= 4)
        for (int k = 0; k < M; ++k) {
            auto delta_of = [&](int cell) {
                int dlt = 0;
                for (int q = m->nu_ptr[k]; q < m->nu_ptr[k + 1]; ++q)
                    if (m->nu_cell[q] == cell) dlt = m->nu_delta[q];
                return dlt;
            };
            uint64_t op[kOpWords] = {};
            for (int r2 = 0; r2 < M && r2 < 4 * kOpWords; ++r2) {
                const int ia = tt.ia[r2], ib = tt.ib[r2], wd = r2 >> 2, sh = 16 * (r2 & 3);
                op[wd] |= (uint64_t)(uint8_t)(int8_t)(ia >= 0 ? delta_of(ia) : 0) << sh;
                op[wd] |= (uint64_t)(uint8_t)(int8_t)(ib >= 0 ? delta_of(ib) : 0) << (sh + 8);
            }
            for (int wd = 0; wd < kOpWords; ++wd) tt.op_pack[k][wd] = op[wd];
        }
        const int s_pad = thread_pad_cells(ncell), m_pad = thread_pad_reactions(std::max(M, 2));
        if (s_pad > 0 && m_pad > 0 && 8 * s_pad + 16 * m_pad <= 64)
            for (int k = 0; k < M; ++k) tt.comb_pack[k] = tt.nu_pack[k] | (tt.op_pack[k][0] << (8 * s_pad));
        for (int c = 0; c < kThreadMaxCells; ++c) {
            tt.obs_of[c] = c < ncell ? m->obs_of_cell[c] : -1;
            tt.init[c] = c < ncell ? m->init[c] : 0;
        }
    }
    return CWC_OK;
}

template <typename T>
size_t push_bytes(std::vector<unsigned char> &blob, const std::vector<T> &v) {
    size_t off = (blob.size() + 255) & ~size_t(255);
    blob.resize(off + std::max<size_t>(v.size() * sizeof(T), 16));
    if (!v.empty()) std::memcpy(blob.data() + off, v.data(), v.size() * sizeof(T));
    return off;
}

// The model's tables on the calling thread's current CUDA device: uploaded
// there on first use (one copy per device, so one handle can serve several
// GPUs of a process), under the handle's mutex (concurrent first calls
// upload once).
cwc_status device_tables(cwc_model_s *m, const WarpTables **out) {
    int ndev = 0;
    cudaError_t e0 = cudaGetDeviceCount(&ndev);
    if (e0 != cudaSuccess || ndev == 0) return fail(CWC_ERR_CUDA, "no CUDA device (there is no CPU fallback)");
    int device = 0;
    cudaError_t e = cudaGetDevice(&device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    std::lock_guard<std::mutex> lock(m->dev_mu);
    auto it = m->dev.find(device);
    if (it != m->dev.end()) {
        *out = &it->second->wt;
        return CWC_OK;
    }
    std::vector<unsigned char> blob;
    std::vector<int2> nu2(m->nu_cell.size());
    for (size_t q = 0; q < nu2.size(); ++q) nu2[q] = make_int2(m->nu_cell[q], m->nu_delta[q]);
    const size_t o_rx = push_bytes(blob, m->rx), o_nup = push_bytes(blob, m->nu_ptr), o_nu = push_bytes(blob, nu2),
                 o_dp = push_bytes(blob, m->dep_ptr), o_dep = push_bytes(blob, m->dep_slot), o_dep16 = push_bytes(blob, m->dep_slot16), o_dep4 = push_bytes(blob, m->dep_slot4), o_dep16_4 = push_bytes(blob, m->dep_slot16_4), o_op = push_bytes(blob, m->obs_ptr),
                 o_whdr = push_bytes(blob, m->wseg_hdr), o_wnu = push_bytes(blob, m->wseg_nu),
                 o_wd16 = push_bytes(blob, m->wseg_dep16), o_wd32 = push_bytes(blob, m->wseg_dep32),
                 o_oc = push_bytes(blob, m->obs_cells), o_init = push_bytes(blob, m->init),
                 o_wnu8 = push_bytes(blob, m->wseg_nu8), o_wd4 = push_bytes(blob, m->wseg_dep4),
                 o_wd8 = push_bytes(blob, m->wseg_dep8);
    std::unique_ptr<cwc_model_s::DevCopy> dc(new (std::nothrow) cwc_model_s::DevCopy());
    if (!dc) return fail(CWC_ERR_NOMEM, "host allocation");
    e = cudaMalloc(&dc->buf.p, blob.size());
    if (e == cudaErrorMemoryAllocation) return fail(CWC_ERR_NOMEM, "model tables: device allocation");
    if (e != cudaSuccess) return cuda_fail(e, "model tables: cudaMalloc");
    e = cudaMemcpy(dc->buf.p, blob.data(), blob.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "model tables: cudaMemcpy");
    unsigned char *b = (unsigned char *)dc->buf.p;
    WarpTables &w = dc->wt;
    w = m->wt;
    w.rx = (const ReactionDesc *)(b + o_rx);
    w.nu_ptr = (const int32_t *)(b + o_nup);
    w.nu = (const int2 *)(b + o_nu);
    w.dep_ptr = (const int32_t *)(b + o_dp);
    w.dep = (const int2 *)(b + o_dep);
    w.dep16 = (const int2 *)(b + o_dep16);
    w.dep4 = (const int4 *)(b + o_dep4);
    w.dep16_4 = (const int4 *)(b + o_dep16_4);
    w.obs_ptr = (const int32_t *)(b + o_op);
    w.obs_cells = (const int32_t *)(b + o_oc);
    w.init = (const int32_t *)(b + o_init);
    w.hdr = (const int4 *)(b + o_whdr);
    w.nuw = (const int2 *)(b + o_wnu);
    w.depw16 = (const int4 *)(b + o_wd16);
    w.depw32 = (const int4 *)(b + o_wd32);
    w.nuw8 = (const int2 *)(b + o_wnu8);
    w.depw4 = (const int4 *)(b + o_wd4);
    w.depw8 = (const int4 *)(b + o_wd8);
    *out = &dc->wt;
    m->dev.emplace(device, std::move(dc));
    return CWC_OK;
}

// ---- launch planning ----------------------------------------------------------
struct Plan {
    int path = 0;
    int64_t G = 0, R = 0;
    int64_t n_launch = 0;  // trajectories in this launch (resumable runs: the live ones)
    int32_t P = 1, J = 0;
    int64_t n_stat_cells = 0;  // P * (J+1) * O
    // thread path
    int threads = 128;
    int s_pad = 0, m_pad = 0;
    // warp path
    int warps_per_block = 4;
    int blocks = 0;
    // stats
    int stats_smem = 0;
    int ws = 0;
    int seg2 = 0;  // warp path: two trajectories per warp
    int grp8 = 0;  // warp path: eight trajectories per warp (4-lane groups)
    int grp4 = 0;  // warp path: four trajectories per warp (8-lane groups)
    int nt = 1;    // thread path, single-warp kernel: trajectories per lane
    StatLayout st{};
    int64_t cells_per_part = 0;
    int n_parts = 1;
    int64_t traj_per_part = 0;
    size_t smem_bytes = 0;
    // workspace layout
    size_t off_rates = 0, off_parts = 0, off_trace = 0, off_counter = 0, off_order = 0, off_smctr = 0, off_stats = 0,
           total = 0;
};

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

// the planner's automatic choice of the 4-lane-group kernel: networks of up
// to 128 reactions (B4 <= 32).  Measured (tools/warp8_crossover.py,
// profiles/r02/warp8/): 1.2-1.45x the two-per-warp kernel up to M = 128,
// slower from M ~ 160 on (C4, M = 256: 3.15e9 vs 4.59e9 -- its 16 KB of
// propensities per warp leave 9 warps per SM, too few to hide latency)
constexpr int kWarp8AutoMaxB4 = 32;
// ... and of the 8-lane-group kernel beyond that (up to 256 reactions)
constexpr bool kWarp4Auto = false;

const char *env(const char *k) {
    const char *v = std::getenv(k);
    return (v && *v) ? v : nullptr;
}

int sm_count() {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

// resumable = cwc_run_* (global statistics accumulators, no warp-specialised
// kernel, n_launch = live trajectories of this launch; -1 = all G)
cwc_status plan_run(const cwc_model_s *m, int64_t n_replicas, const cwc_sweep *sweep, double t_end, double dt,
                    const cwc_sim_opts *opts, bool host_stats, Plan &pl, bool resumable = false,
                    int64_t n_launch = -1) {
    if (!m) return fail(CWC_ERR_INVALID, "model is NULL");
    if (!(t_end > 0.0) || !std::isfinite(t_end)) return fail(CWC_ERR_INVALID, "t_end must be finite and > 0");
    if (!(dt > 0.0) || !std::isfinite(dt)) return fail(CWC_ERR_INVALID, "sample_dt must be finite and > 0");
    if (dt > t_end) return fail(CWC_ERR_INVALID, "sample_dt must be <= t_end");
    if (n_replicas < 1) return fail(CWC_ERR_INVALID, "n_replicas must be >= 1");
    const double Jd = std::floor(t_end / dt);
    if (Jd > 2e9) return fail(CWC_ERR_INVALID, "too many samples");
    pl.J = (int32_t)Jd;
    pl.P = 1;
    if (sweep) {
        if (sweep->n_points < 1) return fail(CWC_ERR_INVALID, "sweep.n_points must be >= 1");
        if (sweep->n_swept < 0 || (sweep->n_swept > 0 && (!sweep->rule || !sweep->value)))
            return fail(CWC_ERR_INVALID, "bad sweep arrays");
        for (int i = 0; i < sweep->n_swept; ++i)
            if (sweep->rule[i] < 0 || sweep->rule[i] >= m->n_rules) return fail(CWC_ERR_INVALID, "sweep rule id out of range");
        for (long long i = 0; i < (long long)sweep->n_points * sweep->n_swept; ++i)
            if (!finite_pos(sweep->value[i])) return fail(CWC_ERR_INVALID, "sweep value must be finite and >= 2^-1021");
        pl.P = sweep->n_points;
    }
    pl.R = n_replicas;
    if ((double)pl.P * (double)n_replicas >= 4294967296.0)  // statistics words take < 2^32 adds
        return fail(CWC_ERR_INVALID, "too many trajectories in one call (shard the run: replica_offset)");
    pl.G = (int64_t)pl.P * n_replicas;
    if (resumable && opts && opts->n_trace > 0) return fail(CWC_ERR_INVALID, "resumable runs do not trace (n_trace must be 0)");
    const int64_t NL = (n_launch < 0) ? pl.G : std::min<int64_t>(n_launch, pl.G);  // trajectories launched
    pl.n_launch = NL;
    const int64_t J1 = (int64_t)pl.J + 1;
    const int O = m->n_obs;
    pl.n_stat_cells = (int64_t)pl.P * J1 * O;
    const int nsm = sm_count();

    int force = opts ? opts->force_path : CWC_PATH_AUTO;
    const int kern = opts ? opts->kernel : CWC_KERNEL_AUTO;
    const int smode = opts ? opts->stats_mode : CWC_STATS_AUTO;
    const int wpb = opts ? opts->warps_per_block : 0;
    const int bps = opts ? opts->blocks_per_sm : 0;
    if (kern < CWC_KERNEL_AUTO || kern > CWC_KERNEL_WARP4) return fail(CWC_ERR_INVALID, "bad kernel");
    if (smode < CWC_STATS_AUTO || smode > CWC_STATS_GLOBAL) return fail(CWC_ERR_INVALID, "bad stats_mode");
    if (wpb < 0 || wpb > 4) return fail(CWC_ERR_INVALID, "warps_per_block must be in [0, 4]");
    if (bps < 0 || bps > 32) return fail(CWC_ERR_INVALID, "blocks_per_sm must be in [0, 32]");
    if (force != CWC_PATH_AUTO && force != CWC_PATH_THREAD && force != CWC_PATH_WARP) return fail(CWC_ERR_INVALID, "bad force_path");
    if (kern == CWC_KERNEL_THREAD_WS || kern == CWC_KERNEL_THREAD || kern == CWC_KERNEL_THREAD2 ||
        kern == CWC_KERNEL_THREAD_WS2) {
        if (force == CWC_PATH_WARP) return fail(CWC_ERR_INVALID, "kernel does not match force_path");
        force = CWC_PATH_THREAD;
    } else if (kern == CWC_KERNEL_WARP2 || kern == CWC_KERNEL_WARP || kern == CWC_KERNEL_WARP8 || kern == CWC_KERNEL_WARP4) {
        if (force == CWC_PATH_THREAD) return fail(CWC_ERR_INVALID, "kernel does not match force_path");
        force = CWC_PATH_WARP;
    }
    if (force == CWC_PATH_THREAD && !m->thread_ok) return fail(CWC_ERR_INVALID, "thread path cannot run this model (too many cells/reactions/observables)");
    pl.path = (force == CWC_PATH_AUTO) ? (m->thread_ok ? CWC_PATH_THREAD : CWC_PATH_WARP) : force;
    const int bt = opts ? opts->block_threads : 0;
    if (bt != 0 && (bt < 32 || bt > 256 || bt % 32)) return fail(CWC_ERR_INVALID, "block_threads must be a multiple of 32 in [32, 256]");
    // exact integer moments: every per-cell sum of observables (< 2^vbits)
    // over all replicas of the (sharded) run must fit int64 (stage 2 and the
    // multi-GPU merge narrow the exact sum to int64)
    {
        const double r_all = (opts && opts->replicas_total > 0) ? (double)opts->replicas_total : (double)n_replicas;
        if (r_all * std::ldexp(1.0, m->vbits) >= 9.2e18)
            return fail(CWC_ERR_INVALID, "observable sums over the replicas could exceed int64 (fewer replicas per point)");
    }
    if (resumable && smode == CWC_STATS_SHARED) return fail(CWC_ERR_INVALID, "resumable runs accumulate in global memory (stats_mode)");
    const size_t smem_cap = 200 * 1024;

    if (pl.path == CWC_PATH_THREAD) {
        pl.s_pad = thread_pad_cells(m->n_cells);
        pl.m_pad = thread_pad_reactions(std::max(m->M, 2));
        if (pl.s_pad < 0 || pl.m_pad < 0) return fail(CWC_ERR_INVALID, "thread path padding");
        // one-warp CTAs: the block scheduler then spreads trajectories of
        // unequal length (sweeps: 17x spread in C3) evenly over the SMs and
        // refills SMs as warps finish; the thread path is latency-bound, so
        // nothing is gained from larger CTAs
        int T = bt ? bt : 32;
        // warp-specialised producer/consumer CTAs (2 warps per 32 trajectories,
        // ssa_thread_ws.cuh) while at most two of them
        // share an SM (their consumer and producer warps then own their
        // sub-partitions: C1); beyond that the single-warp kernel, whose
        // warps carry their own draws, is faster (measured with the
        // table-driven log: C2 at 16384 replicas 8.58e10 vs 8.41e10
        // firings/s; one lone CTA 274 vs 355 cycles per firing)
        bool ws = !bt && (pl.G + 31) / 32 <= 2ll * nsm;
        // two trajectories per consumer lane (ssa_thread_ws2.cuh) only on
        // request: measured 2x slower per trajectory on C2 (a consumer with
        // two interleaved chains takes ~650 cycles per firing pair, against
        // ~290 per firing with one: the consumer is throughput-, not
        // latency-bound), with one or two producer warps alike
        int ws2 = 0;
        if (kern == CWC_KERNEL_THREAD_WS2) {
            if (resumable || bt || pl.m_pad > 8)
                return fail(CWC_ERR_INVALID, "kernel THREAD_WS2 needs M <= 8, a one-shot run and no block_threads");
            ws2 = 1;
        }
        if (ws2) ws = true;
        if (kern == CWC_KERNEL_THREAD_WS) {
            if (resumable) return fail(CWC_ERR_INVALID, "resumable runs do not use the warp-specialised kernel");
            if (bt && bt != 32 * kWsGroups) return fail(CWC_ERR_INVALID, "the warp-specialised kernel has a fixed CTA shape (block_threads)");
            ws = true;
        } else if (kern == CWC_KERNEL_THREAD || kern == CWC_KERNEL_THREAD2) {
            ws = false;
        }
        if (resumable) ws = false;
        if (kern == CWC_KERNEL_THREAD_WS || kern == CWC_KERNEL_THREAD) ws2 = 0;
        if (ws) T = ws2 ? 64 : 32 * kWsGroups;
        pl.ws = ws ? (ws2 ? 2 : 1) : 0;
        pl.threads = T;
        // single-warp kernel: two trajectories per lane (ssa_thread_impl.cuh
        // NT) only on request -- measured 3x slower on C2/C3 (the doubled
        // per-trajectory state spills at 255 registers)
        pl.nt = (!ws && !resumable && pl.m_pad <= 8 && kern == CWC_KERNEL_THREAD2) ? 2 : 1;
        if (kern == CWC_KERNEL_THREAD2 && pl.nt != 2)
            return fail(CWC_ERR_INVALID, "kernel THREAD2 needs M <= 8 and a one-shot run");
        const int64_t blocks = (NL + (int64_t)T * pl.nt - 1) / ((int64_t)T * pl.nt);  // (ws2: T = 64 trajectories)
        if (blocks > 0x7fffffffll) return fail(CWC_ERR_INVALID, "too many trajectories for one launch");
        pl.blocks = (int)blocks;
        // points touched by one block
        int64_t np_max = 1;
        const int64_t TB = (int64_t)T * pl.nt;  // trajectories per block
        for (int64_t b = 0; b < blocks; ++b) {
            const int64_t pf = (b * TB) / pl.R, plst = (std::min<int64_t>((b + 1) * TB, pl.G) - 1) / pl.R;
            np_max = std::max(np_max, plst - pf + 1);
            if (np_max >= pl.P) break;
        }
        const int64_t cells = stat_cells_round(np_max * J1 * O);
        const StatLayout lay_s = stat_layout(true, m->vbits), lay_g = stat_layout(false, m->vbits);
        const size_t smem = (size_t)stat_bytes(lay_s, cells);
        // beyond the statistics part: the draw ring + staging of the
        // warp-specialised CTA, or the record staging of each warp
        const size_t extra = (ws ? (pl.ws == 2 ? kWs2RingBytes : kWsRingBytes) : (size_t)(T / 32) * kStageLL * sizeof(long long)) +
                             kNegLogSmemBytes;
        // One global part (fire-and-forget 64-bit REDs to L2) by default:
        // measured faster than per-CTA shared-memory parts on every config
        // (profiles/r02/stats_modes.json: C1 4.60e9 vs 4.17e9, C2 8.95e10 vs
        // 4.56e10, C3 6.77 vs 7.27 ms per step); crossings are too rare for
        // L2 contention, and shared parts cost occupancy, zeroing and a
        // larger stage 2.  CWC_STATS_SHARED keeps the block-level reduction
        // available (same results bit for bit).
        bool use_smem = false;
        if (smode == CWC_STATS_SHARED) {
            if (smem + extra > smem_cap) return fail(CWC_ERR_INVALID, "stats_mode SHARED: the part does not fit in shared memory");
            use_smem = true;
        }
        if (smode == CWC_STATS_GLOBAL || O == 0 || resumable) use_smem = false;
        if (use_smem) {
            pl.stats_smem = 1;
            pl.st = lay_s;
            pl.cells_per_part = std::max<int64_t>(cells, 4);
            pl.n_parts = pl.blocks;
            pl.traj_per_part = (int64_t)T * pl.nt;
            pl.smem_bytes = smem + extra;
        } else {
            pl.stats_smem = 0;
            pl.st = lay_g;
            pl.cells_per_part = std::max<int64_t>(stat_cells_round(pl.n_stat_cells), 4);
            // one global part: its 64-bit words take 2^32 adds of 32-bit limbs
            // (G < 2^32), and crossings are far too rare to contend in L2
            pl.n_parts = 1;
            pl.traj_per_part = 0;
            pl.smem_bytes = extra;
        }
    } else {
        const WarpTables &w = m->wt;
        int W = bt ? std::min(bt / 32, 4) : 4;  // ssa_warp_kernel is built for <= 128 threads
        if (wpb) W = wpb;
        pl.warps_per_block = W;
        // two trajectories per warp (16-lane segments) when a segment's chunks
        // stay short (M <= 256)
        bool seg2 = w.B16 <= 16;
        // eight trajectories per warp (4-lane groups) for M <= 256 one-shot
        // runs with one global statistics part (ssa_warp8.cu)
        const bool grp_ok = w.B4 <= 64 && !resumable && smode != CWC_STATS_SHARED;
        bool grp8 = grp_ok, grp4 = false;
        if (kern == CWC_KERNEL_WARP2) {
            if (!seg2) return fail(CWC_ERR_INVALID, "kernel WARP2 needs M <= 256");
            grp8 = false;
        } else if (kern == CWC_KERNEL_WARP) {
            seg2 = false;
            grp8 = false;
        } else if (kern == CWC_KERNEL_WARP8) {
            if (!grp8) return fail(CWC_ERR_INVALID, "kernel WARP8 needs M <= 256, a one-shot run and global statistics");
        } else if (kern == CWC_KERNEL_WARP4) {
            if (!grp_ok) return fail(CWC_ERR_INVALID, "kernel WARP4 needs M <= 256, a one-shot run and global statistics");
            grp8 = false;
            grp4 = true;
        } else if (kern == CWC_KERNEL_AUTO) {
            grp8 = grp_ok && w.B4 <= kWarp8AutoMaxB4;
            grp4 = grp_ok && !grp8 && kWarp4Auto;
        }
        if (grp8 || grp4) seg2 = false;
        pl.seg2 = seg2 ? 1 : 0;
        pl.grp8 = grp8 ? 1 : 0;
        pl.grp4 = grp4 ? 1 : 0;
        if ((grp8 || grp4) && !wpb) W = 1;
        pl.warps_per_block = W;
        const size_t per_warp = (grp8 || grp4) ? ((group_smem_per_warp(w, grp8 ? 4 : 8) + 15) & ~(size_t)15)
                                               : (seg2 ? warp2_smem_per_warp(w) : warp_smem_per_warp(w));
        const int64_t cells = std::max<int64_t>(stat_cells_round(pl.n_stat_cells), 4);
        const StatLayout lay_s = stat_layout(true, m->vbits), lay_g = stat_layout(false, m->vbits);
        const size_t stats = (size_t)stat_bytes(lay_s, cells);
        // one global part by default (see the thread path; C4 4.58e9 vs
        // 0.86e9, C5 1.50e9 vs 0.46e9 with shared-memory parts, which halve
        // the resident warps)
        bool use_smem = false;
        if (smode == CWC_STATS_SHARED) {
            if (stats + W * per_warp > smem_cap) return fail(CWC_ERR_INVALID, "stats_mode SHARED: the part does not fit in shared memory");
            use_smem = true;
        }
        if (smode == CWC_STATS_GLOBAL || O == 0 || resumable || grp8 || grp4) use_smem = false;
        pl.stats_smem = use_smem ? 1 : 0;
        pl.st = use_smem ? lay_s : lay_g;
        pl.cells_per_part = cells;
        pl.smem_bytes = (use_smem ? stats : 0) + W * per_warp;
        if (pl.smem_bytes > smem_cap + 27 * 1024) return fail(CWC_ERR_UNSUPPORTED, "warp path: per-warp state does not fit in shared memory");
        // persistent grid: resident blocks on all SMs
        int per_sm = 1;
        // occupancy by shared memory / threads
        const int by_smem = (int)std::max<size_t>(1, (228 * 1024) / (pl.smem_bytes + 1024));
        const int by_threads = std::max(1, 2048 / (W * 32));
        per_sm = std::min(std::min(by_smem, by_threads), 32);
        if (bps) per_sm = std::min(per_sm, bps);
        int64_t blocks = (int64_t)nsm * per_sm;
        const int tpw = grp8 ? 8 : grp4 ? 4 : (seg2 ? 2 : 1);  // trajectories per warp
        blocks = std::min<int64_t>(blocks, (NL + (int64_t)W * tpw - 1) / ((int64_t)W * tpw));
        pl.blocks = (int)std::max<int64_t>(1, blocks);
        pl.threads = W * 32;
        // a shared-memory part takes <= 2^16 trajectories (16-bit limbs); the
        // kernel caps each CTA at that, so the grid must cover G with it
        if (use_smem && (int64_t)pl.blocks * kSmemPartMaxTraj < pl.G) {
            if (smode == CWC_STATS_SHARED) return fail(CWC_ERR_INVALID, "stats_mode SHARED: too many trajectories per CTA part");
            use_smem = false;
            pl.stats_smem = 0;
            pl.st = lay_g;
            pl.smem_bytes = W * per_warp;
        }
        pl.traj_per_part = 0;
        if (use_smem) {
            pl.n_parts = pl.blocks;
        } else {
            pl.n_parts = 1;  // one global part (see the thread path)
        }
    }

    // workspace
    size_t off = 0;
    pl.off_rates = off;  // rates [P][M] then rates_h [P][M]
    off = align256(off + 2 * sizeof(double) * (size_t)pl.P * std::max(m->M, 1));
    pl.off_parts = off;
    off = align256(off + (size_t)stat_bytes(pl.st, pl.cells_per_part) * pl.n_parts);
    pl.off_trace = off;
    off = align256(off + sizeof(int64_t) * (size_t)std::max(opts ? opts->n_trace : 0, 1));
    pl.off_counter = off;
    off = align256(off + 16);
    pl.off_order = off;
    if (pl.path == CWC_PATH_THREAD && pl.P > 1) off = align256(off + sizeof(int32_t) * (size_t)pl.blocks);
    pl.off_smctr = off;
    if (pl.ws) off = align256(off + sizeof(unsigned) * 1024);
    pl.off_stats = off;
    if (host_stats) off = align256(off + (size_t)32 * std::max<int64_t>(pl.n_stat_cells, 1));
    pl.total = off;
    return CWC_OK;
}

// per-point flat rates [P][M] (host expansion of the sweep),
// followed by the same with A + A entries halved ([P][M], exact: the segment
// kernel forms k/2 RN(x (x - 1)) == k RN(x (x - 1) / 2))
std::vector<double> expand_rates(const cwc_model_s *m, const Plan &pl, const cwc_sweep *sweep) {
    const int M = m->M;
    const size_t PM = (size_t)pl.P * std::max(M, 1);
    std::vector<double> rates(2 * PM, 0.0);
    std::vector<double> rule_rates(m->rule_rate);
    for (int p = 0; p < pl.P; ++p) {
        if (sweep)
            for (int i = 0; i < sweep->n_swept; ++i) rule_rates[sweep->rule[i]] = sweep->value[(size_t)p * sweep->n_swept + i];
        for (int k = 0; k < M; ++k) {
            const double r = rule_rates[m->entry_rule[k]];
            rates[(size_t)p * M + k] = r;
            rates[PM + (size_t)p * M + k] = (m->rx[k].kind >> 1) ? r * 0.5 : r;
        }
    }
    return rates;
}

// Expected work of each point's trajectories: the total propensity a0(x0)
// (firings per unit time at t = 0), the longest-first dispatch key for sweeps.
std::vector<double> point_a0(const cwc_model_s *m, const Plan &pl, const std::vector<double> &rates) {
    const int M = m->M;
    std::vector<double> a0p(pl.P, 0.0);
    for (int p = 0; p < pl.P; ++p) {
        double a0 = 0.0;
        for (int k = 0; k < M; ++k) {
            const ReactionDesc &r = m->rx[k];
            const double xa = r.ia < m->n_cells ? (double)m->init[r.ia] : 1.0;
            const double xb = r.ib < m->n_cells ? (double)m->init[r.ib] - (r.kind & 1) : 1.0;
            a0 += rates[(size_t)p * M + k] * xa * xb / ((r.kind >> 1) ? 2.0 : 1.0);
        }
        a0p[p] = a0;
    }
    return a0p;
}

// Groups of T consecutive trajectories in longest-expected-first order.
std::vector<int32_t> lpt_groups(const Plan &pl, const std::vector<double> &a0p, int64_t T) {
    const int64_t n_groups = (pl.G + T - 1) / T;
    std::vector<std::pair<double, int32_t>> w8(n_groups);
    for (int64_t b = 0; b < n_groups; ++b) {
        double s = 0.0;
        const int64_t ge = std::min<int64_t>((b + 1) * T, pl.G);
        for (int64_t gg = b * T; gg < ge; ++gg) s += a0p[gg / pl.R];
        w8[b] = {-s, (int32_t)b};
    }
    std::stable_sort(w8.begin(), w8.end());
    std::vector<int32_t> order(n_groups);
    for (int64_t b = 0; b < n_groups; ++b) order[b] = w8[b].second;
    return order;
}

// Sharding and optional outputs of opts (both one-shot and resumable runs).
cwc_status apply_shard(RunParams &rp, const cwc_sim_opts *opts, int64_t n_replicas) {
    if (!opts) return CWC_OK;
    if (opts->replicas_total != 0) {
        if (opts->replica_offset < 0 || opts->replicas_total < opts->replica_offset + n_replicas)
            return fail(CWC_ERR_INVALID, "replica_offset + n_replicas must be <= replicas_total");
        rp.R_total = opts->replicas_total;
        rp.r_off = opts->replica_offset;
    } else if (opts->replica_offset != 0) {
        return fail(CWC_ERR_INVALID, "replica_offset needs replicas_total");
    }
    rp.out_traj = opts->out_traj;
    rp.out_firings = opts->out_firings;
    rp.out_status = opts->out_status;
    return CWC_OK;
}

cudaError_t launch_ssa(const cwc_model_s *m, const WarpTables &wt, const Plan &pl, const RunParams &rp,
                       cudaStream_t stream) {
    if (pl.path == CWC_PATH_THREAD)
        return launch_ssa_thread(pl.s_pad, pl.m_pad, rp, m->tt, pl.threads, pl.smem_bytes, stream);
    if (pl.grp8 || pl.grp4)
        return launch_ssa_group(pl.grp8 ? 4 : 8, rp, wt, pl.blocks, pl.warps_per_block, pl.smem_bytes, stream);
    return pl.seg2 ? launch_ssa_warp2(rp, wt, pl.blocks, pl.warps_per_block, pl.smem_bytes, stream)
                   : launch_ssa_warp(rp, wt, pl.blocks, pl.warps_per_block, pl.smem_bytes, stream);
}

cwc_status run(cwc_model m, int64_t n_replicas, const cwc_sweep *sweep, double t_end, double dt, uint64_t seed,
               void *stream_, cwc_stats st, void *ws, size_t ws_bytes, const cwc_sim_opts *opts, bool host_stats,
               cwc_stats host_out) {
    if (!m) return fail(CWC_ERR_INVALID, "model is NULL");
    const WarpTables *dwt = nullptr;  // tables go to the device on first use (host-only creation needs no GPU)
    cwc_status su = device_tables(m, &dwt);
    if (su != CWC_OK) return su;
    Plan pl;
    cwc_status s = plan_run(m, n_replicas, sweep, t_end, dt, opts, host_stats, pl);
    if (s != CWC_OK) return s;
    if (!ws && pl.total > 0) return fail(CWC_ERR_INVALID, "workspace is NULL");
    if (ws_bytes < pl.total) return fail(CWC_ERR_INVALID, "workspace too small: need " + std::to_string(pl.total) + " bytes");
    if (opts && opts->n_trace > 0 && (!opts->trace_g || !opts->trace_buf || !opts->trace_len || opts->trace_cap < 1))
        return fail(CWC_ERR_INVALID, "trace arguments incomplete");
    if (pl.n_stat_cells > 0 && (!st.count || !st.sum || !st.sumsq)) return fail(CWC_ERR_INVALID, "stats pointers are NULL");
    cudaStream_t stream = (cudaStream_t)stream_;
    unsigned char *w = (unsigned char *)ws;

    // per-point rates (and, for sweeps on the thread path, the dispatch
    // order) through the model's pinned staging (cwc_model_s::Stage)
    const bool want_order = pl.path == CWC_PATH_THREAD && pl.P > 1;
    const int T_order = pl.ws == 2 ? 64 : pl.ws ? 32 * kWsGroups : pl.threads * pl.nt;
    cudaError_t e = cudaSuccess;
    {
        uint64_t key = 0xcbf29ce484222325ull;
        const int64_t shape[6] = {pl.P, m->M, pl.R, pl.blocks, want_order ? T_order : 0, sweep ? sweep->n_swept : -1};
        key = fnv1a(key, shape, sizeof(shape));
        if (sweep && sweep->n_swept > 0) {
            key = fnv1a(key, sweep->rule, sizeof(int32_t) * sweep->n_swept);
            key = fnv1a(key, sweep->value, sizeof(double) * (size_t)sweep->n_points * sweep->n_swept);
        }
        int device = 0;
        if ((e = cudaGetDevice(&device)) != cudaSuccess) return cuda_fail(e, "cwc_simulate: cudaGetDevice");
        std::lock_guard<std::mutex> lock(m->stage_mu);
        cwc_model_s::Stage &sg = m->stage[device];
        if (!sg.valid || sg.key != key) {
            if (sg.done && (e = cudaEventSynchronize(sg.done)) != cudaSuccess) return cuda_fail(e, "cwc_simulate: staging");
            const std::vector<double> rates = expand_rates(m, pl, sweep);
            std::vector<int32_t> order;
            // Parameter sweeps: trajectory lengths differ by point (C3: 17x),
            // and CTAs start in blockIdx order as the SMs free up.  Dispatch
            // the groups longest-expected-first (LPT), estimating a group's
            // work by the total propensity a0(x0) of its trajectories' points
            // (firings per unit time at t = 0).  Trajectory ids -- hence the
            // RNG streams and every result -- are unchanged; only the start
            // order moves.
            if (want_order) order = lpt_groups(pl, point_a0(m, pl, rates), T_order);
            sg.rates_bytes = sizeof(double) * rates.size();
            sg.order_off = align256(sg.rates_bytes);
            sg.order_bytes = sizeof(int32_t) * order.size();
            const size_t need = sg.order_off + sg.order_bytes;
            if (need > sg.cap) {
                if (sg.pinned) cudaFreeHost(sg.pinned);
                sg.pinned = nullptr;
                sg.cap = 0;
                sg.valid = false;
                if ((e = cudaHostAlloc((void **)&sg.pinned, need, cudaHostAllocDefault)) != cudaSuccess)
                    return cuda_fail(e, "cwc_simulate: pinned staging");
                sg.cap = need;
            }
            std::memcpy(sg.pinned, rates.data(), sg.rates_bytes);
            if (!order.empty()) std::memcpy(sg.pinned + sg.order_off, order.data(), sg.order_bytes);
            if (!sg.done && (e = cudaEventCreateWithFlags(&sg.done, cudaEventDisableTiming)) != cudaSuccess)
                return cuda_fail(e, "cwc_simulate: staging event");
            sg.key = key;
            sg.valid = true;
        }
        e = cudaMemcpyAsync(w + pl.off_rates, sg.pinned, sg.rates_bytes, cudaMemcpyHostToDevice, stream);
        if (e == cudaSuccess && want_order)
            e = cudaMemcpyAsync(w + pl.off_order, sg.pinned + sg.order_off, sg.order_bytes, cudaMemcpyHostToDevice, stream);
        if (e == cudaSuccess) e = cudaEventRecord(sg.done, stream);
        if (e != cudaSuccess) return cuda_fail(e, "cwc_simulate: rates upload");
    }

    RunParams rp{};
    rp.G = pl.G;
    rp.R = pl.R;
    rp.R_total = pl.R;
    rp.r_off = 0;
    rp.P = pl.P;
    rp.J = pl.J;
    rp.dt = dt;
    rp.seed = seed;
    set_round_keys(rp);
    rp.rates = (const double *)(w + pl.off_rates);
    rp.rates_h = rp.rates + (size_t)pl.P * std::max(m->M, 1);
    rp.n_launch = pl.G;
    rp.j_stop = (int64_t)pl.J + 1;
    rp.parts = w + pl.off_parts;
    rp.cells_per_part = pl.cells_per_part;
    rp.st = pl.st;
    rp.ws = pl.ws;
    rp.thread_nt = pl.nt;
    rp.stats_smem = pl.stats_smem;
    rp.n_parts = pl.n_parts;
    rp.traj_per_part = pl.traj_per_part;
    rp.next_traj = (unsigned long long *)(w + pl.off_counter);
#ifdef CWC_DEBUG_KNOBS  // debug builds only (tools/ws_prof.py): consumer cycle accounting buffer
    if (const char *e = env("CWC_PROF_PTR")) rp.prof = (unsigned long long *)std::strtoull(e, nullptr, 0);
#endif
    if (opts) {
        s = apply_shard(rp, opts, n_replicas);
        if (s != CWC_OK) return s;
        if (opts->n_trace > 0) {
            e = cudaMemcpyAsync(w + pl.off_trace, opts->trace_g, sizeof(int64_t) * opts->n_trace, cudaMemcpyHostToDevice, stream);
            if (e != cudaSuccess) return cuda_fail(e, "cwc_simulate: trace ids upload");
            e = cudaMemsetAsync(opts->trace_len, 0, sizeof(int64_t) * opts->n_trace, stream);
            if (e != cudaSuccess) return cuda_fail(e, "cwc_simulate: trace_len");
            rp.trace_g = (const int64_t *)(w + pl.off_trace);
            rp.n_trace = opts->n_trace;
            rp.trace_cap = opts->trace_cap;
            rp.trace_buf = opts->trace_buf;
            rp.trace_len = opts->trace_len;
        }
    }
    if (!pl.stats_smem) {
        e = cudaMemsetAsync(w + pl.off_parts, 0, (size_t)stat_bytes(pl.st, pl.cells_per_part) * pl.n_parts, stream);
        if (e != cudaSuccess) return cuda_fail(e, "cwc_simulate: zero partials");
    }
    if (want_order) rp.cta_order = (const int32_t *)(w + pl.off_order);
    // Alternating consumer/producer placement per SM (CWC_WS_MIX=1) was
    // measured slower on C2: a producer's fp64-heavy log stream on the same
    // sub-partition delays the consumer's fp64 chain more than a second
    // consumer does.  Kept as an experiment switch.
#ifdef CWC_DEBUG_KNOBS
    if (pl.ws && env("CWC_WS_MIX") && std::atoi(env("CWC_WS_MIX")) != 0) {
        e = cudaMemsetAsync(w + pl.off_smctr, 0, sizeof(unsigned) * 1024, stream);
        if (e != cudaSuccess) return cuda_fail(e, "cwc_simulate: SM counters");
        rp.sm_ctr = (unsigned *)(w + pl.off_smctr);
    }
#endif
    e = cudaMemsetAsync(w + pl.off_counter, 0, 16, stream);
    if (e != cudaSuccess) return cuda_fail(e, "cwc_simulate: counter");

    cudaEvent_t ev0 = opts ? (cudaEvent_t)opts->ev_kernel_begin : nullptr;
    cudaEvent_t ev1 = opts ? (cudaEvent_t)opts->ev_kernel_end : nullptr;
    if (ev0 && (e = cudaEventRecord(ev0, stream)) != cudaSuccess) return cuda_fail(e, "cwc_simulate: ev_kernel_begin");
    e = launch_ssa(m, *dwt, pl, rp, stream);
    if (e != cudaSuccess) return cuda_fail(e, "cwc_simulate: SSA kernel launch");
    if (ev1 && (e = cudaEventRecord(ev1, stream)) != cudaSuccess) return cuda_fail(e, "cwc_simulate: ev_kernel_end");
    cwc_stats dst = st;
    if (host_stats) {
        unsigned char *sb = w + pl.off_stats;
        dst.count = (int64_t *)sb;
        dst.sum = (int64_t *)(sb + 8 * pl.n_stat_cells);
        dst.sumsq = (uint64_t *)(sb + 16 * pl.n_stat_cells);
    }
    if (pl.n_stat_cells > 0) {
        cudaEvent_t es0 = opts ? (cudaEvent_t)opts->ev_stage2_begin : nullptr;
        cudaEvent_t es1 = opts ? (cudaEvent_t)opts->ev_stage2_end : nullptr;
        if (es0 && (e = cudaEventRecord(es0, stream)) != cudaSuccess) return cuda_fail(e, "cwc_simulate: ev_stage2_begin");
        e = launch_stats_stage2(rp, m->n_obs, dst.count, dst.sum, dst.sumsq, stream);
        if (e != cudaSuccess) return cuda_fail(e, "cwc_simulate: stage-2 launch");
        if (es1 && (e = cudaEventRecord(es1, stream)) != cudaSuccess) return cuda_fail(e, "cwc_simulate: ev_stage2_end");
        if (host_stats) {
            const size_t n8 = 8 * (size_t)pl.n_stat_cells;
            if ((e = cudaMemcpyAsync(host_out.count, dst.count, n8, cudaMemcpyDeviceToHost, stream)) != cudaSuccess ||
                (e = cudaMemcpyAsync(host_out.sum, dst.sum, n8, cudaMemcpyDeviceToHost, stream)) != cudaSuccess ||
                (e = cudaMemcpyAsync(host_out.sumsq, dst.sumsq, 2 * n8, cudaMemcpyDeviceToHost, stream)) != cudaSuccess)
                return cuda_fail(e, "cwc_simulate_host: stats download");
        }
    }
    return CWC_OK;
}

// ---- resumable runs (cwc_run_*) -------------------------------------------------
// One caller-owned device buffer: header (live count, dispatch counter,
// compaction count), per-point rates, the global statistics part, the
// per-trajectory state (x [G][n_cells] int32, t, n, j), two live lists
// (current, compaction target) and the compaction's scratch.
struct StateLayout {
    size_t hdr = 0, rates = 0, parts = 0, x = 0, t = 0, n = 0, j = 0, live0 = 0, live1 = 0, temp = 0, temp_bytes = 0,
           total = 0;
};
constexpr size_t kHdrLive = 0, kHdrCounter = 16, kHdrOut = 32, kHdrPending = 40, kHdrPrint = 64, kHdrBytes = 256;

// Run fingerprint at header offset kHdrPrint, written by cwc_run_init and
// checked by every later call on the state: layout version, the plan's
// shape, the shard, a hash of the flat model tables and of the per-point
// rates, and the seed (recorded by the first advance, checked by the next).
constexpr uint64_t kPrintMagic = 0x43574352554e0004ull;  // "CWCRUN" + layout version 4
struct RunPrint {
    uint64_t magic;
    int64_t G, J, n_cells, M, P, O, R_total, r_off;
    uint64_t tables_hash, rates_hash;
    uint64_t seed, seed_set;
};
static_assert(kHdrPrint + sizeof(RunPrint) <= kHdrBytes, "header too small");


StateLayout state_layout(const cwc_model_s *m, const Plan &pl) {
    StateLayout l;
    const size_t G = (size_t)pl.G;
    size_t off = 0;
    l.hdr = off;
    off = align256(off + kHdrBytes);
    l.rates = off;  // rates [P][M] then rates_h [P][M]
    off = align256(off + 2 * sizeof(double) * (size_t)pl.P * std::max(m->M, 1));
    l.parts = off;
    off = align256(off + (size_t)stat_bytes(pl.st, pl.cells_per_part) * pl.n_parts);
    l.x = off;
    off = align256(off + sizeof(int32_t) * G * (size_t)std::max(m->n_cells, 1));
    l.t = off;
    off = align256(off + sizeof(double) * G);
    l.n = off;
    off = align256(off + sizeof(int64_t) * G);
    l.j = off;
    off = align256(off + sizeof(int32_t) * G);
    l.live0 = off;
    off = align256(off + sizeof(int64_t) * G);
    l.live1 = off;
    off = align256(off + sizeof(int64_t) * G);
    l.temp = off;
    l.temp_bytes = compact_temp_bytes((long long)G);
    off = align256(off + l.temp_bytes);
    l.total = off;
    return l;
}

cwc_status run_prepare(cwc_model m, int64_t n_replicas, const cwc_sweep *sweep, double t_end, double dt,
                       const cwc_sim_opts *opts, const void *state, size_t state_bytes, Plan &pl, StateLayout &sl,
                       const WarpTables **dwt) {
    if (!m) return fail(CWC_ERR_INVALID, "model is NULL");
    cwc_status s = plan_run(m, n_replicas, sweep, t_end, dt, opts, false, pl, true, -1);
    if (s != CWC_OK) return s;
    sl = state_layout(m, pl);
    if (!state) return fail(CWC_ERR_INVALID, "state is NULL");
    if (state_bytes < sl.total) return fail(CWC_ERR_INVALID, "state too small: need " + std::to_string(sl.total) + " bytes");
    return device_tables(m, dwt);
}

RunPrint run_print(const cwc_model_s *m, const Plan &pl, const cwc_sim_opts *opts, const std::vector<double> &rates) {
    RunPrint f{};
    f.magic = kPrintMagic;
    f.G = pl.G;
    f.J = pl.J;
    f.n_cells = m->n_cells;
    f.M = m->M;
    f.P = pl.P;
    f.O = m->n_obs;
    f.R_total = (opts && opts->replicas_total) ? opts->replicas_total : pl.R;
    f.r_off = opts ? opts->replica_offset : 0;
    uint64_t h = 0xcbf29ce484222325ull;
    h = fnv_vec(h, m->entry_rule);
    h = fnv_vec(h, m->re_cell);
    h = fnv_vec(h, m->re_mult);
    h = fnv_vec(h, m->nu_cell);
    h = fnv_vec(h, m->nu_delta);
    h = fnv_vec(h, m->init);
    h = fnv_vec(h, m->obs_of_cell);
    f.tables_hash = h;
    f.rates_hash = fnv_vec(0xcbf29ce484222325ull, rates);
    return f;
}

// Read the state header (synchronises the stream) and check the fingerprint
// against this call's arguments (and seed, when seed_check).
cwc_status check_print(const cwc_model_s *m, const Plan &pl, const cwc_sim_opts *opts, const cwc_sweep *sweep,
                       const StateLayout &sl, const unsigned char *st, cudaStream_t stream, bool seed_check,
                       uint64_t seed, unsigned char (&hdr)[kHdrBytes], const char *who) {
    cudaError_t e = cudaMemcpyAsync(hdr, st + sl.hdr, kHdrBytes, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return cuda_fail(e, (std::string(who) + ": state header").c_str());
    RunPrint have;
    std::memcpy(&have, hdr + kHdrPrint, sizeof(have));
    const RunPrint want = run_print(m, pl, opts, expand_rates(m, pl, sweep));
    if (have.magic != kPrintMagic) return fail(CWC_ERR_INVALID, std::string(who) + ": state not initialised by cwc_run_init (or corrupt)");
    if (have.G != want.G || have.J != want.J || have.n_cells != want.n_cells || have.M != want.M || have.P != want.P ||
        have.O != want.O || have.R_total != want.R_total || have.r_off != want.r_off ||
        have.tables_hash != want.tables_hash || have.rates_hash != want.rates_hash)
        return fail(CWC_ERR_INVALID, std::string(who) + ": arguments differ from the ones the state was initialised with "
                    "(model, n_replicas, sweep, t_end, sample_dt, replica shard)");
    if (seed_check && have.seed_set && have.seed != seed)
        return fail(CWC_ERR_INVALID, std::string(who) + ": seed differs from the run's earlier advances");
    return CWC_OK;
}

RunParams run_params(const cwc_model_s *m, const Plan &pl, const StateLayout &sl, unsigned char *st, double dt,
                     uint64_t seed) {
    RunParams rp{};
    rp.G = pl.G;
    rp.R = pl.R;
    rp.R_total = pl.R;
    rp.r_off = 0;
    rp.P = pl.P;
    rp.J = pl.J;
    rp.dt = dt;
    rp.seed = seed;
    set_round_keys(rp);
    rp.rates = (const double *)(st + sl.rates);
    rp.rates_h = rp.rates + (size_t)pl.P * std::max(m->M, 1);
    rp.parts = st + sl.parts;
    rp.st = pl.st;
    rp.cells_per_part = pl.cells_per_part;
    rp.stats_smem = 0;
    rp.ws = 0;
    rp.n_parts = pl.n_parts;
    rp.traj_per_part = 0;
    rp.next_traj = (unsigned long long *)(st + sl.hdr + kHdrCounter);
    rp.n_launch = pl.n_launch;
    rp.rs_live = (const int64_t *)(st + sl.live0);
    rp.rs_x = (int32_t *)(st + sl.x);
    rp.rs_t = (double *)(st + sl.t);
    rp.rs_n = (int64_t *)(st + sl.n);
    rp.rs_j = (int32_t *)(st + sl.j);
    rp.quantum = 0;
    rp.j_stop = (int64_t)pl.J + 1;
    (void)m;
    return rp;
}

}  // namespace

extern "C" {

cwc_status cwc_run_state_size(cwc_model m, int64_t n_replicas, const cwc_sweep *sweep, double t_end,
                              double sample_dt, const cwc_sim_opts *opts, size_t *bytes) {
    if (!bytes) return fail(CWC_ERR_INVALID, "bytes is NULL");
    if (!m) return fail(CWC_ERR_INVALID, "model is NULL");
    Plan pl;
    cwc_status s = plan_run(m, n_replicas, sweep, t_end, sample_dt, opts, false, pl, true, -1);
    if (s != CWC_OK) return s;
    *bytes = state_layout(m, pl).total;
    return CWC_OK;
}

cwc_status cwc_run_init(cwc_model m, int64_t n_replicas, const cwc_sweep *sweep, double t_end, double sample_dt,
                        const cwc_sim_opts *opts, void *state, size_t state_bytes, void *cuda_stream) {
    Plan pl;
    StateLayout sl;
    const WarpTables *dwt = nullptr;
    cwc_status s = run_prepare(m, n_replicas, sweep, t_end, sample_dt, opts, state, state_bytes, pl, sl, &dwt);
    if (s != CWC_OK) return s;
    cudaStream_t stream = (cudaStream_t)cuda_stream;
    unsigned char *st = (unsigned char *)state;
    const std::vector<double> rates = expand_rates(m, pl, sweep);
    cudaError_t e = cudaMemcpyAsync(st + sl.rates, rates.data(), sizeof(double) * rates.size(), cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return cuda_fail(e, "cwc_run_init: rates upload");
    e = cudaMemsetAsync(st + sl.parts, 0, (size_t)stat_bytes(pl.st, pl.cells_per_part) * pl.n_parts, stream);
    if (e != cudaSuccess) return cuda_fail(e, "cwc_run_init: zero accumulators");
    // sweeps: the live list starts longest-expected-first, in groups of 32
    // (a warp of the thread path); compaction keeps that order
    const bool lpt = pl.P > 1;
    e = launch_state_init(pl.G, m->n_cells, dwt->init, (int32_t *)(st + sl.x), (double *)(st + sl.t),
                          (int64_t *)(st + sl.n), (int32_t *)(st + sl.j), lpt ? nullptr : (int64_t *)(st + sl.live0),
                          stream);
    if (e != cudaSuccess) return cuda_fail(e, "cwc_run_init: state");
    if (lpt) {
        const int64_t T = 32;
        const std::vector<int32_t> order = lpt_groups(pl, point_a0(m, pl, rates), T);
        std::vector<int64_t> live;
        live.reserve(pl.G);
        for (int32_t b : order)
            for (int64_t gg = b * T; gg < std::min<int64_t>((b + 1) * T, pl.G); ++gg) live.push_back(gg);
        // pageable source: cudaMemcpyAsync has copied it when it returns
        e = cudaMemcpyAsync(st + sl.live0, live.data(), sizeof(int64_t) * live.size(), cudaMemcpyHostToDevice, stream);
        if (e != cudaSuccess) return cuda_fail(e, "cwc_run_init: live list");
    }
    // header: live count, dispatch counter, fingerprint (the call then
    // synchronises: the host header must outlive the copy)
    unsigned char hdr[kHdrBytes] = {};
    const int64_t live_n[2] = {pl.G, 0};
    std::memcpy(hdr + kHdrLive, live_n, sizeof(live_n));
    const RunPrint f = run_print(m, pl, opts, rates);
    std::memcpy(hdr + kHdrPrint, &f, sizeof(f));
    e = cudaMemcpyAsync(st + sl.hdr, hdr, kHdrBytes, cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return cuda_fail(e, "cwc_run_init: header");
    return CWC_OK;
}

cwc_status cwc_run_advance(cwc_model m, int64_t n_replicas, const cwc_sweep *sweep, double t_end, double sample_dt,
                           uint64_t seed, const cwc_sim_opts *opts, int64_t quantum, int64_t j_stop, void *state,
                           size_t state_bytes, void *cuda_stream, int64_t *n_pending) {
    Plan pl0;
    StateLayout sl;
    const WarpTables *dwt = nullptr;
    cwc_status s = run_prepare(m, n_replicas, sweep, t_end, sample_dt, opts, state, state_bytes, pl0, sl, &dwt);
    if (s != CWC_OK) return s;
    if (quantum < 0) return fail(CWC_ERR_INVALID, "quantum must be >= 0");
    if (j_stop == 0) j_stop = (int64_t)pl0.J + 1;
    if (j_stop < 1 || j_stop > (int64_t)pl0.J + 1) return fail(CWC_ERR_INVALID, "j_stop must be in [1, J+1] (or 0)");
    cudaStream_t stream = (cudaStream_t)cuda_stream;
    unsigned char *st = (unsigned char *)state;
    unsigned char hdr[kHdrBytes];
    s = check_print(m, pl0, opts, sweep, sl, st, stream, true, seed, hdr, "cwc_run_advance");
    if (s != CWC_OK) return s;
    int64_t nl = 0;
    std::memcpy(&nl, hdr + kHdrLive, sizeof(nl));
    if (nl < 0 || nl > pl0.G) return fail(CWC_ERR_INVALID, "state header corrupt (live count out of range)");
    cudaError_t e = cudaSuccess;
    {
        RunPrint f;
        std::memcpy(&f, hdr + kHdrPrint, sizeof(f));
        if (!f.seed_set) {  // the first advance records the run's seed
            f.seed = seed;
            f.seed_set = 1;
            e = cudaMemcpyAsync(st + sl.hdr + kHdrPrint, &f, sizeof(f), cudaMemcpyHostToDevice, stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
            if (e != cudaSuccess) return cuda_fail(e, "cwc_run_advance: header");
        }
    }
    int64_t n_out = 0;
    if (nl > 0) {
        Plan pl;
        s = plan_run(m, n_replicas, sweep, t_end, sample_dt, opts, false, pl, true, nl);
        if (s != CWC_OK) return s;
        RunParams rp = run_params(m, pl, sl, st, sample_dt, seed);
        s = apply_shard(rp, opts, n_replicas);
        if (s != CWC_OK) return s;
        rp.quantum = quantum;
        rp.j_stop = j_stop;
        e = cudaMemsetAsync(st + sl.hdr + kHdrCounter, 0, 16, stream);
        if (e != cudaSuccess) return cuda_fail(e, "cwc_run_advance: counter");
        cudaEvent_t ev0 = opts ? (cudaEvent_t)opts->ev_kernel_begin : nullptr;
        cudaEvent_t ev1 = opts ? (cudaEvent_t)opts->ev_kernel_end : nullptr;
        if (ev0 && (e = cudaEventRecord(ev0, stream)) != cudaSuccess) return cuda_fail(e, "cwc_run_advance: ev_kernel_begin");
        e = launch_ssa(m, *dwt, pl, rp, stream);
        if (e != cudaSuccess) return cuda_fail(e, "cwc_run_advance: SSA kernel launch");
        if (ev1 && (e = cudaEventRecord(ev1, stream)) != cudaSuccess) return cuda_fail(e, "cwc_run_advance: ev_kernel_end");
        // compaction: live1 = unfinished entries of live0 (order kept)
        int64_t *cnt = (int64_t *)(st + sl.hdr + kHdrOut);
        e = launch_compact((const int64_t *)(st + sl.live0), nl, (int64_t *)(st + sl.live1), cnt, rp.rs_j, pl.J,
                           st + sl.temp, sl.temp_bytes, stream);
        if (e != cudaSuccess) return cuda_fail(e, "cwc_run_advance: compaction");
        unsigned long long *pend = (unsigned long long *)(st + sl.hdr + kHdrPending);
        int64_t n_unfinished = 0;
        e = cudaMemcpyAsync(&n_unfinished, cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) return cuda_fail(e, "cwc_run_advance: live count");
        if (n_unfinished > 0) {
            e = cudaMemcpyAsync(st + sl.live0, st + sl.live1, sizeof(int64_t) * (size_t)n_unfinished, cudaMemcpyDeviceToDevice, stream);
            if (e != cudaSuccess) return cuda_fail(e, "cwc_run_advance: live list");
        }
        e = cudaMemcpyAsync(st + sl.hdr + kHdrLive, cnt, sizeof(int64_t), cudaMemcpyDeviceToDevice, stream);
        if (e != cudaSuccess) return cuda_fail(e, "cwc_run_advance: header");
        if (n_unfinished > 0 && j_stop <= (int64_t)pl0.J) {  // pending: unfinished and below the window bound
            e = launch_count_below((const int64_t *)(st + sl.live0), n_unfinished, rp.rs_j, (int32_t)j_stop, pend, stream);
            unsigned long long np = 0;
            if (e == cudaSuccess) e = cudaMemcpyAsync(&np, pend, sizeof(np), cudaMemcpyDeviceToHost, stream);
            if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
            if (e != cudaSuccess) return cuda_fail(e, "cwc_run_advance: pending count");
            n_out = (int64_t)np;
        } else {
            n_out = n_unfinished;
        }
    }
    if (n_pending) *n_pending = n_out;
    return CWC_OK;
}

cwc_status cwc_run_stats(cwc_model m, int64_t n_replicas, const cwc_sweep *sweep, double t_end, double sample_dt,
                         const cwc_sim_opts *opts, const void *state, size_t state_bytes, cwc_stats out_stats,
                         void *cuda_stream) {
    Plan pl;
    StateLayout sl;
    const WarpTables *dwt = nullptr;
    cwc_status s = run_prepare(m, n_replicas, sweep, t_end, sample_dt, opts, state, state_bytes, pl, sl, &dwt);
    if (s != CWC_OK) return s;
    unsigned char hdr[kHdrBytes];
    s = check_print(m, pl, opts, sweep, sl, (const unsigned char *)state, (cudaStream_t)cuda_stream, false, 0, hdr,
                    "cwc_run_stats");
    if (s != CWC_OK) return s;
    if (pl.n_stat_cells == 0) return CWC_OK;
    if (!out_stats.count || !out_stats.sum || !out_stats.sumsq) return fail(CWC_ERR_INVALID, "stats pointers are NULL");
    const RunParams rp = run_params(m, pl, sl, (unsigned char *)state, sample_dt, 0);
    cudaError_t e = launch_stats_stage2(rp, m->n_obs, out_stats.count, out_stats.sum, out_stats.sumsq, (cudaStream_t)cuda_stream);
    if (e != cudaSuccess) return cuda_fail(e, "cwc_run_stats: stage-2 launch");
    return CWC_OK;
}

cwc_status cwc_model_create(const cwc_model_desc *desc, cwc_model *out) {
    if (!out) return fail(CWC_ERR_INVALID, "out is NULL");
    *out = nullptr;
    cwc_model_s *m = new (std::nothrow) cwc_model_s();
    if (!m) return fail(CWC_ERR_NOMEM, "host allocation");
    cwc_status s = build_model(desc, m);
    if (s != CWC_OK) {
        delete m;
        return s;
    }
    *out = m;
    g_err.clear();
    return CWC_OK;
}

void cwc_model_destroy(cwc_model model) { delete model; }

cwc_status cwc_model_info_get(cwc_model m, cwc_model_info *info) {
    if (!m || !info) return fail(CWC_ERR_INVALID, "NULL argument");
    info->n_cells = m->n_cells;
    info->n_reactions = m->M;
    info->n_obs = m->n_obs;
    info->n_rules = m->n_rules;
    info->path = m->thread_ok ? CWC_PATH_THREAD : CWC_PATH_WARP;
    info->thread_path_ok = m->thread_ok ? 1 : 0;
    info->max_deps = m->max_deps;
    info->n_nu = (int32_t)m->nu_cell.size();
    info->n_deps = (int64_t)m->dep.size();
    return CWC_OK;
}

cwc_status cwc_model_get_flat(cwc_model m, int32_t *entry_rule, int32_t *entry_context, int32_t *entry_child,
                              int32_t *re_ptr, int32_t *re_cell, int32_t *re_mult, int32_t *nu_ptr, int32_t *nu_cell,
                              int32_t *nu_delta, int32_t *dep_ptr, int32_t *dep) {
    if (!m) return fail(CWC_ERR_INVALID, "model is NULL");
    auto cp = [](int32_t *dst, const std::vector<int32_t> &v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(int32_t));
    };
    cp(entry_rule, m->entry_rule);
    cp(entry_context, m->entry_ctx);
    cp(entry_child, m->entry_child);
    cp(re_ptr, m->re_ptr);
    cp(re_cell, m->re_cell);
    cp(re_mult, m->re_mult);
    cp(nu_ptr, m->nu_ptr);
    cp(nu_cell, m->nu_cell);
    cp(nu_delta, m->nu_delta);
    cp(dep_ptr, m->dep_ptr);
    cp(dep, m->dep);
    return CWC_OK;
}

cwc_status cwc_plan(cwc_model m, int64_t n_replicas, const cwc_sweep *sweep, double t_end, double sample_dt,
                    const cwc_sim_opts *opts, cwc_plan_info *info) {
    if (!info) return fail(CWC_ERR_INVALID, "info is NULL");
    Plan pl;
    cwc_status s = plan_run(m, n_replicas, sweep, t_end, sample_dt, opts, false, pl);
    if (s != CWC_OK) return s;
    info->kernel = pl.path == CWC_PATH_THREAD
                       ? (pl.ws == 2 ? CWC_KERNEL_THREAD_WS2 : pl.ws ? CWC_KERNEL_THREAD_WS
                                                                   : (pl.nt == 2 ? CWC_KERNEL_THREAD2 : CWC_KERNEL_THREAD))
                       : (pl.grp8 ? CWC_KERNEL_WARP8 : pl.grp4 ? CWC_KERNEL_WARP4 : pl.seg2 ? CWC_KERNEL_WARP2 : CWC_KERNEL_WARP);
    info->blocks = pl.path == CWC_PATH_THREAD
                       ? (pl.ws == 2 ? (int32_t)((pl.G + 63) / 64)
                                     : pl.ws ? (int32_t)((pl.G + 32 * kWsGroups - 1) / (32 * kWsGroups)) : pl.blocks)
                       : pl.blocks;
    info->threads = pl.path == CWC_PATH_THREAD ? (pl.ws == 2 ? 32 * (1 + kWs2Producers) : pl.ws ? 32 * (1 + kWsProducers) * kWsGroups : pl.threads)
                                               : pl.threads;
    info->stats_shared = pl.stats_smem;
    info->smem_bytes = (int64_t)pl.smem_bytes;
    info->n_parts = pl.n_parts;
    info->part_cells = pl.cells_per_part;
    info->word_bytes = pl.st.wb;
    info->words_per_cell = stat_words(pl.st);
    info->n_stat_cells = pl.n_stat_cells;
    info->workspace_bytes = (int64_t)pl.total;
    return CWC_OK;
}

cwc_status cwc_simulate_workspace_size(cwc_model m, int64_t n_replicas, const cwc_sweep *sweep, double t_end,
                                       double sample_dt, const cwc_sim_opts *opts, size_t *bytes) {
    if (!bytes) return fail(CWC_ERR_INVALID, "bytes is NULL");
    Plan pl;
    cwc_status s = plan_run(m, n_replicas, sweep, t_end, sample_dt, opts, false, pl);
    if (s != CWC_OK) return s;
    *bytes = pl.total;
    return CWC_OK;
}

cwc_status cwc_simulate_host_workspace_size(cwc_model m, int64_t n_replicas, const cwc_sweep *sweep, double t_end,
                                            double sample_dt, size_t *bytes) {
    if (!bytes) return fail(CWC_ERR_INVALID, "bytes is NULL");
    Plan pl;
    cwc_status s = plan_run(m, n_replicas, sweep, t_end, sample_dt, nullptr, true, pl);
    if (s != CWC_OK) return s;
    *bytes = pl.total;
    return CWC_OK;
}

cwc_status cwc_simulate(cwc_model m, int64_t n_replicas, const cwc_sweep *sweep, double t_end, double sample_dt,
                        uint64_t seed, void *cuda_stream, cwc_stats out_stats, void *workspace, size_t workspace_bytes,
                        const cwc_sim_opts *opts) {
    return run(m, n_replicas, sweep, t_end, sample_dt, seed, cuda_stream, out_stats, workspace, workspace_bytes, opts,
               false, cwc_stats{});
}

cwc_status cwc_simulate_host(cwc_model m, int64_t n_replicas, const cwc_sweep *sweep, double t_end, double sample_dt,
                             uint64_t seed, void *cuda_stream, cwc_stats host_stats, void *workspace,
                             size_t workspace_bytes) {
    if (!host_stats.count || !host_stats.sum || !host_stats.sumsq) return fail(CWC_ERR_INVALID, "host stats pointers are NULL");
    return run(m, n_replicas, sweep, t_end, sample_dt, seed, cuda_stream, host_stats, workspace, workspace_bytes, nullptr,
               true, host_stats);
}

cwc_status cwc_stats_finalize(const cwc_stats *stats, int64_t n_cells, double *mean, double *var, double *ci90,
                              void *cuda_stream) {
    if (!stats || n_cells < 0) return fail(CWC_ERR_INVALID, "bad arguments");
    if (n_cells > 0 && (!stats->count || !stats->sum || !stats->sumsq)) return fail(CWC_ERR_INVALID, "stats pointers are NULL");
    cudaError_t e = launch_stats_finalize(stats->count, stats->sum, stats->sumsq, n_cells, mean, var, ci90,
                                          (cudaStream_t)cuda_stream);
    if (e != cudaSuccess) return cuda_fail(e, "cwc_stats_finalize");
    return CWC_OK;
}

cwc_status cwc_philox_blocks(uint64_t seed, const int64_t *g, const int64_t *n, int64_t count, uint32_t *out,
                             void *cuda_stream) {
    if (count < 0 || (count > 0 && (!g || !n || !out))) return fail(CWC_ERR_INVALID, "bad arguments");
    cudaError_t e = launch_philox_blocks(seed, g, n, count, out, (cudaStream_t)cuda_stream);
    if (e != cudaSuccess) return cuda_fail(e, "cwc_philox_blocks");
    return CWC_OK;
}

cwc_status cwc_draws(uint64_t seed, const int64_t *g, const int64_t *n, int64_t count, double *E, double *u2,
                     void *cuda_stream) {
    if (count < 0 || (count > 0 && (!g || !n || !E || !u2))) return fail(CWC_ERR_INVALID, "bad arguments");
    cudaError_t e = launch_draws(seed, g, n, count, E, u2, (cudaStream_t)cuda_stream);
    if (e != cudaSuccess) return cuda_fail(e, "cwc_draws");
    return CWC_OK;
}

cwc_status cwc_block_draws(const uint32_t *words, int64_t count, double *u1, double *u2, double *E, void *cuda_stream) {
    if (count < 0 || (count > 0 && (!words || !u1 || !u2 || !E))) return fail(CWC_ERR_INVALID, "bad arguments");
    cudaError_t e = launch_block_draws(words, count, u1, u2, E, (cudaStream_t)cuda_stream);
    if (e != cudaSuccess) return cuda_fail(e, "cwc_block_draws");
    return CWC_OK;
}

cwc_status cwc_tau_div(const double *num, const double *den, int64_t count, double *q, void *cuda_stream) {
    if (count < 0 || (count > 0 && (!num || !den || !q))) return fail(CWC_ERR_INVALID, "bad arguments");
    cudaError_t e = launch_tau_div(num, den, count, q, (cudaStream_t)cuda_stream);
    if (e != cudaSuccess) return cuda_fail(e, "cwc_tau_div");
    return CWC_OK;
}

const char *cwc_last_error(void) { return g_err.c_str(); }

}  // extern "C"
