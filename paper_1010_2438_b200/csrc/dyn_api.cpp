// dyn_api.cpp -- the C ABI of the dynamic-topology path (include/cwc_dyn.h;
// SURVEY 8(f) NEXT-4): model compiler (validation, dense per-rule tables,
// structural classification, rule dependency masks), per-device upload,
// launch planning, and cwc_dyn_simulate (SSA kernel + the stage-2 reduction
// of stats.cu).
#include <cmath>
#include <cstring>
#include <algorithm>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "cwc_dyn.h"
#include "cwc_internal.h"
#include "dyn_internal.h"

using namespace cwc;
using namespace cwc::dyn;

namespace {

cwc_status fail(cwc_status s, const std::string &msg) {
    set_last_error(msg);
    return s;
}
cwc_status cuda_fail(cudaError_t e, const char *where) {
    set_last_error(std::string(where) + ": " + cudaGetErrorString(e));
    return CWC_ERR_CUDA;
}

struct DevBuf {
    void *p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

template <typename T>
size_t push(std::vector<unsigned char> &blob, const std::vector<T> &v) {
    const size_t off = (blob.size() + 255) & ~size_t(255);
    blob.resize(off + std::max<size_t>(v.size() * sizeof(T), 16));
    if (!v.empty()) std::memcpy(blob.data() + off, v.data(), v.size() * sizeof(T));
    return off;
}

}  // namespace

struct cwc_dyn_model_s {
    int32_t A = 0, n_labels = 0, R = 0, O = 0, n0 = 0, max_keys = 0, n_structural = 0;
    std::vector<int4> rule;
    std::vector<double> rate;
    std::vector<int32_t> lhs, rhs, dctx, dwrap, dcont;
    std::vector<int4> ctor_hdr, ctor;
    std::vector<int32_t> ctor_atoms;
    std::vector<int32_t> init_label, init_depth, init_wrap, init_cont;
    std::vector<int32_t> obs_ptr;
    std::vector<int4> obs_key;
    struct DevCopy {
        DevBuf buf;
        DynTables t{};
    };
    std::mutex mu;
    std::map<int, std::unique_ptr<DevCopy>> dev;
};

namespace {

bool rate_ok(double v) { return std::isfinite(v) && v >= 0x1.0p-1021; }

cwc_status compile(const cwc_dyn_model_desc *d, cwc_dyn_model_s *m) {
    if (!d) return fail(CWC_ERR_INVALID, "desc is NULL");
    const int A = d->n_atoms, NL = d->n_labels, C = d->n_comps, R = d->n_rules, O = d->n_obs;
    if (A < 1) return fail(CWC_ERR_INVALID, "n_atoms must be >= 1");
    if (A > CWC_DYN_MAX_ATOMS) return fail(CWC_ERR_UNSUPPORTED, "n_atoms > CWC_DYN_MAX_ATOMS");
    if (NL < 1 || NL > 255) return fail(CWC_ERR_INVALID, "n_labels must be in [1, 255]");
    if (C < 1) return fail(CWC_ERR_INVALID, "the term needs its top level (n_comps >= 1)");
    if (C > CWC_DYN_MAX_CAP) return fail(CWC_ERR_UNSUPPORTED, "initial term larger than CWC_DYN_MAX_CAP compartments");
    if (R < 0) return fail(CWC_ERR_INVALID, "n_rules < 0");
    if (R > CWC_DYN_MAX_RULES) return fail(CWC_ERR_UNSUPPORTED, "n_rules > CWC_DYN_MAX_RULES");
    if (O < 0) return fail(CWC_ERR_INVALID, "n_obs < 0");
    if (O > CWC_DYN_MAX_OBS) return fail(CWC_ERR_UNSUPPORTED, "n_obs > CWC_DYN_MAX_OBS");
    if (!d->comp_label || !d->comp_parent || !d->comp_wrap || !d->comp_content)
        return fail(CWC_ERR_INVALID, "term arrays are NULL");
    // ---- initial term: preorder tree ----
    if (d->comp_parent[0] != -1 || d->comp_label[0] != 0) return fail(CWC_ERR_INVALID, "compartment 0 must be the top level (label 0, parent -1)");
    std::vector<int32_t> depth(C, 0), chain{0};  // chain = ancestors of the last compartment
    for (int c = 1; c < C; ++c) {
        const int p = d->comp_parent[c];
        if (p < 0 || p >= c) return fail(CWC_ERR_INVALID, "comp_parent[c] must be in [0, c)");
        while (!chain.empty() && chain.back() != p) chain.pop_back();
        if (chain.empty()) return fail(CWC_ERR_INVALID, "compartments are not in preorder (a subtree is not contiguous)");
        chain.push_back(c);
        depth[c] = depth[p] + 1;
        if (depth[c] > CWC_DYN_MAX_DEPTH) return fail(CWC_ERR_UNSUPPORTED, "initial term nested deeper than CWC_DYN_MAX_DEPTH");
        if (d->comp_label[c] < 1 || d->comp_label[c] >= NL) return fail(CWC_ERR_INVALID, "compartment label out of range [1, n_labels)");
    }
    for (int i = 0; i < C * A; ++i)
        if (d->comp_wrap[i] < 0 || d->comp_content[i] < 0) return fail(CWC_ERR_INVALID, "negative initial count");
    for (int a = 0; a < A; ++a)
        if (d->comp_wrap[a] != 0) return fail(CWC_ERR_INVALID, "the top level has no wrap");
    m->A = A;
    m->n_labels = NL;
    m->R = R;
    m->O = O;
    m->n0 = C;
    m->init_label.assign(d->comp_label, d->comp_label + C);
    m->init_depth = depth;
    m->init_wrap.assign(d->comp_wrap, d->comp_wrap + (size_t)C * A);
    m->init_cont.assign(d->comp_content, d->comp_content + (size_t)C * A);
    // ---- rules ----
    if (R > 0 && (!d->rule_label || !d->rule_comp_label || !d->rate || !d->rule_flags || !d->lhs_ptr || !d->rhs_ptr ||
                  !d->ctor_ptr))
        return fail(CWC_ERR_INVALID, "rule arrays are NULL");
    m->lhs.assign((size_t)R * 3 * A, 0);
    m->rhs.assign((size_t)R * A, 0);
    m->dctx.assign((size_t)R * A, 0);
    m->dwrap.assign((size_t)R * A, 0);
    m->dcont.assign((size_t)R * A, 0);
    m->rule.assign(R, make_int4(0, 0, 0, 0));
    m->rate.assign(R, 0.0);
    m->ctor_hdr.assign(R, make_int4(0, 0, -1, 0));
    std::vector<bool> structural(R, true);
    for (int r = 0; r < R; ++r) {
        const int L = d->rule_label[r], Lc = d->rule_comp_label[r], fl = d->rule_flags[r];
        const std::string at = " (rule " + std::to_string(r) + ")";
        if (L < 0 || L >= NL) return fail(CWC_ERR_INVALID, "rule_label out of range" + at);
        if (Lc != -1 && (Lc < 1 || Lc >= NL)) return fail(CWC_ERR_INVALID, "rule_comp_label must be -1 or in [1, n_labels)" + at);
        if (!rate_ok(d->rate[r])) return fail(CWC_ERR_INVALID, "rate must be finite and >= 2^-1021" + at);
        if (fl & ~7) return fail(CWC_ERR_INVALID, "unknown rule flag" + at);
        if ((fl & (CWC_DYN_RELEASE_W | CWC_DYN_RELEASE_Y)) && Lc < 0)
            return fail(CWC_ERR_INVALID, "W / Y released by a rule without a child pattern" + at);
        int *lhs = &m->lhs[(size_t)r * 3 * A];
        int order = 0;
        for (int q = d->lhs_ptr[r]; q < d->lhs_ptr[r + 1]; ++q) {
            const int side = d->lhs_side[q], atom = d->lhs_atom[q], mult = d->lhs_mult[q];
            if (side < 0 || side > 2) return fail(CWC_ERR_INVALID, "lhs_side out of range" + at);
            if (side != CWC_DYN_CTX && Lc < 0) return fail(CWC_ERR_INVALID, "wrap / content pattern atoms on a rule without a child pattern" + at);
            if (atom < 0 || atom >= A) return fail(CWC_ERR_INVALID, "lhs_atom out of range" + at);
            if (mult < 1) return fail(CWC_ERR_INVALID, "lhs_mult must be >= 1" + at);
            lhs[side * A + atom] += mult;
            order += mult;
            if (order > 2) return fail(CWC_ERR_UNSUPPORTED, "reaction order > 2" + at);
        }
        for (int q = d->rhs_ptr[r]; q < d->rhs_ptr[r + 1]; ++q) {
            const int atom = d->rhs_atom[q], mult = d->rhs_mult[q];
            if (atom < 0 || atom >= A) return fail(CWC_ERR_INVALID, "rhs_atom out of range" + at);
            if (mult < 1) return fail(CWC_ERR_INVALID, "rhs_mult must be >= 1" + at);
            m->rhs[(size_t)r * A + atom] += mult;
        }
        const int c0 = d->ctor_ptr[r], c1 = d->ctor_ptr[r + 1];
        if (c1 - c0 > CWC_DYN_MAX_CTORS) return fail(CWC_ERR_UNSUPPORTED, "more than CWC_DYN_MAX_CTORS constructors" + at);
        if (c1 < c0) return fail(CWC_ERR_INVALID, "ctor_ptr not ascending" + at);
        int usedW = (fl & CWC_DYN_RELEASE_W) ? 1 : 0, usedY = (fl & CWC_DYN_RELEASE_Y) ? 1 : 0, inplace = -1;
        const int first = (int)m->ctor.size();
        for (int c = c0; c < c1; ++c) {
            const int cl = d->ctor_label[c], cf = d->ctor_flags[c];
            if (cl < 1 || cl >= NL) return fail(CWC_ERR_INVALID, "ctor_label out of range [1, n_labels)" + at);
            if (cf & ~3) return fail(CWC_ERR_INVALID, "unknown constructor flag" + at);
            if (cf && Lc < 0) return fail(CWC_ERR_INVALID, "constructor carries W / Y on a rule without a child pattern" + at);
            usedW += (cf & CWC_DYN_CTOR_W) ? 1 : 0;
            usedY += (cf & CWC_DYN_CTOR_Y) ? 1 : 0;
            if (cf == (CWC_DYN_CTOR_W | CWC_DYN_CTOR_Y) && inplace < 0) inplace = first + (c - c0);
            std::vector<int32_t> atoms(2 * A, 0);
            for (int q = d->ctor_atom_ptr[c]; q < d->ctor_atom_ptr[c + 1]; ++q) {
                const int side = d->ctor_side[q], atom = d->ctor_atom[q], mult = d->ctor_mult[q];
                if (side != CWC_DYN_WRAP && side != CWC_DYN_CONTENT) return fail(CWC_ERR_INVALID, "ctor_side must be WRAP or CONTENT" + at);
                if (atom < 0 || atom >= A) return fail(CWC_ERR_INVALID, "ctor_atom out of range" + at);
                if (mult < 1) return fail(CWC_ERR_INVALID, "ctor_mult must be >= 1" + at);
                atoms[(side == CWC_DYN_WRAP ? 0 : A) + atom] += mult;
            }
            m->ctor.push_back(make_int4(cl, cf, 0, 0));
            m->ctor_atoms.insert(m->ctor_atoms.end(), atoms.begin(), atoms.end());
        }
        if (usedW > 1 || usedY > 1) return fail(CWC_ERR_INVALID, "W and Y are each used at most once (reading D3)" + at);
        m->ctor_hdr[r] = make_int4(first, c1 - c0, inplace, 0);
        // factors of h (order <= 2: at most two)
        int fac[2] = {0, 0}, nf = 0;
        for (int side = 0; side < 3; ++side)
            for (int a = 0; a < A; ++a)
                if (lhs[side * A + a] > 0) fac[nf++] = side | (a << 4) | (lhs[side * A + a] << 12);
        const bool X = fl & CWC_DYN_KEEP_X, rel = fl & (CWC_DYN_RELEASE_W | CWC_DYN_RELEASE_Y);
        bool ns = false;
        if (X && !rel) {
            if (Lc < 0 && c1 == c0) ns = true;
            if (Lc >= 0 && c1 - c0 == 1 && inplace == first && m->ctor[first].x == Lc) ns = true;
        }
        structural[r] = !ns;
        for (int a = 0; a < A; ++a) {
            m->dctx[(size_t)r * A + a] = m->rhs[(size_t)r * A + a] - lhs[a];
            if (ns && Lc >= 0) {
                m->dwrap[(size_t)r * A + a] = m->ctor_atoms[(size_t)first * 2 * A + a] - lhs[A + a];
                m->dcont[(size_t)r * A + a] = m->ctor_atoms[(size_t)first * 2 * A + A + a] - lhs[2 * A + a];
            }
        }
        const int single = (L == 0 && Lc < 0) ? 1 : 0;
        m->rule[r] = make_int4(L | ((Lc + 1) << 8) | (nf << 16) | (fl << 20) | ((ns ? 0 : 1) << 24) | (single << 25),
                               fac[0], fac[1], 0);
        m->rate[r] = d->rate[r];
        m->n_structural += ns ? 0 : 1;
    }
    // dependency masks of the non-structural rules: rules whose pattern reads
    // a (label, side, atom) the firing changes
    for (int mu = 0; mu < R; ++mu) {
        if (structural[mu]) continue;
        const int Lm = rd_label(m->rule[mu].x), Lcm = rd_comp(m->rule[mu].x);
        unsigned mask = 0;
        for (int r = 0; r < R; ++r) {
            const int L = rd_label(m->rule[r].x), Lc = rd_comp(m->rule[r].x);
            const int *lhs = &m->lhs[(size_t)r * 3 * A];
            bool dep = false;
            for (int a = 0; a < A && !dep; ++a) {
                const int dc = m->dctx[(size_t)mu * A + a], dw = m->dwrap[(size_t)mu * A + a], dt = m->dcont[(size_t)mu * A + a];
                // changed: (Lm, content, a) if dc; (Lcm, wrap, a) if dw; (Lcm, content, a) if dt
                if (dc && lhs[a] && L == Lm) dep = true;                       // r's context content
                if (dc && Lc >= 0 && lhs[2 * A + a] && Lc == Lm) dep = true;   // r's child content
                if (Lcm >= 0 && dw && Lc >= 0 && lhs[A + a] && Lc == Lcm) dep = true;
                if (Lcm >= 0 && dt && lhs[a] && L == Lcm) dep = true;
                if (Lcm >= 0 && dt && Lc >= 0 && lhs[2 * A + a] && Lc == Lcm) dep = true;
            }
            if (dep) mask |= 1u << r;
        }
        m->rule[mu].w = (int)mask;
    }
    // ---- observables ----
    m->obs_ptr.assign(1, 0);
    if (O > 0 && (!d->obs_ptr || !d->obs_kind || !d->obs_label || !d->obs_atom))
        return fail(CWC_ERR_INVALID, "observable arrays are NULL");
    for (int o = 0; o < O; ++o) {
        const int k0 = d->obs_ptr[o], k1 = d->obs_ptr[o + 1];
        if (k1 < k0) return fail(CWC_ERR_INVALID, "obs_ptr not ascending");
        if (k1 - k0 > CWC_DYN_MAX_KEYS) return fail(CWC_ERR_UNSUPPORTED, "more than CWC_DYN_MAX_KEYS keys in one observable");
        m->max_keys = std::max(m->max_keys, k1 - k0);
        for (int k = k0; k < k1; ++k) {
            const int kind = d->obs_kind[k], lab = d->obs_label[k], atom = d->obs_atom[k];
            if (kind < 0 || kind > 2) return fail(CWC_ERR_INVALID, "obs_kind out of range");
            if (lab < 0 || lab >= NL || (kind != CWC_DYN_OBS_CONTENT && lab < 1))
                return fail(CWC_ERR_INVALID, "obs_label out of range (wrap / count keys need label >= 1)");
            if (kind != CWC_DYN_OBS_COUNT && (atom < 0 || atom >= A)) return fail(CWC_ERR_INVALID, "obs_atom out of range");
            m->obs_key.push_back(make_int4(kind, lab, kind == CWC_DYN_OBS_COUNT ? 0 : atom, 0));
        }
        m->obs_ptr.push_back((int)m->obs_key.size());
    }
    return CWC_OK;
}

cwc_status device_tables(cwc_dyn_model_s *m, const DynTables **out) {
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) return fail(CWC_ERR_CUDA, "no CUDA device (there is no CPU fallback)");
    int device = 0;
    if ((e = cudaGetDevice(&device)) != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    std::lock_guard<std::mutex> lock(m->mu);
    auto it = m->dev.find(device);
    if (it != m->dev.end()) {
        *out = &it->second->t;
        return CWC_OK;
    }
    std::vector<unsigned char> blob;
    const size_t o_rule = push(blob, m->rule), o_rate = push(blob, m->rate), o_lhs = push(blob, m->lhs),
                 o_rhs = push(blob, m->rhs), o_dctx = push(blob, m->dctx), o_dw = push(blob, m->dwrap),
                 o_dc = push(blob, m->dcont), o_ch = push(blob, m->ctor_hdr), o_ct = push(blob, m->ctor),
                 o_ca = push(blob, m->ctor_atoms), o_il = push(blob, m->init_label), o_id = push(blob, m->init_depth),
                 o_iw = push(blob, m->init_wrap), o_ic = push(blob, m->init_cont), o_op = push(blob, m->obs_ptr),
                 o_ok = push(blob, m->obs_key);
    std::unique_ptr<cwc_dyn_model_s::DevCopy> dc(new (std::nothrow) cwc_dyn_model_s::DevCopy());
    if (!dc) return fail(CWC_ERR_NOMEM, "host allocation");
    e = cudaMalloc(&dc->buf.p, blob.size());
    if (e == cudaErrorMemoryAllocation) return fail(CWC_ERR_NOMEM, "dynamic model tables: device allocation");
    if (e != cudaSuccess) return cuda_fail(e, "dynamic model tables: cudaMalloc");
    if ((e = cudaMemcpy(dc->buf.p, blob.data(), blob.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
        return cuda_fail(e, "dynamic model tables: cudaMemcpy");
    const unsigned char *b = (const unsigned char *)dc->buf.p;
    DynTables &t = dc->t;
    t.A = m->A;
    t.R = m->R;
    t.O = m->O;
    t.n0 = m->n0;
    t.max_keys = m->max_keys;
    t.rule = (const int4 *)(b + o_rule);
    t.rate = (const double *)(b + o_rate);
    t.lhs = (const int32_t *)(b + o_lhs);
    t.rhs = (const int32_t *)(b + o_rhs);
    t.dctx = (const int32_t *)(b + o_dctx);
    t.dwrap = (const int32_t *)(b + o_dw);
    t.dcont = (const int32_t *)(b + o_dc);
    t.ctor_hdr = (const int4 *)(b + o_ch);
    t.ctor = (const int4 *)(b + o_ct);
    t.ctor_atoms = (const int32_t *)(b + o_ca);
    t.init_label = (const int32_t *)(b + o_il);
    t.init_depth = (const int32_t *)(b + o_id);
    t.init_wrap = (const int32_t *)(b + o_iw);
    t.init_cont = (const int32_t *)(b + o_ic);
    t.obs_ptr = (const int32_t *)(b + o_op);
    t.obs_key = (const int4 *)(b + o_ok);
    *out = &dc->t;
    m->dev.emplace(device, std::move(dc));
    return CWC_OK;
}

struct DynPlan {
    int64_t G = 0, r_off = 0;
    int32_t J = 0, cap = CWC_DYN_MAX_CAP, wpb = 4, blocks = 0, vbits = 31;
    size_t smem = 0;
    StatLayout st{};
    int64_t cells = 0, n_stat_cells = 0;
    size_t off_part = 0, off_counter = 0, total = 0;
};

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

// with_device: also size the persistent grid from the device's occupancy
cwc_status plan(const cwc_dyn_model_s *m, int64_t n_replicas, double t_end, double dt, const cwc_dyn_opts *o,
                bool with_device, DynPlan &pl) {
    if (!m) return fail(CWC_ERR_INVALID, "model is NULL");
    if (!(t_end > 0.0) || !std::isfinite(t_end)) return fail(CWC_ERR_INVALID, "t_end must be finite and > 0");
    if (!(dt > 0.0) || !std::isfinite(dt)) return fail(CWC_ERR_INVALID, "sample_dt must be finite and > 0");
    if (dt > t_end) return fail(CWC_ERR_INVALID, "sample_dt must be <= t_end");
    if (n_replicas < 1) return fail(CWC_ERR_INVALID, "n_replicas must be >= 1");
    const double Jd = std::floor(t_end / dt);
    if (Jd > 2147483000.0) return fail(CWC_ERR_INVALID, "too many samples");
    pl.J = (int32_t)Jd;
    pl.G = n_replicas;
    if (o) {
        const int64_t tot = o->replicas_total ? o->replicas_total : n_replicas;
        if (o->replica_offset < 0 || tot < n_replicas || o->replica_offset > tot - n_replicas)
            return fail(CWC_ERR_INVALID, "replica shard outside [0, replicas_total)");
        pl.r_off = o->replica_offset;
        if (o->capacity) pl.cap = o->capacity;
        if (o->warps_per_block) pl.wpb = o->warps_per_block;
    }
    if (pl.cap < m->n0 || pl.cap > CWC_DYN_MAX_CAP)
        return fail(CWC_ERR_INVALID, "capacity must be in [initial compartments, CWC_DYN_MAX_CAP]");
    if (pl.wpb < 1 || pl.wpb > 8) return fail(CWC_ERR_INVALID, "warps_per_block must be in [1, 8]");
    if (o && o->blocks_per_sm < 0) return fail(CWC_ERR_INVALID, "blocks_per_sm must be >= 0");
    const size_t per_warp = dyn_smem_per_warp(m->A, m->R);
    while (pl.wpb > 1 && per_warp * pl.wpb > 227 * 1024) --pl.wpb;
    pl.smem = per_warp * pl.wpb;
    // observables: sums of <= max_keys keys over <= cap compartments of int32 counts
    int kb = 0;
    while ((1ll << kb) < (long long)pl.cap * std::max(1, m->max_keys)) ++kb;
    pl.vbits = 31 + kb;
    if ((double)pl.G * std::ldexp(1.0, pl.vbits) >= std::ldexp(1.0, 63))
        return fail(CWC_ERR_INVALID, "n_replicas too large: the exact moments could exceed int64");
    pl.st = stat_layout(false, pl.vbits);
    pl.n_stat_cells = (int64_t)(pl.J + 1) * m->O;
    pl.cells = stat_cells_round(std::max<int64_t>(pl.n_stat_cells, 1));
    pl.off_part = 0;
    pl.off_counter = align256((size_t)stat_bytes(pl.st, pl.cells));
    pl.total = pl.off_counter + 256;
    if (with_device) {
        int dev = 0, sms = 148, occ = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if ((e = cudaFuncSetAttribute(dyn_kernel_fn(), cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)) != cudaSuccess)
            return cuda_fail(e, "cwc_dyn: kernel attribute");
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, dyn_kernel_fn(), 32 * pl.wpb, pl.smem)) != cudaSuccess)
            return cuda_fail(e, "cwc_dyn: occupancy");
        if (occ < 1) return fail(CWC_ERR_UNSUPPORTED, "cwc_dyn: kernel does not fit on an SM");
        int bps = occ;
        if (o && o->blocks_per_sm) bps = std::min(bps, o->blocks_per_sm);
        int64_t blocks = (int64_t)sms * bps;
        blocks = std::min<int64_t>(blocks, (pl.G + pl.wpb - 1) / pl.wpb);
        pl.blocks = (int32_t)std::max<int64_t>(blocks, 1);
    }
    return CWC_OK;
}

}  // namespace

extern "C" {

cwc_status cwc_dyn_model_create(const cwc_dyn_model_desc *desc, cwc_dyn_model *out) {
    if (!out) return fail(CWC_ERR_INVALID, "out is NULL");
    *out = nullptr;
    std::unique_ptr<cwc_dyn_model_s> m(new (std::nothrow) cwc_dyn_model_s());
    if (!m) return fail(CWC_ERR_NOMEM, "host allocation");
    cwc_status s = compile(desc, m.get());
    if (s != CWC_OK) return s;
    *out = m.release();
    set_last_error("");
    return CWC_OK;
}

void cwc_dyn_model_destroy(cwc_dyn_model model) { delete model; }

cwc_status cwc_dyn_info_get(cwc_dyn_model m, int64_t n_replicas, double t_end, double sample_dt,
                            const cwc_dyn_opts *opts, cwc_dyn_info *info) {
    if (!m || !info) return fail(CWC_ERR_INVALID, "model or info is NULL");
    std::memset(info, 0, sizeof(*info));
    info->n_atoms = m->A;
    info->n_labels = m->n_labels;
    info->n_rules = m->R;
    info->n_obs = m->O;
    info->n_structural = m->n_structural;
    info->capacity = CWC_DYN_MAX_CAP;
    if (n_replicas > 0) {
        DynPlan pl;
        int ndev = 0;
        const bool dev = cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0;
        cwc_status s = plan(m, n_replicas, t_end, sample_dt, opts, dev, pl);
        if (s != CWC_OK) return s;
        info->blocks = pl.blocks;
        info->threads = 32 * pl.wpb;
        info->capacity = pl.cap;
        info->smem_bytes = (int64_t)pl.smem;
        info->n_stat_cells = pl.n_stat_cells;
        info->workspace_bytes = (int64_t)pl.total;
    }
    return CWC_OK;
}

cwc_status cwc_dyn_workspace_size(cwc_dyn_model m, int64_t n_replicas, double t_end, double sample_dt,
                                  const cwc_dyn_opts *opts, size_t *bytes) {
    if (!bytes) return fail(CWC_ERR_INVALID, "bytes is NULL");
    DynPlan pl;
    cwc_status s = plan(m, n_replicas, t_end, sample_dt, opts, false, pl);
    if (s != CWC_OK) return s;
    *bytes = pl.total;
    return CWC_OK;
}

cwc_status cwc_dyn_simulate(cwc_dyn_model m, int64_t n_replicas, double t_end, double sample_dt, uint64_t seed,
                            void *cuda_stream, cwc_stats out_stats, void *workspace, size_t workspace_bytes,
                            const cwc_dyn_opts *opts) {
    if (!m) return fail(CWC_ERR_INVALID, "model is NULL");
    const DynTables *t = nullptr;
    cwc_status s = device_tables(m, &t);
    if (s != CWC_OK) return s;
    DynPlan pl;
    if ((s = plan(m, n_replicas, t_end, sample_dt, opts, true, pl)) != CWC_OK) return s;
    if (!workspace) return fail(CWC_ERR_INVALID, "workspace is NULL");
    if (workspace_bytes < pl.total) return fail(CWC_ERR_INVALID, "workspace too small: need " + std::to_string(pl.total) + " bytes");
    if (pl.n_stat_cells > 0 && (!out_stats.count || !out_stats.sum || !out_stats.sumsq))
        return fail(CWC_ERR_INVALID, "stats pointers are NULL");
    cudaStream_t stream = (cudaStream_t)cuda_stream;
    unsigned char *w = (unsigned char *)workspace;
    cudaError_t e = cudaMemsetAsync(w, 0, pl.total, stream);
    if (e != cudaSuccess) return cuda_fail(e, "cwc_dyn_simulate: zero workspace");
    DynParams P{};
    P.G = pl.G;
    P.r_off = pl.r_off;
    P.J = pl.J;
    P.cap = pl.cap;
    P.dt = sample_dt;
    P.seed = seed;
    P.part = w + pl.off_part;
    P.st = pl.st;
    P.cells = pl.cells;
    P.next_traj = (unsigned long long *)(w + pl.off_counter);
    if (opts) {
        P.out_traj = opts->out_traj;
        P.out_firings = opts->out_firings;
        P.out_status = opts->out_status;
    }
    cudaEvent_t ev0 = opts ? (cudaEvent_t)opts->ev_kernel_begin : nullptr;
    cudaEvent_t ev1 = opts ? (cudaEvent_t)opts->ev_kernel_end : nullptr;
    if (ev0 && (e = cudaEventRecord(ev0, stream)) != cudaSuccess) return cuda_fail(e, "cwc_dyn_simulate: ev_kernel_begin");
    if ((e = launch_dyn_ssa(P, *t, pl.blocks, pl.wpb, pl.smem, stream)) != cudaSuccess)
        return cuda_fail(e, "cwc_dyn_simulate: SSA kernel launch");
    if (ev1 && (e = cudaEventRecord(ev1, stream)) != cudaSuccess) return cuda_fail(e, "cwc_dyn_simulate: ev_kernel_end");
    if (pl.n_stat_cells > 0) {
        RunParams rp{};
        rp.G = pl.G;
        rp.R = pl.G;
        rp.R_total = pl.G;
        rp.P = 1;
        rp.J = pl.J;
        rp.parts = P.part;
        rp.st = pl.st;
        rp.cells_per_part = pl.cells;
        rp.n_parts = 1;
        rp.traj_per_part = 0;
        if ((e = launch_stats_stage2(rp, m->O, out_stats.count, out_stats.sum, out_stats.sumsq, stream)) != cudaSuccess)
            return cuda_fail(e, "cwc_dyn_simulate: stage-2 launch");
    }
    return CWC_OK;
}

}  // extern "C"
