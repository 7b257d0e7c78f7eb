// plan.cpp -- host-side gather-scatter and halo planning (no device needed).
//
// Builds, from the global node ids of one rank's elements:
//   * the canonical local gather-scatter map (reading 7; P:198-200
//     "C0 continuity ... unit-depth stencils"): runs = all local copies of one
//     gid, runs ordered by first touch (smallest local index), copies ascending;
//   * for nranks > 1, the halo plan: which runs are shared with which ranks,
//     per-neighbour send/receive slot lists in ascending gid order, and the
//     per-run summation order (ascending rank) so every rank computes the same
//     bits for the same node;
//   * owner flags for the owner-copy inner product (reading 8);
//   * the element order [boundary | interior] used to overlap the halo
//     exchange with interior-element Ax.
// Validation: N in [1,15], gid >= 0, copies of one gid with equal
// coordinates (1e-9 * diameter) and equal Dirichlet flags.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "nek.h"
#include "nek_plan_impl.h"

namespace nekb200 {

// Stable LSD radix sort of local indices by gid (16-bit digits, only as many
// passes as the largest gid needs).  Ties keep ascending l because the input
// order is ascending l and every pass is stable.
static void radix_sort_by_gid(const std::vector<int64_t> &gid, std::vector<int32_t> &order)
{
    const size_t n = gid.size();
    order.resize(n);
    for (size_t l = 0; l < n; ++l) order[l] = (int32_t)l;
    if (n < 2) return;
    uint64_t mx = 0;
    for (size_t l = 0; l < n; ++l) mx = std::max<uint64_t>(mx, (uint64_t)gid[l]);
    std::vector<int32_t> tmp(n);
    std::vector<size_t> cnt(65537);
    for (int shift = 0; shift < 64 && (mx >> shift) != 0; shift += 16) {
        std::fill(cnt.begin(), cnt.end(), 0);
        for (size_t a = 0; a < n; ++a) cnt[(((uint64_t)gid[order[a]] >> shift) & 0xffff) + 1]++;
        for (int d = 0; d < 65536; ++d) cnt[d + 1] += cnt[d];
        for (size_t a = 0; a < n; ++a) tmp[cnt[((uint64_t)gid[order[a]] >> shift) & 0xffff]++] = order[a];
        order.swap(tmp);
    }
}

int plan_build_local(nek_plan *p, int64_t E, int N, const int64_t *gid, const uint8_t *dirichlet,
                     const double *xyz)
{
    if (N < 1 || N > 15) { p->err = "order N=" + std::to_string(N) + " outside [1,15]"; return NEK_EORDER; }
    if (E < 0 || (E > 0 && !gid)) { p->err = "bad E or null gid"; return NEK_EINVAL; }
    p->E = E; p->N = N; p->Nq = N + 1; p->P3 = p->Nq * p->Nq * p->Nq;
    const int64_t n = E * p->P3;
    if (n >= (int64_t)1 << 31) { p->err = "more than 2^31-1 local points on one rank"; return NEK_EINVAL; }
    p->n = n;
    p->gid.assign(gid, gid + n);
    for (int64_t l = 0; l < n; ++l)
        if (p->gid[l] < 0) { p->err = "negative gid at local index " + std::to_string(l); return NEK_EINVAL; }
    p->mask.assign(n, 0);
    if (dirichlet) for (int64_t l = 0; l < n; ++l) p->mask[l] = dirichlet[l] ? 1 : 0;

    radix_sort_by_gid(p->gid, p->sorted);
    // runs over the sorted order (every gid, singletons included)
    p->run_start.clear();
    for (int64_t a = 0; a < n;) {
        int64_t b = a + 1;
        while (b < n && p->gid[p->sorted[b]] == p->gid[p->sorted[a]]) ++b;
        p->run_start.push_back(a);
        a = b;
    }
    const int64_t nr = (int64_t)p->run_start.size();
    p->run_start.push_back(n);
    p->run_of.assign(n, 0);
    for (int64_t r = 0; r < nr; ++r)
        for (int64_t a = p->run_start[r]; a < p->run_start[r + 1]; ++a) p->run_of[p->sorted[a]] = (int32_t)r;

    // topology checks: equal Dirichlet flags and coordinates on all copies
    double diam = 0.0;
    if (xyz && n > 0) {
        double lo[3], hi[3];
        for (int d = 0; d < 3; ++d) { lo[d] = 1e300; hi[d] = -1e300; }
        for (int d = 0; d < 3; ++d)
            for (int64_t l = 0; l < n; ++l) { lo[d] = std::min(lo[d], xyz[d * n + l]); hi[d] = std::max(hi[d], xyz[d * n + l]); }
        for (int d = 0; d < 3; ++d) diam += (hi[d] - lo[d]) * (hi[d] - lo[d]);
        diam = std::sqrt(diam);
    }
    const double ctol = 1e-9 * diam;
    for (int64_t r = 0; r < nr; ++r) {
        int64_t a0 = p->run_start[r];
        int32_t l0 = p->sorted[a0];
        for (int64_t a = a0 + 1; a < p->run_start[r + 1]; ++a) {
            int32_t l = p->sorted[a];
            if (p->mask[l] != p->mask[l0]) {
                p->err = "inconsistent Dirichlet flags on gid " + std::to_string(p->gid[l0]) + " (local " +
                         std::to_string(l0) + " vs " + std::to_string(l) + ")";
                return NEK_ETOPO;
            }
            if (xyz) {
                double d2 = 0;
                for (int d = 0; d < 3; ++d) { double t = xyz[d * n + l] - xyz[d * n + l0]; d2 += t * t; }
                if (std::sqrt(d2) > ctol) {
                    p->err = "copies of gid " + std::to_string(p->gid[l0]) + " (local " + std::to_string(l0) + ", " +
                             std::to_string(l) + ") differ in coordinates by " + std::to_string(std::sqrt(d2));
                    return NEK_ETOPO;
                }
            }
        }
    }
    // surface runs: first copy lies on an element face (i, j or k in {0, N})
    p->surf_run.clear();
    for (int64_t r = 0; r < nr; ++r) {
        int32_t l = p->sorted[p->run_start[r]];
        int q = l % p->P3, i = q % p->Nq, j = (q / p->Nq) % p->Nq, k = q / (p->Nq * p->Nq);
        if (i == 0 || i == N || j == 0 || j == N || k == 0 || k == N) p->surf_run.push_back((int32_t)r);
    }
    return plan_set_ranks(p, 0, 1, nullptr, nullptr);
}

// Emit runs in first-touch order: walk l ascending, emit run(l) when l is its first copy.
static void emit_first_touch(const nek_plan *p, const std::vector<uint8_t> &sel, std::vector<int32_t> &perm,
                             std::vector<int64_t> &offs, std::vector<int32_t> *run_ids)
{
    perm.clear(); offs.clear();
    if (run_ids) run_ids->clear();
    for (int64_t l = 0; l < p->n; ++l) {
        int32_t r = p->run_of[l];
        if (!sel[r] || p->sorted[p->run_start[r]] != l) continue;
        offs.push_back((int64_t)perm.size());
        for (int64_t a = p->run_start[r]; a < p->run_start[r + 1]; ++a) perm.push_back(p->sorted[a]);
        if (run_ids) run_ids->push_back(r);
    }
    offs.push_back((int64_t)perm.size());
}

int plan_set_ranks(nek_plan *p, int rank, int nranks, const int64_t *counts, const int64_t *const *lists)
{
    if (nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && (!counts || !lists))) {
        p->err = "bad rank/nranks"; return NEK_EINVAL;
    }
    p->rank = rank; p->nranks = nranks;
    const int64_t nr = (int64_t)p->run_start.size() - 1;
    // holders: (run, q) pairs for q != rank, built q-ascending
    std::vector<std::vector<std::pair<int32_t, int32_t>>> pairs_by_q(nranks);  // (run, position in q's list)
    std::vector<int32_t> nhold(nr, 0);
    if (nranks > 1) {
        for (int q = 0; q < nranks; ++q) {
            if (q == rank) continue;
            const int64_t *L = lists[q];
            int64_t nq = counts[q], a = 0, b = 0, ns = (int64_t)p->surf_run.size();
            while (a < ns && b < nq) {
                int32_t r = p->surf_run[a];
                int64_t g = p->gid[p->sorted[p->run_start[r]]];
                if (g < L[b]) ++a;
                else if (L[b] < g) ++b;
                else { pairs_by_q[q].push_back({r, 0}); nhold[r]++; ++a; ++b; }
            }
        }
    }
    // interface runs = runs held by another rank; first-touch order
    std::vector<uint8_t> sel_local(nr, 0), sel_ifc(nr, 0);
    for (int64_t r = 0; r < nr; ++r) {
        int64_t len = p->run_start[r + 1] - p->run_start[r];
        if (nhold[r] > 0) sel_ifc[r] = 1;
        else if (len >= 2) sel_local[r] = 1;
    }
    emit_first_touch(p, sel_local, p->perm, p->offs, nullptr);
    std::vector<int32_t> ifc_runs;
    emit_first_touch(p, sel_ifc, p->ifc_perm, p->ifc_offs, &ifc_runs);
    const int64_t ni = (int64_t)ifc_runs.size();
    std::vector<int32_t> ifc_index(nr, -1);
    p->ifc_gid.resize(ni);
    for (int64_t x = 0; x < ni; ++x) {
        ifc_index[ifc_runs[x]] = (int32_t)x;
        p->ifc_gid[x] = p->gid[p->sorted[p->run_start[ifc_runs[x]]]];
    }
    // neighbours and send slots: for each neighbour q, the shared runs in ascending gid
    // order (pairs_by_q[q] is already gid-ascending because surf_run is).
    p->neighbors.clear(); p->send_offs.assign(1, 0); p->send_run.clear();
    std::vector<std::vector<int64_t>> slot_of(nranks);   // slot of each pair
    for (int q = 0; q < nranks; ++q) {
        if (pairs_by_q[q].empty()) continue;
        p->neighbors.push_back(q);
        for (auto &pr : pairs_by_q[q]) {
            slot_of[q].push_back((int64_t)p->send_run.size());
            p->send_run.push_back(ifc_index[pr.first]);
        }
        p->send_offs.push_back((int64_t)p->send_run.size());
    }
    // contributions per interface run in ascending rank order
    std::vector<int64_t> cstart(ni + 1, 0);
    for (int64_t x = 0; x < ni; ++x) cstart[x + 1] = cstart[x] + 1 + nhold[ifc_runs[x]];
    p->contrib.assign(cstart[ni], INT32_MIN);
    std::vector<int64_t> fill(ni, 0);
    std::vector<uint8_t> own_done(ni, 0);
    for (int q = 0; q < nranks; ++q) {
        if (q == rank) {
            for (int64_t x = 0; x < ni; ++x) { p->contrib[cstart[x] + fill[x]++] = -1; }
            continue;
        }
        for (size_t t = 0; t < pairs_by_q[q].size(); ++t) {
            int32_t x = ifc_index[pairs_by_q[q][t].first];
            p->contrib[cstart[x] + fill[x]++] = (int32_t)slot_of[q][t];
        }
    }
    p->contrib_offs = cstart;
    // owner flags: first local copy of a run, if this rank is the lowest holder
    p->owner.assign(p->n, 0);
    std::vector<int32_t> min_holder(nr, rank);
    for (int q = 0; q < rank; ++q)
        for (auto &pr : pairs_by_q[q]) min_holder[pr.first] = std::min(min_holder[pr.first], q);
    for (int64_t r = 0; r < nr; ++r)
        if (min_holder[r] == rank) p->owner[p->sorted[p->run_start[r]]] = 1;
    // element order: elements with an interface copy first
    std::vector<uint8_t> bnd(p->E, 0);
    for (int32_t l : p->ifc_perm) bnd[l / p->P3] = 1;
    p->elem_order.clear();
    for (int64_t e = 0; e < p->E; ++e) if (bnd[e]) p->elem_order.push_back((int32_t)e);
    p->n_boundary = (int64_t)p->elem_order.size();
    for (int64_t e = 0; e < p->E; ++e) if (!bnd[e]) p->elem_order.push_back((int32_t)e);
    return NEK_OK;
}

}  // namespace nekb200

using namespace nekb200;

template <class T>
static int copy_out(const std::vector<T> &v, void *out)
{
    if (!v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(T));
    return NEK_OK;
}

extern "C" {

int nek_plan_create(nek_plan **out, int64_t E, int N, const int64_t *gid, const uint8_t *dirichlet,
                    const double *xyz)
{
    if (!out) return NEK_EINVAL;
    *out = nullptr;
    nek_plan *p = new (std::nothrow) nek_plan();
    if (!p) return NEK_ENOMEM;
    int st;
    try {
        st = plan_build_local(p, E, N, gid, dirichlet, xyz);
    } catch (const std::bad_alloc &) {
        p->err = "host allocation failed"; st = NEK_ENOMEM;
    }
    *out = p;   // returned even on failure so the caller can read nek_plan_errmsg
    return st;
}

int64_t nek_plan_surface_gids(const nek_plan *p, int64_t *out)
{
    if (!p) return -1;
    if (out)
        for (size_t a = 0; a < p->surf_run.size(); ++a) out[a] = p->gid[p->sorted[p->run_start[p->surf_run[a]]]];
    return (int64_t)p->surf_run.size();
}

int nek_plan_set_ranks(nek_plan *p, int rank, int nranks, const int64_t *counts, const int64_t *const *lists)
{
    if (!p) return NEK_EINVAL;
    try {
        return plan_set_ranks(p, rank, nranks, counts, lists);
    } catch (const std::bad_alloc &) {
        p->err = "host allocation failed"; return NEK_ENOMEM;
    }
}

int64_t nek_plan_size(const nek_plan *p, int what)
{
    if (!p) return -1;
    switch (what) {
    case NEK_PLAN_PERM: return (int64_t)p->perm.size();
    case NEK_PLAN_OFFS: return (int64_t)p->offs.size();
    case NEK_PLAN_IFC_PERM: return (int64_t)p->ifc_perm.size();
    case NEK_PLAN_IFC_OFFS: return (int64_t)p->ifc_offs.size();
    case NEK_PLAN_IFC_GID: return (int64_t)p->ifc_gid.size();
    case NEK_PLAN_NEIGHBORS: return (int64_t)p->neighbors.size();
    case NEK_PLAN_SEND_OFFS: return (int64_t)p->send_offs.size();
    case NEK_PLAN_SEND_RUN: return (int64_t)p->send_run.size();
    case NEK_PLAN_CONTRIB_OFFS: return (int64_t)p->contrib_offs.size();
    case NEK_PLAN_CONTRIB: return (int64_t)p->contrib.size();
    case NEK_PLAN_OWNER: return (int64_t)p->owner.size();
    case NEK_PLAN_ELEM_ORDER: return (int64_t)p->elem_order.size();
    default: return -1;
    }
}

int nek_plan_get(const nek_plan *p, int what, void *out)
{
    if (!p || !out) return NEK_EINVAL;
    switch (what) {
    case NEK_PLAN_PERM: return copy_out(p->perm, out);
    case NEK_PLAN_OFFS: return copy_out(p->offs, out);
    case NEK_PLAN_IFC_PERM: return copy_out(p->ifc_perm, out);
    case NEK_PLAN_IFC_OFFS: return copy_out(p->ifc_offs, out);
    case NEK_PLAN_IFC_GID: return copy_out(p->ifc_gid, out);
    case NEK_PLAN_NEIGHBORS: return copy_out(p->neighbors, out);
    case NEK_PLAN_SEND_OFFS: return copy_out(p->send_offs, out);
    case NEK_PLAN_SEND_RUN: return copy_out(p->send_run, out);
    case NEK_PLAN_CONTRIB_OFFS: return copy_out(p->contrib_offs, out);
    case NEK_PLAN_CONTRIB: return copy_out(p->contrib, out);
    case NEK_PLAN_OWNER: return copy_out(p->owner, out);
    case NEK_PLAN_ELEM_ORDER: return copy_out(p->elem_order, out);
    default: return NEK_EINVAL;
    }
}

const char *nek_plan_errmsg(const nek_plan *p) { return p ? p->err.c_str() : "null plan"; }

void nek_plan_free(nek_plan *p) { delete p; }

}  // extern "C"
