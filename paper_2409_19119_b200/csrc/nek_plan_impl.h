// nek_plan_impl.h -- internal layout of the host plan (see plan.cpp).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

struct nek_plan {
    int64_t E = 0;
    int N = 0, Nq = 0, P3 = 0;
    int64_t n = 0;
    int rank = 0, nranks = 1;
    std::vector<int64_t> gid;
    std::vector<uint8_t> mask;
    std::vector<int32_t> sorted;      // local indices sorted by (gid, l)
    std::vector<int64_t> run_start;   // runs over `sorted` (all gids), plus end sentinel
    std::vector<int32_t> run_of;      // run of each local index
    std::vector<int32_t> surf_run;    // runs on element surfaces, gid-ascending
    // outputs
    std::vector<int32_t> perm;        // local-only shared runs (len >= 2), first-touch order
    std::vector<int64_t> offs;
    std::vector<int32_t> ifc_perm;    // interface runs (gid on another rank too)
    std::vector<int64_t> ifc_offs;
    std::vector<int64_t> ifc_gid;
    std::vector<int32_t> neighbors;
    std::vector<int64_t> send_offs;
    std::vector<int32_t> send_run;
    std::vector<int64_t> contrib_offs;
    std::vector<int32_t> contrib;
    std::vector<uint8_t> owner;
    std::vector<int32_t> elem_order;
    int64_t n_boundary = 0;
    std::string err;
};

namespace nekb200 {
int plan_build_local(nek_plan *p, int64_t E, int N, const int64_t *gid, const uint8_t *dirichlet, const double *xyz);
int plan_set_ranks(nek_plan *p, int rank, int nranks, const int64_t *counts, const int64_t *const *lists);
}
