// dd.cuh -- domain-decomposition (DD) splitting stage solves.
// Placeholder until the strip-block solver lands: every entry reports PRS_EUNSUPPORTED.
#pragma once
#include <cuda_runtime.h>
#include <string>

#include "../../include/prs.h"
#include "common.cuh"

struct prs_ctx;
int prs_internal_prof_begin(prs_ctx *ctx);
int prs_internal_prof_end(prs_ctx *ctx, int kind, double bytes);

namespace prs {

struct DDData {
    const double *sinpi = nullptr;
};

inline int dd_init(DDData &, const prs_problem &, double, double, cudaStream_t, std::string &err) {
    err = "DD splitting is not implemented on the GPU path yet";
    return PRS_EUNSUPPORTED;
}
inline int dd_factors(DDData &, int, double, cudaStream_t, std::string &err) {
    err = "DD splitting is not implemented on the GPU path yet";
    return PRS_EUNSUPPORTED;
}
template <class Fac>
inline int dd_step(DDData &, int, double, Fac *, const double *, double *, long long, const TimeArgs &, int,
                   const double *, double *, const double *, double *, unsigned long long *, cudaStream_t,
                   prs_ctx *, std::string &err, long long &) {
    err = "DD splitting is not implemented on the GPU path yet";
    return PRS_EUNSUPPORTED;
}
inline void dd_free(DDData &) {}

}  // namespace prs
