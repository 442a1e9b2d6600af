#pragma once
// cg_fin.cuh — sharded CG finalisation (rank-order sums of the shards'
// partials into the CG scalars), shared by cg.cu (k_cg_fin, after an NCCL or
// device-copy exchange) and p2p.cu (k_wait_fin, after a peer-memory exchange).

#include "b200.hpp"

namespace b200 {

// g: rank-major partials, `stride` per rank (2 for the norms, else 1)
__device__ __forceinline__ void cg_fin_apply(int what, CgScalars* sc, const double* g, int nranks, double shift) {
    const int stride = what == static_cast<int>(CgFin::Norms) ? 2 : 1;
    double a = 0.0, b = 0.0;
    for (int r = 0; r < nranks; ++r) {
        a += g[r * stride];
        if (stride == 2) b += g[r * stride + 1];
    }
    switch (static_cast<CgFin>(what)) {
    case CgFin::Rho: sc->rho = a; break;
    case CgFin::Alpha:
        sc->d = a;
        sc->rho0 = sc->rho;
        sc->alpha = sc->rho / a;
        break;
    case CgFin::Beta:
        sc->rho = a;
        sc->beta = a / sc->rho0;
        break;
    case CgFin::Rnorm: sc->rnorm = sqrt(a); break;
    case CgFin::Norms:
        sc->t1 = a;
        sc->t2 = 1.0 / sqrt(b);
        sc->zeta = shift + 1.0 / a;
        break;
    }
}

}  // namespace b200
