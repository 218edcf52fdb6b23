// Right-hand-side device functors g(q, t) of q' = v, v' = g(q, t) (Eq. ivp2,
// P:L253) and their Hamiltonians, for the problems with a per-thread state
// (d small).  Canonical op sequences: DESIGN.md "Right-hand sides".
#pragma once
#include "fp64.cuh"

namespace irk {

// Planar Kepler, H = |v|^2/2 - GM/|q| (the 2-body reduction of Eq. Ham2).
struct Kepler {
    static constexpr int d = 2;
    double GM;
    // EXACT = false: branch-free fast paths, `ok` cleared if any needs the exact
    // intrinsic (the caller then re-evaluates with EXACT = true); same bits.
    template <bool EXACT>
    __device__ __forceinline__ void accel(const double *q, double *a, double /*t*/, bool &ok) const {
        double r2 = dfma(q[0], q[0], dmul(q[1], q[1]));
        double r3 = dmul(r2, EXACT ? dsqrt(r2) : dsqrt_fast(r2, ok));
        double w = EXACT ? ddiv(GM, r3) : ddiv_fast(GM, r3, ok);
        a[0] = -dmul(w, q[0]);
        a[1] = -dmul(w, q[1]);
    }
    __device__ __forceinline__ double energy(const double *q, const double *v) const {
        Neumaier n;
        n.add(dmul(0.5, dmul(v[0], v[0])));
        n.add(dmul(0.5, dmul(v[1], v[1])));
        n.add(-ddiv(GM, dsqrt(dfma(q[0], q[0], dmul(q[1], q[1])))));
        return n.result();
    }
};

// Henon-Heiles with the time-dependent coupling of Listing 2:
// aux = lambda + xi sin(t); a1 = -q1 - 2 aux q1 q2; a2 = -q2 - aux (q1^2 - q2^2).
struct HenonHeiles {
    static constexpr int d = 2;
    double lambda, xi;
    template <bool EXACT>
    __device__ __forceinline__ void accel(const double *q, double *a, double t, bool & /*ok*/) const {
        double aux = lambda;
        if (xi != 0.0) aux = dadd(lambda, dmul(xi, sin(t)));  // not bitwise vs libm
        a[0] = dsub(-q[0], dmul(dmul(dmul(2.0, aux), q[0]), q[1]));
        a[1] = dsub(-q[1], dmul(aux, dsub(dmul(q[0], q[0]), dmul(q[1], q[1]))));
    }
    __device__ __forceinline__ double energy(const double *q, const double *v) const {
        Neumaier n;
        n.add(dmul(0.5, dmul(v[0], v[0])));
        n.add(dmul(0.5, dmul(v[1], v[1])));
        n.add(dmul(0.5, dmul(q[0], q[0])));
        n.add(dmul(0.5, dmul(q[1], q[1])));
        n.add(dmul(lambda, dmul(dmul(q[0], q[0]), q[1])));
        n.add(-dmul(lambda, ddiv(dmul(dmul(q[1], q[1]), q[1]), 3.0)));
        return n.result();
    }
};

}  // namespace irk
