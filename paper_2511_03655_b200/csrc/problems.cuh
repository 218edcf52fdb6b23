// Right-hand-side device functors g(q, t) of q' = v, v' = g(q, t) (Eq. ivp2,
// P:L253) and their Hamiltonians, for the problems with a per-thread state
// (d small).  Canonical op sequences: oracle/CANON.md "Right-hand sides".
#pragma once
#include "fp64.cuh"

namespace irk {

// Planar Kepler, H = |v|^2/2 - GM/|q| (the 2-body reduction of Eq. Ham2).
// UNIT_GM: GM == 1 (every Kepler workload here), the division in its reciprocal
// form (drcp_fast, same bits); chosen at launch from the parameter.
template <bool UNIT_GM>
struct KeplerT {
    static constexpr int d = 2;
    static constexpr bool first_order = false;  // g(q, t) of q'' = g: (v, g) in first-order mode
    double GM;
    // EXACT = false: branch-free fast paths, `ok` cleared if any needs the exact
    // intrinsic (the caller then re-evaluates with EXACT = true); same bits.
    template <bool EXACT>
    __device__ __forceinline__ void accel(const double *q, double *a, double /*t*/, bool &ok) const {
        double r2 = dfma(q[0], q[0], dmul(q[1], q[1]));
        double r3, w;
        if (!EXACT && UNIT_GM) {  // one range predicate for the whole chain (fp64.cuh)
            bool unused = true;
            ok = ok && weight_range_ok(r2);
            r3 = dmul(r2, dsqrt_fast(r2, unused));
            w = drcp_fast(r3, unused);
        } else {
            r3 = dmul(r2, EXACT ? dsqrt(r2) : dsqrt_fast(r2, ok));
            w = EXACT ? ddiv(GM, r3) : (UNIT_GM ? drcp_fast(r3, ok) : ddiv_fast(GM, r3, ok));
        }
        // -(w q) as (-w) q: the same bits (round to nearest is sign-symmetric), and the
        // negation is an operand modifier of the DMUL instead of a separate DADD
        a[0] = dmul(-w, q[0]);
        a[1] = dmul(-w, q[1]);
    }
    __device__ __forceinline__ double energy(const double *q, const double *v) const {
        Neumaier n;
        n.add(dmul(0.5, dmul(v[0], v[0])));
        n.add(dmul(0.5, dmul(v[1], v[1])));
        n.add(-ddiv(GM, dsqrt(dfma(q[0], q[0], dmul(q[1], q[1])))));
        return n.result();
    }
};
using Kepler = KeplerT<false>;
using KeplerG1 = KeplerT<true>;

// Canonical sine and cosine (oracle/CANON.md "Canonical sin / cos"): x = k pi/2 + t
// by a three-part Cody-Waite reduction, Taylor polynomials of degree 19 / 20 in
// t on |t| <= pi/4 (Horner in t^2 with fma), quadrant by k mod 4.  All
// operations are IEEE-RN, so the result is the oracle's bit for bit (CUDA's own
// sin/cos differ from libm in the last ulp).
__device__ __forceinline__ void canon_sincos(double x, double &sn, double &cs) {
    const double k = rint(dmul(x, 0x1.45f306dc9c883p-1));                    // RN(2/pi)
    double t = dfma(-k, 0x1.921fb54442d18p+0, x);                            // pi/2 = P1 + P2 + P3
    t = dfma(-k, 0x1.1a62633145c07p-54, t);
    t = dfma(-k, -0x1.f1976b7ed8fbcp-110, t);
    const double z = dmul(t, t);
    // RN((-1)^j / (2j+1)!), j = 9 .. 1  and  RN((-1)^j / (2j)!), j = 10 .. 1
    double ps = -0x1.2f49b46814157p-57;
    ps = dfma(ps, z, 0x1.952c77030ad4ap-49);
    ps = dfma(ps, z, -0x1.ae7f3e733b81fp-41);
    ps = dfma(ps, z, 0x1.6124613a86d09p-33);
    ps = dfma(ps, z, -0x1.ae64567f544e4p-26);
    ps = dfma(ps, z, 0x1.71de3a556c734p-19);
    ps = dfma(ps, z, -0x1.a01a01a01a01ap-13);
    ps = dfma(ps, z, 0x1.1111111111111p-7);
    ps = dfma(ps, z, -0x1.5555555555555p-3);
    const double st = dfma(dmul(t, z), ps, t);
    double pc = 0x1.e542ba4020225p-62;
    pc = dfma(pc, z, -0x1.6827863b97d97p-53);
    pc = dfma(pc, z, 0x1.ae7f3e733b81fp-45);
    pc = dfma(pc, z, -0x1.93974a8c07c9dp-37);
    pc = dfma(pc, z, 0x1.1eed8eff8d898p-29);
    pc = dfma(pc, z, -0x1.27e4fb7789f5cp-22);
    pc = dfma(pc, z, 0x1.a01a01a01a01ap-16);
    pc = dfma(pc, z, -0x1.6c16c16c16c17p-10);
    pc = dfma(pc, z, 0x1.5555555555555p-5);
    pc = dfma(pc, z, -0.5);
    const double ct = dfma(z, pc, 1.0);
    switch ((int)((long long)k & 3)) {
    case 0: sn = st; cs = ct; break;
    case 1: sn = ct; cs = -st; break;
    case 2: sn = -st; cs = -ct; break;
    default: sn = -ct; cs = st; break;
    }
}

// Henon-Heiles with the time-dependent coupling of Listing 2:
// aux = lambda + xi sin(t); a1 = -q1 - 2 aux q1 q2; a2 = -q2 - aux (q1^2 - q2^2).
struct HenonHeiles {
    static constexpr int d = 2;
    static constexpr bool first_order = false;
    double lambda, xi;
    template <bool EXACT>
    __device__ __forceinline__ void accel(const double *q, double *a, double t, bool & /*ok*/) const {
        double aux = lambda;
        if (xi != 0.0) {  // canonical sin (R-12): bitwise the oracle's
            double sn, cs;
            canon_sincos(t, sn, cs);
            aux = dadd(lambda, dmul(xi, sn));
        }
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

// Charged particle near a magnetised Schwarzschild black hole, Eq. Ham_SBH
// (P:L508-518), y = (r, theta | p_r, p_theta), parameters {E, L, beta}.
// Not separable, so it is integrated in first-order mode only (Eqs. IRK_init /
// IRK_FP): rhs() is Hamilton's equations in the canonical order of CANON.md.
struct Schwarzschild {
    static constexpr int d = 2;
    static constexpr bool first_order = true;
    double E, L, beta;
    // EXACT = false: branch-free division fast paths, `ok` cleared if any operand
    // needs the exact intrinsic (the caller re-evaluates with EXACT = true); same bits.
    template <bool EXACT>
    __device__ __forceinline__ void rhs(const double *y, double *f, double /*t*/, bool &ok) const {
        auto dv = [&ok](double num, double den) { return EXACT ? ddiv(num, den) : ddiv_fast(num, den, ok); };
        const double r = y[0], pr = y[2], pth = y[3];
        double s, c;
        canon_sincos(y[1], s, c);
        const double fr = dsub(1.0, dv(2.0, r));
        const double r2 = dmul(r, r), s2 = dmul(s, s);
        const double A = dsub(L, dmul(dmul(0.5, beta), dmul(r2, s2)));
        const double r3 = dmul(r2, r);
        const double t1 = dv(dmul(pr, pr), r2);
        const double t2 = dv(dmul(E, E), dmul(r2, dmul(fr, fr)));
        const double t3 = dv(dmul(pth, pth), r3);
        const double t4 = dv(dmul(beta, A), r);
        const double t5 = dv(dmul(A, A), dmul(r3, s2));
        f[0] = dmul(fr, pr);
        f[1] = dv(pth, r2);
        f[2] = -dsub(dsub(dsub(dadd(t1, t2), t3), t4), t5);
        f[3] = dadd(dv(dmul(dmul(beta, A), c), s), dv(dmul(dmul(A, A), c), dmul(r2, dmul(s2, s))));
    }
    __device__ __forceinline__ double energy(const double *q, const double *p) const {
        const double r = q[0], pr = p[0], pth = p[1];
        double s, c;
        canon_sincos(q[1], s, c);
        const double fr = dsub(1.0, ddiv(2.0, r));
        const double r2 = dmul(r, r), s2 = dmul(s, s);
        const double A = dsub(L, dmul(dmul(0.5, beta), dmul(r2, s2)));
        Neumaier n;
        n.add(dmul(0.5, dmul(fr, dmul(pr, pr))));
        n.add(-dmul(0.5, ddiv(dmul(E, E), fr)));
        n.add(ddiv(dmul(pth, pth), dmul(2.0, r2)));
        n.add(ddiv(dmul(A, A), dmul(2.0, dmul(r2, s2))));
        return n.result();
    }
};

}  // namespace irk
