// lbw_cell.cuh — per-cell D3Q27 physics on a register-resident population
// vector (double f[27]).  Two flavours of every operator:
//
//   Exact  (this header compiled with -fmad=false, see Makefile): a literal
//          transcription of the reference expressions.  C++ and Python share
//          precedence and left-to-right associativity for + - *, so with FMA
//          contraction disabled and no reassociation every rounding matches
//          the numba kernels (fastmath=False, _kernels.py:41) bit for bit.
//          Only multiplications by the constant 0.0 of the velocity tables
//          are dropped (they only ever change the sign of a zero).
//   Fast   (compiled with FMA): the same operator written in raw-moment form
//          (three 3-point axis transforms + binomial shifts), relaxation in
//          unnormalised central moments, FMAs throughout.  ~470 FP64
//          instructions per cell instead of ~1050.
//
// Direction order i = (cx+1)*9 + (cy+1)*3 + (cz+1), opposite = 26-i
// (stencil.py:6-9).  Moment index of kappa[a][b][c] is a*9 + b*3 + c, the
// same flat position as the population with (cx,cy,cz) = (a-1,b-1,c-1), so
// every transform runs in place on the one register array.
#pragma once

namespace lbw {

__host__ __device__ constexpr int cx_of(int i) { return i / 9 - 1; }
__host__ __device__ constexpr int cy_of(int i) { return (i / 3) % 3 - 1; }
__host__ __device__ constexpr int cz_of(int i) { return i % 3 - 1; }
__host__ __device__ constexpr int csq_of(int i) {
    return cx_of(i) * cx_of(i) + cy_of(i) * cy_of(i) + cz_of(i) * cz_of(i);
}
// weight classes |c|^2 = 0,1,2,3 (stencil.py:19-20); correctly rounded quotients
__host__ __device__ constexpr double w_of(int i) {
    return csq_of(i) == 0 ? 8.0 / 27.0
         : csq_of(i) == 1 ? 2.0 / 27.0
         : csq_of(i) == 2 ? 1.0 / 54.0
                          : 1.0 / 216.0;
}
constexpr double kCS2 = 1.0 / 3.0;  // stencil.py:16

struct Relax {
    double omega, w3, w4, w5, w6, dt;
};

struct Macro {
    double rho, ux, uy, uz;
};

// rho and half-force-shifted u (_kernels.py:94-107, 366-380).
// Sums run in direction order; "+= c*f" with c = -1 is "-= f" bitwise.
__device__ __forceinline__ Macro moments_exact(const double (&f)[27], double Fx, double Fy,
                                               double Fz, double dt) {
    double rho = 0.0, mx = 0.0, my = 0.0, mz = 0.0;
#pragma unroll
    for (int i = 0; i < 27; ++i) {
        rho += f[i];
        if (cx_of(i) > 0) mx += f[i];
        if (cx_of(i) < 0) mx -= f[i];
        if (cy_of(i) > 0) my += f[i];
        if (cy_of(i) < 0) my -= f[i];
        if (cz_of(i) > 0) mz += f[i];
        if (cz_of(i) < 0) mz -= f[i];
    }
    const double inv_rho = 1.0 / rho;
    const double hdt = 0.5 * dt;
    Macro m;
    m.rho = rho;
    m.ux = (mx + hdt * Fx) * inv_rho;
    m.uy = (my + hdt * Fy) * inv_rho;
    m.uz = (mz + hdt * Fz) * inv_rho;
    return m;
}

// The force-free half of moments_exact: rho and sum_i f_i c_i with its
// summation order (a flag-ordered chain stores these before the cell's
// force is known and completes u = (m + F dt/2) / rho in the sampling).
__device__ __forceinline__ void raw_sums_exact(const double (&f)[27], double& rho, double& mx,
                                               double& my, double& mz) {
    rho = 0.0;
    mx = my = mz = 0.0;
#pragma unroll
    for (int i = 0; i < 27; ++i) {
        rho += f[i];
        if (cx_of(i) > 0) mx += f[i];
        if (cx_of(i) < 0) mx -= f[i];
        if (cy_of(i) > 0) my += f[i];
        if (cy_of(i) < 0) my -= f[i];
        if (cz_of(i) > 0) mz += f[i];
        if (cz_of(i) < 0) mz -= f[i];
    }
}

// Guo source (_kernels.py:44-52), exact expression order.  Callers skip it
// when F == 0 exactly: every term is then a signed zero.
__device__ __forceinline__ void guo_add_exact(double (&f)[27], double Fx, double Fy, double Fz,
                                              double ux, double uy, double uz, double omega,
                                              double dt) {
    const double pref = (1.0 - 0.5 * omega) * dt;
    const double uF = ux * Fx + uy * Fy + uz * Fz;
#pragma unroll
    for (int i = 0; i < 27; ++i) {
        const double cF = (double)cx_of(i) * Fx + (double)cy_of(i) * Fy + (double)cz_of(i) * Fz;
        const double cu = (double)cx_of(i) * ux + (double)cy_of(i) * uy + (double)cz_of(i) * uz;
        f[i] += pref * w_of(i) * (3.0 * (cF - uF) + 9.0 * cu * cF);
    }
}

// --------------------------------------------------------------- BGK exact
// _kernels.py:55-84
__device__ __forceinline__ Macro bgk_exact(double (&f)[27], double Fx, double Fy, double Fz,
                                           const Relax& r) {
    const Macro m = moments_exact(f, Fx, Fy, Fz, r.dt);
    const double rho = m.rho, ux = m.ux, uy = m.uy, uz = m.uz;
    const double usq = ux * ux + uy * uy + uz * uz;
    if (r.omega == 1.0) {
#pragma unroll
        for (int i = 0; i < 27; ++i) {
            const double cu = (double)cx_of(i) * ux + (double)cy_of(i) * uy + (double)cz_of(i) * uz;
            f[i] = w_of(i) * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * usq);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 27; ++i) {
            const double cu = (double)cx_of(i) * ux + (double)cy_of(i) * uy + (double)cz_of(i) * uz;
            const double feq = w_of(i) * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * usq);
            f[i] += r.omega * (feq - f[i]);
        }
    }
    if (Fx != 0.0 || Fy != 0.0 || Fz != 0.0) guo_add_exact(f, Fx, Fy, Fz, ux, uy, uz, r.omega, r.dt);
    return m;
}

// ---------------------------------------------------------- cumulant exact
// _kernels.py:87-301, expression by expression.
__device__ __forceinline__ Macro cumulant_exact(double (&k)[27], double Fx, double Fy, double Fz,
                                                const Relax& r) {
    const Macro m = moments_exact(k, Fx, Fy, Fz, r.dt);
    const double rho = m.rho, ux = m.ux, uy = m.uy, uz = m.uz;
    const double inv_rho = 1.0 / rho;

    // forward transform z -> y -> x (_kernels.py:109-143)
    {
        const double zm = -1.0 - uz, z0 = -uz, zp = 1.0 - uz;
#pragma unroll
        for (int ab = 0; ab < 9; ++ab) {
            const double f0 = k[ab * 3], f1 = k[ab * 3 + 1], f2 = k[ab * 3 + 2];
            k[ab * 3] = f0 + f1 + f2;
            k[ab * 3 + 1] = f0 * zm + f1 * z0 + f2 * zp;
            k[ab * 3 + 2] = f0 * zm * zm + f1 * z0 * z0 + f2 * zp * zp;
        }
    }
    {
        const double ym = -1.0 - uy, y0 = -uy, yp = 1.0 - uy;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double g0 = k[a * 9 + c], g1 = k[a * 9 + 3 + c], g2 = k[a * 9 + 6 + c];
                k[a * 9 + c] = g0 + g1 + g2;
                k[a * 9 + 3 + c] = g0 * ym + g1 * y0 + g2 * yp;
                k[a * 9 + 6 + c] = g0 * ym * ym + g1 * y0 * y0 + g2 * yp * yp;
            }
    }
    {
        const double xm = -1.0 - ux, x0 = -ux, xp = 1.0 - ux;
#pragma unroll
        for (int bc = 0; bc < 9; ++bc) {
            const double h0 = k[bc], h1 = k[9 + bc], h2 = k[18 + bc];
            k[bc] = h0 + h1 + h2;
            k[9 + bc] = h0 * xm + h1 * x0 + h2 * xp;
            k[18 + bc] = h0 * xm * xm + h1 * x0 * x0 + h2 * xp * xp;
        }
    }
#pragma unroll
    for (int i = 0; i < 27; ++i) k[i] *= inv_rho;

    const double m1x = k[9], m1y = k[3], m1z = k[1];
    const double mu200 = k[18], mu020 = k[6], mu002 = k[2];
    const double mu110 = k[12], mu101 = k[10], mu011 = k[4];
    const double mu210 = k[21], mu201 = k[19], mu120 = k[15];
    const double mu102 = k[11], mu021 = k[7], mu012 = k[5];
    const double mu111 = k[13];

    // moments -> cumulants (_kernels.py:168-188)
    const double c220 = k[24] - mu200 * mu020 - 2.0 * mu110 * mu110;
    const double c202 = k[20] - mu200 * mu002 - 2.0 * mu101 * mu101;
    const double c022 = k[8] - mu020 * mu002 - 2.0 * mu011 * mu011;
    const double c211 = k[22] - mu200 * mu011 - 2.0 * mu110 * mu101;
    const double c121 = k[16] - mu020 * mu101 - 2.0 * mu110 * mu011;
    const double c112 = k[14] - mu002 * mu110 - 2.0 * mu101 * mu011;
    const double c221 = (k[25] - mu200 * mu021 - mu020 * mu201
                         - 4.0 * mu110 * mu111 - 2.0 * mu101 * mu120 - 2.0 * mu011 * mu210);
    const double c212 = (k[23] - mu200 * mu012 - mu002 * mu210
                         - 4.0 * mu101 * mu111 - 2.0 * mu110 * mu102 - 2.0 * mu011 * mu201);
    const double c122 = (k[17] - mu020 * mu102 - mu002 * mu120
                         - 4.0 * mu011 * mu111 - 2.0 * mu110 * mu012 - 2.0 * mu101 * mu021);
    const double c222 = (k[26]
                         - (mu200 * c022 + mu020 * c202 + mu002 * c220
                            + 4.0 * mu110 * c112 + 4.0 * mu101 * c121 + 4.0 * mu011 * c211)
                         - (2.0 * mu210 * mu012 + 2.0 * mu201 * mu021
                            + 2.0 * mu120 * mu102 + 4.0 * mu111 * mu111)
                         - (mu200 * mu020 * mu002 + 2.0 * mu200 * mu011 * mu011
                            + 2.0 * mu020 * mu101 * mu101 + 2.0 * mu002 * mu110 * mu110
                            + 8.0 * mu110 * mu101 * mu011));

    // relax (_kernels.py:190-218)
    const double r2 = 1.0 - r.omega, r3 = 1.0 - r.w3, r4 = 1.0 - r.w4;
    const double r5 = 1.0 - r.w5, r6 = 1.0 - r.w6;
    const double c200p = mu200 + r.omega * (kCS2 - mu200);
    const double c020p = mu020 + r.omega * (kCS2 - mu020);
    const double c002p = mu002 + r.omega * (kCS2 - mu002);
    const double c110p = r2 * mu110, c101p = r2 * mu101, c011p = r2 * mu011;
    const double c210p = r3 * mu210, c201p = r3 * mu201, c120p = r3 * mu120;
    const double c102p = r3 * mu102, c021p = r3 * mu021, c012p = r3 * mu012;
    const double c111p = r3 * mu111;
    const double c220p = r4 * c220, c202p = r4 * c202, c022p = r4 * c022;
    const double c211p = r4 * c211, c121p = r4 * c121, c112p = r4 * c112;
    const double c221p = r5 * c221, c212p = r5 * c212, c122p = r5 * c122;
    const double c222p = r6 * c222;

    // cumulants -> moments (_kernels.py:220-262)
    k[0] = 1.0;
    k[9] = r2 * m1x;
    k[3] = r2 * m1y;
    k[1] = r2 * m1z;
    k[18] = c200p;
    k[6] = c020p;
    k[2] = c002p;
    k[12] = c110p;
    k[10] = c101p;
    k[4] = c011p;
    k[21] = c210p;
    k[19] = c201p;
    k[15] = c120p;
    k[11] = c102p;
    k[7] = c021p;
    k[5] = c012p;
    k[13] = c111p;
    k[24] = c220p + c200p * c020p + 2.0 * c110p * c110p;
    k[20] = c202p + c200p * c002p + 2.0 * c101p * c101p;
    k[8] = c022p + c020p * c002p + 2.0 * c011p * c011p;
    k[22] = c211p + c200p * c011p + 2.0 * c110p * c101p;
    k[16] = c121p + c020p * c101p + 2.0 * c110p * c011p;
    k[14] = c112p + c002p * c110p + 2.0 * c101p * c011p;
    k[25] = (c221p + c200p * c021p + c020p * c201p
             + 4.0 * c110p * c111p + 2.0 * c101p * c120p + 2.0 * c011p * c210p);
    k[23] = (c212p + c200p * c012p + c002p * c210p
             + 4.0 * c101p * c111p + 2.0 * c110p * c102p + 2.0 * c011p * c201p);
    k[17] = (c122p + c020p * c102p + c002p * c120p
             + 4.0 * c011p * c111p + 2.0 * c110p * c012p + 2.0 * c101p * c021p);
    k[26] = (c222p
             + (c200p * c022p + c020p * c202p + c002p * c220p
                + 4.0 * c110p * c112p + 4.0 * c101p * c121p + 4.0 * c011p * c211p)
             + (2.0 * c210p * c012p + 2.0 * c201p * c021p
                + 2.0 * c120p * c102p + 4.0 * c111p * c111p)
             + (c200p * c020p * c002p + 2.0 * c200p * c011p * c011p
                + 2.0 * c020p * c101p * c101p + 2.0 * c002p * c110p * c110p
                + 8.0 * c110p * c101p * c011p));
#pragma unroll
    for (int i = 0; i < 27; ++i) k[i] *= rho;

    // backward transform x -> y -> z (_kernels.py:269-298); the per-axis
    // coefficient subexpressions are hoisted (pure CSE, same roundings).
    {
        const double a = 1.0 - 2.0 * ux, b = ux * ux - ux, c = 1.0 - ux * ux, d = 2.0 * ux;
        const double e = 1.0 + 2.0 * ux, g = ux * ux + ux;
#pragma unroll
        for (int bc = 0; bc < 9; ++bc) {
            const double m0 = k[bc], m1 = k[9 + bc], m2 = k[18 + bc];
            k[bc] = 0.5 * (m2 - a * m1 + b * m0);
            k[9 + bc] = c * m0 - d * m1 - m2;
            k[18 + bc] = 0.5 * (m2 + e * m1 + g * m0);
        }
    }
    {
        const double a = 1.0 - 2.0 * uy, b = uy * uy - uy, c = 1.0 - uy * uy, d = 2.0 * uy;
        const double e = 1.0 + 2.0 * uy, g = uy * uy + uy;
#pragma unroll
        for (int x = 0; x < 3; ++x)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                const double m0 = k[x * 9 + cc], m1 = k[x * 9 + 3 + cc], m2 = k[x * 9 + 6 + cc];
                k[x * 9 + cc] = 0.5 * (m2 - a * m1 + b * m0);
                k[x * 9 + 3 + cc] = c * m0 - d * m1 - m2;
                k[x * 9 + 6 + cc] = 0.5 * (m2 + e * m1 + g * m0);
            }
    }
    {
        const double a = 1.0 - 2.0 * uz, b = uz * uz - uz, c = 1.0 - uz * uz, d = 2.0 * uz;
        const double e = 1.0 + 2.0 * uz, g = uz * uz + uz;
#pragma unroll
        for (int ab = 0; ab < 9; ++ab) {
            const double m0 = k[ab * 3], m1 = k[ab * 3 + 1], m2 = k[ab * 3 + 2];
            k[ab * 3] = 0.5 * (m2 - a * m1 + b * m0);
            k[ab * 3 + 1] = c * m0 - d * m1 - m2;
            k[ab * 3 + 2] = 0.5 * (m2 + e * m1 + g * m0);
        }
    }
    if (Fx != 0.0 || Fy != 0.0 || Fz != 0.0) guo_add_exact(k, Fx, Fy, Fz, ux, uy, uz, r.omega, r.dt);
    return m;
}

// ====================================================================== fast
// Same operator, FMA form.  Used only in the translation unit compiled with
// contraction enabled (lbw_kernels_fast.cu).

// 3-point raw transform along one axis on (f-, f0, f+) -> (m0, m1, m2)
__device__ __forceinline__ void raw3(double& a, double& b, double& c) {
    const double s = c + a;   // f+ + f-
    const double d = c - a;   // f+ - f-
    a = s + b;                // m0
    b = d;                    // m1
    c = s;                    // m2
}
// raw -> central about u: k1 = m1 - u m0, k2 = m2 - 2u m1 + u^2 m0
__device__ __forceinline__ void shift3(double& m0, double& m1, double& m2, double u, double u2) {
    const double k1 = fma(-u, m0, m1);
    const double k2 = fma(u2, m0, fma(-2.0 * u, m1, m2));
    m1 = k1;
    m2 = k2;
}
// central -> raw about u: m1 = k1 + u k0, m2 = k2 + 2u k1 + u^2 k0
__device__ __forceinline__ void unshift3(double& k0, double& k1, double& k2, double u, double u2) {
    const double m1 = fma(u, k0, k1);
    const double m2 = fma(u2, k0, fma(2.0 * u, k1, k2));
    k1 = m1;
    k2 = m2;
}
// raw -> populations: f- = (m2 - m1)/2, f0 = m0 - m2, f+ = (m2 + m1)/2
__device__ __forceinline__ void unraw3(double& a, double& b, double& c) {
    const double m0 = a, m1 = b, m2 = c;
    const double h = 0.5 * m2;
    a = fma(-0.5, m1, h);
    b = m0 - m2;
    c = fma(0.5, m1, h);
}

template <int AXIS, typename Fn>
__device__ __forceinline__ void for_axis_triples(double (&k)[27], Fn fn) {
    // AXIS 0: x (stride 9), 1: y (stride 3), 2: z (stride 1)
#pragma unroll
    for (int t = 0; t < 9; ++t) {
        const int o = AXIS == 2 ? t * 3 : (AXIS == 1 ? (t / 3) * 9 + (t % 3) : t);
        const int s = AXIS == 2 ? 1 : (AXIS == 1 ? 3 : 9);
        fn(k[o], k[o + s], k[o + 2 * s]);
    }
}

__device__ __forceinline__ void guo_add_fast(double (&f)[27], double Fx, double Fy, double Fz,
                                             double ux, double uy, double uz, double omega,
                                             double dt) {
    const double pref = (1.0 - 0.5 * omega) * dt;
    const double uF = ux * Fx + uy * Fy + uz * Fz;
#pragma unroll
    for (int i = 0; i < 27; ++i) {
        const double cF = (cx_of(i) ? cx_of(i) * Fx : 0.0) + (cy_of(i) ? cy_of(i) * Fy : 0.0) +
                          (cz_of(i) ? cz_of(i) * Fz : 0.0);
        const double cu = (cx_of(i) ? cx_of(i) * ux : 0.0) + (cy_of(i) ? cy_of(i) * uy : 0.0) +
                          (cz_of(i) ? cz_of(i) * uz : 0.0);
        f[i] += (pref * w_of(i)) * (3.0 * (cF - uF) + 9.0 * cu * cF);
    }
}

// Raw moments of the populations, in place; returns rho and u.
__device__ __forceinline__ Macro raw_moments_fast(double (&k)[27], double Fx, double Fy, double Fz,
                                                  double dt) {
    auto raw = [](double& a, double& b, double& c) { raw3(a, b, c); };
    for_axis_triples<2>(k, raw);
    for_axis_triples<1>(k, raw);
    for_axis_triples<0>(k, raw);
    Macro m;
    m.rho = k[0];
    const double inv_rho = 1.0 / m.rho;
    const double hdt = 0.5 * dt;
    m.ux = fma(hdt, Fx, k[9]) * inv_rho;
    m.uy = fma(hdt, Fy, k[3]) * inv_rho;
    m.uz = fma(hdt, Fz, k[1]) * inv_rho;
    return m;
}

__device__ __forceinline__ Macro cumulant_fast(double (&k)[27], double Fx, double Fy, double Fz,
                                               const Relax& r) {
    const Macro m = raw_moments_fast(k, Fx, Fy, Fz, r.dt);
    const double rho = m.rho, ux = m.ux, uy = m.uy, uz = m.uz;
    const double inv_rho = 1.0 / rho;
    const double ux2 = ux * ux, uy2 = uy * uy, uz2 = uz * uz;
    // central moments (unnormalised): shifts commute, apply per axis
    for_axis_triples<2>(k, [&](double& a, double& b, double& c) { shift3(a, b, c, uz, uz2); });
    for_axis_triples<1>(k, [&](double& a, double& b, double& c) { shift3(a, b, c, uy, uy2); });
    for_axis_triples<0>(k, [&](double& a, double& b, double& c) { shift3(a, b, c, ux, ux2); });

    const double k200 = k[18], k020 = k[6], k002 = k[2];
    const double k110 = k[12], k101 = k[10], k011 = k[4];
    const double k210 = k[21], k201 = k[19], k120 = k[15];
    const double k102 = k[11], k021 = k[7], k012 = k[5];
    const double k111 = k[13];

    // unnormalised cumulants C = rho * c
    const double C220 = fma(-(fma(2.0 * k110, k110, k200 * k020)), inv_rho, k[24]);
    const double C202 = fma(-(fma(2.0 * k101, k101, k200 * k002)), inv_rho, k[20]);
    const double C022 = fma(-(fma(2.0 * k011, k011, k020 * k002)), inv_rho, k[8]);
    const double C211 = fma(-(fma(2.0 * k110, k101, k200 * k011)), inv_rho, k[22]);
    const double C121 = fma(-(fma(2.0 * k110, k011, k020 * k101)), inv_rho, k[16]);
    const double C112 = fma(-(fma(2.0 * k101, k011, k002 * k110)), inv_rho, k[14]);
    const double C221 = fma(-(k200 * k021 + k020 * k201 + 4.0 * k110 * k111 +
                              2.0 * (k101 * k120 + k011 * k210)),
                            inv_rho, k[25]);
    const double C212 = fma(-(k200 * k012 + k002 * k210 + 4.0 * k101 * k111 +
                              2.0 * (k110 * k102 + k011 * k201)),
                            inv_rho, k[23]);
    const double C122 = fma(-(k020 * k102 + k002 * k120 + 4.0 * k011 * k111 +
                              2.0 * (k110 * k012 + k101 * k021)),
                            inv_rho, k[17]);
    const double A = k200 * C022 + k020 * C202 + k002 * C220 +
                     4.0 * (k110 * C112 + k101 * C121 + k011 * C211);
    const double B = 2.0 * (k210 * k012 + k201 * k021 + k120 * k102) + 4.0 * k111 * k111;
    const double D = k200 * k020 * k002 +
                     2.0 * (k200 * k011 * k011 + k020 * k101 * k101 + k002 * k110 * k110) +
                     8.0 * k110 * k101 * k011;
    const double C222 = k[26] - (A + B) * inv_rho - D * (inv_rho * inv_rho);

    // relax
    const double r2 = 1.0 - r.omega, r3 = 1.0 - r.w3, r4 = 1.0 - r.w4;
    const double r5 = 1.0 - r.w5, r6 = 1.0 - r.w6;
    const double rcs2 = rho * kCS2;
    const double K200 = fma(r.omega, rcs2 - k200, k200);
    const double K020 = fma(r.omega, rcs2 - k020, k020);
    const double K002 = fma(r.omega, rcs2 - k002, k002);
    const double K110 = r2 * k110, K101 = r2 * k101, K011 = r2 * k011;
    const double K210 = r3 * k210, K201 = r3 * k201, K120 = r3 * k120;
    const double K102 = r3 * k102, K021 = r3 * k021, K012 = r3 * k012;
    const double K111 = r3 * k111;
    const double P220 = r4 * C220, P202 = r4 * C202, P022 = r4 * C022;
    const double P211 = r4 * C211, P121 = r4 * C121, P112 = r4 * C112;
    const double P221 = r5 * C221, P212 = r5 * C212, P122 = r5 * C122;
    const double P222 = r6 * C222;

    // back to central moments
    k[0] = rho;
    k[9] = r2 * k[9];
    k[3] = r2 * k[3];
    k[1] = r2 * k[1];
    k[18] = K200;
    k[6] = K020;
    k[2] = K002;
    k[12] = K110;
    k[10] = K101;
    k[4] = K011;
    k[21] = K210;
    k[19] = K201;
    k[15] = K120;
    k[11] = K102;
    k[7] = K021;
    k[5] = K012;
    k[13] = K111;
    k[24] = fma(fma(2.0 * K110, K110, K200 * K020), inv_rho, P220);
    k[20] = fma(fma(2.0 * K101, K101, K200 * K002), inv_rho, P202);
    k[8] = fma(fma(2.0 * K011, K011, K020 * K002), inv_rho, P022);
    k[22] = fma(fma(2.0 * K110, K101, K200 * K011), inv_rho, P211);
    k[16] = fma(fma(2.0 * K110, K011, K020 * K101), inv_rho, P121);
    k[14] = fma(fma(2.0 * K101, K011, K002 * K110), inv_rho, P112);
    k[25] = fma(K200 * K021 + K020 * K201 + 4.0 * K110 * K111 + 2.0 * (K101 * K120 + K011 * K210),
                inv_rho, P221);
    k[23] = fma(K200 * K012 + K002 * K210 + 4.0 * K101 * K111 + 2.0 * (K110 * K102 + K011 * K201),
                inv_rho, P212);
    k[17] = fma(K020 * K102 + K002 * K120 + 4.0 * K011 * K111 + 2.0 * (K110 * K012 + K101 * K021),
                inv_rho, P122);
    {
        const double Ap = K200 * P022 + K020 * P202 + K002 * P220 +
                          4.0 * (K110 * P112 + K101 * P121 + K011 * P211);
        const double Bp = 2.0 * (K210 * K012 + K201 * K021 + K120 * K102) + 4.0 * K111 * K111;
        const double Dp = K200 * K020 * K002 +
                          2.0 * (K200 * K011 * K011 + K020 * K101 * K101 + K002 * K110 * K110) +
                          8.0 * K110 * K101 * K011;
        k[26] = P222 + (Ap + Bp) * inv_rho + Dp * (inv_rho * inv_rho);
    }

    // central -> raw -> populations, x then y then z
    for_axis_triples<0>(k, [&](double& a, double& b, double& c) { unshift3(a, b, c, ux, ux2); });
    for_axis_triples<1>(k, [&](double& a, double& b, double& c) { unshift3(a, b, c, uy, uy2); });
    for_axis_triples<2>(k, [&](double& a, double& b, double& c) { unshift3(a, b, c, uz, uz2); });
    auto unraw = [](double& a, double& b, double& c) { unraw3(a, b, c); };
    for_axis_triples<0>(k, unraw);
    for_axis_triples<1>(k, unraw);
    for_axis_triples<2>(k, unraw);

    if (Fx != 0.0 || Fy != 0.0 || Fz != 0.0) guo_add_fast(k, Fx, Fy, Fz, ux, uy, uz, r.omega, r.dt);
    return m;
}

__device__ __forceinline__ Macro bgk_fast(double (&f)[27], double Fx, double Fy, double Fz,
                                          const Relax& r) {
    double rho = 0.0, jx = 0.0, jy = 0.0, jz = 0.0;
#pragma unroll
    for (int i = 0; i < 27; ++i) {
        rho += f[i];
        if (cx_of(i)) jx += cx_of(i) * f[i];
        if (cy_of(i)) jy += cy_of(i) * f[i];
        if (cz_of(i)) jz += cz_of(i) * f[i];
    }
    const double inv_rho = 1.0 / rho;
    const double hdt = 0.5 * r.dt;
    Macro m;
    m.rho = rho;
    m.ux = fma(hdt, Fx, jx) * inv_rho;
    m.uy = fma(hdt, Fy, jy) * inv_rho;
    m.uz = fma(hdt, Fz, jz) * inv_rho;
    const double ux = m.ux, uy = m.uy, uz = m.uz;
    const double base = 1.0 - 1.5 * (ux * ux + uy * uy + uz * uz);
    const double one_m_omega = 1.0 - r.omega;
#pragma unroll
    for (int i = 0; i < 27; ++i) {
        const double cu = (cx_of(i) ? cx_of(i) * ux : 0.0) + (cy_of(i) ? cy_of(i) * uy : 0.0) +
                          (cz_of(i) ? cz_of(i) * uz : 0.0);
        const double feq = (w_of(i) * rho) * fma(4.5 * cu, cu, fma(3.0, cu, base));
        f[i] = fma(r.omega, feq, one_m_omega * f[i]);
    }
    if (Fx != 0.0 || Fy != 0.0 || Fz != 0.0) guo_add_fast(f, Fx, Fy, Fz, ux, uy, uz, r.omega, r.dt);
    return m;
}

}  // namespace lbw
