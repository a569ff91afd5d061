// lbw_chain.cuh — device code of the actuator chain:
// the turbine-tree walk and point kinematics, macro sampling at the
// trilinear cube, polar lookup and blade-element force, and the per-axis
// deposit kernels.  Included once per arithmetic flavour after
// lbw_sweep.cuh (internal linkage inside the flavour namespace): the
// standalone chain kernels use the exact copy (lbw_alm.cu, -fmad=false),
// the fused step kernel the copy of its own translation unit.
#pragma once
#include <climits>
#include <cstdio>

// Inlining of the chain's device functions: by default the compiler decides
// and two rare paths stay out of line.  A TU whose kernels pass their
// parameter structs to these functions defines both macros as
// __forceinline__: an out-of-line call taking a reference to a kernel
// parameter makes the compiler copy the parameter block to local memory,
// and every field access becomes a local load instead of a constant-bank
// operand (measured: 2-3x on the chain's latency).
#ifndef LBW_CHAIN_FN
#define LBW_CHAIN_FN __device__
#endif
#ifndef LBW_CHAIN_COLD
#define LBW_CHAIN_COLD __device__ __noinline__
#endif

#include "../../include/lbw.h"
#include "lbw_alm_dev.h"

namespace lbw {
namespace LBW_FLAVOR {
namespace {

// ------------------------------------------------------------ 3x3 algebra
// row-major 3x3; C = A B with a fixed (a0 b0 + a1 b1) + a2 b2 order
LBW_CHAIN_FN void mm3(const double* A, const double* B, double* C) {
    double t[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            t[i * 3 + j] = A[i * 3] * B[j] + A[i * 3 + 1] * B[3 + j] + A[i * 3 + 2] * B[6 + j];
    for (int k = 0; k < 9; ++k) C[k] = t[k];
}
LBW_CHAIN_FN void mv3(const double* A, const double* v, double* out) {
    double t[3];
    for (int i = 0; i < 3; ++i) t[i] = A[i * 3] * v[0] + A[i * 3 + 1] * v[1] + A[i * 3 + 2] * v[2];
    for (int i = 0; i < 3; ++i) out[i] = t[i];
}
LBW_CHAIN_FN void cross3(const double* a, const double* b, double* out) {
    const double c0 = a[1] * b[2] - a[2] * b[1];
    const double c1 = a[2] * b[0] - a[0] * b[2];
    const double c2 = a[0] * b[1] - a[1] * b[0];
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
}
// Gram-Schmidt on the columns (turbine.py:83-90)
LBW_CHAIN_FN void reorth(double* T) {
    double c0[3] = {T[0], T[3], T[6]}, c1[3] = {T[1], T[4], T[7]};
    const double n0 = sqrt(c0[0] * c0[0] + c0[1] * c0[1] + c0[2] * c0[2]);
    for (int i = 0; i < 3; ++i) c0[i] /= n0;
    const double d = c0[0] * c1[0] + c0[1] * c1[1] + c0[2] * c1[2];
    for (int i = 0; i < 3; ++i) c1[i] = c1[i] - d * c0[i];
    const double n1 = sqrt(c1[0] * c1[0] + c1[1] * c1[1] + c1[2] * c1[2]);
    for (int i = 0; i < 3; ++i) c1[i] /= n1;
    double c2[3];
    cross3(c0, c1, c2);
    for (int i = 0; i < 3; ++i) {
        T[i * 3] = c0[i];
        T[i * 3 + 1] = c1[i];
        T[i * 3 + 2] = c2[i];
    }
}
// numpy float remainder (npy_divmod): result takes the divisor's sign
LBW_CHAIN_FN double np_mod(double a, double b) {
    double m = fmod(a, b);
    if (m != 0.0) {
        if ((b < 0) != (m < 0)) m += b;
    } else {
        m = copysign(0.0, b);
    }
    return m;
}

// Warp-cooperative 3x3 algebra on shared memory for the tree walk: every
// lane of the warp calls; lanes 0..8 (0..2) own one entry each, with the
// per-entry arithmetic of mm3 / mv3 / cross3 / drifted (bit-identical).
LBW_CHAIN_FN void wmm3(const double* A, const double* B, double* C, int lane) {
    double t = 0.0;
    if (lane < 9) {
        const int i = lane / 3, j = lane % 3;
        t = A[i * 3] * B[j] + A[i * 3 + 1] * B[3 + j] + A[i * 3 + 2] * B[6 + j];
    }
    __syncwarp();
    if (lane < 9) C[lane] = t;
    __syncwarp();
}
LBW_CHAIN_FN void wmv3(const double* A, const double* v, double* out, int lane) {
    double t = 0.0;
    if (lane < 3) t = A[lane * 3] * v[0] + A[lane * 3 + 1] * v[1] + A[lane * 3 + 2] * v[2];
    __syncwarp();
    if (lane < 3) out[lane] = t;
    __syncwarp();
}
LBW_CHAIN_FN void wcross3(const double* a, const double* b, double* out, int lane) {
    double t = 0.0;
    if (lane == 0) t = a[1] * b[2] - a[2] * b[1];
    if (lane == 1) t = a[2] * b[0] - a[0] * b[2];
    if (lane == 2) t = a[0] * b[1] - a[1] * b[0];
    __syncwarp();
    if (lane < 3) out[lane] = t;
    __syncwarp();
}
// max |T^T T - I| > 1e-12 (turbine.py:_DRIFT_TOL)
LBW_CHAIN_FN bool wdrifted(const double* T, int lane) {
    bool over = false;
    if (lane < 9) {
        const int i = lane / 3, j = lane % 3;
        double s = T[i] * T[j] + T[3 + i] * T[3 + j] + T[6 + i] * T[6 + j];
        if (i == j) s -= 1.0;
        over = fabs(s) > 1e-12;   // max(...) > tol, NaN entries ignored as fmax does
    }
    return __any_sync(0xffffffffu, over);
}
LBW_CHAIN_FN void wreorth(double* T, int lane) {
    __syncwarp();
    if (lane == 0) reorth(T);
    __syncwarp();
}


// One component of the tree walk (turbine.py:259-311, sim.py:167-191) by
// one warp: lanes 0..8 own the entries of each 3x3 product (the per-entry
// arithmetic of mm3 / mv3 / cross3, bit-identical to a serial walk).
LBW_CHAIN_FN void walk_component(const KinDev& k, double* prm, double* cs, int c, int advance,
                               const double* off, const double* orient, double* wt,
                               const double* I3s, const double* zero3s, int lane) {
    double* tmp9 = wt;
    double* tmp9b = wt + 9;
    double* tmp3 = wt + 18;
    double* tmp3b = wt + 21;
    double* q = prm + c * kKP;
    double* s = cs + c * kCS;
    const int par = (int)q[34];
    const double* Pp = par >= 0 ? cs + par * kCS + CS_P : zero3s;
    const double* PT = par >= 0 ? cs + par * kCS + CS_T : I3s;
    const double* Pv = par >= 0 ? cs + par * kCS + CS_V : zero3s;
    const double* Pw = par >= 0 ? cs + par * kCS + CS_W : zero3s;
    double* spin = q + 25;
    const double rate = q[15];
    if (advance && rate != 0.0) {
        wmm3(spin, q + 16, spin, lane);
        if (wdrifted(spin, lane)) wreorth(spin, lane);
    }
    double* Tp_rp = tmp3;
    double* Tp_Tr = tmp9;
    wmv3(PT, q, Tp_rp, lane);
    wmm3(PT, q + 3, Tp_Tr, lane);
    if (lane < 3) s[CS_P + lane] = Pp[lane] + Tp_rp[lane];
    wmm3(Tp_Tr, spin, s + CS_T, lane);
    if (wdrifted(s + CS_T, lane)) wreorth(s + CS_T, lane);
    wcross3(Pw, Tp_rp, tmp3b, lane);
    if (lane < 3) {
        s[CS_V + lane] = Pv[lane] + tmp3b[lane];
        s[CS_W + lane] = Pw[lane];
        s[CS_AX + lane] = par >= 0 ? cs[par * kCS + CS_AX + lane] : 0.0;
    }
    if (lane == 0) s[CS_HAX] = par >= 0 ? cs[par * kCS + CS_HAX] : 0.0;
    __syncwarp();
    if (rate != 0.0) {
        wmv3(Tp_Tr, q + 12, s + CS_AX, lane);
        if (lane == 0) s[CS_HAX] = 1.0;
        if (lane < 3) s[CS_W + lane] = s[CS_W + lane] + s[CS_AX + lane] * rate;
        __syncwarp();
    }
    if (lane < 9) s[CS_R + lane] = spin[lane];
    __syncwarp();
    const int first = (int)q[35];
    if (q[36] != 0.0) {
        // disk centre (update_disk, turbine.py:237-241) and its velocity
        double* Tc_p = tmp3;
        double* TcT = tmp9b;
        wmv3(s + CS_T, q + 37, Tc_p, lane);
        if (lane < 3) s[CS_SP + lane] = s[CS_P + lane] + Tc_p[lane];
        wmm3(s + CS_T, q + 40, TcT, lane);
        wmm3(TcT, spin, s + CS_ST, lane);
        wcross3(s + CS_W, Tc_p, tmp3b, lane);
        if (lane < 3) s[CS_VS + lane] = s[CS_V + lane] + tmp3b[lane];
        __syncwarp();
    } else if (first >= 0) {
        const double* W = s + CS_T;
        double* Tp_o0 = tmp3;
        double* Tp_O0 = tmp9b;
        wmv3(W, off + (int64_t)first * 3, Tp_o0, lane);
        if (lane < 3) s[CS_SP + lane] = s[CS_P + lane] + Tp_o0[lane];
        wmm3(W, orient + (int64_t)first * 9, Tp_O0, lane);
        wmm3(Tp_O0, spin, s + CS_ST, lane);
        wcross3(s + CS_W, Tp_o0, tmp3b, lane);
        if (lane < 3) {
            s[CS_VS + lane] = s[CS_V + lane] + tmp3b[lane];
            s[CS_WS + lane] = s[CS_W + lane];
        }
        __syncwarp();
        if (rate != 0.0) {
            wmv3(Tp_O0, q + 12, tmp3b, lane);
            if (lane < 3) s[CS_WS + lane] = s[CS_WS + lane] + tmp3b[lane] * rate;
            __syncwarp();
        }
    }
}

// KK: tree walk + point kinematics, one CTA.  The component parameters and
// state are staged in shared memory (the walk itself is one thread: a chain
// of dependent 3x3 products down the tree); points are then evaluated in
// parallel.  Layout per component in smem: params[kKP] then state[kCS].
// rel_p 3, rel_T 9, axis 3, rate 1, rstep 9, spin 9, parent 1, first 1, is_disk 1, disk p 3, T 9
LBW_CHAIN_FN void kinematics_cta(const KinDev& k, const AlmDev& a, const Geom& g, int per_x,
                               int advance, double* ksm, int tid, int nthr) {
#ifdef LBW_KK_PROF
    long long t0 = clock64();
#endif
    double* prm = ksm;                         // (nc, kKP)
    double* cs = ksm + (size_t)k.nc * kKP;     // (nc, kCS)
    // per-point constants staged too when they fit (k.stage_points): every
    // global load of the kernel is then issued in this one parallel pass
    double* sm_off = cs + (size_t)k.nc * kCS;            // (P,3)
    double* sm_orient = sm_off + (size_t)a.n * 3;        // (P,9)
    double* sm_lframe = sm_orient + (size_t)a.n * 9;     // (P,9)
    int32_t* sm_comp = reinterpret_cast<int32_t*>(sm_lframe + (size_t)a.n * 9);  // (P)
    // walk schedule (always staged, after the point block or after cs)
    int32_t* sm_order = k.stage_points ? sm_comp + a.n
                                       : reinterpret_cast<int32_t*>(cs + (size_t)k.nc * kCS);
    int32_t* sm_static = sm_order + k.nc;
    int32_t* sm_lstart = sm_static + k.nc;
    const double* off = k.stage_points ? sm_off : k.off;
    const double* orient = k.stage_points ? sm_orient : k.orient;
    const double* lframe = k.stage_points ? sm_lframe : k.lframe;
    const int32_t* point_comp = k.stage_points ? sm_comp : k.point_comp;
    {
        // constant image + the dynamic spins / static components' state: all
        // loads of a round issued before its shared stores
        constexpr int U = 8;
        const int n_prm = k.nc * kKP, n_img = n_prm + k.img_tail_words;
        long long* dst_prm = reinterpret_cast<long long*>(prm);
        long long* dst_tail = reinterpret_cast<long long*>(k.stage_points ? sm_off : (double*)sm_order);
        for (int i0 = tid; i0 < n_img; i0 += U * nthr) {
            long long v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * nthr;
                if (i < n_img) v[u] = i < n_prm ? k.img_prm[i] : k.img_tail[i - n_prm];
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * nthr;
                if (i < n_prm) dst_prm[i] = v[u];
                else if (i < n_img) dst_tail[i - n_prm] = v[u];
            }
        }
        __syncthreads();
        for (int i = tid; i < k.nc * 9; i += nthr) prm[(i / 9) * kKP + 25 + i % 9] = k.spin[i];
        if (k.skip_static)
            for (int i = tid; i < k.nc * kCS; i += nthr)
                if (sm_static[i / kCS]) cs[i] = k.cs[i];
    }
    __syncthreads();
#ifdef LBW_KK_PROF
    long long t1 = clock64();
#endif
    {
        // level by level: the components of one depth in parallel, one warp
        // each.  Components whose world transform never changes (no
        // rotation on their path) keep the state of the first launch.
        __shared__ double I3s[9], zero3s[3];
        __shared__ double wtmp[32][24];   // one per warp (up to 1024 threads)
        const int lane = tid & 31, warp = tid >> 5, nwarp = nthr >> 5;
        if (tid < 9) I3s[tid] = (tid % 4 == 0) ? 1.0 : 0.0;
        if (tid < 3) zero3s[tid] = 0.0;
        __syncthreads();
        for (int L = 0; L < k.nlevels; ++L) {
            for (int j = sm_lstart[L] + warp; j < sm_lstart[L + 1]; j += nwarp) {
                const int c = sm_order[j];
                if (k.skip_static && sm_static[c]) continue;
                walk_component(k, prm, cs, c, advance, off, orient, wtmp[warp], I3s, zero3s, lane);
            }
            __syncthreads();
        }
    }
#ifdef LBW_KK_PROF
    long long t2 = clock64();
#endif
    // persist spin + component state (downloadable), evaluate the points
    for (int i = tid; i < k.nc * 9; i += nthr)
        k.spin[i] = k.spin_hist[(int64_t)k.hist_slot * k.nc * 9 + i] =
            prm[(i / 9) * kKP + 25 + i % 9];
    for (int i = tid; i < k.nc * kCS; i += nthr)
        k.cs[i] = k.cs_hist[(int64_t)k.hist_slot * k.nc * kCS + i] = cs[i];
#ifdef LBW_KK_PROF
    long long t3 = clock64();
#endif
    const int64_t dims[3] = {g.nxg, g.ny, g.nz};
    const int per[3] = {per_x, g.per_y, g.per_z};
    __shared__ int box_lo, box_hi;
    if (tid == 0) {
        box_lo = INT_MAX;
        box_hi = INT_MIN;
    }
    __syncthreads();
    for (int p = tid; p < a.n; p += nthr) {
        const int c = point_comp[p];
        const double* s = cs + c * kCS;
        const int kk = p - k.line_first[c];
        double pos[3], fr[9], vel[3];
        const bool disk = prm[c * kKP + 36] != 0.0;
        if (disk) {
            // world = centre.p + offs @ centre.T^T (sim.py:182-187); the disk
            // axis (centre frame +x) rides in the e_chord slot
            double rel[3];
            mv3(s + CS_ST, off + (int64_t)p * 3, rel);
            for (int i = 0; i < 3; ++i) pos[i] = s[CS_SP + i] + rel[i];
            for (int i = 0; i < 3; ++i) vel[i] = s[CS_VS + i];
            const double fr_d[9] = {s[CS_ST], s[CS_ST + 3], s[CS_ST + 6], 0, 1, 0, 0, 0, 1};
            for (int i = 0; i < 9; ++i) fr[i] = fr_d[i];
        } else if (kk == 0) {
            for (int i = 0; i < 3; ++i) pos[i] = s[CS_SP + i];
            for (int i = 0; i < 9; ++i) fr[i] = s[CS_ST + i];
            for (int i = 0; i < 3; ++i) vel[i] = s[CS_VS + i];
        } else {
            double rel[3], tmp[9], cr[3];
            mv3(s + CS_ST, off + (int64_t)p * 3, rel);
            for (int i = 0; i < 3; ++i) pos[i] = s[CS_SP + i] + rel[i];
            mm3(s + CS_ST, orient + (int64_t)p * 9, tmp);
            mm3(tmp, s + CS_R, fr);
            cross3(s + CS_WS, rel, cr);
            for (int i = 0; i < 3; ++i) vel[i] = s[CS_VS + i] + cr[i];
        }
        double* out = a.kin + (int64_t)p * kKin;
        for (int i = 0; i < 3; ++i) {
            double lat = pos[i] / k.dx;
            if (per[i]) lat = np_mod(lat, (double)dims[i]);
            else if (!(lat >= 0.0 && lat < (double)dims[i])) atomicOr(a.error_flags, 2);
            out[i] = lat;
            out[3 + i] = vel[i];
            out[15 + i] = pos[i];
            if (i == 0 && k.box) {
                // planes the chain reads (sampling cube + pull sources) or
                // writes (deposit rows) for this point
                const int64_t n0 = (int64_t)floor(lat);
                int64_t lo = n0 - k.box_halo - g.x0, hi = n0 + k.box_halo - g.x0;
                if (lo < 0 || hi >= g.nxl) {   // wraps or leaves the slab: gate all planes
                    if (per_x || lo < 0) lo = 0;
                    if (per_x || hi >= g.nxl) hi = g.nxl - 1;
                }
                atomicMin(&box_lo, (int)(lo < 0 ? 0 : lo));
                atomicMax(&box_hi, (int)(hi > g.nxl - 1 ? g.nxl - 1 : hi));
            }
        }
        if (disk) {
            for (int i = 0; i < 9; ++i) out[6 + i] = fr[i];
        } else {
            for (int f = 0; f < 3; ++f) mv3(fr, lframe + (int64_t)p * 9 + f * 3, out + 6 + 3 * f);
        }
    }
    if (k.box) {
        __syncthreads();
        if (tid == 0) {
            k.box[0] = box_lo;
            k.box[1] = box_hi;
        }
    }
#ifdef LBW_KK_PROF
    __syncthreads();
    if (tid == 0)
        printf("KKPROF stage %lld walk %lld persist %lld points %lld\n", t1 - t0, t2 - t1, t3 - t2,
               clock64() - t3);
#endif
}

LBW_CHAIN_COLD void load_cell_general(const void* buf, const Geom& g, bool pull, int x,
                                               int y, int z, double (&f)[27]) {
    if (pull) load_cell_any<true>(buf, g, x, y, z, f);
    else load_cell_any<false>(buf, g, x, y, z, f);
}

// Macro (rho, u) of global cell (gx,gy,gz), following the ghost semantics
// of PdfField.macro (fields.py:35-36, halo.py:144-160).  Returns MA_REMOTE
// (nothing written) when the cell belongs to another slab, MA_OWNED for a
// cell of this slab, MA_CONST for a ghost value every slab knows.  Values
// are those the reference's macro array of the storage dtype holds.
LBW_CHAIN_FN int macro_at_raw(const Geom& g, const MacroDev& m, int64_t gx, int64_t gy, int64_t gz,
                            double out[4]);
LBW_CHAIN_FN int macro_at(const Geom& g, const MacroDev& m, int64_t gx, int64_t gy, int64_t gz,
                        double out[4]) {
    const int code = macro_at_raw(g, m, gx, gy, gz, out);
    if (code != MA_REMOTE && g.single)
        for (int k = 0; k < 4; ++k) out[k] = stored<float>(out[k]);
    return code;
}
LBW_CHAIN_FN int macro_at_raw(const Geom& g, const MacroDev& m, int64_t gx, int64_t gy, int64_t gz,
                            double out[4]) {
    const double ghost0[4] = {1.0, 0.0, 0.0, 0.0};
    auto put = [&](const double* v) {
        for (int k = 0; k < 4; ++k) out[k] = v[k];
    };
    if (gx < 0 || gx >= g.nxg) {
        if (m.per_x) {
            gx = gx < 0 ? gx + g.nxg : gx - g.nxg;
        } else if (m.inflow && gx < 0) {
            if (m.bc_set) {
                out[0] = 1.0;
                out[1] = m.u_in[0];
                out[2] = m.u_in[1];
                out[3] = m.u_in[2];
            } else {
                put(ghost0);
            }
            return MA_CONST;
        } else if (m.inflow && gx >= g.nxg && m.bc_set) {
            gx = g.nxg - 1;
        } else {
            put(ghost0);
            return MA_CONST;
        }
    }
    if (gy < 0 || gy >= g.ny) {
        if (!g.per_y) { put(ghost0); return MA_CONST; }
        gy = gy < 0 ? gy + g.ny : gy - g.ny;
    }
    if (gz < 0 || gz >= g.nz) {
        if (!g.per_z) { put(ghost0); return MA_CONST; }
        gz = gz < 0 ? gz + g.nz : gz - g.nz;
    }
    const int64_t x = gx - g.x0;
    if (x < 0 || x >= g.nxl) return MA_REMOTE;
    if (m.kind == MS_UNIFORM) {
        put(m.uniform);
        return MA_OWNED;
    }
    const int64_t cell = (x * g.ny + gy) * g.nz + gz;
    if (m.kind == MS_DENSE) {
        put(m.dense + cell * 4);
        return MA_OWNED;
    }
    // the row key and the 27 populations are loaded together (one DRAM
    // round trip); the force sum over the staged deposit data follows
    const uint64_t key = m.fv.row_key ? m.fv.row_key[x * g.ny + gy] : 0ull;
    double f[27];
    // interior cells take the compact branch-free pull; cells at boundaries
    // (x faces, non-periodic y / z, walls) the general one, out of line so
    // this kernel's code stays small
    if (m.pull && pull_is_simple(g, (int)x, (int)gy, (int)gz)) {
        if (g.single)
            load_cell_simple(static_cast<const float*>(m.buf), g, (int)x, (int)gy, (int)gz, f);
        else
            load_cell_simple(static_cast<const double*>(m.buf), g, (int)x, (int)gy, (int)gz, f);
    } else {
        load_cell_general(m.buf, g, m.pull != 0, (int)x, (int)gy, (int)gz, f);
    }
    double Fx, Fy, Fz;
    if (g.single) force_from_key<float>(m.fv, g, key, (int)x, (int)gy, (int)gz, Fx, Fy, Fz);
    else force_from_key<double>(m.fv, g, key, (int)x, (int)gy, (int)gz, Fx, Fy, Fz);
    const Macro mm = moments_exact(f, Fx, Fy, Fz, 1.0);
    out[0] = mm.rho;
    out[1] = mm.ux;
    out[2] = mm.uy;
    out[3] = mm.uz;
    return MA_OWNED;
}

__device__ __forceinline__ double dot3(const double* a, const double* b) {
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

// np.interp on one value (numpy compiled_base.c arr_interp semantics)
// Roma 3-point kernel (actuator.py:100-110)
__device__ __forceinline__ double roma(double r) {
    const double a = fabs(r);
    if (a <= 0.5) return (1.0 + sqrt(1.0 - 3.0 * (a * a))) / 3.0;
    if (a <= 1.5) {
        const double b = 1.0 - a;
        return (5.0 - 3.0 * a - sqrt(1.0 - 3.0 * (b * b))) / 6.0;
    }
    return 0.0;
}

// Per-point data that does not depend on the flow, loaded at the start of
// K4 so its latency overlaps the sampling loads: the point's polar table
// sits in registers (one row per lane) when it has at most 32 rows.
struct PointStatic {
    int pid, off, rows;
    double chord, elen, twist;
    double xl, cll, cdl;   // this lane's polar row
};
__device__ __forceinline__ PointStatic load_static(const AlmDev& a, int p, int lane) {
    PointStatic ps;
    ps.pid = a.polar_index[p];
    ps.chord = a.chord[p];
    ps.elen = a.elen[p];
    ps.twist = a.twist[p];
    ps.off = ps.rows = 0;
    ps.xl = ps.cll = ps.cdl = 0.0;
    if (ps.pid >= 0) {
        ps.off = a.polar_offset[ps.pid];
        ps.rows = a.polar_rows[ps.pid];
        if (lane < ps.rows) {
            ps.xl = a.p_alpha[ps.off + lane];
            ps.cll = a.p_cl[ps.off + lane];
            ps.cdl = a.p_cd[ps.off + lane];
        }
    }
    return ps;
}

// polar row r of the point: from the lanes' registers (<= 32 rows) or memory
__device__ __forceinline__ void polar_row(const AlmDev& a, const PointStatic& ps, int r,
                                          double& x, double& cl, double& cd) {
    if (ps.rows <= 32) {
        x = __shfl_sync(0xffffffffu, ps.xl, r);
        cl = __shfl_sync(0xffffffffu, ps.cll, r);
        cd = __shfl_sync(0xffffffffu, ps.cdl, r);
    } else {
        x = a.p_alpha[ps.off + r];
        cl = a.p_cl[ps.off + r];
        cd = a.p_cd[ps.off + r];
    }
}

// np.interp (polars.py:65-80) of cl and cd at x for the whole warp: the
// bracketing row (largest j with xp[j] <= x; tables are increasing) is
// counted with a ballot instead of a binary search of dependent loads.
LBW_CHAIN_FN void polar_interp(const AlmDev& a, const PointStatic& ps, double x, int lane,
                             double& cl, double& cd) {
    const int n = ps.rows;
    double x0, c0l, c0d, xn, cnl, cnd;
    polar_row(a, ps, 0, x0, c0l, c0d);
    polar_row(a, ps, n - 1, xn, cnl, cnd);
    int cnt = 0;
    if (n <= 32) {
        cnt = __popc(__ballot_sync(0xffffffffu, lane < n && ps.xl <= x));
    } else {
        for (int k0 = 0; k0 < n; k0 += 32) {
            const int k = k0 + lane;
            cnt += __popc(__ballot_sync(0xffffffffu, k < n && a.p_alpha[ps.off + k] <= x));
        }
    }
    const int j = cnt > 0 ? (cnt - 1 < n - 2 ? cnt - 1 : n - 2) : 0;
    double xa, cla, cda, xb, clb, cdb;
    polar_row(a, ps, j, xa, cla, cda);
    polar_row(a, ps, j + 1, xb, clb, cdb);
    auto one = [&](double fa, double fb, double f0, double fn) -> double {
        if (isnan(x)) return x;
        if (x < x0) return f0;
        if (x > xn) return fn;
        if (x == xn) return fn;
        if (xa == x) return fa;
        const double slope = (fb - fa) / (xb - xa);
        double r = slope * (x - xa) + fa;
        if (isnan(r)) {
            r = slope * (x - xb) + fb;
            if (isnan(r) && fa == fb) r = fa;
        }
        return r;
    };
    cl = one(cla, clb, c0l, cnl);
    cd = one(cda, cdb, c0d, cnd);
}

// blade-element force on the BLADE (actuator.py:117-146, sim.py:218-235),
// evaluated by a whole warp (identical values on every lane; lane 0 raises
// the flags).  kr: the point's kinematics row.
LBW_CHAIN_FN void blade_force_warp(const AlmDev& a, const PointStatic& ps, const double* kr,
                                 const double* acc, double* blade, int lane) {
    blade[0] = blade[1] = blade[2] = 0.0;
    if (ps.pid < 0) return;
    const double* vel = kr + 3;
    const double* ec = kr + 6;
    const double* en = kr + 9;
    const double* es = kr + 12;
    double urel[3];
    for (int c = 0; c < 3; ++c) urel[c] = acc[1 + c] * a.vscale - vel[c];
    const double along = dot3(urel, es);
    double up[3];
    for (int c = 0; c < 3; ++c) up[c] = urel[c] - along * es[c];
    const double speed = sqrt(dot3(up, up));
    if (!(speed >= 1e-12)) return;  // DEGENERATE_SPEED (actuator.py:30)
    const double phi = atan2(dot3(up, en), dot3(up, ec));
    double alpha = phi - ps.twist;
    double ed[3], el[3];
    for (int c = 0; c < 3; ++c) ed[c] = up[c] / speed;
    cross3(es, ed, el);
    double x0, c0l, c0d, xn, cnl, cnd;
    polar_row(a, ps, 0, x0, c0l, c0d);
    polar_row(a, ps, ps.rows - 1, xn, cnl, cnd);
    if (alpha < x0 || alpha > xn) {
        if (lane == 0) atomicOr(&a.clamp_flags[ps.pid], 1);
        alpha = fmin(fmax(alpha, x0), xn);
    }
    double cl, cd;
    polar_interp(a, ps, alpha, lane, cl, cd);
    const double rho_phys = acc[0] * a.rho_ref;
    if (!(rho_phys > 0.0) && lane == 0) atomicOr(a.error_flags, 1);
    const double scale = 0.5 * rho_phys * speed * speed * ps.chord * ps.elen;
    for (int c = 0; c < 3; ++c) blade[c] = scale * (cl * el[c] + cd * ed[c]);
}

// per-axis deposit cells + weights, images across periodic faces computed
// from the shifted position pos - w*L (actuator.py:190-195, 330-332)
// Gaussian kernel (extension): cells j with |x - (j + 1/2)| <= 3 eps,
// weights exp(-(r/eps)^2) normalised over that support (per axis, so the
// deposited momentum equals the point force for interior points).
__device__ __forceinline__ void gaussian_support(double xs, double eps, int64_t& jlo,
                                                 int64_t& jhi, double& inv_sum) {
    const double R = 3.0 * eps;
    jlo = (int64_t)ceil(xs - 0.5 - R);
    jhi = (int64_t)floor(xs - 0.5 + R);
    double sum = 0.0;
    for (int64_t j = jlo; j <= jhi; ++j) {
        const double r = (xs - ((double)j + 0.5)) / eps;
        sum += exp(-r * r);
    }
    inv_sum = 1.0 / sum;
}

LBW_CHAIN_FN void deposit_axis(double x, int64_t L, int periodic, int kernel, double eps, int kw,
                             int32_t* dc, double* dw) {
    int cnt = 0;
    for (int q = 0; q < kw; ++q) {
        dc[q] = -1;
        dw[q] = 0.0;
    }
    const int nimg = periodic ? 3 : 1;
    for (int im = 0; im < nimg; ++im) {
        const double w = im == 0 ? 0.0 : (im == 1 ? 1.0 : -1.0);
        const double xs = im == 0 ? x : x - w * (double)L;
        if (kernel == LBW_SPREAD_GAUSSIAN) {
            int64_t jlo, jhi;
            double inv_sum;
            gaussian_support(xs, eps, jlo, jhi, inv_sum);
            for (int64_t j = jlo; j <= jhi; ++j) {
                if (j < 0 || j >= L || cnt >= kw) continue;
                const double r = (xs - ((double)j + 0.5)) / eps;
                dc[cnt] = (int32_t)j;
                dw[cnt] = exp(-r * r) * inv_sum;
                ++cnt;
            }
            continue;
        }
        const double n0f = floor(xs);
        const int64_t n0 = (int64_t)n0f;
        const double r[3] = {xs - (n0f - 0.5), xs - (n0f + 0.5), xs - (n0f + 1.5)};
        for (int q = 0; q < 3; ++q) {
            const int64_t c = n0 - 1 + q;
            if (c < 0 || c >= L) continue;
            const double wt = roma(r[q]);
            if (wt == 0.0 || cnt >= kw) continue;
            dc[cnt] = (int32_t)c;
            dw[cnt] = wt;
            ++cnt;
        }
    }
}

// (x,y) row of deposit pair q = p*9 + k (k: 3 x-cells x 3 y-cells of point
// p) as a slab row index, or -1 when it is not a cell of this slab.
__device__ __forceinline__ int32_t pair_row(const AlmDev& a, const Geom& g, int q) {
    const int kw = a.kw, kk = kw * kw;
    const int32_t* dc = a.dep_cell + (int64_t)(q / kk) * 3 * kw;
    const int k = q % kk;
    const int32_t cxg = dc[k / kw], cy = dc[kw + k % kw];
    const int64_t x = (int64_t)cxg - g.x0;
    if (cxg < 0 || cy < 0 || x < 0 || x >= g.nxl) return -1;
    return (int32_t)(x * g.ny + cy);
}


// deposit cells of a wide (Gaussian) kernel, stored straight to the point's
// deposit arrays; out of line to keep the Roma path of K4 compact
LBW_CHAIN_COLD void deposit_axis_wide(const AlmDev& a, int p, int k, double x, int64_t L,
                                               int per) {
    const int kw = a.kw;
    int32_t dc[kMaxKw];
    double dw[kMaxKw];
    deposit_axis(x, L, per, a.kernel, a.eps, kw, dc, dw);
    for (int q = 0; q < kw; ++q) {
        a.dep_cell[(int64_t)p * 3 * kw + kw * k + q] = dc[q];
        a.dep_w[(int64_t)p * 3 * kw + kw * k + q] = dw[q];
    }
}

// K4: one warp per point
// phase 0: single slab, everything in one pass.  Multi-slab: phase 1 only
// computes the cube values of this slab's cells and stores them into the
// local and both neighbours' cube buffers; phase 2 (after the neighbours'
// stores are visible) continues from the cube buffer.

// Where the sampled macro of global cell (gx,gy,gz) comes from, with the
// ghost rules of macro_at_raw in steady state (the x-face BC has run):
// MA_CONST with its value in out, or MA_OWNED with the slab-local cell.
__device__ __forceinline__ int corner_map(const Geom& g, int per_x, int inflow, const double* u_in,
                                          int64_t gx, int64_t gy, int64_t gz, int& x, int& y,
                                          int& z, double out[4]) {
    out[0] = 1.0;
    out[1] = out[2] = out[3] = 0.0;
    if (gx < 0 || gx >= g.nxg) {
        if (per_x) {
            gx = gx < 0 ? gx + g.nxg : gx - g.nxg;
        } else if (inflow && gx < 0) {
            out[1] = u_in[0];
            out[2] = u_in[1];
            out[3] = u_in[2];
            return MA_CONST;
        } else if (inflow && gx >= g.nxg) {
            gx = g.nxg - 1;
        } else {
            return MA_CONST;
        }
    }
    if (gy < 0 || gy >= g.ny) {
        if (!g.per_y) return MA_CONST;
        gy = gy < 0 ? gy + g.ny : gy - g.ny;
    }
    if (gz < 0 || gz >= g.nz) {
        if (!g.per_z) return MA_CONST;
        gz = gz < 0 ? gz + g.nz : gz - g.nz;
    }
    x = (int)(gx - g.x0);
    y = (int)gy;
    z = (int)gz;
    return MA_OWNED;
}

// Sampled macro from the pool the previous sweep filled (fused step):
// the (rho, u) its collide computed for the keyed rows, already rounded
// to the storage type as the reference's macro array holds them.
__device__ __forceinline__ int pool_macro(const Geom& g, const FsPool& pl, int per_x, int64_t gx,
                                          int64_t gy, int64_t gz, double out[4], int pc = -1) {
    int x = 0, y = 0, z = 0;
    const int code = corner_map(g, per_x, pl.inflow, pl.u_in, gx, gy, gz, x, y, z, out);
    if (code != MA_OWNED) return code;
    const uint64_t key = __ldcg(reinterpret_cast<const unsigned long long*>(pl.skey) +
                                (int64_t)x * g.ny + y);
    if ((uint32_t)(key >> 32) != pl.tag) {
        atomicOr(pl.error_flags, 8);
        return code;
    }
    const double* b = pl.spool + (int64_t)(uint32_t)key * 4 * g.zp + z;
#pragma unroll
    for (int q = 0; q < 4; ++q) out[q] = __ldcg(b + (int64_t)q * g.zp);
    if (pl.raw) {
        // out = (rho, mx, my, mz); the force of the previous sweep at the
        // cell, then u exactly as moments_exact forms it (dt = 1)
        double F[3];
        const int nt = (pl.cf_n && pc >= 0) ? pl.cf_n[pc] : -1;
        if (nt >= 0) {
            // the listed deposit terms, in actuator_force_k's order
            F[0] = F[1] = F[2] = 0.0;
            for (int t = 0; t < nt; ++t) {
                const int p = pl.cf_p[(int64_t)pc * kCornerTerms + t];
                const double w = pl.cf_w[(int64_t)pc * kCornerTerms + t];
                for (int c = 0; c < 3; ++c) {
                    const double v = __dadd_rn(F[c], __dmul_rn(w, pl.fv.flat[p * 3 + c]));
                    F[c] = g.single ? (double)(float)v : v;
                }
            }
        } else {
            const uint64_t fkey = pl.fv.row_key ? pl.fv.row_key[(int64_t)x * g.ny + y] : 0ull;
            if (g.single) force_from_key<float>(pl.fv, g, fkey, x, y, z, F[0], F[1], F[2]);
            else force_from_key<double>(pl.fv, g, fkey, x, y, z, F[0], F[1], F[2]);
        }
        const double inv_rho = 1.0 / out[0];
        const double hdt = 0.5 * 1.0;
        for (int q = 0; q < 3; ++q) out[1 + q] = (out[1 + q] + hdt * F[q]) * inv_rho;
        if (g.single)
            for (int q = 0; q < 4; ++q) out[q] = stored<float>(out[q]);
    }
    return MA_OWNED;
}

// Flow-independent per-point inputs, loaded by the kernel before anything
// that waits (kinematics row one value per lane, polar / chord data).
struct PointInputs {
    double kv;
    PointStatic ps;
    bool disk;
#ifdef LBW_K4_PROF
    long long t0, t1;
#endif
};
__device__ __forceinline__ PointInputs load_point_inputs(const AlmDev& a, int p, int lane) {
    PointInputs in;
    in.kv = lane < 15 ? a.kin[(int64_t)p * kKin + lane] : 0.0;
    in.ps = load_static(a, p, lane);
    in.disk = a.point_ring != nullptr && a.point_ring[p] >= 0;
    return in;
}

LBW_CHAIN_FN void point_warp(const AlmDev& a, const Geom& g, const MacroDev& m, const ForceSet& s,
                           int phase, const CubeArgs& cube, int p, int lane,
                           const PointInputs& in, const FsPool* pool = nullptr,
                           bool geometry = true) {
    const PointStatic& ps = in.ps;
    const bool disk = in.disk;
    double kr[15];
    for (int k = 0; k < 15; ++k) kr[k] = __shfl_sync(0xffffffffu, in.kv, k);
#ifdef LBW_K4_PROF
    const long long t2 = clock64();   // kinematics row available
#endif
    const double* kin = kr;
    // deposit cells / Roma weights per axis (lanes 8..10), kept in registers
    // for the row tags below and stored for the sweep / fill / next sample
    const int kw = a.kw;
    int32_t dcl[3] = {-1, -1, -1};   // Roma: kept in registers for the row tags
    if (geometry && phase != 1 && lane >= 8 && lane <= 10) {
        const int k = lane - 8;
        const int64_t L = k == 0 ? g.nxg : (k == 1 ? g.ny : g.nz);
        const int per = k == 0 ? m.per_x : (k == 1 ? g.per_y : g.per_z);
        if (kw == 3) {
            double dwl[3];
            deposit_axis(kin[k], L, per, LBW_SPREAD_ROMA, 0.0, 3, dcl, dwl);
            for (int q = 0; q < 3; ++q) {
                a.dep_cell[(int64_t)p * 9 + 3 * k + q] = dcl[q];
                a.dep_w[(int64_t)p * 9 + 3 * k + q] = dwl[q];
            }
        } else {
            deposit_axis_wide(a, p, k, kin[k], L, per);
        }
    }
    int64_t j0[3];
    double t[3];
    for (int k = 0; k < 3; ++k) {
        const double fl = floor(kin[k] - 0.5);
        j0[k] = (int64_t)fl;
        t[k] = kin[k] - 0.5 - fl;
    }
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    bool have = true;  // this lane's cube cell is this step's value
    if (phase == 2) {
        if (lane < 8) {
            for (int q = 0; q < 4; ++q) v[q] = cube.local[((int64_t)p * 8 + lane) * 4 + q];
            have = cube.tag_local[(int64_t)p * 8 + lane] == cube.epoch;
        }
    } else if (lane < 8) {
        const int64_t cgx = j0[0] + ((lane >> 2) & 1), cgy = j0[1] + ((lane >> 1) & 1),
                      cgz = j0[2] + (lane & 1);
        const int code = pool ? pool_macro(g, *pool, m.per_x, cgx, cgy, cgz, v, p * 8 + lane)
                              : macro_at(g, m, cgx, cgy, cgz, v);
        if (phase == 1) {
            const int64_t o = ((int64_t)p * 8 + lane) * 4;
            if (code != MA_REMOTE) {
                for (int q = 0; q < 4; ++q) cube.local[o + q] = v[q];
                cube.tag_local[(int64_t)p * 8 + lane] = cube.epoch;
            }
            if (code == MA_OWNED)
                for (int side = 0; side < 2; ++side)
                    if (cube.peer[side]) {
                        for (int q = 0; q < 4; ++q) cube.peer[side][o + q] = v[q];
                        cube.tag_peer[side][(int64_t)p * 8 + lane] = cube.epoch;
                    }
        }
    }
    if (phase == 1) return;
    const bool complete = __all_sync(0xffffffffu, have);
#ifdef LBW_K4_PROF
    const long long t3 = clock64();   // cube macro done
#endif
    // lane 0: trilinear sum in (dx,dy,dz) lexicographic order (actuator.py:88-92)
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int c = 0; c < 8; ++c) {
        double vc[4];
        for (int q = 0; q < 4; ++q) vc[q] = __shfl_sync(0xffffffffu, v[q], c);
        const double wx = (c >> 2) & 1 ? t[0] : 1.0 - t[0];
        const double wy = (c >> 1) & 1 ? t[1] : 1.0 - t[1];
        const double wz = c & 1 ? t[2] : 1.0 - t[2];
        const double w = wx * wy * wz;
        for (int q = 0; q < 4; ++q) acc[q] += w * vc[q];
    }
    if (s.flag_rows && phase != 1) {
        // tag this step's rows (benign race: equal values); for the Roma
        // kernel the x / y cells come from lanes 8 / 9 by shuffle
        if (kw == 3) {
            int32_t cx[3], cy[3];
            for (int q = 0; q < 3; ++q) {
                cx[q] = __shfl_sync(0xffffffffu, dcl[q], 8);
                cy[q] = __shfl_sync(0xffffffffu, dcl[q], 9);
            }
            if (lane < 9) {
                const int32_t cxg = cx[lane / 3], cyy = cy[lane % 3];
                const int64_t x = (int64_t)cxg - g.x0;
                LBW_CHECK(cyy < g.ny);
                if (cxg >= 0 && cyy >= 0 && x >= 0 && x < g.nxl)
                    s.row_key[x * g.ny + cyy] = row_key_of(s.tag, 0);
            }
        } else {
            __syncwarp();   // the deposit cells stored above are visible to the warp
            for (int t = lane; t < kw * kw; t += 32) {
                const int32_t row = pair_row(a, g, p * kw * kw + t);
                if (row >= 0) s.row_key[row] = row_key_of(s.tag, 0);
            }
        }
    }
    // Multi-slab: only points whose Roma support reaches this slab (their
    // sampling cube is then complete: own + neighbour cells) are evaluated;
    // per-point outputs come from the slab owning floor(x).  (Warp-uniform.)
    const int64_t n0 = (int64_t)floor(kin[0]);
    const int64_t ox = n0 - g.x0;
    const bool owner = phase == 0 || (ox >= 0 && ox < g.nxl);
    bool relevant = phase == 0;
    for (int dxc = -a.halo_x; dxc <= a.halo_x && !relevant; ++dxc) {
        int64_t c = n0 + dxc;
        if (m.per_x) c = (c % g.nxg + g.nxg) % g.nxg;
        relevant = c - g.x0 >= 0 && c - g.x0 < g.nxl;
    }
    double blade[3] = {0.0, 0.0, 0.0};
    if (relevant && !disk) blade_force_warp(a, ps, kin, acc, blade, lane);
#ifdef LBW_K4_PROF
    const long long t4 = clock64();
    if (lane == 0 && p == 0 && (a.step % 50) == 0)
        printf("K4PROF step %lld inputs+stage %lld kin %lld cube %lld blade %lld\n", (long long)a.step,
               in.t1 - in.t0, t2 - in.t1, t3 - t2, t4 - t3);
#endif
    if (lane == 0) {
        for (int q = 0; q < 4; ++q) a.samples[p * 4 + q] = owner ? acc[q] : 0.0;
        for (int c = 0; c < 3; ++c) {
            a.blade[p * 3 + c] = owner ? blade[c] : 0.0;
            a.flat[p * 3 + c] = -blade[c] * a.dt2 / a.den;  // units.py:69
            if (a.loads_row) a.loads_row[p * 3 + c] = owner ? blade[c] : 0.0;
        }
        if (disk) {
            // ring averages need every sample of the ring, owned or not
            for (int q = 0; q < 4; ++q) a.ring_samples[p * 4 + q] = acc[q];
            a.ring_sample_ok[p] = complete ? 1 : 0;
        }
    }
}

// K4d: actuator-disk rings (actuator.py:149-183), one thread per ring, fixed
// summation order.  Fluid force per sample = direction * thrust/area_ring *
// area_i * axis; the blade force is its negation (sim.py:236-244).
// Slab-local view of a disk point (multi-slab): its Roma support reaches
// this slab / floor(x) lies in it.
LBW_CHAIN_FN bool point_relevant(const Geom& g, int per_x, int halo, double x) {
    const int64_t n0 = (int64_t)floor(x);
    for (int dxc = -halo; dxc <= halo; ++dxc) {
        int64_t c = n0 + dxc;
        if (per_x) c = (c % g.nxg + g.nxg) % g.nxg;
        if (c - g.x0 >= 0 && c - g.x0 < g.nxl) return true;
    }
    return false;
}

LBW_CHAIN_FN void disk_ring(const AlmDev& a, const Geom& g, int per_x, int linked, int r) {
    const int first = a.ring_first[r], cnt = a.ring_count[r];
    const double ct = a.ring_ct[r];
    if (linked) {
        // across slabs: the ring's samples must all be known here (owned by
        // this slab or a neighbour) if any of its forces land here
        bool all_ok = true, needed = false;
        for (int i = 0; i < cnt; ++i) {
            const int p = first + i;
            all_ok &= a.ring_sample_ok[p] != 0;
            needed |= point_relevant(g, per_x, a.halo_x, a.kin[(int64_t)p * kKin]);
        }
        if (!needed) {
            for (int i = 0; i < cnt; ++i)
                for (int c = 0; c < 3; ++c) {
                    a.blade[(first + i) * 3 + c] = 0.0;
                    a.flat[(first + i) * 3 + c] = 0.0;
                }
            return;
        }
        if (!all_ok) {
            atomicOr(a.error_flags, 4);
            return;
        }
    }
    const double* k0 = a.kin + (int64_t)first * kKin;
    double axis[3] = {k0[6], k0[7], k0[8]};
    const double nrm = sqrt(dot3(axis, axis));
    for (int c = 0; c < 3; ++c) axis[c] = axis[c] / nrm;
    if (ct == 0.0) return;  // forces stay zero
    const double ind = (1.0 - sqrt(1.0 - ct)) / 2.0;
    double ring_area = 0.0, su = 0.0, srho = 0.0;
    for (int i = 0; i < cnt; ++i) {
        const int p = first + i;
        const double ar = a.area[p];
        double up[3];
        for (int c = 0; c < 3; ++c) up[c] = a.ring_samples[p * 4 + 1 + c] * a.vscale;
        ring_area += ar;
        su += dot3(up, axis) * ar;
        srho += a.ring_samples[p * 4] * a.rho_ref * ar;
    }
    const double u_d = su / ring_area;
    const double rho = srho / ring_area;
    const double u_inf = u_d / (1.0 - ind);
    const double thrust = 0.5 * rho * u_inf * u_inf * ct * ring_area;
    const double direction = u_d != 0.0 ? (u_d > 0.0 ? -1.0 : 1.0) : 0.0;
    const double per_area = thrust / ring_area;
    for (int i = 0; i < cnt; ++i) {
        const int p = first + i;
        const int64_t ox = (int64_t)floor(a.kin[(int64_t)p * kKin]) - g.x0;
        const bool owner = !linked || (ox >= 0 && ox < g.nxl);
        for (int c = 0; c < 3; ++c) {
            const double f = direction * per_area * a.area[p] * axis[c];
            a.blade[p * 3 + c] = owner ? -f : 0.0;
            a.flat[p * 3 + c] = f * a.dt2 / a.den;
        }
    }
}

// Flow-independent geometry of step j for the fused step (KK, after the
// CTA's kinematics): per point the per-axis deposit cells and weights
// (actuator.py:190-195), the force rows its deposit touches (tag j+1, the
// rows sweep j sums point forces in), and the rows of its sampling cube
// (sample keys: sweep j-1 stores its macro there for K4(j)).  Rows shared
// by several points get one key each write; any writer's slot is valid.
LBW_CHAIN_FN void fs_geometry(const FsGeom& geo, const AlmDev& a, const Geom& g, int per_x, int tid,
                            int nthr) {
    // whole CTA; one thread per (point, axis), then per (point, corner row)
    // and per deposit (x, y) pair: a point's three axes are independent
    // chains of sqrt / division latency, so they run side by side
    __shared__ int32_t s_dc[2][kOnTheFlyMaxPoints * kMaxKw];   // x / y deposit cells
    const int kw = a.kw;
    for (int t = tid; t < 3 * a.n; t += nthr) {
        const int p = t / 3, k = t % 3;
        const double xk = a.kin[(int64_t)p * kKin + k];
        const int64_t L = k == 0 ? g.nxg : (k == 1 ? g.ny : g.nz);
        const int per = k == 0 ? per_x : (k == 1 ? g.per_y : g.per_z);
        int32_t dc[kMaxKw];
        double dw[kMaxKw];
        deposit_axis(xk, L, per, a.kernel, a.eps, kw, dc, dw);
        for (int q = 0; q < kw; ++q) {
            geo.dep_cell[((int64_t)p * 3 + k) * kw + q] = dc[q];
            geo.dep_w[((int64_t)p * 3 + k) * kw + q] = dw[q];
            if (k < 2) s_dc[k][p * kw + q] = dc[q];
        }
    }
    const double zero3[3] = {0.0, 0.0, 0.0};
    for (int t = tid; t < 4 * a.n; t += nthr) {
        const int p = t >> 2, c = t & 3;
        const double* kr = a.kin + (int64_t)p * kKin;
        const int64_t j0x = (int64_t)floor(kr[0] - 0.5), j0y = (int64_t)floor(kr[1] - 0.5);
        int x = 0, y = 0, z = 0;
        double v[4];
        if (corner_map(g, per_x, geo.inflow, zero3, j0x + (c >> 1), j0y + (c & 1), 0, x, y, z,
                       v) == MA_OWNED)
            geo.skey[(int64_t)x * g.ny + y] = row_key_of(geo.tag, p * 4 + c);
    }
    __syncthreads();
    for (int t = tid; t < a.n * kw * kw; t += nthr) {
        const int p = t / (kw * kw), i = (t / kw) % kw, l = t % kw;
        const int32_t cxg = s_dc[0][p * kw + i], cy = s_dc[1][p * kw + l];
        const int64_t x = (int64_t)cxg - g.x0;
        if (cxg >= 0 && cy >= 0 && x >= 0 && x < g.nxl)
            geo.frow_key[x * g.ny + cy] = row_key_of(geo.tag, 0);
    }
}

}  // namespace
}  // namespace LBW_FLAVOR
}  // namespace lbw
