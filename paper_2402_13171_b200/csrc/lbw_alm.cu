// lbw_alm.cu — actuator-line coupling on the device (compiled with
// -fmad=false like the exact sweep: the per-point arithmetic follows the
// reference expression order).  Per step, three small launches precede
// the sweep:
//
//   KK  k_kinematics       (device kinematics mode) one CTA: advance every
//                          component's spin by R(axis, rate dt), compose the
//                          world frames down the tree, then every point's
//                          position, velocity and chord/normal/span frame
//                          (turbine.py:227-311, sim.py:167-191)
//   K4  k_alm_points       one warp per point: lanes 0-7 recompute the
//                          previous step's macro at the 8 sampling-cube cells
//                          from the retained population buffer (SURVEY.md
//                          App. A.7); lane 0 interpolates, evaluates angle of
//                          attack, polar and blade-element force
//                          (actuator.py:70-146, polars.py:65-80,
//                          sim.py:210-235); lanes 0-2 build the per-axis Roma
//                          deposit lists with periodic images
//                          (actuator.py:100-110, 190-195, 297-341); lane 0
//                          claims a pool slot for every touched (x,y) row
//   K5  k_alm_fill         one CTA per claimed row: per cell, the sum of
//                          (wx*wy)*wz*F over the points in ascending global id
//                          from 0.0 (actuator.py:204-247) — deterministic, no
//                          float atomics.  CTA 0 also clears the other force
//                          set (last read by this step's K4) for the next step.
#include <algorithm>
#include <climits>
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <vector>

#include "lbw_domain.h"

#define LBW_FAST 0
#include "lbw_sweep.cuh"
#define LBW_CHAIN_FN __device__ __forceinline__
#define LBW_CHAIN_COLD __device__ __forceinline__
#include "lbw_chain.cuh"

namespace lbw {

struct AlmState {
    int32_t n = 0, n_polars = 0;
    double *chord = nullptr, *elen = nullptr, *twist = nullptr;
    int32_t *polar_index = nullptr, *polar_offset = nullptr, *polar_rows = nullptr;
    double *p_alpha = nullptr, *p_cl = nullptr, *p_cd = nullptr;
    double* kin = nullptr;       // (kSlots,P,18): slot m % kSlots (kinematics run ahead)
    double *samples = nullptr;   // (2,P,4)
    double *blade = nullptr;     // (2,P,3)
    double *flat = nullptr;      // (P,3)
    double* cube = nullptr;      // (2,P,8,4) sampled cube values + (2,P,8) tags (multi-slab)
    double* ring_samples = nullptr;
    int32_t* ring_sample_ok = nullptr;
    int32_t* dep_cell = nullptr;
    double* dep_w = nullptr;
    int32_t *clamp_flags = nullptr, *error_flags = nullptr;
    int32_t *point_ring = nullptr, *ring_first = nullptr, *ring_count = nullptr;
    double *area = nullptr, *ring_ct = nullptr;
    int32_t n_rings = 0;
    double vscale = 0, rho_ref = 0, dt2 = 0, den = 0;
    ForceSet set[2];
    // Few points: the sweep sums a tagged cell's force from the points'
    // deposit data itself (no fill kernel, no pool); many points: K5 fills
    // per-row pools.
    bool on_the_fly = false;
    int32_t kw = 3, kernel = 0, halo_x = 1;
    double eps = 0.0;
    double* h_ring = nullptr;   // pinned (kRing, P, 18)
    cudaEvent_t ring_ev[kRing] = {};
    int ring_pos = 0;
    int64_t kin_queued_step = -1;  // host kinematics uploaded for this step
    int64_t ready_step = -1;       // step whose actuator chain is queued and valid
    // device kinematics run on their own stream, one step ahead
    cudaStream_t kin_stream = nullptr;
    cudaEvent_t ev_kin_done = nullptr;
    cudaEvent_t ev_chain_done[2] = {nullptr, nullptr};  // chain of a step parity done
    int64_t kin_valid[kSlots] = {-1, -1, -1, -1, -1, -1};  // step whose kinematics kin[slot] holds
    // sweep gate (alm_gate): chain-done flag, per-slot x range of each step's
    // deposits and sampling, KK completion per slot
    uint32_t* gate_flag = nullptr;
    int32_t* gate_box = nullptr;     // (3, 2) local planes, inclusive
    cudaEvent_t ev_kin_step[kSlots] = {};
    // per-step blade-force series (lbw_alm_record_loads)
    double* h_loads = nullptr;   // pinned (loads_cap, P, 3)
    double* d_loads = nullptr;   // its device mapping (the fused step writes it in-kernel)
    int64_t loads_cap = 0, loads_from = 0;
    // device kinematics
    bool kin_device = false;
    int32_t nc = 0;
    int32_t *k_parent = nullptr, *k_line_first = nullptr, *k_line_count = nullptr;
    int32_t* k_point_comp = nullptr;
    double *k_rel_p = nullptr, *k_rel_T = nullptr, *k_axis = nullptr, *k_rate = nullptr;
    double *k_rstep = nullptr, *k_spin = nullptr, *k_off = nullptr, *k_orient = nullptr;
    double *k_lframe = nullptr, *k_cs = nullptr;
    double *k_spin_hist = nullptr, *k_cs_hist = nullptr;
    int32_t* k_is_disk = nullptr;
    double* k_disk_center = nullptr;
    double k_dx = 1.0;
    int64_t kin_state_step = 0;  // step whose kinematics the device spins represent
    bool kin_stage_points = false;
    int32_t *k_order = nullptr, *k_level_start = nullptr, *k_static = nullptr;
    int32_t k_nlevels = 0;
    bool kin_static_ready = false;   // static components' state computed once
    size_t kin_smem = 0;
    long long* k_img_prm = nullptr;    // constant smem image of the kinematics CTA (kinematics_cta)
    long long* k_img_tail = nullptr;
    int32_t k_img_words = 0;
    // fused step (lbw_fused.cuh): per-step geometry in slots j % kSlots, sample
    // pools by parity, task counters of two consecutive launches
    bool fs_alloc = false;
    int32_t* fs_dep_cell = nullptr;   // (3,P,3,kw)
    double* fs_dep_w = nullptr;       // (3,P,3,kw)
    uint64_t* fs_frow = nullptr;      // (3, rows)
    uint64_t* fs_skey = nullptr;      // (3, rows)
    double* fs_spool = nullptr;       // (2, 4P, 4, zp)
    uint32_t* fs_ctr = nullptr;       // (2, 2)
    int64_t fs_next = -1;             // step the pipeline is primed for
    unsigned long long* fs_prof = nullptr;   // (256, 8) timeline ring (LBW_FUSED_PROF)
    // chain B (flag-ordered, alm_chainb_*): flags [0] KK done (j+1), [1] K4
    // done (j+1), [2] samples of step j stored (j), [3] sample-warp count,
    // [4] K4 count, [5] a bounded wait expired; sample warps per geometry slot
    uint32_t* cb_flags = nullptr;
    int32_t* cb_pool_tiles = nullptr;   // (kSlots)
    bool loop_loaded = false;           // sweep kernels loaded (lazy module loading)
    int64_t cb_loop_end = -1;           // resident chain queued up to (excluding) this step
    cudaStream_t loop_stream = nullptr; // its stream, on the chain's SMs
    cudaEvent_t loop_ev = nullptr;      // stream handover per-step chain <-> loop
    bool loop_last = false;             // the last chain launch was the loop
    int loop_fit = -1;                  // resident chain fits the chain's SMs (-1: not checked)
    int32_t* cb_box_h = nullptr;        // (kSlots, 2) pinned, device-mapped: [x_first, x_len] hint per KK
    int32_t* cb_cf_n = nullptr;         // (kSlots, P, 8) corner-force term counts
    int16_t* cb_cf_p = nullptr;         // (kSlots, P, 8, kCornerTerms)
    double* cb_cf_w = nullptr;
    int32_t* cb_box_d = nullptr;
    int64_t cb_next = -1;               // step the chain-B pipeline is primed for
    int64_t fs_prof_n = 0;
    std::vector<void*> allocs;

    // device view for step m: outputs by parity, kinematics by m % kSlots
    AlmDev dev(int64_t m) const {
        const int parity = (int)(m & 1);
        AlmDev a;
        a.n = n;
        a.chord = chord;
        a.elen = elen;
        a.twist = twist;
        a.polar_index = polar_index;
        a.polar_offset = polar_offset;
        a.polar_rows = polar_rows;
        a.p_alpha = p_alpha;
        a.p_cl = p_cl;
        a.p_cd = p_cd;
        a.vscale = vscale;
        a.rho_ref = rho_ref;
        a.dt2 = dt2;
        a.den = den;
        a.kin = kin + (size_t)(m % kSlots) * n * kKin;
        a.samples = samples + (size_t)parity * n * 4;
        a.blade = blade + (size_t)parity * n * 3;
        a.flat = flat + (size_t)parity * n * 3;
        a.dep_cell = dep_cell + (size_t)parity * n * 3 * kw;
        a.dep_w = dep_w + (size_t)parity * n * 3 * kw;
        a.kw = kw;
        a.kernel = kernel;
        a.eps = eps;
        a.halo_x = halo_x;
        a.clamp_flags = clamp_flags;
        a.step = m;
        a.ring_samples = ring_samples;
        a.ring_sample_ok = ring_sample_ok;
        a.error_flags = error_flags;
        a.loads_row = nullptr;
        a.point_ring = point_ring;
        a.area = area;
        a.n_rings = n_rings;
        a.ring_first = ring_first;
        a.ring_count = ring_count;
        a.ring_ct = ring_ct;
        return a;
    }
    KinDev kdev() const {
        KinDev k;
        k.nc = nc;
        k.parent = k_parent;
        k.rel_p = k_rel_p;
        k.rel_T = k_rel_T;
        k.axis = k_axis;
        k.rate = k_rate;
        k.rstep = k_rstep;
        k.spin = k_spin;
        k.line_first = k_line_first;
        k.line_count = k_line_count;
        k.point_comp = k_point_comp;
        k.off = k_off;
        k.orient = k_orient;
        k.lframe = k_lframe;
        k.is_disk = k_is_disk;
        k.disk_center = k_disk_center;
        k.cs = k_cs;
        k.spin_hist = k_spin_hist;
        k.cs_hist = k_cs_hist;
        k.hist_slot = 0;
        k.box = nullptr;
        k.box_halo = halo_x + 2;
        k.stage_points = kin_stage_points ? 1 : 0;
        k.order = k_order;
        k.level_start = k_level_start;
        k.nlevels = k_nlevels;
        k.is_static = k_static;
        k.skip_static = 0;
        k.dx = k_dx;
        k.img_prm = k_img_prm;
        k.img_tail = k_img_tail;
        k.img_tail_words = k_img_words;
        return k;
    }
};

namespace {

__global__ void k_kinematics(KinDev k, AlmDev a, Geom g, int per_x, int advance) {
    extern __shared__ double ksm[];
    LBW_TRACE_BEGIN(1, a.step);
    kinematics_cta(k, a, g, per_x, advance, ksm, (int)threadIdx.x, (int)blockDim.x);
    LBW_TRACE_END(1, a.step);
}

__global__ void k_alm_points(AlmDev a, Geom g, MacroDev m, ForceSet s, int phase, CubeArgs cube) {
    extern __shared__ double alm_sm[];
    const int p = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    LBW_TRACE_BEGIN(2, a.step);
    // The sampled cells lie in the rows the previous step's points forced:
    // their force is summed from that step's deposit data (actuator view),
    // which is staged in shared memory first -- one parallel load instead
    // of a dependent global load per point inside every cube cell.
    // flow-independent loads of this warp's point are issued first, so their
    // latency overlaps the staging below
    const int lane = threadIdx.x & 31;
    PointInputs in{};
#ifdef LBW_K4_PROF
    const long long t0 = clock64();
#endif
    if (p < a.n) in = load_point_inputs(a, p, lane);
    const ForceView& fv = m.fv;
    if (fv.row_key != nullptr && fv.pool == nullptr && fv.npts > 0 && fv.npts <= kOnTheFlyMaxPoints &&
        phase != 2) {
        const int n = fv.npts, nd = n * 3 * fv.kw;
        double* w = alm_sm;                                   // (n, 3, kw)
        double* fl = w + nd;                                  // (n, 3)
        int32_t* dc = reinterpret_cast<int32_t*>(fl + n * 3); // (n, 3, kw)
        // every load of a thread is issued before its first shared store
        // (one DRAM round trip, not one per loop iteration)
        constexpr int U = 8;
        const int nb = (int)blockDim.x, n3 = n * 3;
        for (int i0 = threadIdx.x; i0 < nd || i0 < n3; i0 += U * nb) {
            double wv[U], flv[U];
            int32_t cv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * nb;
                if (i < nd) {
                    wv[u] = fv.dep_w[i];
                    cv[u] = fv.dep_cell[i];
                }
                if (i < n3) flv[u] = fv.flat[i];
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * nb;
                if (i < nd) {
                    w[i] = wv[u];
                    dc[i] = cv[u];
                }
                if (i < n3) fl[i] = flv[u];
            }
        }
        __syncthreads();
        m.fv.dep_w = w;
        m.fv.flat = fl;
        m.fv.dep_cell = dc;
    }
    if (p >= a.n) return;  // uniform per warp
#ifdef LBW_K4_PROF
    in.t0 = t0;
    in.t1 = clock64();
#endif
    point_warp(a, g, m, s, phase, cube, p, lane, in);
    LBW_TRACE_END(2, a.step);
}

__global__ void k_alm_disks(AlmDev a, Geom g, int per_x, int linked) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    LBW_TRACE_BEGIN(3, a.step);
    if (r < a.n_rings) disk_ring(a, g, per_x, linked, r);
    LBW_TRACE_END(3, a.step);
}

// Fused-step priming (lbw_fused.cuh): kinematics (when not yet computed)
// and the flow-independent geometry of step j, one CTA on the main stream.
__global__ void k_fs_prime(KinDev k, AlmDev a, Geom g, int per_x, int advance, int do_kin,
                           FsGeom geo) {
    extern __shared__ double psm[];
    if (do_kin) {
        kinematics_cta(k, a, g, per_x, advance, psm, (int)threadIdx.x, (int)blockDim.x);
        __syncthreads();
    }
    fs_geometry(geo, a, g, per_x, (int)threadIdx.x, (int)blockDim.x);
}

// ---------------------------------------------------------------- chain B
// Flags of the flag-ordered chain (AlmState::cb_flags): [0] kinematics of
// step j done = j+1, [1] point forces (K4) of step j done = j+1, [2] force-
// free sample sums of step j stored by sweep j-1 = j, [3] sample-tile count
// of the running sweep, [4] K4 warp count, [5] a bounded wait expired,
// [6] geometry of step j done = j+1 (published in step order).

// Geometry of step j (one CTA, kinematics of j done): deposit geometry and
// row keys (fs_geometry), the number of sweep tiles holding rows of step j's
// sampling cubes, the plane-order hint, then "geometry(j) done" = j+1 once
// geometry(j-1) has published (flags are maxima: publish in step order).
struct CornerLists {
    const int32_t* prev_cell;   // deposit cells / weights of the step before J
    const double* prev_w;       // (nullptr: not built)
    const double* ckin;         // kinematics rows of step J (its sampling corners)
    uint32_t ckin_value;        // wait for "kinematics done" >= this first (0: no wait)
    uint32_t k4_value;          // ... and for "K4 done" >= this (the slot's last reader)
    int32_t* n;                 // (P, 8)
    int16_t* p;                 // (P, 8, kCornerTerms)
    double* w;
    int32_t inflow;
    double u_in[3];
};

// For each sampling corner of this step: the previous step's deposit terms
// reaching that cell, in the order actuator_force_k adds them (ascending
// point, the last x / y match, every z match), weight (wx wy) wz rounded as
// there -- so the sampling sums a few terms instead of scanning the points.
__device__ __forceinline__ void cb_corner_lists(const AlmDev& a, const Geom& g, int per_x,
                                                const CornerLists& L, int tid, int nthr) {
    const int kw = a.kw;
    for (int q = tid; q < 8 * a.n; q += nthr) {
        const int pt = q >> 3, c = q & 7;
        const double* kr = L.ckin + (int64_t)pt * kKin;
        int64_t j0[3];
        for (int k = 0; k < 3; ++k) j0[k] = (int64_t)floor(kr[k] - 0.5);
        int x = 0, y = 0, z = 0;
        double v[4];
        const int code = corner_map(g, per_x, L.inflow, L.u_in, j0[0] + ((c >> 2) & 1),
                                    j0[1] + ((c >> 1) & 1), j0[2] + (c & 1), x, y, z, v);
        int cnt = 0;
        if (code == MA_OWNED) {
            const int64_t xg = g.x0 + x;
            for (int p = 0; p < a.n && cnt >= 0; ++p) {
                const int32_t* dc = L.prev_cell + (int64_t)p * 3 * kw;
                const double* dw = L.prev_w + (int64_t)p * 3 * kw;
                double wx = 0.0, wy = 0.0;
                bool hx = false, hy = false;
                for (int t = 0; t < kw; ++t) {
                    if (dc[t] == xg) { hx = true; wx = dw[t]; }
                    if (dc[kw + t] == y) { hy = true; wy = dw[kw + t]; }
                }
                if (!(hx && hy)) continue;
                const double wxy = __dmul_rn(wx, wy);
                for (int t = 0; t < kw; ++t) {
                    if (dc[2 * kw + t] != z) continue;
                    if (cnt >= kCornerTerms) { cnt = -1; break; }
                    L.p[(int64_t)q * kCornerTerms + cnt] = (int16_t)p;
                    L.w[(int64_t)q * kCornerTerms + cnt] = __dmul_rn(wxy, dw[2 * kw + t]);
                    ++cnt;
                }
            }
        }
        L.n[q] = cnt;
    }
}

__device__ __forceinline__ void cb_geometry_body(const AlmDev& a, const Geom& g, int per_x,
                                                 const FsGeom& geo, int warps_row,
                                                 int32_t* pool_tiles, uint32_t* flags,
                                                 uint32_t value, int32_t* box_hint,
                                                 const CornerLists& cl) {
    __shared__ uint32_t pairs[4 * kOnTheFlyMaxPoints];
    __shared__ uint32_t dup[4 * kOnTheFlyMaxPoints];
    __shared__ int cnt, blo, bhi;
    const int tid = (int)threadIdx.x, nthr = (int)blockDim.x;
    const int nq = 4 * a.n;
    if (tid == 0) {
        cnt = 0;
        blo = INT_MAX;
        bhi = INT_MIN;
    }
    fs_geometry(geo, a, g, per_x, tid, nthr);   // synchronises the CTA
    if (cl.prev_cell) {
        if (tid == 0) {
            int32_t* err = reinterpret_cast<int32_t*>(flags + 5);
            if (cl.ckin_value) gate_wait(flags, cl.ckin_value, err, 33);
            if (cl.k4_value) gate_wait(flags + 1, cl.k4_value, err, 34);
        }
        __syncthreads();
        cb_corner_lists(a, g, per_x, cl, tid, nthr);
    }
    // sampling rows -> sweep tiles (x plane, y block), and the plane range
    // of the points relative to point 0 (wrapped on a periodic x axis)
    const double zero3[3] = {0.0, 0.0, 0.0};
    const int64_t c0 = (int64_t)floor(a.kin[0]);
    for (int q = tid; q < nq; q += nthr) {
        const double* kr = a.kin + (int64_t)(q >> 2) * kKin;
        const int c = q & 3;
        const int64_t j0x = (int64_t)floor(kr[0] - 0.5), j0y = (int64_t)floor(kr[1] - 0.5);
        int x = 0, y = 0, z = 0;
        double v[4];
        pairs[q] = corner_map(g, per_x, geo.inflow, zero3, j0x + (c >> 1), j0y + (c & 1), 0, x, y,
                              z, v) == MA_OWNED
                       ? ((uint32_t)x << 16) | (uint32_t)y
                       : 0xffffffffu;
        dup[q] = 0u;
        if (c == 0) {
            int64_t dlt = (int64_t)floor(kr[0]) - c0;
            if (per_x) dlt = ((dlt + g.nxg / 2) % g.nxg + g.nxg) % g.nxg - g.nxg / 2;
            atomicMin(&blo, (int)dlt);
            atomicMax(&bhi, (int)dlt);
        }
    }
    __syncthreads();
    // distinct rows: every pair (r < q) compared once, spread over the CTA
    const int npair = nq * (nq - 1) / 2;
    for (int t = tid; t < npair; t += nthr) {
        int q = (int)((1.0 + sqrt(1.0 + 8.0 * (double)t)) * 0.5);
        while (q * (q - 1) / 2 > t) --q;
        while ((q + 1) * q / 2 <= t) ++q;
        const int r = t - q * (q - 1) / 2;
        if (pairs[q] == pairs[r]) dup[q] = 1u;
    }
    __syncthreads();
    for (int q = tid; q < nq; q += nthr)
        if (pairs[q] != 0xffffffffu && !dup[q]) atomicAdd(&cnt, 1);
    __syncthreads();
    if (tid == 0) {
        *pool_tiles = cnt * warps_row;   // sweep warps that store samples
        gate_wait(flags + 6, value - 1u, reinterpret_cast<int32_t*>(flags + 5), 35);
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + 6), "r"(value) : "memory");
        if (box_hint) {   // a hint in mapped host memory: after the release, no fence
            const int h = a.halo_x + 1;
            const int64_t first = c0 + blo - h - g.x0;
            const int len = (int)min((int64_t)(bhi - blo + 2 * h + 1), (int64_t)g.nxl);
            box_hint[0] = (int32_t)(((first % g.nxl) + g.nxl) % g.nxl);
            box_hint[1] = len;
        }
    }
}

// Kinematics of step j (one CTA), then "kinematics(j) done" = j+1.
__device__ __forceinline__ void cb_kin_body(const KinDev& k, const AlmDev& a, const Geom& g,
                                            int per_x, int advance, int do_kin, uint32_t* flags,
                                            uint32_t value, double* csm) {
    const int tid = (int)threadIdx.x, nthr = (int)blockDim.x;
    if (do_kin) kinematics_cta(k, a, g, per_x, advance, csm, tid, nthr);
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags), "r"(value) : "memory");
    }
}

// priming: kinematics + geometry of step j in one CTA, serially
__global__ void k_cb_kk(KinDev k, AlmDev a, Geom g, int per_x, int advance, int do_kin,
                        FsGeom geo, int warps_row, int32_t* pool_tiles, uint32_t* flags,
                        uint32_t value, int32_t* box_hint, CornerLists cl) {
    extern __shared__ double csm[];
    LBW_TRACE_BEGIN(1, a.step);
    cb_kin_body(k, a, g, per_x, advance, do_kin, flags, value, csm);
    __syncthreads();
    cb_geometry_body(a, g, per_x, geo, warps_row, pool_tiles, flags, value, box_hint, cl);
    LBW_TRACE_END(1, a.step);
}

struct CbChainArgs {
    Geom g;
    int32_t role;               // 0: K4(j), 1: kinematics(jk), 2: geometry(jk)
    // K4(j): 4 points (warps) per CTA
    AlmDev a;
    MacroDev md;
    FsPool pool;
    int32_t use_pool;
    const uint32_t* box_flag;   // sums of step j stored: *box_flag >= box_value
    uint32_t box_value;
    const int32_t* pool_tiles;  // of step j (0: nothing to wait for)
    uint32_t* flags;            // chain-B flags
    uint32_t k4_value;
    // kinematics / geometry of step jk (one CTA)
    int32_t kk_advance, kk_do_kin;
    KinDev k;
    AlmDev akk;
    FsGeom geo;
    int32_t per_x, warps_row;
    int32_t* pool_tiles_kk;
    uint32_t kin_value;         // jk + 1
    uint32_t slot_value;        // the slot of step jk is free once box >= slot_value
    int32_t* box_hint;          // (2) plane-order hint of step jk (mapped host memory)
    CornerLists cl;             // geometry: corner-force lists of step jk
};

// The chain of step j: three launches on the actuator stream -- K4(j),
// kinematics(j+4), geometry(j+3) -- ordered only by the flags: each waits
// in-kernel for what it reads, then lets the next launch on the stream be
// scheduled (griddepcontrol.launch_dependents; never griddepcontrol.wait),
// so only the kinematics (the turbine state advances step by step) and the
// point forces (each step samples the previous step's forces) form serial
// chains; the geometry of different steps overlaps.
//   K4(j):     geometry(j) done; sums of step j stored by sweep j-1; before
//              its force part, K4(j-1) done
//   kin(jk):   kin(jk-1) done; the slot of step jk free (box >= jk-4: sweep
//              jk-5 started, so sweep jk-6 -- the slot's last reader -- is done)
//   geo(jk):   kin(jk) done; slot free as above
template <int ROLE>
__global__ void __launch_bounds__(128) k_cb_chain(CbChainArgs A) {
    extern __shared__ double csm[];
    const int tid = (int)threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int32_t* err = reinterpret_cast<int32_t*>(A.flags + 5);
    if (ROLE == 1) {
        if (tid == 0) {
            gate_wait(A.flags, A.kin_value - 1u, err);
            gate_wait(A.box_flag, A.slot_value, err);
        }
        __syncthreads();
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        LBW_TRACE_BEGIN(1, A.akk.step);
        cb_kin_body(A.k, A.akk, A.g, A.per_x, A.kk_advance, A.kk_do_kin, A.flags, A.kin_value, csm);
        LBW_TRACE_END(5, A.akk.step);
        return;
    }
    if (ROLE == 2) {
        if (tid == 0) {
            gate_wait(A.flags, A.kin_value, err);
            gate_wait(A.box_flag, A.slot_value, err);
        }
        __syncthreads();
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        cb_geometry_body(A.akk, A.g, A.per_x, A.geo, A.warps_row, A.pool_tiles_kk, A.flags,
                         A.kin_value, A.box_hint, A.cl);
        LBW_TRACE_END(1, A.akk.step);
        return;
    }
    // K4(j).  The force view of step j-1 (it completes the pooled sums) is
    // staged in shared memory while the samples are being waited for.
    double* sw = csm;                                          // (n, 3, kw) weights
    double* sfl = sw + (size_t)A.a.n * 3 * A.a.kw;             // (n, 3) forces
    int32_t* sdc = reinterpret_cast<int32_t*>(sfl + (size_t)A.a.n * 3);  // (n, 3, kw) cells
    const bool stage = false;   // deposit terms come from the corner lists
    if (tid == 0) {
        gate_wait(A.flags + 6, A.k4_value, err);   // geometry(j) done: flag >= j+1
        if (A.use_pool && *(const volatile int32_t*)A.pool_tiles > 0)
            gate_wait(A.box_flag, A.box_value, err);
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int nd = stage ? A.a.n * 3 * A.a.kw : 0;
    for (int i = tid; i < nd; i += (int)blockDim.x) {
        sw[i] = A.pool.fv.dep_w[i];
        sdc[i] = A.pool.fv.dep_cell[i];
    }
    const int p = (int)blockIdx.x * 4 + warp;
    PointInputs in{};
    if (p < A.a.n) in = load_point_inputs(A.a, p, lane);
    if (A.use_pool) {
        if (tid == 0) gate_wait(A.flags + 1, A.k4_value - 1u, err);   // K4(j-1): its forces
        __syncthreads();
        for (int i = tid; i < A.a.n * 3; i += (int)blockDim.x) sfl[i] = A.pool.fv.flat[i];
        __syncthreads();
    }
    if (p >= A.a.n) return;   // uniform per warp
    LBW_TRACE_BEGIN(2, A.a.step);
#ifdef LBW_K4_PROF
    in.t0 = in.t1 = clock64();
#endif
    FsPool pool = A.pool;
    if (stage) {
        pool.fv.dep_w = sw;
        pool.fv.dep_cell = sdc;
    }
    if (A.use_pool) pool.fv.flat = sfl;   // staged after K4(j-1)
    ForceSet none{};
    CubeArgs cube{};
    point_warp(A.a, A.g, A.md, none, 0, cube, p, lane, in, A.use_pool ? &pool : nullptr, false);
    __syncwarp();
    if (lane == 0) {
        // the last point's warp publishes "K4(j) done"
        __threadfence();
        const uint32_t done = atomicAdd(A.flags + 4, 1u) + 1u;
        if (done == (uint32_t)A.a.n) {
            A.flags[4] = 0u;
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(A.flags + 1), "r"(A.k4_value)
                         : "memory");
        }
    }
    LBW_TRACE_END(2, A.a.step);
}

// The whole flag-ordered chain of steps j0 .. j0+nsteps-1 in ONE resident
// launch (a persistent kernel on the chain's SMs; 6 CTAs, clusters of 2):
//   CTAs 0-1 (cluster 0): K4(j), one warp per point, half the points each.
//     Each step's point forces stay in shared memory -- a CTA writes its
//     half into its own and, through distributed shared memory, its
//     partner's copy -- so the next step's sampling completes its sums
//     without a global round trip; steps hand over with a cluster barrier.
//   CTA 2: kinematics of steps j0+4 .. (serial, the turbine state advances)
//   CTAs 3..5: geometry of steps j0+3 .. round robin (one geometry takes
//     longer than a step) and the corner lists of the step after; they
//     publish in step order.
// All ordering is by the chain flags, as with the per-step launches.  One
// kernel instead of three PDL-chained launches per step (a launch chained
// by PDL only overlaps its direct predecessor, so the per-step chain is a
// serial sequence of launch latencies).  Unlike those launches it waits for
// sweeps queued AFTER it: the sweep kernels must be loaded before it runs
// (lazy module loading), and it needs all its CTAs resident (cb_loop_ok).
constexpr int kLoopMaxPoints = 18;
constexpr int kLoopThreads = 32 * ((kLoopMaxPoints + 1) / 2);   // 288
constexpr int kLoopGeoCtas = 3;                                 // geometry CTAs (grid 3 + this, even)
struct CbPersistArgs {
    Geom g;
    AlmDev a0;                 // constants; per-step pointers from the bases below
    KinDev k0;
    double *kin_base, *samples_base, *blade_base, *flat_base, *loads_base;
    int64_t loads_cap;
    FsPool pool0;              // constants (inflow, u_in, error flags, raw)
    uint64_t* skey_base;
    const double* spool_base;
    size_t spool_stride;
    uint64_t* frow_base;
    int32_t* dep_cell_base;
    double* dep_w_base;
    int32_t* cf_n_base;
    int16_t* cf_p_base;
    double* cf_w_base;
    int32_t* pool_tiles;
    int32_t* box_hint;         // (kSlots, 2) mapped host memory
    uint32_t* flags;
    int64_t rows, j0;
    int32_t nsteps, per_x, warps_row, inflow, first_skip_static;
    double u_in[3];
};

__device__ __forceinline__ AlmDev cb_step_view(const CbPersistArgs& P, int64_t j) {
    AlmDev a = P.a0;
    const int n = a.n;
    a.kin = P.kin_base + (size_t)(j % kSlots) * n * kKin;
    a.samples = P.samples_base + (size_t)(j & 1) * n * 4;
    a.blade = P.blade_base + (size_t)(j & 1) * n * 3;
    a.flat = P.flat_base + (size_t)(j & 1) * n * 3;
    a.loads_row = P.loads_base ? P.loads_base + (size_t)(j % P.loads_cap) * n * 3 : nullptr;
    a.step = j;
    return a;
}

__device__ __forceinline__ FsGeom cb_step_geo(const CbPersistArgs& P, int64_t j) {
    const size_t dep = (size_t)P.a0.n * 3 * P.a0.kw;
    FsGeom geo;
    geo.dep_cell = P.dep_cell_base + (size_t)(j % kSlots) * dep;
    geo.dep_w = P.dep_w_base + (size_t)(j % kSlots) * dep;
    geo.frow_key = P.frow_base + (size_t)(j % kSlots) * P.rows;
    geo.skey = P.skey_base + (size_t)(j % kSlots) * P.rows;
    geo.tag = (uint32_t)(j + 1);
    geo.inflow = P.inflow;
    return geo;
}

__global__ void __launch_bounds__(kLoopThreads, 1) k_cb_persist(CbPersistArgs P) {
    namespace cg = cooperative_groups;
    extern __shared__ double csm[];
    __shared__ double sfl[2][3 * kLoopMaxPoints];   // K4: every point's force, by step parity
    const int tid = (int)threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int n = P.a0.n, kw = P.a0.kw;
    int32_t* err = reinterpret_cast<int32_t*>(P.flags + 5);
    if (blockIdx.x == 2) {   // ---------------------------------- kinematics
        for (int st = 0; st < P.nsteps; ++st) {
            const int64_t jk = P.j0 + 4 + st;
            if (tid == 0) gate_wait(P.flags + 2, (uint32_t)(jk - 4), err, 2100 + (int32_t)(jk % 100));   // slot of jk-6 free
            __syncthreads();
            KinDev k = P.k0;
            k.hist_slot = (int32_t)(jk % kSlots);
            k.skip_static = (st > 0 || P.first_skip_static) ? 1 : 0;
            const AlmDev a = cb_step_view(P, jk);
            LBW_TRACE_BEGIN(1, jk);
            cb_kin_body(k, a, P.g, P.per_x, 1, 1, P.flags, (uint32_t)(jk + 1), csm);
            LBW_TRACE_END(5, jk);
            __syncthreads();
        }
        return;
    }
    if (blockIdx.x >= 3) {   // ------------------------------------ geometry
        // kLoopGeoCtas CTAs take the steps round robin (one geometry CTA
        // would take longer than a step); they publish in step order
        for (int st = (int)blockIdx.x - 3; st < P.nsteps; st += kLoopGeoCtas) {
            const int64_t jg = P.j0 + 3 + st;
            if (tid == 0) {
                gate_wait(P.flags, (uint32_t)(jg + 1), err, 3100 + (int32_t)(jg % 100));            // kinematics of jg
                gate_wait(P.flags + 2, (uint32_t)(jg - 4), err, 3200 + (int32_t)(jg % 100));        // its slot free
            }
            __syncthreads();
            const AlmDev a = cb_step_view(P, jg);
            CornerLists cl{};
            cl.prev_cell = cb_step_geo(P, jg).dep_cell;
            cl.prev_w = cb_step_geo(P, jg).dep_w;
            cl.ckin = P.kin_base + (size_t)((jg + 1) % kSlots) * n * kKin;
            cl.ckin_value = (uint32_t)(jg + 2);
            cl.k4_value = (uint32_t)(jg - 4);
            const size_t off = (size_t)((jg + 1) % kSlots) * n * 8;
            cl.n = P.cf_n_base + off;
            cl.p = P.cf_p_base + off * kCornerTerms;
            cl.w = P.cf_w_base + off * kCornerTerms;
            cl.inflow = P.inflow;
            for (int c = 0; c < 3; ++c) cl.u_in[c] = P.u_in[c];
            cb_geometry_body(a, P.g, P.per_x, cb_step_geo(P, jg), P.warps_row,
                             P.pool_tiles + jg % kSlots, P.flags, (uint32_t)(jg + 1),
                             P.box_hint + 2 * (jg % kSlots), cl);
            LBW_TRACE_END(1, jg);
            __syncthreads();
        }
        return;
    }
    // -------------------------------------------------------- K4 (cluster 0)
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned rank = cluster.block_rank();
    const int half = (n + 1) / 2;
    const int p = (int)rank * half + w;
    const bool mine = w < half && p < n;
    double* peer = cluster.map_shared_rank(&sfl[0][0], rank ^ 1u);
    if (tid == 0) gate_wait(P.flags + 1, (uint32_t)P.j0, err, 41);   // K4(j0-1) done
    __syncthreads();
    for (int i = tid; i < 3 * n; i += (int)blockDim.x)
        sfl[(P.j0 - 1) & 1][i] = P.flat_base[(size_t)((P.j0 - 1) & 1) * n * 3 + i];
    cluster.sync();
    const MacroDev md{};
    for (int st = 0; st < P.nsteps; ++st) {
        const int64_t j = P.j0 + st;
        if (tid == 0) {
            gate_wait(P.flags + 6, (uint32_t)(j + 1), err, 4200 + (int32_t)(j % 100));   // geometry(j)
            if (*(const volatile int32_t*)(P.pool_tiles + j % kSlots) > 0)
                gate_wait(P.flags + 2, (uint32_t)j, err, 4300 + (int32_t)(j % 100));       // sums stored by sweep j-1
        }
        __syncthreads();
        if (mine) {
            const AlmDev a = cb_step_view(P, j);
            FsPool pool = P.pool0;
            pool.skey = P.skey_base + (size_t)(j % kSlots) * P.rows;
            pool.spool = P.spool_base + (size_t)(j & 1) * P.spool_stride;
            pool.tag = (uint32_t)(j + 1);
            const FsGeom gp = cb_step_geo(P, j - 1);
            pool.fv = ForceView{gp.frow_key, nullptr, (uint32_t)j};
            pool.fv.npts = n;
            pool.fv.kw = kw;
            pool.fv.dep_cell = gp.dep_cell;
            pool.fv.dep_w = gp.dep_w;
            pool.fv.flat = sfl[(j - 1) & 1];
            pool.cf_n = P.cf_n_base + (size_t)(j % kSlots) * n * 8;
            pool.cf_p = P.cf_p_base + (size_t)(j % kSlots) * n * 8 * kCornerTerms;
            pool.cf_w = P.cf_w_base + (size_t)(j % kSlots) * n * 8 * kCornerTerms;
            LBW_TRACE_BEGIN(2, j);
            const PointInputs in = load_point_inputs(a, p, lane);
            ForceSet none{};
            CubeArgs cube{};
            point_warp(a, P.g, md, none, 0, cube, p, lane, in, &pool, false);
            __syncwarp();
            if (lane < 3) {
                const double v = a.flat[p * 3 + lane];   // this warp's own store
                sfl[j & 1][p * 3 + lane] = v;
                peer[(j & 1) * 3 * kLoopMaxPoints + p * 3 + lane] = v;
            }
            LBW_TRACE_END(2, j);
        }
        cluster.sync();   // both halves of step j's forces in both CTAs
        if (rank == 0 && tid == 0) {
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(P.flags + 1),
                         "r"((uint32_t)(j + 1))
                         : "memory");
        }
    }
}

// one chain launch; pdl: programmatic stream serialisation (actuator stream)
static cudaError_t launch_cb_chain(const CbChainArgs& A, unsigned grid, size_t smem,
                                   cudaStream_t st, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(128, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // one instantiation per role: each gets its own register allocation
    // (the kinematics / geometry CTAs wait resident on the chain's SMs)
    if (A.role == 1) return cudaLaunchKernelEx(&cfg, k_cb_chain<1>, A);
    if (A.role == 2) return cudaLaunchKernelEx(&cfg, k_cb_chain<2>, A);
    return cudaLaunchKernelEx(&cfg, k_cb_chain<0>, A);
}

// K5: one warp per deposit pair q.  The lowest pair touching a row owns it:
// it writes the row's force into pool slot q (per cell, the sum over all
// points touching the row in ascending id, as the reference's spreading
// loop adds them, actuator.py:241-246) and tags the row for this step.  No
// claims, counters or clearing: rows of earlier steps just keep old tags.
constexpr int kFillSmemPairs = 4096;
__global__ void k_alm_fill(AlmDev a, Geom g, ForceSet s) {
    __shared__ int32_t rows_sm[kFillSmemPairs];
    LBW_TRACE_BEGIN(4, a.step);
    const int kw = a.kw, npairs = a.n * kw * kw;
    const bool staged = npairs <= kFillSmemPairs;
    if (staged)
        for (int q = threadIdx.x; q < npairs; q += blockDim.x) rows_sm[q] = pair_row(a, g, q);
    __syncthreads();
    const int q = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (q >= npairs) return;  // uniform per warp
    const int32_t row = staged ? rows_sm[q] : pair_row(a, g, q);
    if (row < 0) return;
    bool dup = false;
    for (int c0 = 0; c0 < q && !dup; c0 += 32) {
        const int q2 = c0 + lane;
        const bool same = q2 < q && (staged ? rows_sm[q2] : pair_row(a, g, q2)) == row;
        dup = __any_sync(0xffffffffu, same);
    }
    if (dup) return;
    const int64_t xg = row / g.ny + g.x0;
    const int32_t y = row % g.ny;
    LBW_CHECK(q >= 0 && q < npairs && row >= 0 && row < (int64_t)g.nxl * g.ny);
    const int64_t row0 = (int64_t)q * 3 * g.zp;
    for (int z0 = 0; z0 < g.nz; z0 += 32) {
        const int z = z0 + lane;
        double F[3] = {0.0, 0.0, 0.0};
        for (int c0 = 0; c0 < a.n; c0 += 32) {
            const int pl = c0 + lane;
            bool hit = false;
            double wxy = 0.0;
            if (pl < a.n) {
                const int32_t* dc = a.dep_cell + (int64_t)pl * 3 * kw;
                const double* dw = a.dep_w + (int64_t)pl * 3 * kw;
                double wx = 0.0, wy = 0.0;
                bool hx = false, hy = false;
                for (int t = 0; t < kw; ++t) {
                    if (dc[t] == xg) { hx = true; wx = dw[t]; }
                    if (dc[kw + t] == y) { hy = true; wy = dw[kw + t]; }
                }
                hit = hx && hy;
                wxy = wx * wy;
            }
            unsigned bal = __ballot_sync(0xffffffffu, hit);
            while (bal) {
                const int src = __ffs(bal) - 1;
                bal &= bal - 1;
                const double w2 = __shfl_sync(0xffffffffu, wxy, src);
                const int p = c0 + src;
                if (z < g.nz) {
                    const int32_t* dc = a.dep_cell + (int64_t)p * 3 * kw + 2 * kw;
                    const double* dw = a.dep_w + (int64_t)p * 3 * kw + 2 * kw;
                    for (int t = 0; t < kw; ++t) {
                        if (dc[t] == z) {
                            const double w = w2 * dw[t];
                            // `force[c] += w * F_lat` on an array of the storage
                            // dtype rounds after every addition (actuator.py:246)
                            if (g.single)
                                for (int c = 0; c < 3; ++c)
                                    F[c] = stored<float>(F[c] + w * a.flat[p * 3 + c]);
                            else
                                for (int c = 0; c < 3; ++c) F[c] += w * a.flat[p * 3 + c];
                        }
                    }
                }
            }
        }
        if (z < g.nz) {
            if (g.single) {
                float* dst = static_cast<float*>(s.pool) + row0;
                for (int c = 0; c < 3; ++c) dst[(int64_t)c * g.zp + z] = (float)F[c];
            } else {
                double* dst = static_cast<double*>(s.pool) + row0;
                for (int c = 0; c < 3; ++c) dst[(int64_t)c * g.zp + z] = F[c];
            }
        }
    }
    if (lane == 0) s.row_key[row] = row_key_of(s.tag, q);
    LBW_TRACE_END(4, a.step);
}

template <class T>
int dev_alloc(lbw_domain* d, AlmState* s, T** p, size_t count) {
    if (count == 0) count = 1;
    if (cudaMalloc((void**)p, count * sizeof(T)) != cudaSuccess) {
        cudaGetLastError();
        set_error("ALM device allocation failed");
        return LBW_ENOMEM;
    }
    s->allocs.push_back(*p);
    d->bytes += (int64_t)(count * sizeof(T));
    return LBW_OK;
}

}  // namespace

bool alm_active(const lbw_domain* d) { return d->alm != nullptr && d->alm->n > 0; }

cudaError_t alm_sync_side(const lbw_domain* d) {
    if (!d->alm) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    if (d->alm->kin_stream && e == cudaSuccess) e = cudaStreamSynchronize(d->alm->kin_stream);
    if (d->alm->loop_stream && e == cudaSuccess) e = cudaStreamSynchronize(d->alm->loop_stream);
    return e;
}

int alm_support_halo(const lbw_domain* d) { return alm_active(d) ? d->alm->halo_x : 0; }

double* alm_cube(const lbw_domain* d) { return alm_active(d) ? d->alm->cube : nullptr; }

void alm_destroy(lbw_domain* d) {
    AlmState* s = d->alm;
    if (!s) return;
    if (s->kin_stream) cudaStreamSynchronize(s->kin_stream);
    if (s->loop_stream) {
        cudaStreamSynchronize(s->loop_stream);
        cudaStreamDestroy(s->loop_stream);
        cudaEventDestroy(s->loop_ev);
    }
    for (void* p : s->allocs) cudaFree(p);
    for (auto& e : s->ring_ev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {s->ev_kin_done, s->ev_chain_done[0], s->ev_chain_done[1]})
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : s->ev_kin_step)
        if (e) cudaEventDestroy(e);
    if (s->kin_stream) cudaStreamDestroy(s->kin_stream);
    if (s->h_ring) cudaFreeHost(s->h_ring);
    if (s->cb_box_h) cudaFreeHost(s->cb_box_h);
    if (s->h_loads) cudaFreeHost(s->h_loads);
    delete s;
    d->alm = nullptr;
}

bool alm_ready(const lbw_domain* d, int64_t m) { return d->alm->ready_step == m; }

int alm_chainb_check(lbw_domain* d);
int alm_check_gate(lbw_domain* d) {
    {
        int rc = alm_chainb_check(d);
        if (rc) return rc;
    }
    if (!alm_active(d) || !d->alm->gate_flag) return LBW_OK;
    int32_t err = 0;
    LBW_CK(cudaMemcpy(&err, d->alm->gate_flag + 1, sizeof(err), cudaMemcpyDeviceToHost));
    if (err) {
        set_error("a sweep's in-kernel wait for the actuator chain expired (results invalid)");
        return LBW_ECUDA;
    }
    return LBW_OK;
}

bool alm_can_prelaunch(const lbw_domain* d) { return d->prelaunch && d->alm->kin_device; }

bool alm_gate(lbw_domain* d, int64_t m, const uint32_t** flag, uint32_t* value,
              const int32_t** box, cudaEvent_t* kin_event) {
    const AlmState* s = d->alm;
    // only with the chain on its own SMs (the waiting CTAs cannot starve
    // it), one slab, device kinematics, and the chain of step m queued last
    if (!s || !s->gate_flag || !d->green_alm || d->linked || !s->kin_device ||
        s->ready_step != m || s->kin_valid[m % kSlots] != m)
        return false;
    *flag = s->gate_flag;
    *value = (uint32_t)d->alm_launches;
    *box = s->gate_box + 2 * (m % kSlots);
    *kin_event = s->ev_kin_step[m % kSlots];
    return true;
}

ForceView alm_force_view(const lbw_domain* d, int64_t m) {
    const AlmState* s = d->alm;
    ForceView v = s->set[m & 1].view((uint32_t)(m + 1));
    if (s->on_the_fly) {
        const AlmDev a = s->dev(m);
        v.pool = nullptr;
        v.npts = s->n;
        v.kw = s->kw;
        v.dep_cell = a.dep_cell;
        v.dep_w = a.dep_w;
        v.flat = a.flat;
    }
    return v;
}

int alm_invalidate(lbw_domain* d) {
    d->touched = true;
    if (!alm_active(d)) return LBW_OK;
    LBW_CK(cudaStreamSynchronize(d->alm_stream));
    LBW_CK(alm_sync_side(d));
    if (d->alm->kin_stream) LBW_CK(cudaStreamSynchronize(d->alm->kin_stream));
    d->alm->ready_step = -1;
    d->alm->fs_next = -1;
    d->alm->cb_next = -1;
    d->alm->cb_loop_end = -1;
    return LBW_OK;
}

// KK for step j on the kinematics stream.  Kinematics do not depend on the
// flow, so step j+1's are computed while step j's chain and sweep run; the
// buffer kin[j&1] is free once the chain of step j-2 (its last reader) is
// done.
static int kin_launch(lbw_domain* d, int64_t j) {
    AlmState* s = d->alm;
    if (j < s->kin_state_step || j > s->kin_state_step + 1) {
        set_error("device kinematics can only advance one step at a time");
        return LBW_ESTATE;
    }
    const int advance = j > s->kin_state_step ? 1 : 0;
    LBW_CK(cudaStreamWaitEvent(s->kin_stream, s->ev_chain_done[j & 1], 0));
    const size_t ksm = s->kin_smem;
    KinDev kd = s->kdev();
    kd.hist_slot = (int32_t)(j % kSlots);
    kd.box = s->gate_box ? s->gate_box + 2 * (j % kSlots) : nullptr;
    kd.skip_static = s->kin_static_ready ? 1 : 0;
    k_kinematics<<<1, 256, ksm, s->kin_stream>>>(kd, s->dev(j), d->g,
                                                  d->desc.periodic[0] ? 1 : 0, advance);
    count_launch();
    LBW_CK(cudaGetLastError());
    LBW_CK(cudaEventRecord(s->ev_kin_done, s->kin_stream));
    if (s->ev_kin_step[j % kSlots]) LBW_CK(cudaEventRecord(s->ev_kin_step[j % kSlots], s->kin_stream));
    s->kin_static_ready = true;
    s->kin_state_step = j;
    s->kin_valid[j % kSlots] = j;
    return LBW_OK;
}

// sampling source of the next actuator step (the macro of the last collide)
static MacroDev make_macro_dev(const lbw_domain* d) {
    MacroDev md{};
    md.kind = d->msrc.kind;
    for (int k = 0; k < 4; ++k) md.uniform[k] = d->msrc.uniform[k];
    md.buf = d->buf[d->msrc.buf];
    md.pull = d->msrc.pull ? 1 : 0;
    md.fv = d->msrc.fv;
    md.dense = d->macro_dense;
    md.bc_set = d->steps_done > 0 ? 1 : 0;
    for (int k = 0; k < 3; ++k) md.u_in[k] = d->desc.u_in[k];
    md.inflow = d->desc.boundary == LBW_BC_INFLOW_OUTFLOW ? 1 : 0;
    md.per_x = d->desc.periodic[0] ? 1 : 0;
    return md;
}

// ------------------------------------------------------------ fused step
// One launch per step (lbw_fused.cuh) on a single slab with device
// kinematics and at most 64 actuator points without disks: sweep m, the
// point forces of step m, kinematics + geometry of step m+2.

bool alm_fused_eligible(const lbw_domain* d) {
    const AlmState* s = d->alm;
    return d->fused && s && s->n > 0 && s->kin_device && s->on_the_fly && s->n_rings == 0 &&
           !d->linked && !d->user_active && d->prelaunch && s->kin_smem <= 24 * 1024;
}

bool alm_after_fused(const lbw_domain* d) {
    return alm_active(d) && d->alm->fs_next == d->step && d->step > 0;
}

static int fs_allocate(lbw_domain* d) {
    AlmState* s = d->alm;
    const int64_t rows = (int64_t)d->g.nxl * d->g.ny;
    const size_t dep = (size_t)kSlots * s->n * 3 * s->kw;
    int rc = LBW_OK;
    auto A = [&](auto** p, size_t n) {
        if (rc == LBW_OK) rc = dev_alloc(d, s, p, n);
    };
    A(&s->fs_dep_cell, dep);
    A(&s->fs_dep_w, dep);
    A(&s->fs_frow, (size_t)kSlots * rows);
    A(&s->fs_skey, (size_t)kSlots * rows);
    A(&s->fs_spool, (size_t)2 * 4 * s->n * 4 * d->g.zp);
    A(&s->fs_ctr, 6);   // [task, done] x 2 launches + a scratch pair
    if (rc) return rc;
    // keys with tag 0xffffffff match no step (tags are step + 1)
    LBW_CK(cudaMemset(s->fs_frow, 0xff, (size_t)kSlots * rows * 8));
    LBW_CK(cudaMemset(s->fs_skey, 0xff, (size_t)kSlots * rows * 8));
    LBW_CK(cudaMemset(s->fs_ctr, 0, 24));
    if (getenv("LBW_FUSED_PROF")) {
        rc = dev_alloc(d, s, &s->fs_prof, (size_t)256 * 8);
        if (rc) return rc;
    }
    s->fs_alloc = true;
    return LBW_OK;
}

// geometry slots of step j (written by KK(j))
static FsGeom fs_geom(const lbw_domain* d, int64_t j) {
    const AlmState* s = d->alm;
    const int64_t rows = (int64_t)d->g.nxl * d->g.ny;
    const int slot = (int)(j % kSlots);
    const size_t dep = (size_t)s->n * 3 * s->kw;
    FsGeom g;
    g.dep_cell = s->fs_dep_cell + slot * dep;
    g.dep_w = s->fs_dep_w + slot * dep;
    g.frow_key = s->fs_frow + slot * rows;
    g.skey = s->fs_skey + slot * rows;
    g.tag = (uint32_t)(j + 1);
    g.inflow = d->desc.boundary == LBW_BC_INFLOW_OUTFLOW ? 1 : 0;
    return g;
}

// force of sweep m: rows tagged m+1 by KK(m), summed on the fly from the
// deposit geometry of step m and the point forces K4(m) writes
static ForceView fs_view(const lbw_domain* d, int64_t m) {
    const AlmState* s = d->alm;
    const FsGeom g = fs_geom(d, m);
    ForceView v{g.frow_key, nullptr, g.tag};
    v.npts = s->n;
    v.kw = s->kw;
    v.dep_cell = g.dep_cell;
    v.dep_w = g.dep_w;
    v.flat = s->flat + (size_t)(m & 1) * s->n * 3;
    return v;
}

// kinematics (when missing) + geometry of step j, serially on the main stream
static int fs_prime(lbw_domain* d, int64_t j) {
    AlmState* s = d->alm;
    int do_kin = 0, advance = 0;
    if (s->kin_valid[j % kSlots] != j) {
        if (j < s->kin_state_step || j > s->kin_state_step + 1) {
            set_error("device kinematics can only advance one step at a time");
            return LBW_ESTATE;
        }
        advance = j > s->kin_state_step ? 1 : 0;
        do_kin = 1;
    }
    KinDev kd = s->kdev();
    kd.hist_slot = (int32_t)(j % kSlots);
    kd.skip_static = s->kin_static_ready ? 1 : 0;
    k_fs_prime<<<1, 128, do_kin ? s->kin_smem : 0, d->stream>>>(
        kd, s->dev(j), d->g, d->desc.periodic[0] ? 1 : 0, advance, do_kin, fs_geom(d, j));
    count_launch();
    LBW_CK(cudaGetLastError());
    if (do_kin) {
        s->kin_static_ready = true;
        s->kin_state_step = j;
        s->kin_valid[j % kSlots] = j;
    }
    return LBW_OK;
}

// LBW_FUSED_PROF: mean timeline of the last 128 complete launches (rows of
// steps m-130 .. m-3), and the gap from each launch's last CTA to the next
// launch's first CTA
static void fs_prof_report(lbw_domain* d, int64_t m) {
    AlmState* s = d->alm;
    std::vector<unsigned long long> h(256 * 8);
    if (cudaMemcpy(h.data(), s->fs_prof, h.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
        return;
    double acc[5] = {0, 0, 0, 0, 0}, gap = 0.0, span = 0.0;
    int n = 0, ng = 0;
    for (int64_t j = m - 130; j < m - 2; ++j) {
        if (j < 1) continue;
        const unsigned long long* r = &h[(size_t)(j % 256) * 8];
        const unsigned long long* q = &h[(size_t)((j + 1) % 256) * 8];
        if (r[0] == ~0ull || r[5] == 0) continue;
        const double t0 = (double)r[0];
        for (int k = 0; k < 5; ++k) acc[k] += r[k + 1] ? (double)r[k + 1] - t0 : 0.0;
        ++n;
        if (q[0] != ~0ull && q[5] != 0) {
            gap += (double)q[0] - (double)r[5];
            span += (double)q[0] - t0;
            ++ng;
        }
    }
    if (!n) return;
    fprintf(stderr,
            "FUSEDPROF %d launches (us after first CTA): KK start %.2f end %.2f | tasks done %.2f "
            "| force-tile wait end %.2f | last CTA end %.2f || next launch start-to-start %.2f, "
            "last CTA end -> next first CTA %.2f\n",
            n, acc[0] / n / 1e3, acc[1] / n / 1e3, acc[2] / n / 1e3, acc[3] / n / 1e3,
            acc[4] / n / 1e3, ng ? span / ng / 1e3 : 0.0, ng ? gap / ng / 1e3 : 0.0);
}

int alm_fused_launch(lbw_domain* d, bool pull, ForceView* fv_out) {
    AlmState* s = d->alm;
    const int64_t m = d->step;
    if (!s->fs_alloc) {
        int rc = fs_allocate(d);
        if (rc) return rc;
    }
    // primed: the previous launch was fused step m-1 (pool of step m filled,
    // kinematics + geometry of m and m+1 done, counters of m zeroed)
    const bool primed = s->fs_next == m && s->kin_state_step == m + 1 &&
                        s->kin_valid[(m + 1) % kSlots] == m + 1 && s->kin_valid[m % kSlots] == m;
    if (!primed) {
        // whatever the standalone chain queued is finished before its
        // outputs are rewritten here
        LBW_CK(cudaStreamSynchronize(d->alm_stream));
    LBW_CK(alm_sync_side(d));
        if (s->kin_stream) LBW_CK(cudaStreamSynchronize(s->kin_stream));
        int rc = fs_prime(d, m);
        if (!rc) rc = fs_prime(d, m + 1);
        if (rc) return rc;
        LBW_CK(cudaMemsetAsync(s->fs_ctr, 0, 4 * sizeof(uint32_t), d->stream));
    }
    const int per_x = d->desc.periodic[0] ? 1 : 0;
    const int64_t rows = (int64_t)d->g.nxl * d->g.ny;
    FusedArgs A{};
    SweepArgs& w = A.sw;
    w.src = d->buf[d->cur];
    w.dst = d->buf[1 - d->cur];
    w.g = d->g;
    w.fv = fs_view(d, m);
    w.r = d->relax;
    w.x_begin = 0;
    w.x_end = d->g.nxl;
    w.nan_key = d->d_nan;
    w.step = m;
    w.halo = HaloOut{nullptr, nullptr, {nullptr, nullptr}, nullptr, 0u, 0u};
    w.gate_flag = nullptr;
    w.gate_box = nullptr;
    w.gate_value = 0;
    w.reverse = (d->sweep_alt && (m & 1)) ? 1 : 0;
    w.pdl = 1;
    w.gate_error = nullptr;
    A.a = s->dev(m);
    if (s->loads_cap > 0 && s->d_loads)
        A.a.loads_row = s->d_loads + (size_t)(m % s->loads_cap) * s->n * 3;
    A.md = make_macro_dev(d);
    A.use_pool = primed ? 1 : 0;
    A.pool.skey = s->fs_skey + (size_t)(m % kSlots) * rows;
    A.pool.spool = s->fs_spool + (size_t)(m & 1) * 4 * s->n * 4 * d->g.zp;
    A.pool.tag = (uint32_t)(m + 1);
    A.pool.inflow = d->desc.boundary == LBW_BC_INFLOW_OUTFLOW ? 1 : 0;
    for (int k = 0; k < 3; ++k) A.pool.u_in[k] = d->desc.u_in[k];
    A.pool.error_flags = s->error_flags;
    A.ctr = s->fs_ctr + 2 * (m & 1);
    A.ctr_next = s->fs_ctr + 2 * ((m + 1) & 1);
    A.skey_next = s->fs_skey + (size_t)((m + 1) % kSlots) * rows;
    A.spool_next = s->fs_spool + (size_t)((m + 1) & 1) * 4 * s->n * 4 * d->g.zp;
    A.store_tag = (uint32_t)(m + 2);
    // KK(m+2) rewrites the geometry slot of step m-1, which a priming
    // launch's sampling reads (the force view of sweep m-1): not then
    A.kk_on = primed ? 1 : 0;
    A.k = s->kdev();
    A.k.hist_slot = (int32_t)((m + 2) % kSlots);
    A.k.skip_static = s->kin_static_ready ? 1 : 0;
    A.a_kk = s->dev(m + 2);
    A.geo = fs_geom(d, m + 2);
    A.per_x = per_x;
    A.n_kk = primed ? 1 : 0;
    A.n_help = (s->n + 3) / 4;
    A.prof = nullptr;
    A.prof_next = nullptr;
    if (s->fs_prof) {
        A.prof = s->fs_prof + (size_t)(m % 256) * 8;
        A.prof_next = s->fs_prof + (size_t)((m + 1) % 256) * 8;
        if (!primed) {
            unsigned long long init[8] = {~0ull, 0, 0, 0, 0, 0, 0, 0};
            LBW_CK(cudaMemcpyAsync(A.prof, init, sizeof init, cudaMemcpyHostToDevice, d->stream));
        }
        if (++s->fs_prof_n % 200 == 0) {
            LBW_CK(cudaStreamSynchronize(d->stream));
            fs_prof_report(d, m);
        }
    }
    const size_t smem = primed ? s->kin_smem : 0;
    auto launch = [&](const FusedArgs& X, size_t sm) {
        return d->desc.mode == LBW_MODE_FAST ? launch_fused_fast(d->desc.op, pull, X, sm, d->stream)
                                             : launch_fused_exact(d->desc.op, pull, X, sm, d->stream);
    };
    if (!primed) {
        // Priming: K4(m) samples by recomputation from buffers this sweep
        // may overwrite (the sampling source is the previous sweep's input,
        // i.e. this sweep's output buffer): it runs first, as a launch of
        // the point tasks alone, which leaves the counters of step m at
        // [n, n] -- the sweep launch then neither claims nor waits.
        FusedArgs T = A;
        T.sw.x_end = T.sw.x_begin;    // no sweep tiles
        T.n_kk = 0;
        T.kk_on = 0;
        T.ctr_next = s->fs_ctr + 4;   // scratch: nothing to reset for a successor
        LBW_CK(launch(T, 0));
        A.n_help = 0;
    }
    LBW_CK(launch(A, smem));
    if (primed) {
        s->kin_static_ready = true;
        s->kin_state_step = m + 2;
        s->kin_valid[(m + 2) % kSlots] = m + 2;
    } else {
        int rc = fs_prime(d, m + 2);
        if (rc) return rc;
    }
    s->fs_next = m + 1;
    s->ready_step = -1;
    *fv_out = w.fv;
    return LBW_OK;
}

// ------------------------------------------------------------ chain B
// The actuator chain ordered by in-kernel flags instead of per-step stream
// events (single slab, device kinematics, <= 64 points, no disks):
//
//   actuator stream: chain(m+1) = K4(m+1) + KK(m+5): waits in-kernel until
//                    sweep m has stored the (rho, u) of step m+1's sampling
//                    rows, then point forces of step m+1 from those samples,
//                    and kinematics + geometry four steps ahead (slot j % 6)
//   main stream:     sweep m: tiles read the geometry once KK(m+1) is done,
//                    force tiles wait for K4(m); sampling-row tiles store
//                    their macro; consecutive sweeps stay PDL-chained
//
// so the chain of step m+1 starts as soon as sweep m has passed the rotor's
// planes, and the main stream never waits for another stream.

// Used on slabs below 1.5 M cells, where the chain's latency sets the step
// time.  On larger slabs the sweep hides the event-ordered chain, and the
// flag-ordered one costs the sweep ~5 % (C2: 0.2718 vs 0.2863 ms in the
// same run; identical in isolation under ncu, 267.6 vs 268.8 us): its
// chain launches wait resident for a whole sweep, holding registers of
// ~2 SMs, and each CTA's acquire of the geometry flag flushes its SM's L1
// (a relaxed read with L2-only key loads recovers ~1 %).
// LBW_CHAIN_FLAGS: 0 never, 1 always (when eligible), unset: by size.
bool alm_chainb_eligible(const lbw_domain* d) {
    const AlmState* s = d->alm;
    if (!(d->chainb && s && s->n > 0 && s->kin_device && s->on_the_fly && s->n_rings == 0 &&
          !d->linked && !d->user_active && d->prelaunch && s->kin_smem <= 48 * 1024))
        return false;
    // forced (LBW_CHAIN_FLAGS=1) it also runs under a profiler that
    // serialises kernels: every wait is on work launched earlier
    if (d->chainb_forced) return true;
    if (tool_injected()) return false;
    return (int64_t)d->g.nxl * d->g.ny * d->g.nz < 1500000;
}

bool alm_after_chainb(const lbw_domain* d) {
    return alm_active(d) && d->alm->cb_next == d->step && d->step > 0;
}

static int cb_allocate(lbw_domain* d) {
    AlmState* s = d->alm;
    if (!s->fs_alloc) {
        int rc = fs_allocate(d);
        if (rc) return rc;
    }
    if (!s->cb_flags) {
        int rc = dev_alloc(d, s, &s->cb_flags, 8);
        if (!rc) rc = dev_alloc(d, s, &s->cb_pool_tiles, kSlots);
        const size_t nc8 = (size_t)kSlots * s->n * 8;
        if (!rc) rc = dev_alloc(d, s, &s->cb_cf_n, nc8);
        if (!rc) rc = dev_alloc(d, s, &s->cb_cf_p, nc8 * kCornerTerms);
        if (!rc) rc = dev_alloc(d, s, &s->cb_cf_w, nc8 * kCornerTerms);
        if (rc) return rc;
        LBW_CK(cudaMemset(s->cb_flags, 0, 8 * sizeof(uint32_t)));
        LBW_CK(cudaMemset(s->cb_pool_tiles, 0, kSlots * sizeof(int32_t)));
        LBW_CK(cudaHostAlloc(&s->cb_box_h, kSlots * 2 * sizeof(int32_t), cudaHostAllocMapped));
        for (int k = 0; k < 2 * kSlots; ++k) s->cb_box_h[k] = 0;
        void* dp = nullptr;
        LBW_CK(cudaHostGetDevicePointer(&dp, s->cb_box_h, 0));
        s->cb_box_d = static_cast<int32_t*>(dp);
    }
    return LBW_OK;
}

// corner-force lists of step j (from the deposit geometry of step j-1 and
// the sampling corners of step j); built by the geometry kernel of step j
// (priming) or of step j-1 (steady state: it waits for the kinematics of j)
static CornerLists cb_lists(const lbw_domain* d, int64_t j, bool build) {
    const AlmState* s = d->alm;
    CornerLists L{};
    if (build) {
        const FsGeom prev = fs_geom(d, j - 1);
        L.prev_cell = prev.dep_cell;
        L.prev_w = prev.dep_w;
        L.ckin = s->kin + (size_t)(j % kSlots) * s->n * kKin;
    }
    const size_t off = (size_t)(j % kSlots) * s->n * 8;
    L.n = s->cb_cf_n + off;
    L.p = s->cb_cf_p + off * kCornerTerms;
    L.w = s->cb_cf_w + off * kCornerTerms;
    L.inflow = d->desc.boundary == LBW_BC_INFLOW_OUTFLOW ? 1 : 0;
    for (int k = 0; k < 3; ++k) L.u_in[k] = d->desc.u_in[k];
    return L;
}

// KK(j) of chain B on stream st
static int cb_kk(lbw_domain* d, int64_t j, cudaStream_t st, bool lists) {
    AlmState* s = d->alm;
    int do_kin = 0, advance = 0;
    if (s->kin_valid[j % kSlots] != j) {
        if (j < s->kin_state_step || j > s->kin_state_step + 1) {
            set_error("device kinematics can only advance one step at a time");
            return LBW_ESTATE;
        }
        advance = j > s->kin_state_step ? 1 : 0;
        do_kin = 1;
    }
    KinDev kd = s->kdev();
    kd.hist_slot = (int32_t)(j % kSlots);
    kd.skip_static = s->kin_static_ready ? 1 : 0;
    const int warps_row = (int)((d->g.nz + 31) / 32);
    k_cb_kk<<<1, 128, do_kin ? s->kin_smem : 0, st>>>(
        kd, s->dev(j), d->g, d->desc.periodic[0] ? 1 : 0, advance, do_kin, fs_geom(d, j),
        warps_row, s->cb_pool_tiles + j % kSlots, s->cb_flags, (uint32_t)(j + 1),
        s->cb_box_d + 2 * (j % kSlots), cb_lists(d, j, lists));
    count_launch();
    LBW_CK(cudaGetLastError());
    if (do_kin) {
        s->kin_static_ready = true;
        s->kin_state_step = j;
        s->kin_valid[j % kSlots] = j;
    }
    return LBW_OK;
}

// The chain launch of step j (K4(j) [+ KK(j+4) when kk]) on stream st;
// use_pool: samples stored by sweep j-1, else recomputed from msrc (priming)
static int cb_loop_stream(lbw_domain* d);

// launch configuration of the resident chain (k_cb_persist)
static void loop_config(const AlmState* s, cudaLaunchConfig_t& cfg, cudaLaunchAttribute& attr) {
    cfg = {};
    cfg.gridDim = dim3(3 + kLoopGeoCtas, 1, 1);
    cfg.blockDim = dim3(kLoopThreads, 1, 1);
    cfg.dynamicSmemBytes = s->kin_smem;   // <= 48 KB (cb_loop_ok)
    cfg.stream = s->loop_stream;
    attr = {};
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 2;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
}

// the resident chain: only on the chain's own SMs (its CTAs beside the
// sweep's could starve for registers), <= kLoopMaxPoints points, and only
// when all its CTAs fit there at once (they wait on each other)
static bool cb_loop_ok(lbw_domain* d) {
    AlmState* s = d->alm;
    if (!(d->chain_loop && d->green_alm && s->n <= kLoopMaxPoints && s->kin_smem <= 48 * 1024))
        return false;
    if (s->loop_fit < 0) {
        s->loop_fit = 0;
        if (cb_loop_stream(d) == LBW_OK) {
            cudaLaunchConfig_t cfg;
            cudaLaunchAttribute attr;
            loop_config(s, cfg, attr);
            int clusters = 0;
            if (cudaOccupancyMaxActiveClusters(&clusters, k_cb_persist, &cfg) == cudaSuccess &&
                2 * clusters >= 3 + kLoopGeoCtas)
                s->loop_fit = 1;
        }
        cudaGetLastError();
    }
    return s->loop_fit == 1;
}

static int cb_loop_stream(lbw_domain* d) {
    AlmState* s = d->alm;
    if (!s->loop_stream) {
        s->loop_stream = green_alm_stream(d);
        if (!s->loop_stream) {
            set_error("no stream on the actuator chain's SMs");
            return LBW_ECUDA;
        }
        LBW_CK(cudaEventCreateWithFlags(&s->loop_ev, cudaEventDisableTiming));
    }
    return LBW_OK;
}

// Hand the chain over between the per-step launches (actuator stream) and
// the resident loop (its own stream): the kinematics of either side advance
// the state the other one continues from.  Waiting for the other stream is
// safe both ways: all either side waits for is already queued.
static int cb_stream_handover(lbw_domain* d, bool to_loop) {
    AlmState* s = d->alm;
    if (s->loop_last == to_loop) return LBW_OK;
    cudaStream_t from = to_loop ? d->alm_stream : s->loop_stream;
    cudaStream_t to = to_loop ? s->loop_stream : d->alm_stream;
    LBW_CK(cudaEventRecord(s->loop_ev, from));
    LBW_CK(cudaStreamWaitEvent(to, s->loop_ev, 0));
    s->loop_last = to_loop;
    return LBW_OK;
}

// the sweeps the resident chain waits for are queued after it: their
// kernels must be loaded before it runs (lazy module loading)
static int cb_preload(lbw_domain* d) {
    AlmState* s = d->alm;
    if (!s->loop_loaded) {
        LBW_CK(d->desc.mode == LBW_MODE_FAST ? preload_sweep_cb_fast(d->desc.op, d->g.single)
                                             : preload_sweep_cb_exact(d->desc.op, d->g.single));
        s->loop_loaded = true;
    }
    return LBW_OK;
}

static int cb_persist(lbw_domain* d, int64_t j0, int32_t nsteps) {
    AlmState* s = d->alm;
    {
        int rc = cb_loop_stream(d);
        if (rc) return rc;
    }
    {
        int rc = cb_preload(d);
        if (rc) return rc;
    }
    {
        int rc = cb_stream_handover(d, true);
        if (rc) return rc;
    }
    // the kinematics of j0+4 .. j0+nsteps+3 advance the state one step each
    if (s->kin_state_step != j0 + 3 || s->kin_valid[(j0 + 4) % kSlots] == j0 + 4) {
        set_error("persistent chain: unexpected kinematics state");
        return LBW_ESTATE;
    }
    CbPersistArgs P{};
    P.g = d->g;
    P.a0 = s->dev(j0);
    P.k0 = s->kdev();
    P.kin_base = s->kin;
    P.samples_base = s->samples;
    P.blade_base = s->blade;
    P.flat_base = s->flat;
    P.loads_base = (s->loads_cap > 0 && s->d_loads) ? s->d_loads : nullptr;
    P.loads_cap = s->loads_cap > 0 ? s->loads_cap : 1;
    P.inflow = d->desc.boundary == LBW_BC_INFLOW_OUTFLOW ? 1 : 0;
    for (int k = 0; k < 3; ++k) P.u_in[k] = P.pool0.u_in[k] = d->desc.u_in[k];
    P.pool0.inflow = P.inflow;
    P.pool0.error_flags = s->error_flags;
    P.pool0.raw = 1;
    P.rows = (int64_t)d->g.nxl * d->g.ny;
    P.skey_base = s->fs_skey;
    P.spool_base = s->fs_spool;
    P.spool_stride = (size_t)4 * s->n * 4 * d->g.zp;
    P.frow_base = s->fs_frow;
    P.dep_cell_base = s->fs_dep_cell;
    P.dep_w_base = s->fs_dep_w;
    P.cf_n_base = s->cb_cf_n;
    P.cf_p_base = s->cb_cf_p;
    P.cf_w_base = s->cb_cf_w;
    P.pool_tiles = s->cb_pool_tiles;
    P.box_hint = s->cb_box_d;
    P.flags = s->cb_flags;
    P.j0 = j0;
    P.nsteps = nsteps;
    P.per_x = d->desc.periodic[0] ? 1 : 0;
    P.warps_row = (int32_t)((d->g.nz + 31) / 32);
    P.first_skip_static = s->kin_static_ready ? 1 : 0;
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute attr;
    loop_config(s, cfg, attr);
    LBW_CK(cudaLaunchKernelEx(&cfg, k_cb_persist, P));
    count_launch();
    s->kin_static_ready = true;
    for (int64_t jk = j0 + 4; jk < j0 + 4 + nsteps; ++jk) s->kin_valid[jk % kSlots] = jk;
    s->kin_state_step = j0 + 3 + nsteps;
    s->cb_loop_end = j0 + nsteps;
    s->ready_step = -1;
    return LBW_OK;
}

static int cb_chain(lbw_domain* d, int64_t j, cudaStream_t st, bool use_pool, bool kk,
                    bool k4 = true) {
    AlmState* s = d->alm;
    const int64_t rows = (int64_t)d->g.nxl * d->g.ny;
    CbChainArgs A{};
    A.g = d->g;
    A.a = s->dev(j);
    if (s->loads_cap > 0 && s->d_loads)
        A.a.loads_row = s->d_loads + (size_t)(j % s->loads_cap) * s->n * 3;
    A.md = make_macro_dev(d);
    A.pool.skey = s->fs_skey + (size_t)(j % kSlots) * rows;
    A.pool.spool = s->fs_spool + (size_t)(j & 1) * 4 * s->n * 4 * d->g.zp;
    A.pool.tag = (uint32_t)(j + 1);
    A.pool.inflow = d->desc.boundary == LBW_BC_INFLOW_OUTFLOW ? 1 : 0;
    for (int k = 0; k < 3; ++k) A.pool.u_in[k] = d->desc.u_in[k];
    A.pool.error_flags = s->error_flags;
    A.pool.raw = 1;
    A.pool.fv = fs_view(d, j - 1);
    {
        const CornerLists L = cb_lists(d, j, false);
        A.pool.cf_n = L.n;
        A.pool.cf_p = L.p;
        A.pool.cf_w = L.w;
    }
    A.use_pool = use_pool ? 1 : 0;
    A.box_flag = s->cb_flags + 2;
    A.box_value = (uint32_t)j;
    A.pool_tiles = s->cb_pool_tiles + j % kSlots;
    A.flags = s->cb_flags;
    A.k4_value = (uint32_t)(j + 1);
    A.per_x = d->desc.periodic[0] ? 1 : 0;
    A.warps_row = (int32_t)((d->g.nz + 31) / 32);
    // K4(j); priming (on the main stream) is an ordinary launch: it samples
    // by recomputation from buffers the previous sweep wrote
    A.role = 0;
    const size_t k4_smem = (size_t)s->n * (3 * s->kw * 12 + 24);
    if (k4) {
        LBW_CK(launch_cb_chain(A, (unsigned)((s->n + 3) / 4), k4_smem, st, use_pool));
        count_launch();
    }
    if (kk) {
        // kinematics of step j+4 (serial chain) and geometry of step j+3
        const int64_t jk = j + 4;
        CbChainArgs B = A;
        B.role = 1;
        if (s->kin_valid[jk % kSlots] != jk) {
            if (jk < s->kin_state_step || jk > s->kin_state_step + 1) {
                set_error("device kinematics can only advance one step at a time");
                return LBW_ESTATE;
            }
            B.kk_do_kin = 1;
            B.kk_advance = jk > s->kin_state_step ? 1 : 0;
        }
        B.k = s->kdev();
        B.k.hist_slot = (int32_t)(jk % kSlots);
        B.k.skip_static = s->kin_static_ready ? 1 : 0;
        B.akk = s->dev(jk);
        B.kin_value = (uint32_t)(jk + 1);
        B.slot_value = (uint32_t)(jk - 4);
        LBW_CK(launch_cb_chain(B, 1, B.kk_do_kin ? s->kin_smem : 0, st, true));
        count_launch();
        if (B.kk_do_kin) {
            s->kin_static_ready = true;
            s->kin_state_step = jk;
            s->kin_valid[jk % kSlots] = jk;
        }
        const int64_t jg = j + 3;
        CbChainArgs C = A;
        C.role = 2;
        C.akk = s->dev(jg);
        C.geo = fs_geom(d, jg);
        C.pool_tiles_kk = s->cb_pool_tiles + jg % kSlots;
        C.kin_value = (uint32_t)(jg + 1);
        C.slot_value = (uint32_t)(jg - 4);
        C.box_hint = s->cb_box_d + 2 * (jg % kSlots);
        // lists of step jg+1: its kinematics first, and the slot's last
        // reader K4(jg+1-6) done
        C.cl = cb_lists(d, jg + 1, true);
        C.cl.ckin_value = (uint32_t)(jg + 2);
        C.cl.k4_value = (uint32_t)(jg - 4);
        LBW_CK(launch_cb_chain(C, 1, 0, st, true));
        count_launch();
    }
    s->ready_step = -1;
    return LBW_OK;
}

int alm_chainb_before(lbw_domain* d, SweepArgs* a) {
    AlmState* s = d->alm;
    const int64_t m = d->step;
    int rc = cb_allocate(d);
    if (rc) return rc;
    if (s->cb_next != m) {
        // priming: anything the standalone chain queued finishes first; the
        // geometry of steps m .. m+4 and the forces of step m (sampled by
        // recomputation from the last collide's input) go on the main stream
        LBW_CK(cudaStreamSynchronize(d->alm_stream));
    LBW_CK(alm_sync_side(d));
        if (s->kin_stream) LBW_CK(cudaStreamSynchronize(s->kin_stream));
        LBW_CK(cudaMemsetAsync(s->cb_flags + 3, 0, 2 * sizeof(uint32_t), d->stream));
        // kinematics + geometry of m .. m+4 (geometry publishes in step
        // order: restart its flag at m)
        rc = stream_write32(d->stream, s->cb_flags + 6, (uint32_t)m);
        for (int64_t j = m; j <= m + 4 && !rc; ++j) rc = cb_kk(d, j, d->stream, j > m);
        if (!rc) rc = cb_chain(d, m, d->stream, false, false);
        if (rc) return rc;
        // the chains queued from now on (actuator stream) read what these
        // priming kernels wrote: kinematics, geometry, pool-tile counts
        // (so does the resident chain's stream: cb_loop_ok creates it if
        // the kinematics configuration did not)
        (void)cb_loop_ok(d);
        LBW_CK(cudaEventRecord(d->ev_main, d->stream));
        LBW_CK(cudaStreamWaitEvent(d->alm_stream, d->ev_main, 0));
        if (s->loop_stream) LBW_CK(cudaStreamWaitEvent(s->loop_stream, d->ev_main, 0));
        s->loop_last = false;
        s->cb_loop_end = -1;
    }
    const int64_t rows = (int64_t)d->g.nxl * d->g.ny;
    a->fv = fs_view(d, m);
    a->gate_flag = nullptr;
    a->gate_box = nullptr;
    a->gate_value = 0;
    a->gate_error = reinterpret_cast<int32_t*>(s->cb_flags + 5);
    a->pdl = 1;
    a->kin_flag = s->cb_flags + 6;      // geometry of step m+2 done (for sweep m+1)
    a->kin_value = (uint32_t)(m + 3);
    a->k4_flag = s->cb_flags + 1;
    a->k4_value = (uint32_t)(m + 1);
    a->skey = s->fs_skey + (size_t)((m + 1) % kSlots) * rows;
    a->spool = s->fs_spool + (size_t)((m + 1) & 1) * 4 * s->n * 4 * d->g.zp;
    a->store_tag = (uint32_t)(m + 2);
    a->pool_cnt = s->cb_flags + 3;
    a->pool_tiles = s->cb_pool_tiles + (m + 1) % kSlots;
    a->box_flag = s->cb_flags + 2;
    a->box_value = (uint32_t)(m + 1);
    // plane order: the rotor's planes first.  A hint only -- whatever KK
    // wrote into the mapped host copy most recently for step m+1's slot
    // (possibly a few steps old while the host runs ahead of the GPU);
    // every dependency is guarded by the flags, not by the order
    const volatile int32_t* hb = s->cb_box_h + 2 * ((m + 1) % kSlots);
    const int32_t nx = d->g.nxl, h0 = hb[0], h1 = hb[1];
    a->x_first = ((h0 % nx) + nx) % nx;
    a->x_len = h1 > 0 && h1 <= nx ? h1 : nx;
    return LBW_OK;
}

int alm_chainb_after(lbw_domain* d, int64_t m, int32_t remaining) {
    AlmState* s = d->alm;
    // the chain of step m+1 (K4(m+1), kinematics(m+5), geometry(m+4)) on
    // the actuator stream, ordered by flags only -- or, for a call of >= 4
    // steps, the whole chain of its remaining steps as one resident kernel
    int rc = LBW_OK;
    if (cb_loop_ok(d) && remaining >= 4) {
        // one persistent chain launch covers this call's remaining steps
        if (s->cb_loop_end <= m + 1 || s->cb_next != m) rc = cb_persist(d, m + 1, remaining);
    } else if (s->cb_loop_end > m + 1 && s->cb_next == m) {
        // still inside the last loop's steps (a short call after a long one)
    } else {
        rc = cb_stream_handover(d, false);
        if (!rc) rc = cb_chain(d, m + 1, d->alm_stream, true, true);
    }
    if (rc) return rc;
    s->cb_next = m + 1;
    return LBW_OK;
}

int alm_chainb_check(lbw_domain* d) {
    if (!alm_active(d) || !d->alm->cb_flags) return LBW_OK;
    uint32_t err = 0;
    LBW_CK(cudaMemcpy(&err, d->alm->cb_flags + 5, sizeof(err), cudaMemcpyDeviceToHost));
    if (err) {
        // the error word holds the first expired wait's site (x100) + step % 100
        uint32_t f[7] = {};
        cudaMemcpy(f, d->alm->cb_flags, sizeof f, cudaMemcpyDeviceToHost);
        char msg[256];
        snprintf(msg, sizeof msg,
                 "an in-kernel wait of the flag-ordered actuator chain expired (results invalid; "
                 "wait site %u, flags kin %u k4 %u box %u geometry %u)",
                 f[5], f[0], f[1], f[2], f[6]);
        set_error(msg);
        return LBW_ECUDA;
    }
    return LBW_OK;
}

int alm_launch(lbw_domain* d, int64_t m) {
    AlmState* s = d->alm;
    const Geom& g = d->g;
    cudaStream_t st = d->alm_stream;
    const int par = (int)(m & 1);
    const AlmDev a = s->dev(m);
    const int per_x = d->desc.periodic[0] ? 1 : 0;
    // this step's use of force set m&1: rows tagged m+1
    ForceSet fs = s->set[par];
    fs.tag = (uint32_t)(m + 1);
    fs.flag_rows = s->on_the_fly ? 1 : 0;
    if (s->kin_device) {
        if (s->kin_valid[m % kSlots] != m) {
            int rc = kin_launch(d, m);
            if (rc) return rc;
        }
        LBW_CK(cudaStreamWaitEvent(st, s->ev_kin_done, 0));
    } else if (s->kin_queued_step != m) {
        set_error("actuator step without kinematics: call lbw_alm_set_kinematics first");
        return LBW_ESTATE;
    }
    MacroDev md = make_macro_dev(d);
    // one warp per CTA: fits in the registers a full sweep leaves free
    const int threads = 32;
    const size_t pts_smem =
        (md.fv.row_key != nullptr && md.fv.pool == nullptr && md.fv.npts <= kOnTheFlyMaxPoints)
            ? (size_t)md.fv.npts * ((3 * md.fv.kw + 3) * sizeof(double) +
                                    3 * md.fv.kw * sizeof(int32_t))
            : 0;
    const unsigned blocks = (unsigned)((s->n * 32 + threads - 1) / threads);
    CubeArgs cube{};
    if (d->linked) {
        const size_t off = (size_t)par * s->n * 32;
        const size_t tags = (size_t)2 * s->n * 32;   // tags follow the values
        const size_t toff = (size_t)par * s->n * 8;
        cube.local = s->cube + off;
        cube.tag_local = reinterpret_cast<int32_t*>(s->cube + tags) + toff;
        for (int side = 0; side < 2; ++side) {
            cube.peer[side] = d->nb_cube[side] ? d->nb_cube[side] + off : nullptr;
            cube.tag_peer[side] = d->nb_cube[side]
                                      ? reinterpret_cast<int32_t*>(d->nb_cube[side] + tags) + toff
                                      : nullptr;
        }
        // epochs count this domain's chain launches: a chain re-launched
        // after a state change (collective on every rank, as SlabSimulation's
        // calls are) waits for the neighbours' re-launch, not their first
        // launch of the same step, whose cube values may be stale
        cube.epoch = (int32_t)(d->alm_launches + 1);
        k_alm_points<<<blocks, threads, pts_smem, st>>>(a, g, md, fs, 1, cube);
        count_launch();
        LBW_CK(cudaGetLastError());
        const uint32_t epoch = (uint32_t)(d->alm_launches + 1);
        int rc = peer_signal(d, st, 1, epoch);
        if (!rc) rc = peer_wait(d, st, 1, epoch);
        if (rc) return rc;
        k_alm_points<<<blocks, threads, pts_smem, st>>>(a, g, md, fs, 2, cube);
    } else {
        k_alm_points<<<blocks, threads, pts_smem, st>>>(a, g, md, fs, 0, cube);
    }
    d->alm_launches += 1;
    if (s->n_rings > 0) {
        k_alm_disks<<<(unsigned)((s->n_rings + 63) / 64), 64, 0, st>>>(a, g, per_x,
                                                                       d->linked ? 1 : 0);
        count_launch();
    }
    if (!s->on_the_fly) {
        k_alm_fill<<<(unsigned)((s->n * s->kw * s->kw + 3) / 4), 128, 0, st>>>(a, g, fs);
        count_launch();
    }
    count_launch();
    LBW_CK(cudaGetLastError());
    LBW_CK(cudaEventRecord(d->ev_alm_done, st));
    if (s->gate_flag) {
        int rc = stream_write32(st, s->gate_flag, (uint32_t)d->alm_launches);
        if (rc) return rc;
    }
    if (s->loads_cap > 0)
        LBW_CK(cudaMemcpyAsync(s->h_loads + (size_t)(m % s->loads_cap) * s->n * 3, a.blade,
                               (size_t)s->n * 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (s->kin_device) {
        LBW_CK(cudaEventRecord(s->ev_chain_done[par], st));
        // prefetch the next step's kinematics while this chain and sweep run
        if (alm_can_prelaunch(d) && s->kin_state_step == m) {
            int rc = kin_launch(d, m + 1);
            if (rc) return rc;
        }
    }
    s->ready_step = m;
    return LBW_OK;
}

}  // namespace lbw

using namespace lbw;

extern "C" {

int lbw_alm_configure(lbw_domain* d, const lbw_alm_desc* desc) {
    LBW_REQ(d && desc, "null argument");
    LBW_REQ(desc->n_points >= 0 && desc->n_points <= 16384, "n_points outside [0, 16384]");
    LBW_REQ(desc->n_polars >= 0, "n_polars must be >= 0");
    LBW_CK(cudaSetDevice(d->device));
    d->touched = true;
    // no SM partition when the fused step will carry the chain (it runs on
    // every SM; lbw_fused.cuh)
    const bool fused_likely = d->fused && !d->linked && desc->n_points <= kOnTheFlyMaxPoints &&
                              !desc->point_ring;
    if (desc->n_points > 0 && !(fused_likely && !getenv("LBW_ALM_SMS"))) {
        int rc_ = green_partition(d, alm_sm_count(d));
        if (rc_) return rc_;
    }
    LBW_CK(cudaStreamSynchronize(d->stream));
    LBW_CK(cudaStreamSynchronize(d->alm_stream));
    LBW_CK(alm_sync_side(d));
    alm_destroy(d);
    const int P = desc->n_points;
    if (P == 0) return LBW_OK;
    for (int p = 0; p < P; ++p)
        LBW_REQ(desc->polar_index[p] >= -1 && desc->polar_index[p] < desc->n_polars,
                "polar index out of range");
    if (desc->point_ring) {
        LBW_REQ(desc->area && desc->n_rings >= 0, "disk rings need areas");
        for (int r = 0; r < desc->n_rings; ++r) {
            LBW_REQ(desc->ring_first[r] >= 0 && desc->ring_count[r] >= 1 &&
                        desc->ring_first[r] + desc->ring_count[r] <= P,
                    "disk ring point range out of bounds");
            LBW_REQ(desc->ring_ct[r] >= 0.0 && desc->ring_ct[r] < 1.0,
                    "thrust coefficient must lie in [0, 1)");
        }
    }
    LBW_REQ(desc->spread_kernel == LBW_SPREAD_ROMA || desc->spread_kernel == LBW_SPREAD_GAUSSIAN,
            "unknown spreading kernel");
    LBW_REQ(desc->spread_kernel != LBW_SPREAD_GAUSSIAN ||
                (desc->spread_epsilon > 0.0 && desc->spread_epsilon <= 2.0),
            "Gaussian spreading width must lie in (0, 2] lattice cells");
    int64_t total_rows = 0;
    for (int k = 0; k < desc->n_polars; ++k) {
        LBW_REQ(desc->polar_rows[k] >= 2, "polar needs at least 2 rows");
        total_rows = std::max<int64_t>(total_rows, (int64_t)desc->polar_offset[k] + desc->polar_rows[k]);
    }
    AlmState* s = new AlmState();
    d->alm = s;
    s->n = P;
    s->n_polars = desc->n_polars;
    s->vscale = desc->velocity_scale;
    s->rho_ref = desc->rho_ref;
    s->dt2 = desc->force_dt2;
    s->den = desc->force_den;
    s->kernel = desc->spread_kernel;
    if (s->kernel == LBW_SPREAD_GAUSSIAN) {
        s->eps = desc->spread_epsilon;
        s->kw = (int32_t)floor(6.0 * s->eps) + 1;      // cells within 3 eps of a point
        s->halo_x = (int32_t)ceil(3.0 * s->eps) + 1;
    }
    int rc = LBW_OK;
    auto A = [&](auto** p, size_t n) {
        if (rc == LBW_OK) rc = dev_alloc(d, s, p, n);
    };
    A(&s->chord, P);
    A(&s->elen, P);
    A(&s->twist, P);
    A(&s->polar_index, P);
    A(&s->polar_offset, std::max(1, desc->n_polars));
    A(&s->polar_rows, std::max(1, desc->n_polars));
    A(&s->p_alpha, std::max<int64_t>(1, total_rows));
    A(&s->p_cl, std::max<int64_t>(1, total_rows));
    A(&s->p_cd, std::max<int64_t>(1, total_rows));
    A(&s->kin, (size_t)kSlots * P * kKin);
    A(&s->samples, (size_t)2 * P * 4);
    A(&s->blade, (size_t)2 * P * 3);
    A(&s->flat, (size_t)2 * P * 3);
    A(&s->cube, (size_t)2 * P * 32 + (size_t)2 * P * 4);   // values, then (2,P,8) int32 tags
    A(&s->ring_samples, (size_t)P * 4);
    A(&s->ring_sample_ok, P);
    A(&s->dep_cell, (size_t)2 * P * 3 * s->kw);
    A(&s->dep_w, (size_t)2 * P * 3 * s->kw);
    A(&s->clamp_flags, std::max(1, desc->n_polars));
    A(&s->error_flags, 1);
    const int R = desc->point_ring ? desc->n_rings : 0;
    if (desc->point_ring) {
        A(&s->point_ring, P);
        A(&s->area, P);
        A(&s->ring_first, std::max(1, R));
        A(&s->ring_count, std::max(1, R));
        A(&s->ring_ct, std::max(1, R));
    }
    // sparse force sets: a point touches at most 3x3 (x,y) rows
    const int64_t rows = (int64_t)d->g.nxl * d->g.ny;
    s->on_the_fly = P <= kOnTheFlyMaxPoints;
    const int64_t cap = s->on_the_fly ? 0 : (int64_t)s->kw * s->kw * P;   // slot = deposit pair
    for (auto& fs : s->set) {
        A(&fs.row_key, rows);
        if (cap) {
            char* pool = nullptr;
            A(&pool, (size_t)cap * 3 * d->g.zp * elem_bytes(d->g));
            fs.pool = pool;
        }
        fs.cap = cap;
    }
    if (rc) {
        alm_destroy(d);
        return rc;
    }
    auto H = [&](void* dst, const void* src, size_t bytes) {
        if (rc == LBW_OK && bytes &&
            cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaGetLastError();
            set_error("ALM upload failed");
            rc = LBW_ECUDA;
        }
    };
    H(s->chord, desc->chord, P * 8);
    H(s->elen, desc->element_length, P * 8);
    H(s->twist, desc->twist, P * 8);
    H(s->polar_index, desc->polar_index, P * 4);
    if (desc->point_ring) {
        H(s->point_ring, desc->point_ring, P * 4);
        H(s->area, desc->area, P * 8);
        if (R) {
            H(s->ring_first, desc->ring_first, R * 4);
            H(s->ring_count, desc->ring_count, R * 4);
            H(s->ring_ct, desc->ring_ct, R * 8);
        }
        s->n_rings = R;
    }
    if (desc->n_polars) {
        H(s->polar_offset, desc->polar_offset, desc->n_polars * 4);
        H(s->polar_rows, desc->polar_rows, desc->n_polars * 4);
        H(s->p_alpha, desc->polar_alpha, total_rows * 8);
        H(s->p_cl, desc->polar_cl, total_rows * 8);
        H(s->p_cd, desc->polar_cd, total_rows * 8);
    }
    if (rc == LBW_OK) {
        for (auto& fs : s->set) {
            // keys with tag 0xffffffff match no step (chain tags are step+1)
            if (cudaMemset(fs.row_key, 0xff, rows * 8) != cudaSuccess) {
                cudaGetLastError();
                rc = LBW_ECUDA;
            }
        }
        if (cudaMemset(s->clamp_flags, 0, std::max(1, desc->n_polars) * 4) != cudaSuccess ||
            cudaMemset(s->error_flags, 0, 4) != cudaSuccess ||
            cudaMemset(s->cube, 0, ((size_t)2 * P * 32 + (size_t)2 * P * 4) * 8) != cudaSuccess ||
            cudaMemset(s->samples, 0, (size_t)2 * P * 32) != cudaSuccess ||
            cudaMemset(s->blade, 0, (size_t)2 * P * 24) != cudaSuccess ||
            cudaMemset(s->kin, 0, (size_t)kSlots * P * kKin * 8) != cudaSuccess ||
            cudaMallocHost(&s->h_ring, (size_t)kRing * P * kKin * 8) != cudaSuccess) {
            cudaGetLastError();
            set_error("ALM initialisation failed");
            rc = LBW_ECUDA;
        }
        for (auto& e : s->ring_ev)
            if (rc == LBW_OK && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
                cudaGetLastError();
                rc = LBW_ECUDA;
            }
    }
    if (rc) {
        alm_destroy(d);
        return rc;
    }
    return LBW_OK;
}

int lbw_alm_configure_kinematics(lbw_domain* d, const lbw_kin_desc* kd) {
    LBW_REQ(d && kd, "null argument");
    LBW_REQ(alm_active(d), "configure the actuator points first");
    AlmState* s = d->alm;
    const int C = kd->n_components, P = s->n;
    LBW_REQ(C >= 1 && C <= 256, "need 1..256 turbine components");
    LBW_REQ(kd->dx > 0.0, "dx must be positive");
    for (int c = 0; c < C; ++c) {
        LBW_REQ(kd->parent[c] >= -1 && kd->parent[c] < c, "components must be in pre-order");
        LBW_REQ(kd->line_first[c] >= -1 && kd->line_first[c] + kd->line_count[c] <= P,
                "line point range out of bounds");
    }
    LBW_CK(cudaSetDevice(d->device));
    LBW_CK(cudaStreamSynchronize(d->stream));
    LBW_CK(cudaStreamSynchronize(d->alm_stream));
    LBW_CK(alm_sync_side(d));
    std::vector<int32_t> point_comp(P, -1);
    for (int c = 0; c < C; ++c)
        for (int k = 0; k < kd->line_count[c]; ++k) point_comp[kd->line_first[c] + k] = c;
    for (int p = 0; p < P; ++p)
        LBW_REQ(point_comp[p] >= 0, "point without a line or disk component");
    int rc = LBW_OK;
    auto A = [&](auto** p, size_t n) {
        if (rc == LBW_OK) rc = dev_alloc(d, s, p, n);
    };
    A(&s->k_parent, C);
    A(&s->k_line_first, C);
    A(&s->k_line_count, C);
    A(&s->k_point_comp, P);
    A(&s->k_rel_p, (size_t)C * 3);
    A(&s->k_rel_T, (size_t)C * 9);
    A(&s->k_axis, (size_t)C * 3);
    A(&s->k_rate, C);
    A(&s->k_rstep, (size_t)C * 9);
    A(&s->k_spin, (size_t)C * 9);
    A(&s->k_off, (size_t)P * 3);
    A(&s->k_orient, (size_t)P * 9);
    A(&s->k_lframe, (size_t)P * 9);
    A(&s->k_cs, (size_t)C * kCS);
    A(&s->k_spin_hist, (size_t)kSlots * C * 9);
    A(&s->k_cs_hist, (size_t)kSlots * C * kCS);
    A(&s->k_is_disk, C);
    A(&s->k_disk_center, (size_t)C * 12);
    A(&s->k_order, C);
    A(&s->k_static, C);
    A(&s->k_level_start, (size_t)C + 1);
    if (rc) return rc;
    // walk schedule: components by depth (parents precede children), and
    // which ones never move (no rotation on the path from the root)
    std::vector<int32_t> depth(C), stat(C), order, lstart;
    for (int c = 0; c < C; ++c) {
        const int pa = kd->parent[c];
        depth[c] = pa < 0 ? 0 : depth[pa] + 1;
        stat[c] = kd->rate[c] == 0.0 && (pa < 0 || stat[pa]);
    }
    const int maxd = *std::max_element(depth.begin(), depth.end());
    for (int L = 0; L <= maxd; ++L) {
        lstart.push_back((int32_t)order.size());
        for (int c = 0; c < C; ++c)
            if (depth[c] == L) order.push_back(c);
    }
    lstart.push_back((int32_t)order.size());
    s->k_nlevels = maxd + 1;
    auto H = [&](void* dst, const void* src, size_t bytes) {
        if (rc == LBW_OK && cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaGetLastError();
            set_error("kinematics upload failed");
            rc = LBW_ECUDA;
        }
    };
    H(s->k_parent, kd->parent, C * 4);
    H(s->k_line_first, kd->line_first, C * 4);
    H(s->k_line_count, kd->line_count, C * 4);
    H(s->k_point_comp, point_comp.data(), P * 4);
    H(s->k_rel_p, kd->rel_p, C * 24);
    H(s->k_rel_T, kd->rel_T, C * 72);
    H(s->k_axis, kd->axis, C * 24);
    H(s->k_rate, kd->rate, C * 8);
    H(s->k_rstep, kd->step_rotation, C * 72);
    H(s->k_spin, kd->spin, C * 72);
    H(s->k_off, kd->offsets, (size_t)P * 24);
    H(s->k_orient, kd->orientations, (size_t)P * 72);
    H(s->k_lframe, kd->local_frames, (size_t)P * 72);
    H(s->k_order, order.data(), (size_t)C * 4);
    H(s->k_static, stat.data(), (size_t)C * 4);
    H(s->k_level_start, lstart.data(), lstart.size() * 4);
    {
        std::vector<int32_t> isd(C, 0);
        std::vector<double> dcen((size_t)C * 12, 0.0);
        for (int c = 0; c < C; ++c) {
            if (kd->is_disk) isd[c] = kd->is_disk[c] ? 1 : 0;
            if (kd->disk_center && isd[c])
                for (int i = 0; i < 12; ++i) dcen[(size_t)c * 12 + i] = kd->disk_center[(size_t)c * 12 + i];
        }
        H(s->k_is_disk, isd.data(), C * 4);
        H(s->k_disk_center, dcen.data(), (size_t)C * 96);
    }
    if (rc) return rc;
    size_t ksm = (size_t)C * (kKP + kCS) * sizeof(double) + (size_t)(3 * C + 1) * 4 + 8;  // +8: the staged image is padded to 8 B
    const size_t kpts = (size_t)P * 21 * sizeof(double) + (size_t)P * sizeof(int32_t);
    s->kin_stage_points = ksm + kpts <= 160 * 1024;
    if (s->kin_stage_points) ksm += kpts;
    if (ksm > 48 * 1024 &&
        cudaFuncSetAttribute(k_kinematics, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)ksm) != cudaSuccess) {
        cudaGetLastError();
        set_error("too many turbine components for the kinematics CTA");
        return LBW_EINVAL;
    }
    s->kin_smem = ksm;
    {
        // the constant part of the CTA's shared-memory image (kinematics_cta)
        std::vector<double> ip((size_t)C * kKP, 0.0);
        for (int c = 0; c < C; ++c) {
            double* q = ip.data() + (size_t)c * kKP;
            for (int i = 0; i < 3; ++i) q[i] = kd->rel_p[c * 3 + i];
            for (int i = 0; i < 9; ++i) q[3 + i] = kd->rel_T[c * 9 + i];
            for (int i = 0; i < 3; ++i) q[12 + i] = kd->axis[c * 3 + i];
            q[15] = kd->rate[c];
            for (int i = 0; i < 9; ++i) q[16 + i] = kd->step_rotation[c * 9 + i];
            for (int i = 0; i < 9; ++i) q[25 + i] = kd->spin[c * 9 + i];   // rewritten per launch
            q[34] = (double)kd->parent[c];
            q[35] = (double)kd->line_first[c];
            const bool disk = kd->is_disk && kd->is_disk[c];
            q[36] = disk ? 1.0 : 0.0;
            for (int i = 0; i < 12; ++i)
                q[37 + i] = (disk && kd->disk_center) ? kd->disk_center[(size_t)c * 12 + i] : 0.0;
        }
        std::vector<char> tail;
        auto put = [&](const void* src, size_t bytes) {
            const char* b = static_cast<const char*>(src);
            tail.insert(tail.end(), b, b + bytes);
        };
        if (s->kin_stage_points) {
            put(kd->offsets, (size_t)P * 24);
            put(kd->orientations, (size_t)P * 72);
            put(kd->local_frames, (size_t)P * 72);
            put(point_comp.data(), (size_t)P * 4);
        }
        put(order.data(), (size_t)C * 4);
        put(stat.data(), (size_t)C * 4);
        put(lstart.data(), lstart.size() * 4);
        tail.resize((tail.size() + 7) / 8 * 8, 0);
        rc = dev_alloc(d, s, &s->k_img_prm, ip.size());
        if (!rc) rc = dev_alloc(d, s, &s->k_img_tail, tail.size() / 8);
        if (rc) return rc;
        H(s->k_img_prm, ip.data(), ip.size() * 8);
        H(s->k_img_tail, tail.data(), tail.size());
        if (rc) return rc;
        s->k_img_words = (int32_t)(tail.size() / 8);
    }
    if (!s->kin_stream) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        s->kin_stream = green_alm_stream(d);   // on the chain's SMs when partitioned
        if ((!s->kin_stream &&
             cudaStreamCreateWithPriority(&s->kin_stream, cudaStreamNonBlocking, hi) != cudaSuccess) ||
            cudaEventCreateWithFlags(&s->ev_kin_done, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->ev_chain_done[0], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->ev_chain_done[1], cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            set_error("kinematics stream/event creation failed");
            return LBW_ECUDA;
        }
    }
    LBW_CK(cudaStreamSynchronize(s->kin_stream));
    // sweep gate (alm_gate): only when the chain has SMs of its own
    const char* ge = getenv("LBW_SWEEP_GATE");
    if (d->green_alm && !(ge && ge[0] == '0') && !s->gate_flag) {
        int rcg = LBW_OK;
        auto G = [&](auto** p, size_t n) {
            if (rcg == LBW_OK) rcg = dev_alloc(d, s, p, n);
        };
        G(&s->gate_flag, 2);   // [0] chain launches done, [1] sweep wait expired
        G(&s->gate_box, 2 * kSlots);
        if (rcg) return rcg;
        for (auto& e : s->ev_kin_step)
            LBW_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        LBW_CK(cudaMemset(s->gate_flag, 0, 2 * sizeof(uint32_t)));
    }
    s->nc = C;
    s->k_dx = kd->dx;
    s->kin_device = true;
    s->kin_state_step = d->step - (kd->advance_first ? 1 : 0);
    for (auto& v : s->kin_valid) v = -1;
    s->kin_static_ready = false;
    s->ready_step = -1;
    s->fs_next = -1;
    s->cb_next = -1;
    // the flag-ordered chain's buffers, and the resident chain's stream and
    // kernels, now rather than inside the first lbw_domain_step
    if (alm_chainb_eligible(d)) {
        int rc = cb_allocate(d);
        if (!rc && cb_loop_ok(d)) rc = cb_preload(d);
        if (rc) return rc;
    }
    return LBW_OK;
}

// step whose turbine state lbw_alm_download_kinematics reports: the
// domain's step, unless the device kinematics have not reached it yet
static int64_t kin_view_step(const lbw_domain* d) {
    return std::min<int64_t>(d->step, d->alm->kin_state_step);
}

// parity of the most recent step's actuator outputs
static int last_parity(const lbw_domain* d) { return d->step > 0 ? (int)((d->step - 1) & 1) : 0; }

int lbw_alm_download_kinematics(lbw_domain* d, double* kin, double* spin, double* comp_state) {
    LBW_REQ(d, "null domain");
    LBW_REQ(alm_active(d), "no actuator points configured");
    AlmState* s = d->alm;
    LBW_CK(cudaSetDevice(d->device));
    LBW_CK(cudaStreamSynchronize(d->stream));
    LBW_CK(cudaStreamSynchronize(d->alm_stream));
    LBW_CK(alm_sync_side(d));
    if (s->kin_stream) LBW_CK(cudaStreamSynchronize(s->kin_stream));
    if (kin)
        LBW_CK(cudaMemcpy(kin, s->kin + (size_t)(d->step > 0 ? (d->step - 1) % kSlots : 0) * s->n * kKin,
                          (size_t)s->n * kKin * 8, cudaMemcpyDeviceToHost));
    // the turbine state of step d->step (what the host objects hold after
    // d->step advances), even when the next step's kinematics already ran
    const int64_t v = kin_view_step(d);
    const bool hist = s->kin_valid[v % kSlots] == v;
    if (spin && s->kin_device)
        LBW_CK(cudaMemcpy(spin, hist ? s->k_spin_hist + (size_t)(v % kSlots) * s->nc * 9 : s->k_spin,
                          (size_t)s->nc * 72, cudaMemcpyDeviceToHost));
    if (comp_state && s->kin_device)
        LBW_CK(cudaMemcpy(comp_state,
                          hist ? s->k_cs_hist + (size_t)(v % kSlots) * s->nc * kCS : s->k_cs,
                          (size_t)s->nc * kCS * 8, cudaMemcpyDeviceToHost));
    return LBW_OK;
}

int64_t lbw_alm_kinematics_step(lbw_domain* d) {
    if (!d || !alm_active(d) || !d->alm->kin_device) return -1;
    return kin_view_step(d);
}

int lbw_alm_set_kinematics(lbw_domain* d, const double* kin) {
    LBW_REQ(d && kin, "null argument");
    LBW_REQ(alm_active(d), "no actuator points configured");
    AlmState* s = d->alm;
    LBW_REQ(!s->kin_device, "kinematics are computed on the device for this domain");
    LBW_CK(cudaSetDevice(d->device));
    const int slot = s->ring_pos;
    s->ring_pos = (s->ring_pos + 1) % kRing;
    LBW_CK(cudaEventSynchronize(s->ring_ev[slot]));
    double* h = s->h_ring + (size_t)slot * s->n * kKin;
    std::memcpy(h, kin, (size_t)s->n * kKin * 8);
    const int64_t m = d->step;
    LBW_CK(cudaMemcpyAsync(s->kin + (size_t)(m % kSlots) * s->n * kKin, h, (size_t)s->n * kKin * 8,
                           cudaMemcpyHostToDevice, d->alm_stream));
    LBW_CK(cudaEventRecord(s->ring_ev[slot], d->alm_stream));
    s->kin_queued_step = m;
    s->ready_step = -1;
    return LBW_OK;
}

int lbw_alm_get(lbw_domain* d, double* rho, double* u, double* blade_force) {
    LBW_REQ(d, "null domain");
    LBW_REQ(alm_active(d), "no actuator points configured");
    AlmState* s = d->alm;
    LBW_CK(cudaSetDevice(d->device));
    LBW_CK(cudaStreamSynchronize(d->stream));
    const int par = last_parity(d);
    std::vector<double> smp((size_t)s->n * 4);
    LBW_CK(cudaMemcpy(smp.data(), s->samples + (size_t)par * s->n * 4, smp.size() * 8,
                      cudaMemcpyDeviceToHost));
    if (blade_force)
        LBW_CK(cudaMemcpy(blade_force, s->blade + (size_t)par * s->n * 3, (size_t)s->n * 24,
                          cudaMemcpyDeviceToHost));
    int32_t err = 0;
    LBW_CK(cudaMemcpy(&err, s->error_flags, 4, cudaMemcpyDeviceToHost));
    for (int p = 0; p < s->n; ++p) {
        if (rho) rho[p] = smp[p * 4];
        if (u)
            for (int c = 0; c < 3; ++c) u[p * 3 + c] = smp[p * 4 + 1 + c];
    }
    if (err & 2) {
        set_error("actuator point outside the non-periodic domain");
        return LBW_EINVAL;
    }
    if (err & 4) {
        set_error("an actuator disk spans more than three x-slabs (its ring averages need "
                  "samples from beyond the neighbouring slabs)");
        return LBW_EINVAL;
    }
    if (err & 8) {
        set_error("internal: a sampled row of the fused step had no pooled macro");
        return LBW_ECUDA;
    }
    if (err & 1) {
        set_error("density must be positive at an actuator point");
        return LBW_EINVAL;
    }
    return LBW_OK;
}

int lbw_alm_record_loads(lbw_domain* d, int64_t capacity) {
    LBW_REQ(d && capacity >= 0, "bad argument");
    LBW_REQ(alm_active(d), "no actuator points configured");
    AlmState* s = d->alm;
    LBW_CK(cudaSetDevice(d->device));
    LBW_CK(cudaStreamSynchronize(d->alm_stream));
    LBW_CK(alm_sync_side(d));
    LBW_CK(cudaStreamSynchronize(d->stream));
    if (s->h_loads) cudaFreeHost(s->h_loads);
    s->h_loads = nullptr;
    s->d_loads = nullptr;
    s->loads_cap = 0;
    if (capacity > 0) {
        LBW_REQ(capacity >= 2, "capacity must be >= 2");
        LBW_CK(cudaMallocHost(&s->h_loads, (size_t)capacity * s->n * 3 * sizeof(double)));
        void* dp = nullptr;
        s->d_loads = cudaHostGetDevicePointer(&dp, s->h_loads, 0) == cudaSuccess
                         ? static_cast<double*>(dp)
                         : nullptr;
        cudaGetLastError();
        s->loads_cap = capacity;
    }
    s->loads_from = d->step;
    // a chain already queued for the next step has not recorded its loads
    s->ready_step = -1;
    return LBW_OK;
}

int lbw_alm_read_loads(lbw_domain* d, double* out, int64_t max_steps, int64_t* first_step,
                       int64_t* n) {
    LBW_REQ(d && out && first_step && n && max_steps >= 0, "null argument");
    LBW_REQ(alm_active(d) && d->alm->loads_cap > 0, "load recording is not enabled");
    AlmState* s = d->alm;
    LBW_CK(cudaSetDevice(d->device));
    const int64_t avail = d->step - s->loads_from;
    LBW_REQ(avail < s->loads_cap || avail == 0,
            "load ring overflow: read the loads at least every capacity-1 steps");
    LBW_CK(cudaStreamSynchronize(d->alm_stream));
    LBW_CK(alm_sync_side(d));
    LBW_CK(cudaStreamSynchronize(d->stream));   // the fused step writes loads in-kernel
    const int64_t k = std::min(avail, max_steps);
    const size_t row = (size_t)s->n * 3;
    for (int64_t i = 0; i < k; ++i) {
        const int64_t st = s->loads_from + i;
        std::memcpy(out + (size_t)i * row, s->h_loads + (size_t)(st % s->loads_cap) * row,
                    row * sizeof(double));
    }
    *first_step = s->loads_from;
    *n = k;
    s->loads_from += k;
    return LBW_OK;
}

int lbw_alm_clamp_flags(lbw_domain* d, int32_t* per_polar) {
    LBW_REQ(d && per_polar, "null argument");
    if (!alm_active(d) || d->alm->n_polars == 0) return LBW_OK;
    LBW_CK(cudaSetDevice(d->device));
    LBW_CK(cudaStreamSynchronize(d->stream));
    LBW_CK(cudaMemcpy(per_polar, d->alm->clamp_flags, d->alm->n_polars * 4,
                      cudaMemcpyDeviceToHost));
    return LBW_OK;
}

}  // extern "C"

LBW_TRACE_EXPORT(alm)

