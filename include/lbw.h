/*
 * lbw.h — C ABI of liblbw.so, the B200 (sm_100a) implementation of the
 * waLBerla-wind / lbwind time-step hot path (D3Q27 cumulant/BGK fp64
 * stream-collide + actuator-line coupling + inflow/outflow + x-slab halo).
 *
 * Conventions
 *   - Every entry point returns 0 on success or a negative LBW_E* code; the
 *     message of the last failure on the calling thread is lbw_last_error().
 *   - Only plain pointers and sizes cross the boundary.  Host pointers are
 *     borrowed for the duration of the call (copy-in / copy-out); device
 *     state is owned by the opaque lbw_domain and freed by
 *     lbw_domain_destroy.
 *   - Host arrays use the reference's layouts: populations (..., 27) with the
 *     direction axis fastest in the D3Q27 order i = (cx+1)*9 + (cy+1)*3 +
 *     (cz+1)  (/root/reference/pkg/src/lbwind/stencil.py:6), C order over
 *     (x, y, z, component).
 *   - Arithmetic is IEEE fp64.  LBW_MODE_EXACT kernels are compiled without
 *     FMA contraction and follow the reference's expression order, so they
 *     are bit-identical to the numba kernels (fastmath=False,
 *     _kernels.py:41).  LBW_MODE_FAST kernels use a raw-moment/FMA
 *     formulation of the same operator (agrees to ~1e-15 per step).
 *
 * Reference interfaces replaced (see INTEGRATION.md for the bindings):
 *   lbw_collide_cumulant_batch  <- lbwind._kernels.collide_cumulant_batch  (_kernels.py:412)
 *   lbw_collide_bgk_batch       <- lbwind._kernels.collide_bgk_batch       (_kernels.py:400)
 *   lbw_collide_cumulant_block  <- lbwind._kernels.collide_cumulant_block  (_kernels.py:328)
 *   lbw_collide_bgk_block       <- lbwind._kernels.collide_bgk_block       (_kernels.py:304)
 *   lbw_moments_block           <- lbwind._kernels.moments_block           (_kernels.py:357)
 *   lbw_stream_pull_block       <- lbwind._kernels.stream_pull_block       (_kernels.py:383)
 *   lbw_domain_*                <- lbwind.sim.Simulation.step and the per-block
 *                                  state it drives (sim.py:264-300, fields.py:22-94,
 *                                  halo.py:107-160, actuator.py:70-341)
 */
#ifndef LBW_H
#define LBW_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LBW_ABI_VERSION 2

/* status codes */
#define LBW_OK 0
#define LBW_EINVAL -1      /* invalid argument / configuration      -> ConfigError / ValueError */
#define LBW_ECUDA -2       /* CUDA runtime failure                  -> RuntimeError            */
#define LBW_ENONFINITE -3  /* non-finite macro found               -> NumericalAbort          */
#define LBW_ESTATE -4      /* call not valid in the current state   -> RuntimeError            */
#define LBW_ENOMEM -5      /* device allocation failed              -> MemoryError             */
#define LBW_ECOMM -6       /* inter-GPU exchange failure            -> RuntimeError            */

/* collision operators (collision.py:26, OPERATORS) */
#define LBW_OP_BGK 0
#define LBW_OP_CUMULANT 1

/* arithmetic flavour */
#define LBW_MODE_EXACT 0
#define LBW_MODE_FAST 1

/* population / force storage (run.precision, config.py:30, _kernels.py:5-7):
 * arithmetic is fp64 either way; SINGLE stores fp32 and rounds on store */
#define LBW_PREC_DOUBLE 0
#define LBW_PREC_SINGLE 1

/* walls on non-periodic y / z faces (an extension: the reference leaves
 * those ghosts unwritten, i.e. LBW_WALL_NONE) */
#define LBW_WALL_NONE 0      /* zero ghost populations (the reference's semantics) */
#define LBW_WALL_NO_SLIP 1   /* halfway bounce-back                               */
#define LBW_WALL_FREE_SLIP 2 /* specular reflection                               */

/* force spreading kernel (lbw_alm_desc.spread_kernel) */
#define LBW_SPREAD_ROMA 0      /* 3-point Roma kernel (actuator.py:100-110), the reference's */
#define LBW_SPREAD_GAUSSIAN 1  /* isotropic Gaussian exp(-(r/eps)^2), truncated at 3 eps and
                                * normalised per axis (extension)                          */

/* outer boundary along x (halo.py:122-141, BoundarySpec.KINDS) */
#define LBW_BC_PERIODIC 0
#define LBW_BC_INFLOW_OUTFLOW 1

/* ------------------------------------------------------------------ info */

int lbw_abi_version(void);
const char* lbw_last_error(void);
/* number of visible CUDA devices (0 without a GPU; never fails) */
int lbw_device_count(void);
/* number of kernels this library launched since load (all devices) */
int64_t lbw_kernel_launches(void);

/* -------------------------------------------- host-array kernel entry points
 * Drop-in equivalents of the numba kernels.  Arrays are host memory;
 * each call copies in, runs one sm_100a kernel, copies out (not the hot
 * path: the time step uses the lbw_domain API below). */

/* f2 (n,27) updated in place, F2 (n,3), macro2 (n,4) written. */
int lbw_collide_cumulant_batch(double* f2, const double* F2, double* macro2, int64_t n,
                               double omega, double w3, double w4, double w5, double w6,
                               double dt, int mode);
int lbw_collide_bgk_batch(double* f2, const double* F2, double* macro2, int64_t n,
                          double omega, double dt, int mode);

/* ghosted block arrays: f (nx+2,ny+2,nz+2,27), force (..,3), macro (..,4);
 * interior cells [1..n] per axis are processed. */
int lbw_collide_cumulant_block(double* f, const double* force, double* macro,
                               int64_t nx, int64_t ny, int64_t nz,
                               double omega, double w3, double w4, double w5, double w6,
                               double dt, int mode);
int lbw_collide_bgk_block(double* f, const double* force, double* macro,
                          int64_t nx, int64_t ny, int64_t nz, double omega, double dt,
                          int mode);
int lbw_moments_block(const double* f, const double* force, double* macro,
                      int64_t nx, int64_t ny, int64_t nz, double dt);
/* fdst interior <- fsrc[x - c_i]; fsrc's ghost ring must be populated. */
int lbw_stream_pull_block(const double* fsrc, double* fdst, int64_t nx, int64_t ny,
                          int64_t nz);

/* ------------------------------------------------------- device-resident domain
 * One lbw_domain owns one x-slab [slab_x0, slab_x0+slab_nx) of the global
 * lattice on one GPU (the whole lattice when slab_nx == cells[0]).  State
 * between steps is the post-collision population field (two fp64 SoA
 * buffers, layout [x+1][27][y][z]); the reference-visible post-stream
 * state is produced on download. */

typedef struct lbw_domain lbw_domain;

typedef struct lbw_domain_desc {
    int64_t cells[3];        /* global lattice size                          */
    int64_t slab_x0;         /* first global x owned by this domain          */
    int64_t slab_nx;         /* number of x planes owned                     */
    int32_t periodic[3];     /* domain.periodicity (config.py:254-256)      */
    int32_t op;              /* LBW_OP_*                                      */
    int32_t mode;            /* LBW_MODE_*                                    */
    int32_t boundary;        /* LBW_BC_*                                      */
    int32_t device;          /* CUDA device ordinal                          */
    double omega;            /* second-order rate (units.omega)              */
    double rates[4];         /* w3..w6 (run.collision.higher_order_rates)    */
    double u_in[3];          /* inflow velocity, lattice units (halo.py:134) */
    int32_t rank;            /* slab index along x (0 .. nranks-1)           */
    int32_t nranks;          /* number of slabs                              */
    int32_t feq_in_given;    /* 1: use feq_in below for the inflow ghost     */
    double feq_in[27];       /* equilibrium_pdf(1, u_in) as the host computed it */
    int32_t precision;       /* LBW_PREC_* (host arrays stay fp64 either way)  */
    int32_t walls[4];        /* LBW_WALL_* of the y_lo, y_hi, z_lo, z_hi faces   */
    int32_t reserved32;
    int64_t reserved[5];
} lbw_domain_desc;

int lbw_domain_create(const lbw_domain_desc* desc, lbw_domain** out);
int lbw_domain_destroy(lbw_domain* d);
/* raw cudaStream_t the domain launches on (for event timing by callers).
 * lbw_alm_configure may replace the domain's streams (an SM partition for
 * the actuator chain on small slabs): query the stream again after it. */
int lbw_domain_stream(lbw_domain* d, void** stream_out);
/* device bytes held by the domain */
int64_t lbw_domain_device_bytes(lbw_domain* d);

/* Populations of the owned interior, host AoS (slab_nx, ny, nz, 27).
 * upload: sets the pre-collision state f_n (what PdfField.interior holds
 * between steps, fields.py:22-50).  download: returns f_n, i.e. the
 * reference's post-stream state after the last step. */
int lbw_domain_upload_pdf(lbw_domain* d, const double* f_aos);
int lbw_domain_download_pdf(lbw_domain* d, double* f_aos);
/* Every owned cell set to the same 27 populations (uniform initial state,
 * fields.py:54-67 with scalar rho and (3,) u) without a host-sized array. */
int lbw_domain_fill_uniform(lbw_domain* d, const double* f27);
/* Same, but on device buffers already laid out AoS (no host copies). */
int lbw_domain_upload_pdf_device(lbw_domain* d, const double* f_aos_dev);
/* Every owned cell at equilibrium of (rho, u(x)) computed on the device,
 * u(x) = u0 + sum_m a_m sin(k_m . x + phi_m) with x the global cell centre
 * (lattice units): a seeded "turbulent-like" initial field for domains too
 * large for a host array (fields.py:54-67 semantics: the
 * macro field becomes exactly (rho, u), the force is cleared).  modes:
 * n_modes rows of 7 doubles (kx, ky, kz, ax, ay, az, phi), host memory.
 * product: 1 = product equilibrium (cumulant), 0 = polynomial (BGK). */
int lbw_domain_init_modes(lbw_domain* d, double rho, const double* u0, int32_t n_modes,
                          const double* modes, int32_t product);

/* Body force density, host AoS (slab_nx, ny, nz, 3), lattice units.
 * set: the force the next collide applies when no actuator points exist
 * (PdfField.force semantics, fields.py:36).  NULL clears it.
 * download: the force applied by the most recent collide. */
int lbw_domain_set_force(lbw_domain* d, const double* force_aos);
int lbw_domain_download_force(lbw_domain* d, double* force_aos);

/* Macroscopic field sampled by the next actuator step (sim.py:27-28):
 * uniform (rho,u) or dense host AoS (slab_nx, ny, nz, 4); NULL dense +
 * NULL uniform = snapshot the current sampling source. */
int lbw_domain_set_macro(lbw_domain* d, const double* macro_aos, const double* uniform4);
/* The macro field the next actuator step samples (PdfField.macro as the
 * reference holds it between steps: the last collide's (rho, u), the
 * initial condition, or the last recomputed moments), host AoS (..,4). */
int lbw_domain_download_macro(lbw_domain* d, double* macro_aos);
/* (rho, u) of the current state with the current force
 * (moments_block on PdfField.f, sim.py:160-165), host AoS (..,4).  Also
 * makes those moments the next actuator sampling source, as the
 * reference's _recompute_moments does. */
int lbw_domain_recompute_moments(lbw_domain* d, double* macro_aos);

/* Advance nsteps time steps (sim.py:264-300 minus host kinematics).
 * For steps with actuator points, lbw_alm_set_kinematics must have queued
 * that step's kinematics.  Asynchronous: returns once the steps are queued.
 * On a small single slab with device kinematics a call of >= 4 steps may
 * queue one resident actuator-chain kernel that waits in-kernel for the
 * call's later sweeps; all of them are queued before the call returns. */
int lbw_domain_step(lbw_domain* d, int32_t nsteps);
int64_t lbw_domain_step_index(lbw_domain* d);
int lbw_domain_set_step_index(lbw_domain* d, int64_t step);

/* Non-finite check (sim.py:254-262).  Non-blocking unless wait != 0.
 * Returns 1 and fills (step, global cell, field: 0 density / 1 velocity)
 * when a non-finite macro was seen, 0 when none (so far), <0 on error. */
int lbw_domain_poll_nonfinite(lbw_domain* d, int wait, int64_t* step, int64_t* cell3,
                              int32_t* field);
/* After a non-finite report of the last step: present the state the
 * reference leaves when _check_finite raises right after the collide
 * (sim.py:254-262, 281; run.abort: immediate) -- downloads return that
 * step's post-collision populations, not streamed.  Waits for queued work
 * and drops any actuator step queued ahead. */
int lbw_domain_hold_collided(lbw_domain* d);
int lbw_domain_sync(lbw_domain* d);

/* Sweep (K1) timing with CUDA events on the domain stream, for roofline
 * reporting.  enable != 0 starts a fresh accumulation; the query
 * synchronises and returns the summed device time of the sweeps launched
 * since, and how many there were. */
int lbw_domain_sweep_timing(lbw_domain* d, int enable);
int lbw_domain_sweep_time(lbw_domain* d, double* ms_total, int64_t* launches);

/* ---------------------------------------------------------------- actuator line
 * Points are numbered by global id (sim.py:113-143).  Static data once,
 * kinematics every step, results on demand. */

typedef struct lbw_alm_desc {
    int32_t n_points;
    const double* chord;            /* (P,)  m                                  */
    const double* element_length;   /* (P,)  m                                  */
    const double* twist;            /* (P,)  rad                                */
    const int32_t* polar_index;     /* (P,)  -1: no polar -> zero force         */
    int32_t n_polars;
    const int32_t* polar_offset;    /* (n_polars,) start row in the tables      */
    const int32_t* polar_rows;      /* (n_polars,)                              */
    const double* polar_alpha;      /* concatenated alpha (rad), cl, cd         */
    const double* polar_cl;
    const double* polar_cd;
    double velocity_scale;          /* units.velocity_scale = dx/dt (units.py:50) */
    double rho_ref;                 /* units.rho_ref                            */
    double force_dt2;               /* units.dt**2         (units.py:69)        */
    double force_den;               /* units.rho_ref*dx**4 (units.py:69)        */
    /* actuator disks (actuator.py:149-183): points of a ring share a ring
     * id; their force is the ring's momentum-theory thrust spread by area.
     * A disk point's kinematics row carries the disk axis (centre frame's
     * +x, unnormalised) in the e_chord slot. */
    const int32_t* point_ring;      /* (P,) ring id or -1 (line point); may be NULL */
    const double* area;             /* (P,) m^2 (disk samples)                  */
    int32_t n_rings;
    const int32_t* ring_first;      /* (n_rings,) first point id of the ring    */
    const int32_t* ring_count;      /* (n_rings,) sectors                        */
    const double* ring_ct;          /* (n_rings,) thrust coefficient in [0, 1)   */
    int32_t spread_kernel;          /* LBW_SPREAD_*                               */
    int32_t reserved32;
    double spread_epsilon;          /* Gaussian width in lattice cells, (0, 2]    */
    int64_t reserved[6];
} lbw_alm_desc;

int lbw_alm_configure(lbw_domain* d, const lbw_alm_desc* desc);

/* Device-side turbine kinematics (replaces TurbineTopology.advance +
 * Simulation.refresh_points, turbine.py:227-311 / sim.py:167-191, with a
 * one-CTA kernel per step).  Components in pre-order (parent < child),
 * all turbines concatenated; every actuator point belongs to exactly one
 * line component, numbered by global id. */
typedef struct lbw_kin_desc {
    int32_t n_components;
    const int32_t* parent;          /* (C) parent index, -1 for a root          */
    const double* rel_p;            /* (C,3) relative position                  */
    const double* rel_T;            /* (C,3,3) relative orientation             */
    const double* axis;             /* (C,3) unit rotation axis (any if rate 0) */
    const double* rate;             /* (C) rad/s                                */
    const double* step_rotation;    /* (C,3,3) rotation_matrix(axis, rate*dt)   */
    const double* spin;             /* (C,3,3) accumulated spin now             */
    const int32_t* line_first;      /* (C) first point id of the line, or -1    */
    const int32_t* line_count;      /* (C) points of the line                   */
    const double* offsets;          /* (P,3) line offsets from the start point  */
    const double* orientations;     /* (P,3,3) per-point orientations           */
    const double* local_frames;     /* (P,3,3) rows chord, normal, span (local) */
    double dx;                      /* m per cell                               */
    int32_t advance_first;          /* 1: advance by dt before the first step  */
    /* disks: the component's disk centre transform relative to it
     * (DiskSpec.center, turbine.py:150-193) and its sample offsets (in
     * `offsets`, rows line_first .. line_first+line_count) */
    const int32_t* is_disk;         /* (C) 1 for a disk component, else 0      */
    const double* disk_center;      /* (C,12) centre p(3), T(3,3); zeros if none */
    int64_t reserved[8];
} lbw_kin_desc;
int lbw_alm_configure_kinematics(lbw_domain* d, const lbw_kin_desc* desc);
/* current device kinematics: kin (P,18) as in set_kinematics, spin
 * (C,3,3), per-component world state (C,49) — any may be NULL. */
int lbw_alm_download_kinematics(lbw_domain* d, double* kin, double* spin, double* comp_state);
/* step whose kinematics the device spin state represents (the next step's
 * once its actuator chain has been queued ahead of time), or -1 */
int64_t lbw_alm_kinematics_step(lbw_domain* d);
/* kin: (P, 18) = lattice position (wrapped, sim.py:188-191), velocity m/s,
 * e_chord, e_normal, e_span (sim.py:176-181), position m.  Queued for the
 * next step. */
int lbw_alm_set_kinematics(lbw_domain* d, const double* kin);
/* Results of the most recent actuator step (host arrays, may be NULL):
 * sampled rho (P,), sampled u lattice (P,3), blade force N (P,3).  Blocks
 * until that step's ALM kernels finished. */
int lbw_alm_get(lbw_domain* d, double* rho, double* u, double* blade_force);
/* Thrust / power time series without synchronising the step loop: every
 * step's blade forces (P x 3) are copied device->host into a pinned ring of
 * `capacity` steps owned by the domain (0 disables).  read: waits for and
 * returns the steps executed since the last read, out (n, P, 3) with
 * n <= max_steps; more than capacity-1 unread steps is LBW_ESTATE. */
int lbw_alm_record_loads(lbw_domain* d, int64_t capacity);
int lbw_alm_read_loads(lbw_domain* d, double* out, int64_t max_steps, int64_t* first_step,
                       int64_t* n);
/* 1 once any polar lookup clamped alpha (polars.py:68-77 warn-once). */
int lbw_alm_clamp_flags(lbw_domain* d, int32_t* per_polar);

/* ---------------------------------------------------------------- multi-GPU
 * x-slab neighbours on other GPUs of the node (one process per GPU).  Each
 * domain exports an opaque blob (CUDA IPC handles of its population
 * buffers, actuator cube buffer and ordering flags); every rank imports its
 * x neighbours' blobs (NULL where the slab touches a non-periodic face).
 * lbw_domain_step then stores the nine outgoing direction planes of each
 * edge plane straight into the neighbour's ghost plane from inside the
 * sweep kernel, and orders steps with GPU-side waits on counters the
 * neighbours write — no host synchronisation per step.  Configure the
 * actuator points (lbw_alm_configure) before exporting. */
int64_t lbw_peer_blob_bytes(void);
int lbw_domain_export_handle(lbw_domain* d, void* blob, int64_t* blob_bytes);
int lbw_domain_import_peers(lbw_domain* d, const void* lo_blob, const void* hi_blob);

#ifdef __cplusplus
}
#endif
#endif /* LBW_H */
