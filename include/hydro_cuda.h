/*
 * hydro_cuda.h -- C ABI of libhydro_cuda.so, the B200-native (sm_100a, FP64) space-time
 * update of arXiv 2211.13295: MC/WENO3 reconstruction -> ADER predictor -> Rusanov/HLL face
 * fluxes -> flux differencing -> conservative update + global CFL min.
 *
 * This is the drop-in boundary. The reference exposes its hot path as free C++ functions in
 * namespace hydro (proj/include/hydro/ *.hpp, statically linked from libhydro.a); a
 * maintainer swaps proj/src/{fields,boundary,reconstruct,predictor,corrector,stepper}.cpp
 * for the thin C++ shim in paper_2211_13295_b200/shim/hydro_gpu_shim.cpp, which calls the
 * entry points below. Signatures carry plain pointers and sizes only.
 *
 * Layouts are the reference's host layouts (proj/include/hydro/fields.hpp:15-128):
 *   skinny [mz][my][mx][5]        ghosts included, mx = nx + 2*ghost
 *   modal  [mz][my][mx][5][M]     M = 5 (order 2) or 11 (order 3); temporal mode = M-1
 *   fx [nz][ny][nx+1][5], fy [nz][nx][ny+1][5], fz [ny][nx][nz+1][5]
 *   rate   [nz][ny][nx][5]
 *
 * Error convention: every entry point returns an hc_status. HC_UNPHYSICAL replaces
 * hydro::unphysical_error (euler.hpp:33-35) and hc_last_error() returns the reference's
 * message text ("predictor: zone (i,j,k): non-positive density X", corrector.cpp:53-55,
 * :119-120, predictor.cpp:82-84, stepper.cpp:41-42). HC_INVALID replaces
 * std::invalid_argument. There is no CPU fallback: without a CUDA device every compute
 * entry point returns HC_CUDA.
 */
#ifndef HYDRO_CUDA_H
#define HYDRO_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HC_ABI_VERSION 1

typedef enum { HC_OK = 0, HC_UNPHYSICAL = 1, HC_INVALID = 2, HC_CUDA = 3 } hc_status;
/* riemann.hpp:12 SolverChoice; HC_HLLC and HC_HLLI are extensions (the reference has neither,
 * SPEC.md:339) */
typedef enum { HC_RUSANOV = 0, HC_HLL = 1, HC_HLLC = 2, HC_HLLI = 3 } hc_solver_kind;
typedef enum { HC_PERIODIC = 0, HC_OUTFLOW = 1 } hc_boundary; /* boundary.hpp:7 BoundaryKind */

/* PatchGeometry, geometry.hpp:34-65 */
typedef struct {
    int nx, ny, nz, ghost;
    double dx, dy, dz;
    double origin[3];
} hc_geom;

/* LimiterConfig, reconstruct.hpp:11-29 */
typedef struct {
    double cfac_rho, cfac_other, weno_eps;
    double weno_w[3];
} hc_limiter;

/* StepParams (gas, solver, limiter, order), stepper.hpp:39-45 */
typedef struct {
    int order;  /* 2 or 3 */
    int solver; /* hc_solver_kind */
    double gamma;
    hc_limiter lim;
} hc_params;

/* ------------------------------------------------------------------ library */
int hc_abi_version(void);
/* Number of visible CUDA devices (0 on a host without a GPU). */
int hc_device_count(void);
/* Measured FP64 (DFMA) throughput of `device` in TFLOP/s (2 flops per DFMA): the FP64
 * roofline denominator, which MEASURED_PEAKS.json does not carry. */
int hc_fp64_peak(int device, double* tflops);
/* Self-test of the fused kernel's branch-free division / sqrt: q = a/b, s = sqrt(a) through
 * the fast paths, with flags where the IEEE slow path would be taken instead. */
int hc_selftest_fastmath(const double* a, const double* b, size_t n, double* q, int* qslow,
                         double* s, int* sslow);
/* Copies the last error message of the calling thread into buf; returns its status. */
int hc_last_error(char* buf, size_t len);

/* ------------------------------------------------ per-kernel, host buffers
 * One entry point per reference kernel (the hydro:: function cited beside it). Arguments
 * are HOST arrays in the reference layouts; each call stages them through the device
 * (H2D, sm_100a kernel, D2H) and returns the same bits as the reference. */
/* fields.hpp:139 skinny_to_modal */
int hc_skinny_to_modal(const hc_geom* g, int modes, const double* skinny, double* modal);
/* fields.hpp:143 modal_to_skinny */
int hc_modal_to_skinny(const hc_geom* g, int modes, const double* modal, double* skinny);
/* boundary.hpp:12 apply_boundary(SkinnyState&, ...) */
int hc_apply_boundary_skinny(const hc_geom* g, int kind, double* skinny);
/* boundary.hpp:15 apply_boundary(ModalState&, ...) */
int hc_apply_boundary_modal(const hc_geom* g, int modes, int kind, double* modal);
/* reconstruct.hpp:88 limit_patch_o2 */
int hc_limit_patch_o2(const hc_geom* g, double* modal, const hc_limiter* lim);
/* reconstruct.hpp:94 reconstruct_patch_o3 */
int hc_reconstruct_patch_o3(const hc_geom* g, double* modal, const hc_limiter* lim);
/* predictor.hpp:42 predict_patch */
int hc_predict_patch(const hc_geom* g, int modes, double* modal, double dt, double gamma);
/* predictor.hpp:47 zero_temporal_mode */
int hc_zero_temporal_mode(const hc_geom* g, int modes, double* modal);
/* corrector.hpp:15 make_flux_axis */
int hc_make_flux_axis(const hc_geom* g, int modes, const double* modal, int axis, double gamma,
                      int solver, double* out);
/* corrector.hpp:21 make_du_dt */
int hc_make_du_dt(const hc_geom* g, const double* fx, const double* fy, const double* fz,
                  double dt, double* rate);
/* corrector.hpp:27 update_u_timestep (dt_next = min CFL estimate, seed 1.0e32) */
int hc_update_u_timestep(const hc_geom* g, int modes, double* modal, double* skinny,
                         const double* rate, double cfl, double gamma, double* dt_next);
/* stepper.hpp:91 compute_dt_next */
int hc_compute_dt_next(const hc_geom* g, int modes, const double* modal, double gamma,
                       double cfl, double* dt_next);
/* stepper.hpp:60 ader_step: the whole pipeline on device, materialising modal, fluxes and
 * rate exactly as the reference does (all outputs copied back). */
int hc_ader_step(const hc_geom* g, const hc_params* p, double* modal, double* skinny,
                 double* fx, double* fy, double* fz, double* rate, double dt, double cfl,
                 double* dt_next);
/* ader_step plus per-stage device times in StageProfile order (stepper.hpp:15-37):
 * [reconstruct, predict, flux, rate, update, transfer] seconds; stage_seconds may be NULL. */
int hc_ader_step_timed(const hc_geom* g, const hc_params* p, double* modal, double* skinny,
                       double* fx, double* fy, double* fz, double* rate, double dt, double cfl,
                       double* dt_next, double* stage_seconds);
/* predictor.hpp:36-37 predictor_ptwise on one zone's [5][M] modes (temporal mode written) */
int hc_predictor_ptwise(double* zone_v, int modes, double dt, double dx, double dy, double dz,
                        double gamma);
/* stepper.hpp:80-85 rk_save_u0 */
int hc_rk_save_u0(const hc_geom* g, const double* skinny, double* stage_u0);
/* stepper.hpp:75-78 rk_stage (stage coefficients a, b) */
int hc_rk_stage(const hc_geom* g, const hc_params* p, double* modal, double* skinny,
                double* fx, double* fy, double* fz, double* rate, const double* stage_u0,
                double dt, double a, double b);
/* rk_stage plus per-stage device times (as hc_ader_step_timed; zero_temporal_mode counts as
 * "predict", stepper.cpp:110-113) */
int hc_rk_stage_timed(const hc_geom* g, const hc_params* p, double* modal, double* skinny,
                      double* fx, double* fy, double* fz, double* rate, const double* stage_u0,
                      double dt, double a, double b, double* stage_seconds);
/* stepper.hpp:87-89 rk_step (nstages 2 = Heun, 3 = SSP-RK3) */
int hc_rk_step(const hc_geom* g, const hc_params* p, int nstages, double* modal,
               double* skinny, double* fx, double* fy, double* fz, double* rate,
               double* stage_u0, int bc, double dt, double cfl, double* dt_next);

/* harness.cpp:92-103 initial_dt: min CFL estimate over the active zones of a HOST skinny */
int hc_initial_dt(const hc_geom* g, const double* skinny, double gamma, double cfl,
                  double* dt);

/* ------------------------------------------------ host-side initial conditions
 * problems.cpp: sampled on the HOST with libm (exp/pow/remainder) so the inputs are
 * bit-identical to the reference's; not part of the device hot path. */
int hc_init_vortex(const hc_geom* g, double gamma, int order, double t, double* skinny);
int hc_init_sod(const hc_geom* g, double gamma, double* skinny);
int hc_init_constant(const hc_geom* g, double gamma, double* skinny);

/* ------------------------------------------------ per-kernel, device buffers
 * Same kernels on caller-owned DEVICE arrays (reference layouts) on `stream`
 * (a cudaStream_t, NULL = default). Calls that can fail synchronise the stream. */
int hc_dev_skinny_to_modal(const hc_geom* g, int modes, const double* skinny, double* modal,
                           void* stream);
int hc_dev_apply_boundary_skinny(const hc_geom* g, int kind, double* skinny, void* stream);
int hc_dev_reconstruct(const hc_geom* g, int order, double* modal, const hc_limiter* lim,
                       void* stream);
int hc_dev_predict_patch(const hc_geom* g, int modes, double* modal, double dt, double gamma,
                         void* stream);
int hc_dev_make_flux_axis(const hc_geom* g, int modes, const double* modal, int axis,
                          double gamma, int solver, double* out, void* stream);
int hc_dev_make_du_dt(const hc_geom* g, const double* fx, const double* fy, const double* fz,
                      double dt, double* rate, void* stream);
int hc_dev_update_u_timestep(const hc_geom* g, int modes, double* modal, double* skinny,
                             const double* rate, double cfl, double gamma, double* dt_next,
                             void* stream);

/* ------------------------------------------------ device-resident stepper (throughput path)
 * One patch (or one z-slab of a decomposed mesh) whose U_skinny stays in HBM across steps
 * (the paper's skinny trick). A step is ONE fused sm_100a kernel: reconstruction, predictor,
 * three face sweeps, flux differencing, update and the CFL min-reduction, never writing
 * modes/fluxes/rate to HBM. dt -> dt_next hand-off and the t_final clip
 * (harness.cpp:155-170) run on the device, so steps queue without host round trips. */
typedef struct hc_stepper hc_stepper;

typedef struct {
    /* ghost fill per axis before every step: HC_PERIODIC / HC_OUTFLOW, or -1 = caller-filled
     * (the z-slab halo planes of a multi-GPU decomposition). */
    int bc[3];
    /* 1: bit-exact build (no FMA contraction, identical to the reference);
     * 0: FMA-contracted build (<= 1e-13 rel. L1 drift after 200 steps). */
    int exact;
    int device;
    /* 0: ADER one-step (stepper.cpp:49-78); 2: Heun RK2; 3: SSP-RK3 (stepper.cpp:80-157) --
     * every RK stage is one fused launch with the temporal mode zero */
    int integrator;
} hc_stepper_opts;

int hc_stepper_create(const hc_geom* g, const hc_params* p, const hc_stepper_opts* o,
                      hc_stepper** out);
int hc_stepper_destroy(hc_stepper* s);
/* Which fused kernel the stepper launches: kernel = 1 for the persistent ring-free kernel
 * (opt-in with HC_PERSIST=1 in the environment at create time; x/y periodic, nx a multiple
 * of 32, every tile resident; ctas = its grid), 0 for the ring kernel (the default). */
int hc_stepper_info(hc_stepper* s, int* kernel, int* ctas);
/* stream used by every later call (cudaStream_t; NULL = a private stream) */
int hc_stepper_set_stream(hc_stepper* s, void* stream);
/* host skinny [mz][my][mx][5] (ghosts included) <-> device state; async on the stream when the
 * host buffer is pinned */
int hc_stepper_upload(hc_stepper* s, const double* host_skinny);
int hc_stepper_download(hc_stepper* s, double* host_skinny);
/* t, dt of the next step, cfl; t_final <= 0 = fixed step count (no clip) */
int hc_stepper_set_time(hc_stepper* s, double t, double dt, double cfl, double t_final);
/* Enqueue n fused steps (no host sync). */
int hc_stepper_step(hc_stepper* s, int n);
/* One step end to end from HOST memory: H2D of the active zones of host_in (U_skinny
 * layout; ghosts are filled on the device, never transferred), the fused step, D2H of the
 * updated active zones into host_out (may equal host_in; its ghosts are left untouched),
 * pipelined over nchunks z-chunks on three streams so both PCIe directions overlap the
 * kernel. Returns after host_out is complete. */
int hc_stepper_step_host(hc_stepper* s, const double* host_in, double* host_out, int nchunks);
/* Synchronise; report t, dt (of the next step), steps done, and device errors. */
int hc_stepper_sync(hc_stepper* s, double* t, double* dt, long* steps_done);
/* Device pointer of the state the next fused launch reads (the current RK stage's input)
 * and its row pitch in doubles; used for z-halo exchange by the multi-GPU driver. */
int hc_stepper_state(hc_stepper* s, double** dptr, size_t* row_pitch_doubles);
/* Device pointer of the scalar dt_next of the last step (for an all-reduce(min)) and the
 * device pointer of the dt the next step will use. */
int hc_stepper_dt_ptrs(hc_stepper* s, double** dt_next_dev, double** dt_dev);
/* Multi-GPU step split: (1) fill local x/y ghosts [and z if bc[2] >= 0]; caller then fills z
 * halos; (2) run the fused kernel; caller then all-reduces dt_next; (3) advance t/dt. */
int hc_stepper_fill_ghosts(hc_stepper* s);
int hc_stepper_compute(hc_stepper* s);
/* The fused launch over active z planes [kz_first, kz_last) only (last = 1 closes the step or
 * RK stage). Lets a z-slab driver compute the interior planes [G, nz-G) -- whose stencils
 * never touch the z-ghost planes, G = order - 1 + 1 -- while the halo exchange is in flight,
 * then the two boundary ranges. */
int hc_stepper_compute_range(hc_stepper* s, int kz_first, int kz_last, int last);
int hc_stepper_advance(hc_stepper* s);
/* hc_stepper_compute, and when that was the step's last stage also hc_stepper_advance -- for a
 * driver with nothing to reduce in between (one domain): the seam kernel pair then runs the
 * advance in its last CTA, one launch fewer per step. */
int hc_stepper_compute_step(hc_stepper* s);
/* fused launches per step: 1 (ADER), 2 or 3 (RK); a multi-GPU step repeats fill_ghosts +
 * halo exchange + compute per stage, then all-reduce + advance */
int hc_stepper_stages(hc_stepper* s);
/* Number of kernels this library launched on the stepper (diagnostic / bench claim). */
long hc_stepper_launches(hc_stepper* s);
/* Storage layout of the state buffers: rows per plane, doubles per row, planes. */
int hc_stepper_layout(hc_stepper* s, int* my_pad, int* pitch, int* mz);
/* The device state buffers (bufs[3]; unused entries NULL) and how many the integrator uses.
 * Which one is current is decided on the device (hc_stepper_state); drivers that enqueue
 * halo exchanges asynchronously track it as the steps flip it (ADER: every step; RK: never,
 * stage k reads buffer (cur + k) % nbuf). */
int hc_stepper_buffers(hc_stepper* s, double** bufs, int* nbuf);
/* z peer stores, for a stepper with caller-filled z ghosts (bc[2] = -1): from now on every
 * fused step (or RK stage) also writes the final state of its gh lowest active planes into the
 * top ghost planes (gh + nz + k) of lo_bufs[b], and of its gh highest into the bottom ghost
 * planes of hi_bufs[b] -- b = the buffer the step writes, the arrays being the z neighbours'
 * hc_stepper_buffers (same layout; on this device or a peer-accessible one, the caller having
 * enabled peer access). The neighbours' z halos then arrive with the compute: no exchange
 * step; hc_stepper_fill_ghosts fills the x/y ring of the z-ghost planes too. The caller orders
 * the steps of neighbouring steppers (a neighbour's step n + 1 starts after this step n).
 * lo_bufs or hi_bufs NULL: no neighbour on that side (an outflow end). */
int hc_stepper_set_zpeer(hc_stepper* s, double* const* lo_bufs, double* const* hi_bufs);

/* ------------------------------------------------ device-resident patch set
 * PatchSet (transfer.hpp:47-73) with the patches' states resident in HBM: px x py x pz
 * patches of `global` (the split must divide the mesh: transfer.cpp:19-22), each a fused
 * stepper, stepped together on one stream. hc_patchset_step = run_patch_step
 * (transfer.cpp:152-216): exchange_ghosts (one device gather reproducing the x, y, z sweeps of
 * transfer.cpp:94-149), every patch's step (RK: an exchange before every stage), the global
 * dt min, the t/dt hand-off -- no host round trip. Bit-identical to the single-patch run
 * (the reference's split invariance, acceptance criterion 8). */
typedef struct hc_patchset hc_patchset;

int hc_patchset_create(const hc_geom* global, int px, int py, int pz, const hc_params* p,
                       int boundary, int exact, int device, int integrator, hc_patchset** out);
int hc_patchset_destroy(hc_patchset* ps);
/* transfer.cpp:50-76 scatter_to_patches / gather_from_patches between a global HOST
 * SkinnyState [mz][my][mx][5] (active zones only) and the patches' device states */
int hc_patchset_scatter(hc_patchset* ps, const double* global_skinny);
int hc_patchset_gather(hc_patchset* ps, double* global_skinny);
/* One patch's whole HOST SkinnyState [mz][my][mx][5] (its own ghosts included) to (upload = 1)
 * or from (0) its device state: the per-patch residency moves of the C++ drop-in driver
 * (shim/hydro_gpu_transfer.cpp), which keeps the reference's host Patch structures. */
int hc_patchset_patch_io(hc_patchset* ps, int idx, double* host_skinny, int upload);
int hc_patchset_set_time(hc_patchset* ps, double t, double dt, double cfl, double t_final);
int hc_patchset_step(hc_patchset* ps, int n);
int hc_patchset_sync(hc_patchset* ps, double* t, double* dt, long* steps_done);
/* TransferLedger (transfer.hpp:16-24) of the skinny strategy, as the reference counts it:
 * uploads, downloads, scalar_uploads, scalar_downloads, uploads_active_only, steps */
int hc_patchset_ledger(hc_patchset* ps, unsigned long long* counts6);
long hc_patchset_launches(hc_patchset* ps);

/* ------------------------------------------------ fourth-order ADER (extension)
 * NOT in the reference (orders 2-3 only, geometry.hpp:13-27). The reference's ADER structure
 * (one face state per face, the zone mean's tau at the midpoint: predictor.cpp:26-60,
 * corrector.cpp:30-33) is second order in time, whatever the reconstruction order; this step
 * is formally fourth order: a degree-3 WENO-AO + cross-term reconstruction, a local space-time
 * predictor (Picard iterations on 4 x 4 x 4 x 4 Gauss-Legendre space-time nodes), fluxes at the
 * 2 x 2 face x 2 time Gauss points (csrc/ader4.cu). Skinny layout, ghost width 3, the same
 * vortex ICs and time-control semantics as hc_stepper; boundary = HC_PERIODIC / HC_OUTFLOW. */
typedef struct hc_ader4 hc_ader4;
int hc_ader4_create(const hc_geom* g, const hc_params* p, int boundary, int device,
                    hc_ader4** out);
int hc_ader4_destroy(hc_ader4* s);
int hc_ader4_upload(hc_ader4* s, const double* host_skinny);
int hc_ader4_download(hc_ader4* s, double* host_skinny);
int hc_ader4_set_time(hc_ader4* s, double t, double dt, double cfl, double t_final);
int hc_ader4_step(hc_ader4* s, int n);
int hc_ader4_sync(hc_ader4* s, double* t, double* dt, long* steps_done);
long hc_ader4_launches(hc_ader4* s);
/* the cudaStream_t every call of this stepper runs on (for event timing) */
int hc_ader4_stream(hc_ader4* s, void** stream);

/* ------------------------------------------------ multi-GPU z-slab domain
 * The reference's PatchSet split along z -- make_patch_set(global, 1, 1, world)
 * (transfer.hpp:60-61, transfer.cpp:17-47) -- with every patch (slab) on its own GPU, and
 * run_patch_step (transfer.hpp:73, transfer.cpp:152-216) as: x/y ghosts on each device; the
 * z sweep of exchange_ghosts (transfer.cpp:131-149) as whole-plane halo messages straight
 * into the neighbours' ghost planes (ncclSend/ncclRecv in one group, or peer copies for the
 * slabs of one process); the fused step (every RK stage gets its own exchange,
 * transfer.cpp:197-201); the global dt min (transfer.cpp:184) as an 8-byte ncclAllReduce(MIN)
 * on the device; the t/dt hand-off on the device. No host round trip per step. Bit-identical
 * to the single domain. NCCL is opened at run time (libnccl.so.2). */
typedef struct hc_domain hc_domain;

/* HC_XCHG_STORE: the fused kernels store their boundary planes straight into the neighbours'
 * ghost planes (hc_stepper_set_zpeer, NVLink peer memory): the halo transfer rides on the
 * compute, no exchange step; hc_domain_create_local only (every slab in this process). */
typedef enum { HC_XCHG_NCCL = 0, HC_XCHG_PEER = 1, HC_XCHG_STORE = 2 } hc_exchange_kind;

typedef struct {
    int bc[3];       /* per axis HC_PERIODIC / HC_OUTFLOW (z: the global ends) */
    int exact;       /* as hc_stepper_opts */
    int integrator;  /* as hc_stepper_opts */
    int device;      /* hc_domain_create: this rank's GPU */
    int transport;   /* hc_exchange_kind; HC_XCHG_PEER / _STORE only with hc_domain_create_local
                      * (_STORE: `overlap` has nothing to overlap and is ignored) */
    int overlap;     /* 1: the halo exchange runs on a second stream while the interior planes
                      * (whose stencils never reach a z ghost) are updated; then the two
                      * boundary ranges. 0: exchange, then the whole slab. Same bits. */
} hc_domain_opts;

/* An NCCL unique id for hc_domain_create (rank 0 makes it and shares it out of band);
 * len >= 128 (NCCL_UNIQUE_ID_BYTES). */
int hc_nccl_unique_id(unsigned char* id, size_t len);
/* One process per GPU: this process owns slab `rank` of `world` (global.nz % world == 0). */
int hc_domain_create(const hc_geom* global, const hc_params* p, const hc_domain_opts* o,
                     int rank, int world, const unsigned char* nccl_id, hc_domain** out);
/* One process driving `ngpu` GPUs (devices[ngpu]; ncclCommInitAll or peer copies). ngpu = 1
 * with periodic z exchanges the slab's halos with itself through the same calls. */
int hc_domain_create_local(const hc_geom* global, const hc_params* p, const hc_domain_opts* o,
                           int ngpu, const int* devices, hc_domain** out);
int hc_domain_destroy(hc_domain* d);
/* scatter_to_patches / gather_from_patches (transfer.cpp:50-76) for the slabs this process
 * drives: a global HOST SkinnyState [mz][my][mx][5]; only the slabs' active planes move. */
int hc_domain_scatter(hc_domain* d, const double* global_skinny);
int hc_domain_gather(hc_domain* d, double* global_skinny);
int hc_domain_set_time(hc_domain* d, double t, double dt, double cfl, double t_final);
/* run_patch_step x n, enqueued without host synchronisation */
int hc_domain_step(hc_domain* d, int n);
int hc_domain_sync(hc_domain* d, double* t, double* dt, long* steps_done);
/* planes per slab, first global plane of this process's first slab, slabs in this process,
 * which fused kernel steps them (hc_stepper_info) */
int hc_domain_info(hc_domain* d, int* nz_local, int* z0, int* nslabs, int* kernel);
long hc_domain_launches(hc_domain* d);

#ifdef __cplusplus
}
#endif
#endif
