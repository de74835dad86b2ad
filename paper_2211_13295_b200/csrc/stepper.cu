#include <cstdlib>
// stepper.cu -- the device-resident stepper (include/hydro_cuda.h, hc_stepper_*).
//
// U_skinny lives in HBM across steps in two ping-pong buffers laid out like the reference's
// SkinnyState ([z][y][x][5], fields.hpp:47-67) but with rows padded to the tile grid, so the
// fused kernel's halo loads never leave the allocation. One step = ghost fill (a gather that
// reproduces boundary.cpp's x->y->z passes) + the fused kernel + a one-thread "advance" kernel
// that performs the harness's dt/dt_next hand-off and t_final clip on the device
// (harness.cpp:155-170), so any number of steps queue on the stream without a host sync.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "fused_types.cuh"

namespace hc {
namespace {

struct SG {  // storage geometry of the stepper
    int nx, ny, nz, gh, mx, my, mz, my_pad, pitch;
};

__device__ __forceinline__ int map_index(int a, int n, int kind) {
    if (kind == 0) return ((a % n) + n) % n;
    return a < 0 ? 0 : (a >= n ? n - 1 : a);
}

// Ghost gather (see k_fill_ghosts in patch_kernels.cu for why one gather equals the
// reference's sequential x, y, z passes), restricted to storage planes [k_lo, k_hi) and
// enumerating ghost zones only: for an active plane its x/y ghost ring (2*gh full rows +
// 2*gh columns of the ny active rows), for a z-ghost plane the whole plane. bz < 0: z ghosts
// belong to the caller (halo exchange of a z-slab decomposition), which is exactly the x and
// y passes of transfer.cpp:94-130 on this rank.
__device__ __forceinline__ void ghost_copy(double* u, const SG& g, int bx, int by, int bz,
                                           int i, int j, int k) {
    bool ai = i >= g.gh && i < g.gh + g.nx, aj = j >= g.gh && j < g.gh + g.ny,
         ak = k >= g.gh && k < g.gh + g.nz;
    int si = ai ? i : g.gh + map_index(i - g.gh, g.nx, bx);
    int sj = aj ? j : g.gh + map_index(j - g.gh, g.ny, by);
    // bz < 0 (caller-filled z): a z-ghost plane's ring is filled from the plane itself
    int sk = (ak || bz < 0) ? k : g.gh + map_index(k - g.gh, g.nz, bz);
    const double* src = u + (size_t(sk) * g.my_pad + sj) * g.pitch + size_t(si) * NV;
    double* dst = u + (size_t(k) * g.my_pad + j) * g.pitch + size_t(i) * NV;
#pragma unroll
    for (int q = 0; q < NV; ++q) dst[q] = src[q];
}

// blockIdx.y = plane k_lo + y. ring_mode: the planes are active, fill their x/y ghost ring
// (2*gh full rows + 2*gh columns of the ny active rows); otherwise they are z-ghost planes,
// fill every zone.
struct Bufs {
    double* b[3];
};

// Up to four plane ranges of one ghost fill, each in ring mode (the planes are active: their
// x/y ghost ring, 2*gh full rows + 2*gh columns of the ny active rows) or full mode (z-ghost
// planes: every zone). Every ghost zone copies its composed active image (ghost_copy), so the
// ranges are independent and go in ONE launch (three launches per fill before: ~6 us each on
// the launch-bound configs[0] mesh).
struct GhostSegs {
    int lo[4], mode[4];
    unsigned start[5];  // prefix thread counts; start[n] = total
    int n;
};

__global__ void k_stepper_ghosts(Bufs bufs, int nbuf, int rel, const StepCtl* c, SG g, int bx,
                                 int by, int bz, GhostSegs segs) {
    if (c->done) return;
    double* u = bufs.b[(c->cur + rel) % nbuf];
    const unsigned r = blockIdx.x * blockDim.x + threadIdx.x;
    int sg = 0;
    while (sg < segs.n && r >= segs.start[sg + 1]) ++sg;
    if (sg >= segs.n) return;
    const unsigned ring = unsigned(2 * g.gh * (g.mx + g.ny)), plane = unsigned(g.mx * g.my);
    const unsigned loc = r - segs.start[sg];
    const unsigned per = segs.mode[sg] ? ring : plane;
    const int k = segs.lo[sg] + int(loc / per);
    const unsigned t = loc % per;
    int i, j;
    if (!segs.mode[sg]) {
        i = int(t % g.mx);
        j = int(t / g.mx);
    } else {
        const unsigned rows = unsigned(2 * g.gh) * g.mx;
        if (t < rows) {  // full ghost rows j < gh or j >= gh + ny
            const int jr = int(t / g.mx);
            i = int(t % g.mx);
            j = jr < g.gh ? jr : g.ny + jr;
        } else {  // ghost columns of the active rows
            const unsigned tt = t - rows;
            const int col = int(tt % (2 * g.gh));
            j = g.gh + int(tt / (2 * g.gh));
            i = col < g.gh ? col : g.nx + col;
        }
    }
    ghost_copy(u, g, bx, by, bz, i, j, k);
}

// z peer stores after the ring kernel (the seam kernels store in place): the gh lowest /
// highest active planes of the buffer the step wrote, into the z neighbours' ghost planes
__global__ void k_zpeer_planes(const __grid_constant__ FusedArgs a) {
    if (a.ctl->done) return;
    const int kz = int(blockIdx.y);
    if ((kz >= a.gh && kz < a.nz - a.gh) || kz < a.kz_first || kz >= a.kz_last) return;
    const int r = int(blockIdx.x * blockDim.x + threadIdx.x);
    if (r >= a.nx * a.ny) return;
    const int i = r % a.nx, j = r / a.nx;
    const size_t inplane = size_t(j + a.gh) * a.pitch + size_t(i + a.gh) * NV;
    const double* src = a.buf[(a.ctl->cur + a.out_rel) % a.nbuf] +
                        size_t(kz + a.gh) * a.my_pad * a.pitch + inplane;
    double v[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = src[q];
    zpeer_store(a, kz, inplane, v);
}

__global__ void k_advance(StepCtl* c, const ErrBlock* eb, int flip) { advance_ctl(c, eb, flip); }

}  // namespace
}  // namespace hc

using namespace hc;

struct hc_stepper {
    hc_geom g;
    hc_params p;
    hc_stepper_opts o;
    SG sg;
    double* buf[3] = {nullptr, nullptr, nullptr};
    int nbuf = 2;
    int stage = 0;  // next RK stage (host side; 0 for ADER)
    int cur = 0;
    StepCtl* ctl = nullptr;
    ErrBlock* eb = nullptr;
    cudaStream_t st = nullptr;
    bool own_stream = false;
    long launches = 0;
    int tz = 32;
    size_t bytes = 0;
    double cfl = 0.6;
    // pipelined host step (hc_stepper_step_host)
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    std::vector<cudaEvent_t> ev;
    // one whole step captured as a CUDA graph (hc_stepper_step with n > 1)
    cudaGraphExec_t graph = nullptr;
    double graph_cfl = -1.0;
    long graph_launches = 0;  // kernels per replayed step
    // the persistent ring-free kernel (fused_persist.cuh), when the mesh allows it
    bool persist = false;
    PersistLaunch pl{};
    // the ring-free seam kernel pair (fused_seam.cuh; both builds, x/y periodic, nx % 32 == 0)
    bool seam = false;
    SeamArgs sa{};
    int seam_tz = 32;
    CUtensorMap* maps = nullptr;  // device copies of the TMA maps (persist or seam)
    // z peer stores (hc_stepper_set_zpeer): the z neighbours' buffers
    double* zlo[3] = {nullptr, nullptr, nullptr};
    double* zhi[3] = {nullptr, nullptr, nullptr};
    bool zstore = false;
    // enqueue_step: the next whole-range closing launch folds the advance in (seam pair)
    bool fold_next = false;
    bool folded = false;  // ... and it did
};

namespace {

int set_dev(const hc_stepper* s) {
    HC_CUDA(cudaSetDevice(s->o.device));
    return HC_OK;
}

// Planes per CTA z-chunk. Each chunk re-runs reconstruction + predictor on its two z-ring
// planes (~0.6 of a plane's cost each), and the grid runs in waves of `slots` resident CTAs:
// pick the chunk height minimising waves x (tz + 1.2). HC_TZ overrides (tuning).
int choose_tz(int tiles, int nz, int slots, int sms) {
    if (const char* v = std::getenv("HC_TZ"))
        if (std::atoi(v) > 0) return std::max(1, std::min(nz, std::atoi(v)));
    // Thin meshes (fewer planes than the shortest chunk below): as many chunks as keep one CTA
    // per SM -- a CTA's fixed cost (pipeline fill, z-ring planes) is worth ~5 planes, and two
    // co-resident CTAs of a latency-bound launch run slower than one. configs[0] (64 tiles,
    // 4 planes): 2 chunks of 2 planes, measured 1.36 G zone/s vs 1.25 (4 x 1) and 1.14 (1 x 4).
    if (nz < 8) {
        const int chunks = std::max(1, std::min(nz, sms / std::max(1, tiles)));
        return (nz + chunks - 1) / chunks;
    }
    int best = std::min(32, nz);
    double best_cost = 1e300;
    for (int tz = 8; tz <= 96; ++tz) {
        const int chunks = (nz + tz - 1) / tz;
        const int eff = (nz + chunks - 1) / chunks;  // tallest chunk
        const long ctas = long(tiles) * chunks;
        const long waves = (ctas + slots - 1) / slots;
        const double cost = double(waves) * (eff + 1.2);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = eff;
        }
    }
    return std::max(1, std::min(best, nz));
}

FusedArgs fused_args(const hc_stepper* s) {
    FusedArgs a;
    a.buf[0] = s->buf[0];
    a.buf[1] = s->buf[1];
    a.buf[2] = s->buf[2];
    a.nbuf = s->nbuf;
    a.in_rel = 0;
    a.out_rel = 1;
    a.want_dt = 1;
    a.rk_a = 0.0;
    a.rk_b = 1.0;
    a.nx = s->g.nx;
    a.ny = s->g.ny;
    a.nz = s->g.nz;
    a.gh = s->g.ghost;
    a.my_pad = s->sg.my_pad;
    a.pitch = s->sg.pitch;
    a.tz = s->tz;
    a.kz_first = 0;
    a.kz_last = s->g.nz;
    a.dx = s->g.dx;
    a.dy = s->g.dy;
    a.dz = s->g.dz;
    a.idx = 1.0 / s->g.dx;  // predictor.cpp:29
    a.idy = 1.0 / s->g.dy;
    a.idz = 1.0 / s->g.dz;
    a.gamma = s->p.gamma;
    a.cfl = 0.0;  // filled per call from the host copy
    a.lim = Limiter{s->p.lim.cfac_rho, s->p.lim.cfac_other, s->p.lim.weno_eps,
                    s->p.lim.weno_w[0], s->p.lim.weno_w[1], s->p.lim.weno_w[2]};
    a.ctl = s->ctl;
    a.eb = s->eb;
    for (int i = 0; i < 3; ++i) {
        a.zlo[i] = s->zlo[i];
        a.zhi[i] = s->zhi[i];
    }
    a.zstore = s->zstore ? 1 : 0;
    a.fold_adv = 0;
    a.flip = s->o.integrator == 0 ? 1 : 0;
    return a;
}


}  // namespace

// Enables the persistent ring-free kernel (fused_persist.cuh) when the mesh allows it: x and y
// periodic (a tile's neighbour across the mesh edge holds exactly the zone the ring would
// recompute), nx a multiple of the 32-wide tile, 16-byte row pitch (TMA strides), and every
// tile resident at once (nx/32 x nty CTAs within the occupancy). Opt-in (HC_PERSIST=1): it
// is bit-identical to the ring kernel but measured 1.8x slower at 256^3.
static int encode_maps(hc_stepper* s, int box_rows);

static int setup_persist(hc_stepper* s) {
    const char* v = std::getenv("HC_PERSIST");
    if (!v || std::atoi(v) == 0) return HC_OK;
    const hc_geom& g = s->g;
    if (s->o.bc[0] != HC_PERIODIC || s->o.bc[1] != HC_PERIODIC) return HC_OK;
    // TMA boxes start on 16-byte boundaries: tile origins x0 = 32 k and an x halo equal to
    // the storage ghost width, so the box starts at storage column 32 k
    if (g.nx % PX_TX || (s->sg.pitch & 1) || g.ghost != (s->p.order >= 3 ? 3 : 2)) return HC_OK;
    const bool rk = s->o.integrator != 0;
    int bps = 0, sms = 0;
    FusedArgs a = fused_args(s);
    int rc = s->o.exact ? launch_fused_exact(a, s->p.order, s->p.solver, rk, nullptr, nullptr, &bps)
                        : launch_fused_fast(a, s->p.order, s->p.solver, rk, nullptr, nullptr, &bps);
    if (rc) return rc;
    HC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->o.device));
    const long cap = long(bps) * sms;
    const int ntx = g.nx / PX_TX;
    if (cap < ntx) return HC_OK;
    int nty = int(std::min<long>(g.ny, cap / ntx));  // spread over every resident slot
    if (const char* v = std::getenv("HC_PERSIST_NTY"))  // tests: force taller tiles
        nty = std::max(1, std::min(nty, std::atoi(v)));
    if (long(nty) * PX_TYM < g.ny) return HC_OK;    // tiles would exceed 7 rows
    PersistArgs& pa = s->pl.args;
    pa.ntx = ntx;
    pa.nty = nty;
    const size_t tiles = size_t(ntx) * nty;
    const size_t nrec = tiles * PX_SLOTS * PX_REC;
    const size_t nflag = tiles * PX_TYM * PX_FLAG_STRIDE;
    const size_t nscr = tiles * PX_TX * PX_TYM * PX_SCR;
    HC_CUDA(cudaMalloc(&pa.rec, nrec * sizeof(XRec)));
    HC_CUDA(cudaMalloc(&pa.flag, nflag * sizeof(unsigned long long)));
    HC_CUDA(cudaMalloc(&pa.scr, nscr * sizeof(double)));
    HC_CUDA(cudaMalloc(&pa.hdr, sizeof(PersistHdr)));
    HC_CUDA(cudaMemsetAsync(pa.rec, 0, nrec * sizeof(XRec), s->st));
    HC_CUDA(cudaMemsetAsync(pa.flag, 0, nflag * sizeof(unsigned long long), s->st));
    PersistHdr h0{};
    h0.epoch = 1;
    HC_CUDA(cudaMemcpyAsync(pa.hdr, &h0, sizeof h0, cudaMemcpyHostToDevice, s->st));
    int rc2 = encode_maps(s, px_box_h(s->p.order));
    if (rc2) return rc2;
    pa.maps = s->maps;
    s->persist = true;
    return HC_OK;
}

// One TMA tensor map per state buffer, in device memory: dims (x * 5 doubles, y rows, z
// planes), box (32 + 2 gh zones x 5, box_rows rows, 1 plane) -- the plane box of the
// persistent (7 + 2R rows) or the seam (8 + 2R rows) kernel.
static int encode_maps(hc_stepper* s, int box_rows) {
    if (s->maps) return HC_OK;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    HC_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) {
        set_error(HC_CUDA, "cuTensorMapEncodeTiled unavailable");
        return HC_CUDA;
    }
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    const SG& sg = s->sg;
    const cuuint64_t dims[3] = {cuuint64_t(sg.mx) * NV, cuuint64_t(sg.my), cuuint64_t(sg.mz)};
    const cuuint64_t strides[2] = {cuuint64_t(sg.pitch) * sizeof(double),
                                   cuuint64_t(sg.my_pad) * sg.pitch * sizeof(double)};
    const cuuint32_t box[3] = {cuuint32_t(px_box_w(s->p.order) * NV),
                               cuuint32_t(box_rows), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUtensorMap maps[3];
    std::memset(maps, 0, sizeof maps);
    for (int i = 0; i < s->nbuf; ++i) {
        CUresult r = encode(&maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, s->buf[i], dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_error(HC_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
            return HC_CUDA;
        }
    }
    // the maps live in device memory (written before any launch reads them)
    CUtensorMap* dmaps = nullptr;
    HC_CUDA(cudaMalloc(&dmaps, sizeof maps));
    HC_CUDA(cudaMemcpy(dmaps, maps, sizeof maps, cudaMemcpyHostToDevice));
    s->maps = dmaps;
    return HC_OK;
}

static int launch_seam(const hc_stepper* s, const FusedArgs& a, const SeamArgs& sa, bool rk,
                       cudaStream_t st, int* bps = nullptr) {
    return s->o.exact ? launch_seam_exact(a, sa, s->p.order, s->p.solver, rk, st, bps)
                      : launch_seam_fast(a, sa, s->p.order, s->p.solver, rk, st, bps);
}

// Enables the ring-free seam kernel pair (fused_seam.cuh) when the mesh allows it: x and y
// periodic (the zone across the mesh edge is the last tile's edge zone), nx a multiple of 32,
// ny >= 2 (every tile has two rows), storage ghosts equal to the kernel's x halo and an even
// row pitch (TMA box origins on 16-byte boundaries). Both builds; the bit-exact one also keeps
// the edge zones' rate parts (SeamArgs ex / ey). HC_SEAM=0 keeps the ring kernel.
static int setup_seam(hc_stepper* s) {
    int force = -1;
    if (const char* v = std::getenv("HC_SEAM")) force = std::atoi(v) != 0;
    if (force == 0) return HC_OK;
    const hc_geom& g = s->g;
    if (s->persist || g.ny < 2) return HC_OK;
    // the bit-exact build's rate records do not pay at order 2 (cheap predictor): equal for
    // ADER, 7 % slower for RK2 at 256^3 than the exact ring kernel (measured)
    if (force < 0 && s->o.exact && s->p.order == 2) return HC_OK;
    if (s->o.bc[0] != HC_PERIODIC || s->o.bc[1] != HC_PERIODIC) return HC_OK;
    if (g.nx % SEAM_TX || (s->sg.pitch & 1) || g.ghost != (s->p.order >= 3 ? 3 : 2)) return HC_OK;
    const bool rk = s->o.integrator != 0;
    int bps = 0, sms = 148;
    SeamArgs& sa = s->sa;
    sa.nx = g.nx;
    sa.ny = g.ny;
    sa.ntx = g.nx / SEAM_TX;
    sa.nty = (g.ny + SEAM_TYM - 1) / SEAM_TYM;
    int rc = launch_seam(s, fused_args(s), sa, rk, nullptr, &bps);
    if (rc) return rc;
    HC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->o.device));
    if (bps < 1) return HC_OK;
    s->seam_tz = choose_tz(sa.ntx * sa.nty, g.nz, sms * bps, sms);
    if ((rc = encode_maps(s, SEAM_TYM + 2 * (s->p.order >= 3 ? 2 : 1)))) return rc;
    sa.maps = s->maps;
    const size_t nsx = size_t(g.nz) * sa.ntx * g.ny * 2 * NV;
    const size_t nsy = size_t(g.nz) * sa.nty * g.nx * 2 * NV;
    HC_CUDA(cudaMalloc(&sa.sx, nsx * sizeof(double)));
    HC_CUDA(cudaMalloc(&sa.sy, nsy * sizeof(double)));
    HC_CUDA(cudaMemsetAsync(sa.sx, 0, nsx * sizeof(double), s->st));
    HC_CUDA(cudaMemsetAsync(sa.sy, 0, nsy * sizeof(double), s->st));
    sa.ex = sa.ey = nullptr;
    if (s->o.exact) {
        const size_t nex = size_t(g.nz) * sa.ntx * g.ny * 2 * 3 * NV;
        const size_t ney = size_t(g.nz) * sa.nty * g.nx * 2 * 3 * NV;
        HC_CUDA(cudaMalloc(&sa.ex, nex * sizeof(double)));
        HC_CUDA(cudaMalloc(&sa.ey, ney * sizeof(double)));
    }
    s->seam = true;
    return HC_OK;
}

// Configures the fused kernels this stepper will launch (module load, shared-memory opt-in)
// at creation, so the first timed step does not pay for them (the seam kernels are configured
// by setup_seam's occupancy query).
static int preload_kernels(hc_stepper* s) {
    if (s->seam || s->persist) return HC_OK;
    FusedArgs a = fused_args(s);
    a.kz_last = a.kz_first;  // empty range: configure only
    const bool rk = s->o.integrator != 0;
    return s->o.exact ? launch_fused_exact(a, s->p.order, s->p.solver, rk, s->st)
                      : launch_fused_fast(a, s->p.order, s->p.solver, rk, s->st);
}

static size_t state_bytes(const hc_stepper* s) {
    return size_t(s->sg.mz) * s->sg.my * s->sg.mx * NV * sizeof(double);
}

// Reads which buffer is current from the device (steps after t_final or after a failure
// are no-ops, so the host's per-launch guess can be off).
static int refresh_cur(hc_stepper* s) {
    int cur = 0;
    HC_CUDA(cudaMemcpyAsync(&cur, &s->ctl->cur, sizeof cur, cudaMemcpyDeviceToHost, s->st));
    HC_CUDA(cudaStreamSynchronize(s->st));
    s->cur = cur;
    return HC_OK;
}

extern "C" {

int hc_stepper_create(const hc_geom* g, const hc_params* p, const hc_stepper_opts* o,
                      hc_stepper** out) {
    if (!p || !o || !out) {
        set_error(HC_INVALID, "null argument");
        return HC_INVALID;
    }
    // order 4 (the WENO-AO extension, fused stepper only) has order 3's ghost needs
    int rc = validate_geom(g, p->order == 4 ? 3 : p->order);
    if (rc) return rc;
    if (p->solver < HC_RUSANOV || p->solver > HC_HLLI) {
        set_error(HC_INVALID, "unknown riemann solver");
        return HC_INVALID;
    }
    if (o->integrator != 0 && o->integrator != 2 && o->integrator != 3) {
        set_error(HC_INVALID, "integrator must be 0 (ADER), 2 (RK2) or 3 (SSP-RK3)");
        return HC_INVALID;
    }
    // -1 = caller-filled ghosts: z alone (z-slab halos) or all three axes (patch sets)
    for (int a = 0; a < 3; ++a)
        if (o->bc[a] < -1 || o->bc[a] > 1 || (a < 2 && o->bc[a] < 0 && o->bc[2] >= 0) ||
            ((o->bc[0] < 0) != (o->bc[1] < 0))) {
            set_error(HC_INVALID, "bad boundary kind (x/y periodic or outflow, or all -1)");
            return HC_INVALID;
        }
    int ndev = hc_device_count();
    if (ndev == 0 || o->device < 0 || o->device >= ndev) {
        set_error(HC_CUDA, "no CUDA device available for the stepper (there is no CPU path)");
        return HC_CUDA;
    }
    hc_stepper* s = new (std::nothrow) hc_stepper();
    if (!s) {
        set_error(HC_INVALID, "out of host memory");
        return HC_INVALID;
    }
    s->g = *g;
    s->p = *p;
    s->o = *o;
    const bool o3 = p->order >= 3;
    const int TX = o3 ? FusedTile<true>::TX : FusedTile<false>::TX;
    const int TY = o3 ? FusedTile<true>::TY : FusedTile<false>::TY;
    const int G = o3 ? 3 : 2;
    SG& sg = s->sg;
    sg.nx = g->nx;
    sg.ny = g->ny;
    sg.nz = g->nz;
    sg.gh = g->ghost;
    sg.mx = mx_of(*g);
    sg.my = my_of(*g);
    sg.mz = mz_of(*g);
    // The device layout IS the host SkinnyState layout (fields.hpp:47-67): transfers are
    // contiguous plane ranges. Tiles hanging over the x/y edge of the mesh read the next
    // row / plane (those zones are masked), and the last plane's overhang lands in the slack.
    sg.my_pad = sg.my;
    sg.pitch = sg.mx * NV;
    // slack sized for the largest tile any (tuning) build instantiates: 32 x 16
    const size_t slack = size_t(std::max(TY, 16) + 2 * G + 2) * sg.pitch +
                         size_t(std::max(TX, 32) + 2 * G) * NV;
    (void)TX;
    if ((rc = set_dev(s))) {
        delete s;
        return rc;
    }
    {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, o->device);
        const int tiles = ((g->nx + TX - 1) / TX) * ((g->ny + TY - 1) / TY);
        s->tz = choose_tz(tiles, g->nz, sms * FusedTile<true>::MINB, sms);
    }
    s->bytes = (size_t(sg.mz) * sg.my_pad * sg.pitch + slack) * sizeof(double);
    cudaError_t e = cudaMalloc(&s->buf[0], s->bytes);
    if (e == cudaSuccess) e = cudaMalloc(&s->buf[1], s->bytes);
    s->nbuf = o->integrator == 3 ? 3 : 2;
    if (e == cudaSuccess && s->nbuf == 3) e = cudaMalloc(&s->buf[2], s->bytes);
    if (e == cudaSuccess) e = cudaMalloc(&s->ctl, sizeof(StepCtl));
    if (e == cudaSuccess) e = cudaMalloc(&s->eb, sizeof(ErrBlock));
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking);
    if (e == cudaSuccess) {
        s->own_stream = true;
        e = cudaMemsetAsync(s->buf[0], 0, s->bytes, s->st);
    }
    if (e == cudaSuccess) e = cudaMemsetAsync(s->buf[1], 0, s->bytes, s->st);
    if (e == cudaSuccess) e = cudaMemsetAsync(s->eb, 0, sizeof(ErrBlock), s->st);
    if (e == cudaSuccess) {
        StepCtl c{};
        c.acc = 1.0e32;
        c.dt_next = 1.0e32;
        e = cudaMemcpyAsync(s->ctl, &c, sizeof c, cudaMemcpyHostToDevice, s->st);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->st);
    if (e != cudaSuccess) {
        rc = cuda_fail(e, "hc_stepper_create");
        hc_stepper_destroy(s);
        return rc;
    }
    if ((rc = setup_persist(s)) || (rc = setup_seam(s)) || (rc = preload_kernels(s)) ||
        (rc = (cudaStreamSynchronize(s->st) == cudaSuccess
                                              ? HC_OK : cuda_fail(cudaGetLastError(),
                                                                  "persist setup")))) {
        hc_stepper_destroy(s);
        return rc;
    }
    *out = s;
    return HC_OK;
}

int hc_stepper_destroy(hc_stepper* s) {
    if (!s) return HC_OK;
    cudaSetDevice(s->o.device);
    if (s->st) cudaStreamSynchronize(s->st);
    cudaFree(s->buf[0]);
    cudaFree(s->buf[1]);
    cudaFree(s->buf[2]);
    cudaFree(s->ctl);
    cudaFree(s->eb);
    cudaFree(s->pl.args.rec);
    cudaFree(s->pl.args.flag);
    cudaFree(s->pl.args.scr);
    cudaFree(s->pl.args.hdr);
    cudaFree(s->sa.sx);
    cudaFree(s->sa.sy);
    cudaFree(s->sa.ex);
    cudaFree(s->sa.ey);
    cudaFree(s->maps);  // (the persistent kernel's maps are these)
    for (cudaEvent_t e : s->ev) cudaEventDestroy(e);
    if (s->graph) cudaGraphExecDestroy(s->graph);
    if (s->s_h2d) cudaStreamDestroy(s->s_h2d);
    if (s->s_d2h) cudaStreamDestroy(s->s_d2h);
    if (s->own_stream && s->st) cudaStreamDestroy(s->st);
    delete s;
    return HC_OK;
}

int hc_stepper_set_stream(hc_stepper* s, void* stream) {
    int rc = set_dev(s);
    if (rc) return rc;
    HC_CUDA(cudaStreamSynchronize(s->st));
    if (stream) {
        if (s->own_stream) cudaStreamDestroy(s->st);
        s->st = static_cast<cudaStream_t>(stream);
        s->own_stream = false;
    }
    return HC_OK;
}

int hc_stepper_upload(hc_stepper* s, const double* host_skinny) {
    int rc = set_dev(s);
    if (!rc) rc = refresh_cur(s);
    if (rc) return rc;
    HC_CUDA(cudaMemcpyAsync(s->buf[s->cur], host_skinny, state_bytes(s), cudaMemcpyHostToDevice,
                            s->st));
    return HC_OK;
}

int hc_stepper_download(hc_stepper* s, double* host_skinny) {
    int rc = set_dev(s);
    if (!rc) rc = refresh_cur(s);
    if (rc) return rc;
    HC_CUDA(cudaMemcpyAsync(host_skinny, s->buf[s->cur], state_bytes(s), cudaMemcpyDeviceToHost,
                            s->st));
    HC_CUDA(cudaStreamSynchronize(s->st));
    return HC_OK;
}

int hc_stepper_set_time(hc_stepper* s, double t, double dt, double cfl, double t_final) {
    int rc = set_dev(s);
    if (rc) return rc;
    StepCtl c{};
    c.t = t;
    c.dt = dt;
    c.t_final = t_final;
    c.acc = 1.0e32;
    c.dt_next = 1.0e32;
    if (t_final > 0.0) {  // harness.cpp:156-160, applied before the first step too
        double rem = t_final - t;
        if (rem <= 1e-12 * t_final) c.done = 1;
        else if (c.dt >= rem) c.dt = rem;
    }
    s->cfl = cfl;  // TimeState::cfl, a constant of the run
    if ((rc = refresh_cur(s))) return rc;
    c.cur = s->cur;
    HC_CUDA(cudaMemcpyAsync(s->ctl, &c, sizeof c, cudaMemcpyHostToDevice, s->st));
    HC_CUDA(cudaMemsetAsync(s->eb, 0, sizeof(ErrBlock), s->st));
    HC_CUDA(cudaStreamSynchronize(s->st));
    return HC_OK;
}

// Ghost fill of storage planes [k_lo, k_hi): active planes get their x/y ring, z-ghost
// planes (when this stepper owns the z boundary) are filled whole.
static int stage_in_rel(const hc_stepper* s) { return s->o.integrator == 0 ? 0 : s->stage; }

static int fill_planes(hc_stepper* s, int k_lo, int k_hi, cudaStream_t st) {
    const SG& g = s->sg;
    k_lo = std::max(k_lo, 0);
    k_hi = std::min(k_hi, g.mz);
    const int a_lo = std::max(k_lo, g.gh), a_hi = std::min(k_hi, g.gh + g.nz);
    const unsigned ring = unsigned(2 * g.gh * (g.mx + g.ny));
    const unsigned plane = unsigned(g.mx * g.my);
    GhostSegs segs{};
    auto add = [&](int lo, int hi, int ring_mode) {
        if (hi <= lo) return;
        segs.lo[segs.n] = lo;
        segs.mode[segs.n] = ring_mode;
        segs.start[segs.n + 1] = segs.start[segs.n] + unsigned(hi - lo) * (ring_mode ? ring : plane);
        ++segs.n;
    };
    if (s->o.bc[0] >= 0) add(a_lo, a_hi, 1);  // (all -1: a patch set fills every ghost)
    if (s->o.bc[0] >= 0 && s->zstore) {  // z-ghost planes hold the neighbours' active zones
        add(k_lo, std::min(k_hi, g.gh), 1);
        add(std::max(k_lo, g.gh + g.nz), k_hi, 1);
    } else if (s->o.bc[2] >= 0) {
        add(k_lo, std::min(k_hi, g.gh), 0);
        add(std::max(k_lo, g.gh + g.nz), k_hi, 0);
    }
    if (segs.n == 0) return HC_OK;
    Bufs b{{s->buf[0], s->buf[1], s->buf[2]}};
    k_stepper_ghosts<<<(segs.start[segs.n] + 255) / 256, 256, 0, st>>>(
        b, s->nbuf, stage_in_rel(s), s->ctl, g, s->o.bc[0], s->o.bc[1], s->o.bc[2], segs);
    s->launches++;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HC_OK : cuda_fail(e, "k_stepper_ghosts");
}

int hc_stepper_fill_ghosts(hc_stepper* s) {
    int rc = set_dev(s);
    if (rc) return rc;
    return fill_planes(s, 0, s->sg.mz, s->st);
}

// Shu-Osher stage coefficients U' = a U0 + b (U + K(U)) (stepper.cpp:80-86)
static const double kHeun[2][2] = {{0.0, 1.0}, {0.5, 0.5}};
static const double kSsp3[3][2] = {{0.0, 1.0}, {0.75, 0.25}, {1.0 / 3.0, 2.0 / 3.0}};

int hc_stepper_stages(hc_stepper* s) { return s->o.integrator == 0 ? 1 : s->o.integrator; }

// The kernels of one step (or RK stage) over a.kz_first..a.kz_last on stream st: the seam
// pair (main kernel + x and y seam fixes), the persistent kernel, or the ring kernel.
static int launch_step(hc_stepper* s, FusedArgs a, bool rk, cudaStream_t st) {
    int rc;
    if (s->seam) {
        a.tz = s->seam_tz;
        if ((rc = launch_seam(s, a, s->sa, rk, st))) return rc;
        s->launches += 2;
        return HC_OK;
    }
    const PersistLaunch* pl = s->persist ? &s->pl : nullptr;
    rc = s->o.exact ? launch_fused_exact(a, s->p.order, s->p.solver, rk, st, pl)
                    : launch_fused_fast(a, s->p.order, s->p.solver, rk, st, pl);
    if (rc) return rc;
    if (s->zstore) {
        const dim3 grid(unsigned((s->g.nx * s->g.ny + 255) / 256), unsigned(s->g.nz));
        k_zpeer_planes<<<grid, 256, 0, st>>>(a);
        s->launches++;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "k_zpeer_planes");
    }
    s->launches++;
    return HC_OK;
}

// One fused launch: the ADER step, or the next Runge-Kutta stage.
int hc_stepper_compute(hc_stepper* s) { return hc_stepper_compute_range(s, 0, s->g.nz, 1); }

// The fused launch over active planes [kz_first, kz_last) only; `last` = 1 closes the step /
// stage (buffer and stage bookkeeping). Ranges of one step may run in any order: each reads
// the input buffer, writes its own planes of the output buffer and min-reduces into the
// same dt accumulator.
int hc_stepper_compute_range(hc_stepper* s, int kz_first, int kz_last, int last) {
    int rc = set_dev(s);
    if (rc) return rc;
    if (kz_first < 0 || kz_last > s->g.nz || kz_first > kz_last) {
        set_error(HC_INVALID, "compute range outside the active planes");
        return HC_INVALID;
    }
    FusedArgs a = fused_args(s);
    a.cfl = s->cfl;
    a.kz_first = kz_first;
    a.kz_last = kz_last;
    const bool rk = s->o.integrator != 0;
    if (rk) {
        const int ns = s->o.integrator, k = s->stage;
        const double* ab = ns == 2 ? kHeun[k] : kSsp3[k];
        a.in_rel = k;                      // stage k reads the previous stage's result
        a.out_rel = (k + 1) % s->nbuf;     // the last stage lands in buffer cur (in place on U0)
        if (k == ns - 1) a.out_rel = 0;
        a.rk_a = ab[0];
        a.rk_b = ab[1];
        a.want_dt = k == ns - 1;
    }
    s->folded = false;
    // (only where launches dominate: every fix CTA takes a turn on one counter, which costs
    // ~2 us per thousand CTAs -- 2 % of the 256^3 step, more than the launch it saves)
    const SeamArgs& sa = s->sa;
    const long fix_ctas = long((sa.nty * sa.nx + 127) / 128 + (sa.ntx * sa.ny + 127) / 128 +
                               (4 * sa.ntx * sa.nty + 127) / 128) * s->g.nz;
    if (s->fold_next && s->seam && kz_first == 0 && kz_last == s->g.nz && a.want_dt &&
        fix_ctas <= 2048) {
        a.fold_adv = 1;
        s->folded = true;
    }
    if (kz_last > kz_first) {
        if ((rc = launch_step(s, a, rk, s->st))) return rc;
    }
    if (!last) return HC_OK;
    if (rk)
        s->stage = (s->stage + 1) % s->o.integrator;
    else
        s->cur = 1 - s->cur;  // host-side guess; the device's ctl->cur is authoritative
    return HC_OK;
}

// The next stage, and -- when it is the step's last -- the advance: folded into the seam
// pair's last CTA, else k_advance (no all-reduce of dt_next between the two).
int hc_stepper_compute_step(hc_stepper* s) {
    const bool last = s->o.integrator == 0 || s->stage == s->o.integrator - 1;
    if (!last) return hc_stepper_compute(s);
    const char* nf = std::getenv("HC_NO_FOLD");  // (A/B: 1 keeps k_advance)
    s->fold_next = !(nf && std::atoi(nf) != 0);
    int rc = hc_stepper_compute(s);
    s->fold_next = false;
    if (rc) return rc;
    if (s->folded) {
        s->folded = false;
        s->stage = 0;
        return HC_OK;
    }
    return hc_stepper_advance(s);
}

int hc_stepper_advance(hc_stepper* s) {
    int rc = set_dev(s);
    if (rc) return rc;
    k_advance<<<1, 1, 0, s->st>>>(s->ctl, s->eb, s->o.integrator == 0 ? 1 : 0);
    s->launches++;
    s->stage = 0;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HC_OK : cuda_fail(e, "k_advance");
}

static int enqueue_step(hc_stepper* s) {
    const int ns = hc_stepper_stages(s);
    int rc = HC_OK;
    for (int k = 0; k < ns && !rc; ++k) {
        rc = hc_stepper_fill_ghosts(s);  // rk_step: apply_boundary before every stage
        if (!rc) rc = k == ns - 1 ? hc_stepper_compute_step(s) : hc_stepper_compute(s);
    }
    return rc;
}

// Captures one whole step (ghost fills, fused launches, advance) as a CUDA graph. Every
// kernel takes its time control and current buffer from the device StepCtl, so one graph
// replays any number of steps; only the host-side cfl is baked into the launch arguments.
static int capture_step(hc_stepper* s) {
    if (s->graph) {
        cudaGraphExecDestroy(s->graph);
        s->graph = nullptr;
    }
    const long l0 = s->launches;
    const int cur0 = s->cur, stage0 = s->stage;
    cudaGraph_t g = nullptr;
    HC_CUDA(cudaStreamBeginCapture(s->st, cudaStreamCaptureModeThreadLocal));
    int rc = enqueue_step(s);
    cudaError_t e = cudaStreamEndCapture(s->st, &g);
    if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&s->graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
        s->graph = nullptr;
        return cuda_fail(e, "cudaGraphInstantiate");
    }
    s->graph_launches = s->launches - l0;
    s->graph_cfl = s->cfl;
    s->launches = l0;  // nothing ran yet: restore the host bookkeeping
    s->cur = cur0;
    s->stage = stage0;
    return HC_OK;
}

// n steps: plain launches for one step, a replayed CUDA graph of one step otherwise
// (HC_NO_GRAPH=1 disables the graph). Launch-bound meshes (configs[0]: 128 x 128 x 4) gain
// most; at 256^3 the five launches per step are < 1 % of the step.
int hc_stepper_step(hc_stepper* s, int n) {
    int rc = set_dev(s);
    if (rc) return rc;
    static const bool no_graph = [] {
        const char* v = std::getenv("HC_NO_GRAPH");
        return v && std::atoi(v) != 0;
    }();
    if (n <= 1 || no_graph) {
        for (int i = 0; i < n; ++i)
            if ((rc = enqueue_step(s))) return rc;
        return HC_OK;
    }
    if (!s->graph || s->graph_cfl != s->cfl)
        if ((rc = capture_step(s))) return rc;
    for (int i = 0; i < n; ++i) {
        HC_CUDA(cudaGraphLaunch(s->graph, s->st));
        s->launches += s->graph_launches;
        if (s->o.integrator == 0) s->cur = 1 - s->cur;  // host guess, as enqueue_step
    }
    return HC_OK;
}

// Copies storage planes [k_lo, k_hi) between host and device (identical layouts).
static int copy_planes(hc_stepper* s, double* dev, double* host, int k_lo, int k_hi, bool up,
                       cudaStream_t st) {
    if (k_hi <= k_lo) return HC_OK;
    const size_t plane = size_t(s->sg.my) * s->sg.mx * NV;
    const size_t off = size_t(k_lo) * plane, bytes = size_t(k_hi - k_lo) * plane * sizeof(double);
    if (up)
        HC_CUDA(cudaMemcpyAsync(dev + off, host + off, bytes, cudaMemcpyHostToDevice, st));
    else
        HC_CUDA(cudaMemcpyAsync(host + off, dev + off, bytes, cudaMemcpyDeviceToHost, st));
    return HC_OK;
}

// Copies the ACTIVE zones of storage planes [k_lo, k_hi) (clamped to the active planes)
// between the host SkinnyState and the device state: one strided 3D copy, rows of nx zones.
// Ghost zones are never transferred -- the device fills them (fill_planes).
static int copy_active(hc_stepper* s, double* dev, double* host, int k_lo, int k_hi, bool up,
                       cudaStream_t st) {
    const SG& g = s->sg;
    k_lo = std::max(k_lo, g.gh);
    k_hi = std::min(k_hi, g.gh + g.nz);
    if (k_hi <= k_lo) return HC_OK;
    cudaMemcpy3DParms p = {};
    const size_t row = size_t(g.mx) * NV * sizeof(double);
    cudaPitchedPtr hp = make_cudaPitchedPtr(host, row, row, g.my);
    cudaPitchedPtr dp = make_cudaPitchedPtr(dev, size_t(g.pitch) * sizeof(double), row, g.my_pad);
    const cudaPos pos = make_cudaPos(size_t(g.gh) * NV * sizeof(double), g.gh, k_lo);
    p.extent = make_cudaExtent(size_t(g.nx) * NV * sizeof(double), g.ny, k_hi - k_lo);
    if (up) {
        p.srcPtr = hp;
        p.dstPtr = dp;
        p.kind = cudaMemcpyHostToDevice;
    } else {
        p.srcPtr = dp;
        p.dstPtr = hp;
        p.kind = cudaMemcpyDeviceToHost;
    }
    p.srcPos = pos;
    p.dstPos = pos;
    HC_CUDA(cudaMemcpy3DAsync(&p, st));
    return HC_OK;
}

// One ADER step end to end from host memory: H2D of U_skinny, ghost fill, fused update, D2H
// of the updated active planes, pipelined over z-chunks on three streams so the two PCIe
// directions and the kernel overlap (chunk c computes while c+1 uploads and c-1 downloads).
// host_in may equal host_out. Pinned host memory gives the overlap; pageable still works.
int hc_stepper_step_host(hc_stepper* s, const double* host_in, double* host_out, int nchunks) {
    int rc = set_dev(s);
    if (!rc) rc = refresh_cur(s);
    if (rc) return rc;
    if (s->o.bc[2] < 0) {
        set_error(HC_INVALID, "hc_stepper_step_host needs a z boundary owned by the stepper");
        return HC_INVALID;
    }
    if (s->o.integrator != 0) {  // multi-stage: whole-state transfers around the stages
        if ((rc = hc_stepper_upload(s, host_in))) return rc;
        if ((rc = hc_stepper_step(s, 1))) return rc;
        return hc_stepper_download(s, host_out);
    }
    const SG& g = s->sg;
    const int G = s->p.order >= 3 ? 3 : 2;
    nchunks = std::max(1, std::min(nchunks, g.nz / 4));
    if (!s->s_h2d) {
        HC_CUDA(cudaStreamCreateWithFlags(&s->s_h2d, cudaStreamNonBlocking));
        HC_CUDA(cudaStreamCreateWithFlags(&s->s_d2h, cudaStreamNonBlocking));
    }
    const size_t need = size_t(3 * nchunks + 3);
    while (s->ev.size() < need) {
        cudaEvent_t e;
        HC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        s->ev.push_back(e);
    }
    cudaEvent_t* ev_up = s->ev.data();                // [nchunks]
    cudaEvent_t* ev_comp = ev_up + nchunks;           // [nchunks]
    cudaEvent_t ev_start = s->ev[2 * nchunks];
    cudaEvent_t ev_wrap = s->ev[2 * nchunks + 1];
    double* in = s->buf[s->cur];
    double* out = s->buf[1 - s->cur];
    double* hin = const_cast<double*>(host_in);
    // order after previous work on the compute stream (the state must be idle)
    HC_CUDA(cudaEventRecord(ev_start, s->st));
    HC_CUDA(cudaStreamWaitEvent(s->s_h2d, ev_start, 0));
    HC_CUDA(cudaStreamWaitEvent(s->s_d2h, ev_start, 0));
    // Only active zones cross PCIe (ghosts are filled on the device): the top G active planes
    // first -- they feed the periodic bottom ghosts of chunk 0 -- then chunk by chunk.
    const int wrap_lo = g.gh + g.nz - G;
    if ((rc = copy_active(s, in, hin, wrap_lo, g.gh + g.nz, true, s->s_h2d))) return rc;
    HC_CUDA(cudaEventRecord(ev_wrap, s->s_h2d));
    int uploaded = 0;  // storage planes [0, uploaded) are on the device (ghosts once filled)
    for (int c = 0; c < nchunks; ++c) {
        const int c0 = int((long(g.nz) * c) / nchunks), c1 = int((long(g.nz) * (c + 1)) / nchunks);
        const int hi = (c == nchunks - 1) ? g.mz : std::min(g.mz, g.gh + c1 + G);
        if ((rc = copy_active(s, in, hin, uploaded, std::min(hi, wrap_lo), true, s->s_h2d)))
            return rc;
        HC_CUDA(cudaEventRecord(ev_up[c], s->s_h2d));
        HC_CUDA(cudaStreamWaitEvent(s->st, ev_up[c], 0));
        if (c == 0) HC_CUDA(cudaStreamWaitEvent(s->st, ev_wrap, 0));
        if ((rc = fill_planes(s, uploaded, hi, s->st))) return rc;
        uploaded = hi;
        FusedArgs a = fused_args(s);
        a.cfl = s->cfl;
        a.kz_first = c0;
        a.kz_last = c1;
        if ((rc = launch_step(s, a, false, s->st))) return rc;
        HC_CUDA(cudaEventRecord(ev_comp[c], s->st));
        HC_CUDA(cudaStreamWaitEvent(s->s_d2h, ev_comp[c], 0));
        if ((rc = copy_active(s, out, host_out, g.gh + c0, g.gh + c1, false, s->s_d2h))) return rc;
    }
    s->cur = 1 - s->cur;
    if ((rc = hc_stepper_advance(s))) return rc;
    HC_CUDA(cudaStreamSynchronize(s->s_d2h));
    HC_CUDA(cudaStreamSynchronize(s->st));
    return HC_OK;
}

int hc_stepper_sync(hc_stepper* s, double* t, double* dt, long* steps_done) {
    int rc = set_dev(s);
    if (rc) return rc;
    StepCtl c;
    ErrBlock eb;
    HC_CUDA(cudaMemcpyAsync(&c, s->ctl, sizeof c, cudaMemcpyDeviceToHost, s->st));
    HC_CUDA(cudaMemcpyAsync(&eb, s->eb, sizeof eb, cudaMemcpyDeviceToHost, s->st));
    HC_CUDA(cudaStreamSynchronize(s->st));
    s->cur = c.cur;
    if (t) *t = c.t;
    if (dt) *dt = c.dt;
    if (steps_done) *steps_done = long(c.steps);
    if (s->persist) {
        unsigned int to = 0;
        HC_CUDA(cudaMemcpy(&to, &s->pl.args.hdr->timeout, sizeof to, cudaMemcpyDeviceToHost));
        if (to) {
            set_error(HC_CUDA, "persistent fused kernel: a tile-exchange wait timed out "
                               "(CTAs not co-resident); results are invalid");
            return HC_CUDA;
        }
    }
    return report_device_errors(eb);
}

int hc_stepper_info(hc_stepper* s, int* kernel, int* ctas) {
    if (!s) return HC_INVALID;
    if (kernel) *kernel = s->persist ? 1 : (s->seam ? 2 : 0);
    if (ctas) *ctas = s->persist ? s->pl.args.ntx * s->pl.args.nty
                                 : (s->seam ? s->sa.ntx * s->sa.nty : 0);
    return HC_OK;
}

int hc_stepper_state(hc_stepper* s, double** dptr, size_t* row_pitch_doubles) {
    int rc = set_dev(s);
    if (!rc) rc = refresh_cur(s);
    if (rc) return rc;
    if (dptr) *dptr = s->buf[(s->cur + stage_in_rel(s)) % s->nbuf];
    if (row_pitch_doubles) *row_pitch_doubles = size_t(s->sg.pitch);
    return HC_OK;
}

int hc_stepper_set_zpeer(hc_stepper* s, double* const* lo_bufs, double* const* hi_bufs) {
    if (!s || (!lo_bufs && !hi_bufs)) {
        set_error(HC_INVALID, "hc_stepper_set_zpeer: null argument");
        return HC_INVALID;
    }
    if (s->o.bc[2] >= 0 || s->persist) {
        set_error(HC_INVALID, "hc_stepper_set_zpeer needs caller-filled z ghosts (bc[2] = -1) "
                              "and the ring or seam kernel");
        return HC_INVALID;
    }
    for (int i = 0; i < s->nbuf; ++i)
        if ((lo_bufs && !lo_bufs[i]) || (hi_bufs && !hi_bufs[i])) {
            set_error(HC_INVALID, "hc_stepper_set_zpeer: a neighbour buffer is NULL");
            return HC_INVALID;
        }
    for (int i = 0; i < 3; ++i) {
        s->zlo[i] = lo_bufs && i < s->nbuf ? lo_bufs[i] : nullptr;
        s->zhi[i] = hi_bufs && i < s->nbuf ? hi_bufs[i] : nullptr;
    }
    s->zstore = true;
    if (s->graph) {  // a captured step holds the old arguments
        cudaGraphExecDestroy(s->graph);
        s->graph = nullptr;
    }
    return HC_OK;
}

int hc_stepper_buffers(hc_stepper* s, double** bufs, int* nbuf) {
    if (!s) return HC_INVALID;
    if (bufs)
        for (int i = 0; i < 3; ++i) bufs[i] = s->buf[i];
    if (nbuf) *nbuf = s->nbuf;
    return HC_OK;
}

int hc_stepper_dt_ptrs(hc_stepper* s, double** dt_next_dev, double** dt_dev) {
    if (dt_next_dev) *dt_next_dev = &s->ctl->acc;
    if (dt_dev) *dt_dev = &s->ctl->dt;
    return HC_OK;
}

long hc_stepper_launches(hc_stepper* s) { return s ? s->launches : 0; }

int hc_stepper_layout(hc_stepper* s, int* my_pad, int* pitch, int* mz) {
    if (my_pad) *my_pad = s->sg.my_pad;
    if (pitch) *pitch = s->sg.pitch;
    if (mz) *mz = s->sg.mz;
    return HC_OK;
}

}  // extern "C"

// ============================================================================ patch set
// Device-resident PatchSet (transfer.hpp:47-73): px x py x pz patches of one global mesh, each
// an hc_stepper whose state stays in HBM, stepped together on one stream. exchange_ghosts
// (transfer.cpp:94-149: x, y, z sweeps over neighbour patches) is one gather kernel: composing
// the three sweeps, every ghost zone of every patch holds the global active zone at the
// composed mapped coordinates, which lives in a computable source patch. The global dt min of
// run_patch_step (transfer.cpp:184) is a device kernel over the patches' accumulators. The
// TransferLedger is pure accounting (transfer.cpp:160-175) and is reproduced on the host.

namespace hc {
namespace psk {  // (a named namespace: nvcc's stub generator trips over a second anonymous one)

struct PatchDev {
    double* buf[3];
    StepCtl* ctl;
};

struct PSGeom {
    int px, py, pz, lnx, lny, lnz, gnx, gny, gnz;
    int gh, mx, my, mz, my_pad, pitch, nbuf, bc;
};

__device__ __forceinline__ int map_global(int a, int n, int bc) {
    if (bc == HC_PERIODIC) return ((a % n) + n) % n;
    return a < 0 ? 0 : (a >= n ? n - 1 : a);
}

__global__ void k_patch_exchange(const PatchDev* __restrict__ pd, PSGeom g, int rel) {
    const size_t per = size_t(g.mx) * g.my * g.mz;
    const size_t np = size_t(g.px) * g.py * g.pz;
    size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (r >= per * np) return;
    const int p = int(r / per);
    size_t z = r % per;
    const int i = int(z % g.mx), j = int((z / g.mx) % g.my), k = int(z / (size_t(g.mx) * g.my));
    const bool act = i >= g.gh && i < g.gh + g.lnx && j >= g.gh && j < g.gh + g.lny &&
                     k >= g.gh && k < g.gh + g.lnz;
    if (act) return;
    const StepCtl* c = pd[p].ctl;
    if (c->done) return;
    const int pi = p % g.px, pj = (p / g.px) % g.py, pk = p / (g.px * g.py);
    const int gx = map_global(pi * g.lnx + i - g.gh, g.gnx, g.bc);
    const int gy = map_global(pj * g.lny + j - g.gh, g.gny, g.bc);
    const int gz = map_global(pk * g.lnz + k - g.gh, g.gnz, g.bc);
    const int s = ((gz / g.lnz) * g.py + gy / g.lny) * g.px + gx / g.lnx;
    const int is = g.gh + gx % g.lnx, js = g.gh + gy % g.lny, ks = g.gh + gz % g.lnz;
    const double* src = pd[s].buf[(pd[s].ctl->cur + rel) % g.nbuf] +
                        (size_t(ks) * g.my_pad + js) * g.pitch + size_t(is) * NV;
    double* dst = pd[p].buf[(c->cur + rel) % g.nbuf] + (size_t(k) * g.my_pad + j) * g.pitch +
                  size_t(i) * NV;
#pragma unroll
    for (int q = 0; q < NV; ++q) dst[q] = src[q];
}

// run_patch_step's global min (transfer.cpp:184): every patch's accumulator becomes the min
__global__ void k_patch_dt_min(const PatchDev* __restrict__ pd, int np) {
    double m = 1.0e32;
    for (int p = 0; p < np; ++p) m = smin(m, pd[p].ctl->acc);
    for (int p = 0; p < np; ++p) pd[p].ctl->acc = m;
}

}  // namespace psk
}  // namespace hc

using hc::psk::PatchDev;
using hc::psk::PSGeom;

struct hc_patchset {
    hc_geom global;
    hc_params p;
    int px, py, pz, bc, integrator;
    std::vector<hc_stepper*> patches;
    PatchDev* dev = nullptr;  // device table of the patches' buffers / control blocks
    PSGeom pg;
    cudaStream_t st = nullptr;
    int device = 0;
    long launches = 0;
    unsigned long long ledger[6] = {0, 0, 0, 0, 0, 0};  // TransferLedger field order
    long long accounted = 0;  // device steps already entered in the ledger
};

// TransferLedger (transfer.cpp:160-175): per patch per EXECUTED step, skinny strategy. The
// device turns steps after t_final or after a fault into no-ops, so the ledger follows the
// device step counter (read at sync), not the number of steps queued.
static void ps_account(hc_patchset* ps, long long steps_now) {
    const long long d = steps_now - ps->accounted;
    if (d <= 0) return;
    ps->accounted = steps_now;
    const unsigned long long np = ps->patches.size();
    const hc_stepper* s0 = ps->patches[0];
    const unsigned long long total = (unsigned long long)s0->sg.mx * s0->sg.my * s0->sg.mz * NV;
    const unsigned long long active =
        (unsigned long long)ps->pg.lnx * ps->pg.lny * ps->pg.lnz * NV;
    const unsigned long long n = (unsigned long long)d;
    ps->ledger[0] += total * np * n;   // uploads
    ps->ledger[1] += total * np * n;   // downloads
    ps->ledger[2] += np * n;           // scalar_uploads (dt)
    ps->ledger[3] += np * n;           // scalar_downloads (dt_next)
    ps->ledger[4] += active * np * n;  // uploads_active_only
    ps->ledger[5] += n;                // steps
}

static int ps_exchange(hc_patchset* ps, int rel) {
    const size_t n = size_t(ps->pg.mx) * ps->pg.my * ps->pg.mz * ps->patches.size();
    hc::psk::k_patch_exchange<<<unsigned((n + 255) / 256), 256, 0, ps->st>>>(ps->dev, ps->pg, rel);
    ps->launches++;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HC_OK : cuda_fail(e, "k_patch_exchange");
}

extern "C" {

int hc_patchset_create(const hc_geom* global, int px, int py, int pz, const hc_params* p,
                       int boundary, int exact, int device, int integrator, hc_patchset** out) {
    if (!global || !p || !out) {
        set_error(HC_INVALID, "null argument");
        return HC_INVALID;
    }
    if (px < 1 || py < 1 || pz < 1) {  // transfer.cpp:19-20
        set_error(HC_INVALID, "patch split counts must be positive");
        return HC_INVALID;
    }
    if (global->nx % px || global->ny % py || global->nz % pz) {  // transfer.cpp:21-22
        set_error(HC_INVALID, "patch split must divide the mesh evenly");
        return HC_INVALID;
    }
    if (boundary != HC_PERIODIC && boundary != HC_OUTFLOW) {
        set_error(HC_INVALID, "boundary kind must be periodic or outflow");
        return HC_INVALID;
    }
    hc_patchset* ps = new (std::nothrow) hc_patchset;
    if (!ps) {
        set_error(HC_CUDA, "out of host memory");
        return HC_CUDA;
    }
    ps->global = *global;
    ps->p = *p;
    ps->px = px;
    ps->py = py;
    ps->pz = pz;
    ps->bc = boundary;
    ps->integrator = integrator;
    ps->device = device;
    int rc = HC_OK;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ps->st, cudaStreamNonBlocking);
    if (e != cudaSuccess) rc = cuda_fail(e, "hc_patchset_create");
    const int lnx = global->nx / px, lny = global->ny / py, lnz = global->nz / pz;
    for (int pk = 0; pk < pz && !rc; ++pk)
        for (int pj = 0; pj < py && !rc; ++pj)
            for (int pi = 0; pi < px && !rc; ++pi) {  // transfer.cpp:33-47
                hc_geom g = *global;
                g.nx = lnx;
                g.ny = lny;
                g.nz = lnz;
                g.origin[0] = global->origin[0] + pi * lnx * global->dx;
                g.origin[1] = global->origin[1] + pj * lny * global->dy;
                g.origin[2] = global->origin[2] + pk * lnz * global->dz;
                // a single patch owns its boundaries (its ghost fill is exchange_ghosts for
                // one patch, and it can take the ring-free seam kernel); several
                // patches have every ghost filled by the exchange gather
                const int b = px * py * pz == 1 ? boundary : -1;
                hc_stepper_opts o = {{b, b, b}, exact, device, integrator};
                hc_stepper* s = nullptr;
                rc = hc_stepper_create(&g, p, &o, &s);
                if (!rc) {
                    ps->patches.push_back(s);
                    rc = hc_stepper_set_stream(s, ps->st);
                }
            }
    if (!rc) {
        const hc_stepper* s0 = ps->patches[0];
        ps->pg = PSGeom{px, py, pz, lnx, lny, lnz, global->nx, global->ny, global->nz,
                        s0->sg.gh, s0->sg.mx, s0->sg.my, s0->sg.mz, s0->sg.my_pad,
                        s0->sg.pitch, s0->nbuf, boundary};
        std::vector<PatchDev> table;
        for (hc_stepper* s : ps->patches)
            table.push_back(PatchDev{{s->buf[0], s->buf[1], s->buf[2]}, s->ctl});
        e = cudaMalloc(&ps->dev, sizeof(PatchDev) * table.size());
        if (e == cudaSuccess)
            e = cudaMemcpy(ps->dev, table.data(), sizeof(PatchDev) * table.size(),
                           cudaMemcpyHostToDevice);
        if (e != cudaSuccess) rc = cuda_fail(e, "hc_patchset_create");
    }
    if (rc) {
        hc_patchset_destroy(ps);
        return rc;
    }
    *out = ps;
    return HC_OK;
}

int hc_patchset_destroy(hc_patchset* ps) {
    if (!ps) return HC_OK;
    cudaSetDevice(ps->device);
    if (ps->st) cudaStreamSynchronize(ps->st);
    for (hc_stepper* s : ps->patches) hc_stepper_destroy(s);
    cudaFree(ps->dev);
    if (ps->st) cudaStreamDestroy(ps->st);
    delete ps;
    return HC_OK;
}

// scatter_to_patches / gather_from_patches (transfer.cpp:50-76): active zones of a global HOST
// SkinnyState <-> the patches' device states (strided 3D copies, ghosts filled on the device)
static int ps_copy(hc_patchset* ps, double* host, bool up) {
    const hc_geom& G = ps->global;
    const int gh = G.ghost;
    const size_t grow = size_t(G.nx + 2 * gh) * NV * sizeof(double);
    for (size_t idx = 0; idx < ps->patches.size(); ++idx) {
        hc_stepper* s = ps->patches[idx];
        int rc = refresh_cur(s);
        if (rc) return rc;
        const int pi = int(idx % ps->px), pj = int((idx / ps->px) % ps->py),
                  pk = int(idx / (size_t(ps->px) * ps->py));
        cudaMemcpy3DParms m = {};
        cudaPitchedPtr hp = make_cudaPitchedPtr(host, grow, grow, G.ny + 2 * gh);
        cudaPitchedPtr dp = make_cudaPitchedPtr(s->buf[s->cur], size_t(s->sg.pitch) * sizeof(double),
                                                size_t(s->sg.mx) * NV * sizeof(double), s->sg.my_pad);
        const cudaPos hpos = make_cudaPos(size_t(gh + pi * ps->pg.lnx) * NV * sizeof(double),
                                          gh + pj * ps->pg.lny, gh + pk * ps->pg.lnz);
        const cudaPos dpos = make_cudaPos(size_t(gh) * NV * sizeof(double), gh, gh);
        m.extent = make_cudaExtent(size_t(ps->pg.lnx) * NV * sizeof(double), ps->pg.lny, ps->pg.lnz);
        m.srcPtr = up ? hp : dp;
        m.dstPtr = up ? dp : hp;
        m.srcPos = up ? hpos : dpos;
        m.dstPos = up ? dpos : hpos;
        m.kind = up ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
        HC_CUDA(cudaMemcpy3DAsync(&m, ps->st));
    }
    HC_CUDA(cudaStreamSynchronize(ps->st));
    return HC_OK;
}

int hc_patchset_scatter(hc_patchset* ps, const double* global_skinny) {
    HC_CUDA(cudaSetDevice(ps->device));
    return ps_copy(ps, const_cast<double*>(global_skinny), true);
}

int hc_patchset_gather(hc_patchset* ps, double* global_skinny) {
    HC_CUDA(cudaSetDevice(ps->device));
    return ps_copy(ps, global_skinny, false);
}

int hc_patchset_patch_io(hc_patchset* ps, int idx, double* host_skinny, int upload) {
    if (!ps || idx < 0 || idx >= int(ps->patches.size()) || !host_skinny) {
        set_error(HC_INVALID, "hc_patchset_patch_io: bad patch index or buffer");
        return HC_INVALID;
    }
    HC_CUDA(cudaSetDevice(ps->device));
    return upload ? hc_stepper_upload(ps->patches[size_t(idx)], host_skinny)
                  : hc_stepper_download(ps->patches[size_t(idx)], host_skinny);
}

int hc_patchset_set_time(hc_patchset* ps, double t, double dt, double cfl, double t_final) {
    for (hc_stepper* s : ps->patches) {
        int rc = hc_stepper_set_time(s, t, dt, cfl, t_final);
        if (rc) return rc;
    }
    return HC_OK;
}

// run_patch_step (transfer.cpp:152-216) n times, all on the device: exchange_ghosts, every
// patch's fused step (each RK stage after its own exchange), the global dt min, the t/dt
// hand-off; the ledger counts what the reference's TransferLedger would.
int hc_patchset_step(hc_patchset* ps, int n) {
    HC_CUDA(cudaSetDevice(ps->device));
    const int ns = ps->integrator == 0 ? 1 : ps->integrator;
    const int np = int(ps->patches.size());
    for (int it = 0; it < n; ++it) {
        for (int k = 0; k < ns; ++k) {
            int rc = np == 1 ? hc_stepper_fill_ghosts(ps->patches[0])
                             : ps_exchange(ps, ps->integrator == 0 ? 0 : k);
            for (int p = 0; p < np && !rc; ++p) rc = hc_stepper_compute(ps->patches[p]);
            if (rc) return rc;
        }
        hc::psk::k_patch_dt_min<<<1, 1, 0, ps->st>>>(ps->dev, np);
        ps->launches++;
        HC_CUDA(cudaGetLastError());
        for (int p = 0; p < np; ++p) {
            int rc = hc_stepper_advance(ps->patches[p]);
            if (rc) return rc;
        }
    }
    return HC_OK;
}

int hc_patchset_sync(hc_patchset* ps, double* t, double* dt, long* steps_done) {
    int rc = HC_OK;
    long first = -1;
    for (hc_stepper* s : ps->patches) {
        long n = 0;
        int r = hc_stepper_sync(s, t, dt, &n);
        if (first < 0) first = n;
        if (r && !rc) rc = r;
    }
    if (steps_done) *steps_done = first;
    ps_account(ps, first);
    return rc;
}

int hc_patchset_ledger(hc_patchset* ps, unsigned long long* counts) {
    long n = 0;
    int rc = hc_stepper_sync(ps->patches[0], nullptr, nullptr, &n);
    if (rc && rc != HC_UNPHYSICAL) return rc;
    ps_account(ps, n);
    for (int i = 0; i < 6; ++i) counts[i] = ps->ledger[i];
    return HC_OK;
}

long hc_patchset_launches(hc_patchset* ps) {
    long l = ps->launches;
    for (hc_stepper* s : ps->patches) l += s->launches;
    return l;
}

}  // extern "C"
