// patch_kernels.cu -- the per-kernel path: one sm_100a kernel per reference patch kernel,
// operating on the reference's own layouts (fields.hpp:15-128), plus the host-buffer and
// device-buffer C-ABI entry points of include/hydro_cuda.h. Built with --fmad=false so every
// output is bit-identical to the reference (-ffp-contract=off). This path exists so the
// reference API can be swapped in function by function (the drop-in shim)
// and so each kernel is parity-checked in isolation; the throughput path is the fused
// stepper (fused_ader.cuh).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace hc {

namespace {

constexpr int TPB = 256;

struct G {  // device copy of the geometry
    int nx, ny, nz, gh, mx, my, mz;
};
G make_g(const hc_geom& g) { return G{g.nx, g.ny, g.nz, g.ghost, mx_of(g), my_of(g), mz_of(g)}; }

__device__ __forceinline__ size_t zoff(const G& g, int k, int j, int i) {
    return (size_t(k) * g.my + j) * g.mx + i;
}

inline unsigned blocks_for(size_t n) { return unsigned((n + TPB - 1) / TPB); }

// ---------------------------------------------------------------- fields.cpp:12-36
__global__ void k_skinny_to_modal(const double* __restrict__ s, double* __restrict__ m,
                                  size_t n, int modes) {
    size_t id = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (id < n) m[id * modes] = s[id];  // id = zone*5 + q; modal index (zone*5+q)*modes
}

__global__ void k_modal_to_skinny(const double* __restrict__ m, double* __restrict__ s, G g,
                                  int modes) {
    size_t id = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    size_t n = size_t(g.nx) * g.ny * g.nz;
    if (id >= n) return;
    int i = int(id % g.nx), j = int((id / g.nx) % g.ny), k = int(id / (size_t(g.nx) * g.ny));
    size_t z = zoff(g, k + g.gh, j + g.gh, i + g.gh);
#pragma unroll
    for (int q = 0; q < NV; ++q) s[z * NV + q] = m[(z * NV + q) * modes];
}

// ------------------------------------------------------------ boundary.cpp:7-58
__device__ __forceinline__ int map_index(int a, int n, int kind) {
    if (kind == 0) return ((a % n) + n) % n;
    return a < 0 ? 0 : (a >= n ? n - 1 : a);
}

// The reference fills x-ghosts (active y,z), then y-ghosts (full x), then z-ghosts (full
// x,y) in sequence (boundary.cpp:14-39). Composing the three passes, every ghost zone ends
// up holding the active zone at (map(i), map(j), map(k)) with map = identity on active
// indices, so one parallel gather produces the same bits with no ordering between threads.
__global__ void k_fill_ghosts(double* base, G g, int kind, int zstride, int qstride) {
    size_t id = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    size_t n = size_t(g.mx) * g.my * g.mz;
    if (id >= n) return;
    int i = int(id % g.mx), j = int((id / g.mx) % g.my), k = int(id / (size_t(g.mx) * g.my));
    bool ai = i >= g.gh && i < g.gh + g.nx, aj = j >= g.gh && j < g.gh + g.ny,
         ak = k >= g.gh && k < g.gh + g.nz;
    if (ai && aj && ak) return;
    int si = ai ? i : g.gh + map_index(i - g.gh, g.nx, kind);
    int sj = aj ? j : g.gh + map_index(j - g.gh, g.ny, kind);
    int sk = ak ? k : g.gh + map_index(k - g.gh, g.nz, kind);
    const double* src = base + zoff(g, sk, sj, si) * zstride;
    double* dst = base + id * zstride;
#pragma unroll
    for (int q = 0; q < NV; ++q) dst[q * qstride] = src[q * qstride];
}

// -------------------------------------------------------- reconstruct.cpp:7-76
__device__ __forceinline__ bool ring_index(size_t id, const G& g, int& i, int& j, int& k) {
    int rx = g.nx + 2, ry = g.ny + 2, rz = g.nz + 2;
    if (id >= size_t(rx) * ry * rz) return false;
    i = int(id % rx) + g.gh - 1;
    j = int((id / rx) % ry) + g.gh - 1;
    k = int(id / (size_t(rx) * ry)) + g.gh - 1;
    return true;
}

__global__ void k_limit_o2(double* m, G g, Limiter L) {
    int i, j, k;
    if (!ring_index(blockIdx.x * size_t(blockDim.x) + threadIdx.x, g, i, j, k)) return;
    const ptrdiff_t sx = NV * 5, sy = sx * g.mx, sz = sy * g.my;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        double cfac = q == 0 ? L.cfac_rho : L.cfac_other;
        double* zc = m + zoff(g, k, j, i) * NV * 5 + q * 5;
        double u0 = zc[0];
        zc[1] = mc_limiter(zc[sx] - u0, u0 - zc[-sx], cfac);
        zc[2] = mc_limiter(zc[sy] - u0, u0 - zc[-sy], cfac);
        zc[3] = mc_limiter(zc[sz] - u0, u0 - zc[-sz], cfac);
    }
}

__global__ void k_recon_o3(double* m, G g, Limiter L) {
    int i, j, k;
    if (!ring_index(blockIdx.x * size_t(blockDim.x) + threadIdx.x, g, i, j, k)) return;
    const ptrdiff_t sx = NV * 11, sy = sx * g.mx, sz = sy * g.my;
    double* z0 = m + zoff(g, k, j, i) * NV * 11;
    // all 13-point stencils of the 5 variables first (mode 0 is never written here), so the
    // loads are not serialised behind the mode stores of the same array
    double sv[NV][13];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        const double* zc = z0 + q * 11;
        sv[q][0] = zc[0];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const ptrdiff_t sd = d == 0 ? sx : (d == 1 ? sy : sz);
            sv[q][1 + 4 * d] = zc[-2 * sd];
            sv[q][2 + 4 * d] = zc[-sd];
            sv[q][3 + 4 * d] = zc[sd];
            sv[q][4 + 4 * d] = zc[2 * sd];
        }
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        double* zc = z0 + q * 11;
        const double* v = sv[q];
        double ux, uxx, uy, uyy, uz, uzz;
        Fault f;  // careful mode: IEEE division, nothing to report from a reconstruction
        f.clear();
        weno3(v[1], v[2], v[0], v[3], v[4], L, ux, uxx, f);
        weno3(v[5], v[6], v[0], v[7], v[8], L, uy, uyy, f);
        weno3(v[9], v[10], v[0], v[11], v[12], L, uz, uzz, f);
        zc[1] = ux;
        zc[2] = uy;
        zc[3] = uz;
        zc[4] = uxx;
        zc[5] = uyy;
        zc[6] = uzz;
    }
}

// cross modes on active zones (reconstruct.cpp:66-75); dead for the update
// (extrapolate_to_face reads modes 0, 1+a, 4+a only) but part of the API contract.
__global__ void k_recon_o3_cross(double* m, G g) {
    size_t id = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (id >= size_t(g.nx) * g.ny * g.nz) return;
    int i = int(id % g.nx) + g.gh, j = int((id / g.nx) % g.ny) + g.gh,
        k = int(id / (size_t(g.nx) * g.ny)) + g.gh;
    const ptrdiff_t sx = NV * 11, sy = sx * g.mx, sz = sy * g.my;
    double* z0 = m + zoff(g, k, j, i) * NV * 11;
    double c[NV][3];  // all loads (slopes, modes 1-3) before the stores (modes 7-9)
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        const double* zc = z0 + q * 11;
        c[q][0] = 0.25 * ((zc[sy + 1] - zc[-sy + 1]) + (zc[sx + 2] - zc[-sx + 2]));
        c[q][1] = 0.25 * ((zc[sz + 2] - zc[-sz + 2]) + (zc[sy + 3] - zc[-sy + 3]));
        c[q][2] = 0.25 * ((zc[sx + 3] - zc[-sx + 3]) + (zc[sz + 1] - zc[-sz + 1]));
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        double* zc = z0 + q * 11;
        zc[7] = c[q][0];
        zc[8] = c[q][1];
        zc[9] = c[q][2];
    }
}

// ------------------------------------------------------------ predictor.cpp:62-102
template <bool O3>
__global__ void k_predict(double* m, G g, double dt, double idx, double idy, double idz,
                          double gamma, ErrBlock* eb) {
    int i, j, k;
    if (!ring_index(blockIdx.x * size_t(blockDim.x) + threadIdx.x, g, i, j, k)) return;
    constexpr int M = O3 ? 11 : 5;
    double* zp = m + zoff(g, k, j, i) * NV * M;
    double face[6][NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        const double* v = zp + q * M;
        double q0 = O3 ? v[4] : 0.0, q1 = O3 ? v[5] : 0.0, q2 = O3 ? v[6] : 0.0;
        face[0][q] = extrap<O3>(v[0], +1.0, v[1], q0);
        face[1][q] = extrap<O3>(v[0], -1.0, v[1], q0);
        face[2][q] = extrap<O3>(v[0], +1.0, v[2], q1);
        face[3][q] = extrap<O3>(v[0], -1.0, v[2], q1);
        face[4][q] = extrap<O3>(v[0], +1.0, v[3], q2);
        face[5][q] = extrap<O3>(v[0], -1.0, v[3], q2);
    }
    Fault f;
    f.clear();
    double tau[NV];
    predictor<O3>(face, dt, idx, idy, idz, gamma, tau, f);
    if (f.code) {
        record_fault(eb, ST_PREDICT, f, i - g.gh, j - g.gh, k - g.gh, 0);
        return;  // the reference skips the scatter for a failed zone (predictor.cpp:85-87)
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) zp[q * M + M - 1] = tau[q];
}

__global__ void k_zero_tm(double* m, size_t nzones, int modes) {
    size_t id = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (id < nzones * NV) m[id * modes + modes - 1] = 0.0;
}

// ------------------------------------------------------------ corrector.cpp:15-70
template <int A, int SOLVER, bool O3>
__global__ void k_flux(const double* __restrict__ m, G g, double gamma, double* __restrict__ out,
                       ErrBlock* eb) {
    const int n2 = A == 1 ? g.nz : (A == 0 ? g.nz : g.ny);
    const int n1 = A == 0 ? g.ny : g.nx;
    const int nf = (A == 0 ? g.nx : (A == 1 ? g.ny : g.nz)) + 1;
    size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (t >= size_t(n2) * n1 * nf) return;
    // x and y sweeps: face index fastest; z sweep: the x index c1 fastest, so a warp reads
    // adjacent zone records instead of records a plane apart (747 -> 239 us at 128^3; the face
    // index is innermost in the OUTPUT layout only)
    int f, c1, c2;
    if (A != 2) {
        f = int(t % nf);
        c1 = int((t / nf) % n1);
        c2 = int(t / (size_t(nf) * n1));
    } else {
        c1 = int(t % n1);
        f = int((t / n1) % nf);
        c2 = int(t / (size_t(nf) * n1));
    }
    const size_t id = (size_t(c2) * n1 + c1) * nf + f;  // FaceFlux layout, fields.hpp:78
    constexpr int M = O3 ? 11 : 5;
    size_t zl, zr;
    const int gh = g.gh;
    if (A == 0) {
        zl = zoff(g, gh + c2, gh + c1, gh + f - 1);
        zr = zoff(g, gh + c2, gh + c1, gh + f);
    } else if (A == 1) {
        zl = zoff(g, gh + c2, gh + f - 1, gh + c1);
        zr = zoff(g, gh + c2, gh + f, gh + c1);
    } else {
        zl = zoff(g, gh + f - 1, gh + c2, gh + c1);
        zr = zoff(g, gh + f, gh + c2, gh + c1);
    }
    double ul[NV], ur[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        const double* lv = m + zl * NV * M + q * M;
        const double* rv = m + zr * NV * M + q * M;
        ul[q] = extrap<O3>(lv[0], +1.0, lv[1 + A], O3 ? lv[4 + A] : 0.0) + 0.5 * lv[M - 1];
        ur[q] = extrap<O3>(rv[0], -1.0, rv[1 + A], O3 ? rv[4 + A] : 0.0) + 0.5 * rv[M - 1];
    }
    Fault flt;
    flt.clear();
    double fl[NV];
    riemann<SOLVER, A>(ul, ur, gamma, fl, flt);
    if (flt.code) {
        record_fault(eb, ST_FLUX, flt, f, c1, c2, A);
        return;
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) out[id * NV + q] = fl[q];
}

__global__ void k_du_dt(const double* __restrict__ fx, const double* __restrict__ fy,
                        const double* __restrict__ fz, G g, double cx, double cy, double cz,
                        double* __restrict__ rate) {
    size_t id = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    const int nx = g.nx, ny = g.ny, nz = g.nz;
    if (id >= size_t(nx) * ny * nz) return;
    int i = int(id % nx), j = int((id / nx) % ny), k = int(id / (size_t(nx) * ny));
    const double* fxw = fx + ((size_t(k) * ny + j) * (nx + 1) + i) * NV;
    const double* fxe = fxw + NV;
    const double* fys = fy + ((size_t(k) * nx + i) * (ny + 1) + j) * NV;
    const double* fyn = fys + NV;
    const double* fzb = fz + ((size_t(j) * nx + i) * (nz + 1) + k) * NV;
    const double* fzt = fzb + NV;
#pragma unroll
    for (int q = 0; q < NV; ++q)
        rate[id * NV + q] =
            -cx * (fxe[q] - fxw[q]) - cy * (fyn[q] - fys[q]) - cz * (fzt[q] - fzb[q]);
}

__device__ __forceinline__ void block_min_to(double v, double* dst) {
    __shared__ double red[32];
    v = warp_min(v);
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        int nw = (blockDim.x + 31) >> 5;
        v = lane < nw ? red[lane] : 1.0e32;
        v = warp_min(v);
        if (lane == 0) atomic_min_pos(dst, v);
    }
}

__global__ void k_update(double* m, double* s, const double* __restrict__ rate, G g, int modes,
                         double cfl, double dx, double dy, double dz, double gamma,
                         double* dtn, ErrBlock* eb) {
    size_t id = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    double dt1 = 1.0e32;
    if (id < size_t(g.nx) * g.ny * g.nz) {
        int i = int(id % g.nx), j = int((id / g.nx) % g.ny), k = int(id / (size_t(g.nx) * g.ny));
        size_t z = zoff(g, k + g.gh, j + g.gh, i + g.gh);
        double u[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            double v = m[(z * NV + q) * modes] + rate[id * NV + q];
            m[(z * NV + q) * modes] = v;
            s[z * NV + q] = v;
            u[q] = v;
        }
        Fault f;
        f.clear();
        dt1 = eval_tstep(u, cfl, dx, dy, dz, gamma, f);
        if (f.code) {
            record_fault(eb, ST_UPDATE, f, i, j, k, 0);
            dt1 = 1.0e32;
        }
    }
    block_min_to(dt1, dtn);
}

__global__ void k_dt_next(const double* __restrict__ m, G g, int modes, double cfl, double dx,
                          double dy, double dz, double gamma, double* dtn, ErrBlock* eb) {
    size_t id = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    double dt1 = 1.0e32;
    if (id < size_t(g.nx) * g.ny * g.nz) {
        int i = int(id % g.nx), j = int((id / g.nx) % g.ny), k = int(id / (size_t(g.nx) * g.ny));
        size_t z = zoff(g, k + g.gh, j + g.gh, i + g.gh);
        double u[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) u[q] = m[(z * NV + q) * modes];
        Fault f;
        f.clear();
        dt1 = eval_tstep(u, cfl, dx, dy, dz, gamma, f);
        if (f.code) {
            record_fault(eb, ST_DT, f, i, j, k, 0);
            dt1 = 1.0e32;
        }
    }
    block_min_to(dt1, dtn);
}

// stepper.cpp:88-98 rk_save_u0 and :128-141 stage combination
__global__ void k_rk_save(const double* __restrict__ s, double* __restrict__ u0, G g) {
    size_t id = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (id >= size_t(g.nx) * g.ny * g.nz) return;
    int i = int(id % g.nx), j = int((id / g.nx) % g.ny), k = int(id / (size_t(g.nx) * g.ny));
    size_t z = zoff(g, k + g.gh, j + g.gh, i + g.gh);
#pragma unroll
    for (int q = 0; q < NV; ++q) u0[z * NV + q] = s[z * NV + q];
}

__global__ void k_rk_combine(double* m, double* s, const double* __restrict__ u0,
                             const double* __restrict__ rate, G g, int modes, double a,
                             double b) {
    size_t id = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (id >= size_t(g.nx) * g.ny * g.nz) return;
    int i = int(id % g.nx), j = int((id / g.nx) % g.ny), k = int(id / (size_t(g.nx) * g.ny));
    size_t z = zoff(g, k + g.gh, j + g.gh, i + g.gh);
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        double unew = a * u0[z * NV + q] + b * (m[(z * NV + q) * modes] + rate[id * NV + q]);
        m[(z * NV + q) * modes] = unew;
        s[z * NV + q] = unew;
    }
}

// ------------------------------------------------------------------ host plumbing

Limiter to_lim(const hc_limiter* l) {
    return Limiter{l->cfac_rho, l->cfac_other, l->weno_eps, l->weno_w[0], l->weno_w[1],
                   l->weno_w[2]};
}

size_t face_count(const hc_geom& g, int axis) {
    if (axis == 0) return size_t(g.nz) * g.ny * (g.nx + 1);
    if (axis == 1) return size_t(g.nz) * g.nx * (g.ny + 1);
    return size_t(g.ny) * g.nx * (g.nz + 1);
}
size_t active_zones(const hc_geom& g) { return size_t(g.nx) * g.ny * g.nz; }
size_t ring_zones(const hc_geom& g) { return size_t(g.nx + 2) * (g.ny + 2) * (g.nz + 2); }

// Per-thread device scratch for the host-buffer entry points (grow-only, keyed by role).
struct Workspace {
    std::map<std::string, std::pair<void*, size_t>> bufs;
    cudaStream_t stream = nullptr;
    ~Workspace() {
        for (auto& kv : bufs) cudaFree(kv.second.first);
        if (stream) cudaStreamDestroy(stream);
    }
    template <typename T>
    T* get(const char* name, size_t count, int* rc) {
        auto& e = bufs[name];
        size_t bytes = count * sizeof(T) + 16;
        if (e.second < bytes) {
            if (e.first) cudaFree(e.first);
            e.first = nullptr;
            e.second = 0;
            cudaError_t err = cudaMalloc(&e.first, bytes);
            if (err != cudaSuccess) {
                *rc = cuda_fail(err, name);
                return nullptr;
            }
            e.second = bytes;
        }
        return static_cast<T*>(e.first);
    }
};
thread_local Workspace* tl_ws = nullptr;
Workspace& ws() {
    if (!tl_ws) tl_ws = new Workspace();
    return *tl_ws;
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// ErrBlock lifecycle around an error-capable launch sequence
struct ErrScope {
    ErrBlock* d = nullptr;
    cudaStream_t st;
    int rc = HC_OK;
    explicit ErrScope(cudaStream_t s) : st(s) {
        d = ws().get<ErrBlock>("errblock", 1, &rc);
        if (d) {
            cudaError_t e = cudaMemsetAsync(d, 0, sizeof(ErrBlock), st);
            if (e != cudaSuccess) rc = cuda_fail(e, "cudaMemsetAsync(err)");
        }
    }
    int finish() {
        if (rc != HC_OK) return rc;
        ErrBlock h;
        cudaError_t e = cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return cuda_fail(e, "error readback");
        return report_device_errors(h);
    }
};

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HC_OK : cuda_fail(e, what);
}

// ---- device-level drivers (shared by host and device entry points)

int d_skinny_to_modal(const hc_geom& g, int modes, const double* s, double* m, cudaStream_t st) {
    size_t n = total_zones(g) * NV;
    k_skinny_to_modal<<<blocks_for(n), TPB, 0, st>>>(s, m, n, modes);
    return check_launch("k_skinny_to_modal");
}

int d_fill(const hc_geom& g, double* base, int kind, int zstride, int qstride, cudaStream_t st) {
    k_fill_ghosts<<<blocks_for(total_zones(g)), TPB, 0, st>>>(base, make_g(g), kind, zstride,
                                                             qstride);
    return check_launch("k_fill_ghosts");
}

int d_reconstruct(const hc_geom& g, int order, double* m, const Limiter& L, cudaStream_t st) {
    if (order == 2) {
        k_limit_o2<<<blocks_for(ring_zones(g)), TPB, 0, st>>>(m, make_g(g), L);
        return check_launch("k_limit_o2");
    }
    k_recon_o3<<<blocks_for(ring_zones(g)), TPB, 0, st>>>(m, make_g(g), L);
    int rc = check_launch("k_recon_o3");
    if (rc) return rc;
    k_recon_o3_cross<<<blocks_for(active_zones(g)), TPB, 0, st>>>(m, make_g(g));
    return check_launch("k_recon_o3_cross");
}

int d_predict(const hc_geom& g, int modes, double* m, double dt, double gamma, ErrBlock* eb,
              cudaStream_t st) {
    double idx = 1.0 / g.dx, idy = 1.0 / g.dy, idz = 1.0 / g.dz;
    if (modes == 5)
        k_predict<false><<<blocks_for(ring_zones(g)), TPB, 0, st>>>(m, make_g(g), dt, idx, idy,
                                                                    idz, gamma, eb);
    else
        k_predict<true><<<blocks_for(ring_zones(g)), TPB, 0, st>>>(m, make_g(g), dt, idx, idy,
                                                                   idz, gamma, eb);
    return check_launch("k_predict");
}

template <int A, int S, bool O3>
void launch_flux(const hc_geom& g, const double* m, double gamma, double* out, ErrBlock* eb,
                 cudaStream_t st) {
    k_flux<A, S, O3><<<blocks_for(face_count(g, A)), TPB, 0, st>>>(m, make_g(g), gamma, out, eb);
}

int d_flux(const hc_geom& g, int modes, const double* m, int axis, double gamma, int solver,
           double* out, ErrBlock* eb, cudaStream_t st) {
    bool o3 = modes == 11;
#define HC_FLUX_CASE(A, S, O)                                            \
    if (axis == A && solver == S && o3 == O) {                           \
        launch_flux<A, S, O>(g, m, gamma, out, eb, st);                  \
        return check_launch("k_flux");                                   \
    }
    HC_FLUX_CASE(0, 0, false) HC_FLUX_CASE(1, 0, false) HC_FLUX_CASE(2, 0, false)
    HC_FLUX_CASE(0, 1, false) HC_FLUX_CASE(1, 1, false) HC_FLUX_CASE(2, 1, false)
    HC_FLUX_CASE(0, 0, true) HC_FLUX_CASE(1, 0, true) HC_FLUX_CASE(2, 0, true)
    HC_FLUX_CASE(0, 1, true) HC_FLUX_CASE(1, 1, true) HC_FLUX_CASE(2, 1, true)
    HC_FLUX_CASE(0, 2, false) HC_FLUX_CASE(1, 2, false) HC_FLUX_CASE(2, 2, false)
    HC_FLUX_CASE(0, 2, true) HC_FLUX_CASE(1, 2, true) HC_FLUX_CASE(2, 2, true)
    HC_FLUX_CASE(0, 3, false) HC_FLUX_CASE(1, 3, false) HC_FLUX_CASE(2, 3, false)
    HC_FLUX_CASE(0, 3, true) HC_FLUX_CASE(1, 3, true) HC_FLUX_CASE(2, 3, true)
#undef HC_FLUX_CASE
    set_error(HC_INVALID, "bad axis/solver/modes");
    return HC_INVALID;
}

int d_du_dt(const hc_geom& g, const double* fx, const double* fy, const double* fz, double dt,
            double* rate, cudaStream_t st) {
    double cx = dt / g.dx, cy = dt / g.dy, cz = dt / g.dz;  // corrector.cpp:75
    k_du_dt<<<blocks_for(active_zones(g)), TPB, 0, st>>>(fx, fy, fz, make_g(g), cx, cy, cz, rate);
    return check_launch("k_du_dt");
}

int seed_min(double* d, cudaStream_t st) {
    static const double seed = 1.0e32;  // corrector.cpp:98
    HC_CUDA(cudaMemcpyAsync(d, &seed, sizeof seed, cudaMemcpyHostToDevice, st));
    return HC_OK;
}

int d_update(const hc_geom& g, int modes, double* m, double* s, const double* rate, double cfl,
             double gamma, double* dtn, ErrBlock* eb, cudaStream_t st) {
    int rc = seed_min(dtn, st);
    if (rc) return rc;
    k_update<<<blocks_for(active_zones(g)), TPB, 0, st>>>(m, s, rate, make_g(g), modes, cfl, g.dx,
                                                        g.dy, g.dz, gamma, dtn, eb);
    return check_launch("k_update");
}

int d_dt_next(const hc_geom& g, int modes, const double* m, double cfl, double gamma,
              double* dtn, ErrBlock* eb, cudaStream_t st) {
    int rc = seed_min(dtn, st);
    if (rc) return rc;
    k_dt_next<<<blocks_for(active_zones(g)), TPB, 0, st>>>(m, make_g(g), modes, cfl, g.dx, g.dy,
                                                         g.dz, gamma, dtn, eb);
    return check_launch("k_dt_next");
}

int modes_ok(int modes) {
    if (modes == 5 || modes == 11) return HC_OK;
    set_error(HC_INVALID, "modes must be 5 or 11");
    return HC_INVALID;
}

// host <-> device helpers for the host-buffer API
int h2d(void* d, const void* h, size_t bytes, cudaStream_t st) {
    HC_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
    return HC_OK;
}
int d2h(void* h, const void* d, size_t bytes, cudaStream_t st) {
    HC_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st));
    return HC_OK;
}
int sync(cudaStream_t st) {
    HC_CUDA(cudaStreamSynchronize(st));
    return HC_OK;
}
cudaStream_t host_stream(int* rc) {
    Workspace& w = ws();
    if (!w.stream) {
        cudaError_t e = cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) *rc = cuda_fail(e, "cudaStreamCreate");
    }
    return w.stream;
}

#define TRY(x)                 \
    do {                       \
        int rc_ = (x);         \
        if (rc_) return rc_;   \
    } while (0)

// Device buffers sized for one patch, shared by the host-buffer pipeline entry points.
struct PatchBufs {
    double *modal, *skinny, *fx, *fy, *fz, *rate, *u0, *dtn;
};
int patch_bufs(const hc_geom& g, int modes, PatchBufs& b) {
    int rc = HC_OK;
    Workspace& w = ws();
    b.modal = w.get<double>("modal", total_zones(g) * NV * modes, &rc);
    b.skinny = w.get<double>("skinny", total_zones(g) * NV, &rc);
    b.fx = w.get<double>("fx", face_count(g, 0) * NV, &rc);
    b.fy = w.get<double>("fy", face_count(g, 1) * NV, &rc);
    b.fz = w.get<double>("fz", face_count(g, 2) * NV, &rc);
    b.rate = w.get<double>("rate", active_zones(g) * NV, &rc);
    b.u0 = w.get<double>("u0", total_zones(g) * NV, &rc);
    b.dtn = w.get<double>("dtn", 1, &rc);
    return rc;
}

}  // namespace
}  // namespace hc

using namespace hc;

// ====================================================================== C ABI

#define GEOM_OR_FAIL(g, order)            \
    do {                                  \
        int rc_ = validate_geom(g, order); \
        if (rc_) return rc_;              \
    } while (0)

extern "C" {

int hc_skinny_to_modal(const hc_geom* g, int modes, const double* skinny, double* modal) {
    GEOM_OR_FAIL(g, 0);
    TRY(modes_ok(modes));
    int rc = HC_OK;
    cudaStream_t st = host_stream(&rc);
    TRY(rc);
    PatchBufs b;
    TRY(patch_bufs(*g, modes, b));
    size_t nm = total_zones(*g) * NV * modes, ns = total_zones(*g) * NV;
    TRY(h2d(b.modal, modal, nm * 8, st));
    TRY(h2d(b.skinny, skinny, ns * 8, st));
    TRY(d_skinny_to_modal(*g, modes, b.skinny, b.modal, st));
    TRY(d2h(modal, b.modal, nm * 8, st));
    return sync(st);
}

int hc_modal_to_skinny(const hc_geom* g, int modes, const double* modal, double* skinny) {
    GEOM_OR_FAIL(g, 0);
    TRY(modes_ok(modes));
    int rc = HC_OK;
    cudaStream_t st = host_stream(&rc);
    TRY(rc);
    PatchBufs b;
    TRY(patch_bufs(*g, modes, b));
    size_t nm = total_zones(*g) * NV * modes, ns = total_zones(*g) * NV;
    TRY(h2d(b.modal, modal, nm * 8, st));
    TRY(h2d(b.skinny, skinny, ns * 8, st));
    k_modal_to_skinny<<<blocks_for(active_zones(*g)), TPB, 0, st>>>(b.modal, b.skinny,
                                                                    make_g(*g), modes);
    TRY(check_launch("k_modal_to_skinny"));
    TRY(d2h(skinny, b.skinny, ns * 8, st));
    return sync(st);
}

int hc_apply_boundary_skinny(const hc_geom* g, int kind, double* skinny) {
    GEOM_OR_FAIL(g, 0);
    int rc = HC_OK;
    cudaStream_t st = host_stream(&rc);
    TRY(rc);
    PatchBufs b;
    TRY(patch_bufs(*g, 5, b));
    size_t ns = total_zones(*g) * NV;
    TRY(h2d(b.skinny, skinny, ns * 8, st));
    TRY(d_fill(*g, b.skinny, kind, NV, 1, st));
    TRY(d2h(skinny, b.skinny, ns * 8, st));
    return sync(st);
}

int hc_apply_boundary_modal(const hc_geom* g, int modes, int kind, double* modal) {
    GEOM_OR_FAIL(g, 0);
    TRY(modes_ok(modes));
    int rc = HC_OK;
    cudaStream_t st = host_stream(&rc);
    TRY(rc);
    PatchBufs b;
    TRY(patch_bufs(*g, modes, b));
    size_t nm = total_zones(*g) * NV * modes;
    TRY(h2d(b.modal, modal, nm * 8, st));
    TRY(d_fill(*g, b.modal, kind, NV * modes, modes, st));
    TRY(d2h(modal, b.modal, nm * 8, st));
    return sync(st);
}

static int host_reconstruct(const hc_geom* g, int order, double* modal, const hc_limiter* lim) {
    GEOM_OR_FAIL(g, order);
    int modes = order == 2 ? 5 : 11;
    int rc = HC_OK;
    cudaStream_t st = host_stream(&rc);
    TRY(rc);
    PatchBufs b;
    TRY(patch_bufs(*g, modes, b));
    size_t nm = total_zones(*g) * NV * modes;
    TRY(h2d(b.modal, modal, nm * 8, st));
    TRY(d_reconstruct(*g, order, b.modal, to_lim(lim), st));
    TRY(d2h(modal, b.modal, nm * 8, st));
    return sync(st);
}
int hc_limit_patch_o2(const hc_geom* g, double* modal, const hc_limiter* lim) {
    return host_reconstruct(g, 2, modal, lim);
}
int hc_reconstruct_patch_o3(const hc_geom* g, double* modal, const hc_limiter* lim) {
    return host_reconstruct(g, 3, modal, lim);
}

int hc_predict_patch(const hc_geom* g, int modes, double* modal, double dt, double gamma) {
    GEOM_OR_FAIL(g, 0);
    TRY(modes_ok(modes));
    int rc = HC_OK;
    cudaStream_t st = host_stream(&rc);
    TRY(rc);
    PatchBufs b;
    TRY(patch_bufs(*g, modes, b));
    size_t nm = total_zones(*g) * NV * modes;
    TRY(h2d(b.modal, modal, nm * 8, st));
    ErrScope es(st);
    TRY(es.rc);
    TRY(d_predict(*g, modes, b.modal, dt, gamma, es.d, st));
    TRY(d2h(modal, b.modal, nm * 8, st));
    return es.finish();
}

int hc_zero_temporal_mode(const hc_geom* g, int modes, double* modal) {
    GEOM_OR_FAIL(g, 0);
    TRY(modes_ok(modes));
    int rc = HC_OK;
    cudaStream_t st = host_stream(&rc);
    TRY(rc);
    PatchBufs b;
    TRY(patch_bufs(*g, modes, b));
    size_t nm = total_zones(*g) * NV * modes;
    TRY(h2d(b.modal, modal, nm * 8, st));
    k_zero_tm<<<blocks_for(total_zones(*g) * NV), TPB, 0, st>>>(b.modal, total_zones(*g), modes);
    TRY(check_launch("k_zero_tm"));
    TRY(d2h(modal, b.modal, nm * 8, st));
    return sync(st);
}

int hc_make_flux_axis(const hc_geom* g, int modes, const double* modal, int axis, double gamma,
                      int solver, double* out) {
    GEOM_OR_FAIL(g, 0);
    TRY(modes_ok(modes));
    if (axis < 0 || axis > 2) {
        set_error(HC_INVALID, "axis must be 0, 1 or 2");
        return HC_INVALID;
    }
    int rc = HC_OK;
    cudaStream_t st = host_stream(&rc);
    TRY(rc);
    PatchBufs b;
    TRY(patch_bufs(*g, modes, b));
    double* f = axis == 0 ? b.fx : (axis == 1 ? b.fy : b.fz);
    size_t nm = total_zones(*g) * NV * modes, nf = face_count(*g, axis) * NV;
    TRY(h2d(b.modal, modal, nm * 8, st));
    TRY(h2d(f, out, nf * 8, st));  // failed faces keep the caller's values, as the reference
    ErrScope es(st);
    TRY(es.rc);
    TRY(d_flux(*g, modes, b.modal, axis, gamma, solver, f, es.d, st));
    TRY(d2h(out, f, nf * 8, st));
    return es.finish();
}

int hc_make_du_dt(const hc_geom* g, const double* fx, const double* fy, const double* fz,
                  double dt, double* rate) {
    GEOM_OR_FAIL(g, 0);
    int rc = HC_OK;
    cudaStream_t st = host_stream(&rc);
    TRY(rc);
    PatchBufs b;
    TRY(patch_bufs(*g, 5, b));
    TRY(h2d(b.fx, fx, face_count(*g, 0) * NV * 8, st));
    TRY(h2d(b.fy, fy, face_count(*g, 1) * NV * 8, st));
    TRY(h2d(b.fz, fz, face_count(*g, 2) * NV * 8, st));
    TRY(d_du_dt(*g, b.fx, b.fy, b.fz, dt, b.rate, st));
    TRY(d2h(rate, b.rate, active_zones(*g) * NV * 8, st));
    return sync(st);
}

int hc_update_u_timestep(const hc_geom* g, int modes, double* modal, double* skinny,
                         const double* rate, double cfl, double gamma, double* dt_next) {
    GEOM_OR_FAIL(g, 0);
    TRY(modes_ok(modes));
    int rc = HC_OK;
    cudaStream_t st = host_stream(&rc);
    TRY(rc);
    PatchBufs b;
    TRY(patch_bufs(*g, modes, b));
    size_t nm = total_zones(*g) * NV * modes, ns = total_zones(*g) * NV;
    TRY(h2d(b.modal, modal, nm * 8, st));
    TRY(h2d(b.skinny, skinny, ns * 8, st));
    TRY(h2d(b.rate, rate, active_zones(*g) * NV * 8, st));
    ErrScope es(st);
    TRY(es.rc);
    TRY(d_update(*g, modes, b.modal, b.skinny, b.rate, cfl, gamma, b.dtn, es.d, st));
    TRY(d2h(modal, b.modal, nm * 8, st));
    TRY(d2h(skinny, b.skinny, ns * 8, st));
    TRY(d2h(dt_next, b.dtn, 8, st));
    return es.finish();
}

int hc_compute_dt_next(const hc_geom* g, int modes, const double* modal, double gamma,
                       double cfl, double* dt_next) {
    GEOM_OR_FAIL(g, 0);
    TRY(modes_ok(modes));
    int rc = HC_OK;
    cudaStream_t st = host_stream(&rc);
    TRY(rc);
    PatchBufs b;
    TRY(patch_bufs(*g, modes, b));
    TRY(h2d(b.modal, modal, total_zones(*g) * NV * modes * 8, st));
    ErrScope es(st);
    TRY(es.rc);
    TRY(d_dt_next(*g, modes, b.modal, cfl, gamma, b.dtn, es.d, st));
    TRY(d2h(dt_next, b.dtn, 8, st));
    return es.finish();
}

// stepper.cpp:49-78, every intermediate materialised as in the reference
// CUDA events bracketing the stages of one host-buffer pipeline call, reported in the
// order of StageProfile (stepper.hpp:15-37): reconstruct, predict, flux, rate, update,
// transfer (host<->device staging and skinny_to_modal).
struct StageEvents {
    cudaEvent_t e[8];
    bool ok = false;
    StageEvents() {
        ok = true;
        for (auto& x : e) ok = ok && cudaEventCreate(&x) == cudaSuccess;
    }
    ~StageEvents() {
        for (auto& x : e) cudaEventDestroy(x);
    }
    void mark(int i, cudaStream_t st) { cudaEventRecord(e[i], st); }
    float ms(int a, int b) {
        float v = 0.f;
        cudaEventElapsedTime(&v, e[a], e[b]);
        return v;
    }
};

int hc_ader_step_timed(const hc_geom* g, const hc_params* p, double* modal, double* skinny,
                       double* fx, double* fy, double* fz, double* rate, double dt, double cfl,
                       double* dt_next, double* stage_seconds) {
    GEOM_OR_FAIL(g, p->order);
    int modes = p->order == 2 ? 5 : 11;
    int rc = HC_OK;
    cudaStream_t st = host_stream(&rc);
    TRY(rc);
    PatchBufs b;
    TRY(patch_bufs(*g, modes, b));
    StageEvents ev;
    size_t nm = total_zones(*g) * NV * modes, ns = total_zones(*g) * NV;
    ev.mark(0, st);
    TRY(h2d(b.modal, modal, nm * 8, st));
    TRY(h2d(b.skinny, skinny, ns * 8, st));
    TRY(h2d(b.fx, fx, face_count(*g, 0) * NV * 8, st));
    TRY(h2d(b.fy, fy, face_count(*g, 1) * NV * 8, st));
    TRY(h2d(b.fz, fz, face_count(*g, 2) * NV * 8, st));
    ErrScope es(st);
    TRY(es.rc);
    TRY(d_skinny_to_modal(*g, modes, b.skinny, b.modal, st));
    ev.mark(1, st);
    TRY(d_reconstruct(*g, p->order, b.modal, to_lim(&p->lim), st));
    ev.mark(2, st);
    TRY(d_predict(*g, modes, b.modal, dt, p->gamma, es.d, st));
    ev.mark(3, st);
    // the reference throws out of predict_patch before touching the fluxes
    rc = es.finish();
    if (rc) {
        d2h(modal, b.modal, nm * 8, st);
        sync(st);
        return rc;
    }
    TRY(d_flux(*g, modes, b.modal, 0, p->gamma, p->solver, b.fx, es.d, st));
    TRY(d_flux(*g, modes, b.modal, 1, p->gamma, p->solver, b.fy, es.d, st));
    TRY(d_flux(*g, modes, b.modal, 2, p->gamma, p->solver, b.fz, es.d, st));
    ev.mark(4, st);
    TRY(d_du_dt(*g, b.fx, b.fy, b.fz, dt, b.rate, st));
    ev.mark(5, st);
    TRY(d_update(*g, modes, b.modal, b.skinny, b.rate, cfl, p->gamma, b.dtn, es.d, st));
    ev.mark(6, st);
    TRY(d2h(modal, b.modal, nm * 8, st));
    TRY(d2h(skinny, b.skinny, ns * 8, st));
    TRY(d2h(fx, b.fx, face_count(*g, 0) * NV * 8, st));
    TRY(d2h(fy, b.fy, face_count(*g, 1) * NV * 8, st));
    TRY(d2h(fz, b.fz, face_count(*g, 2) * NV * 8, st));
    TRY(d2h(rate, b.rate, active_zones(*g) * NV * 8, st));
    TRY(d2h(dt_next, b.dtn, 8, st));
    ev.mark(7, st);
    rc = es.finish();
    if (stage_seconds && ev.ok) {
        stage_seconds[0] = ev.ms(1, 2) * 1e-3;
        stage_seconds[1] = ev.ms(2, 3) * 1e-3;
        stage_seconds[2] = ev.ms(3, 4) * 1e-3;
        stage_seconds[3] = ev.ms(4, 5) * 1e-3;
        stage_seconds[4] = ev.ms(5, 6) * 1e-3;
        stage_seconds[5] = (ev.ms(0, 1) + ev.ms(6, 7)) * 1e-3;
    }
    return rc;
}

int hc_ader_step(const hc_geom* g, const hc_params* p, double* modal, double* skinny,
                 double* fx, double* fy, double* fz, double* rate, double dt, double cfl,
                 double* dt_next) {
    return hc_ader_step_timed(g, p, modal, skinny, fx, fy, fz, rate, dt, cfl, dt_next,
                              nullptr);
}

// predictor.cpp:26-60 on one zone (the reference tests call predictor_ptwise directly)
int hc_predictor_ptwise(double* zone_v, int modes, double dt, double dx, double dy, double dz,
                        double gamma) {
    TRY(modes_ok(modes));
    int rc = HC_OK;
    cudaStream_t st = host_stream(&rc);
    TRY(rc);
    double* d = ws().get<double>("zone", NV * 11, &rc);
    TRY(rc);
    ErrScope es(st);
    TRY(es.rc);
    TRY(h2d(d, zone_v, NV * modes * 8, st));
    // a 1x1x1 "patch" whose single ring zone is the zone itself
    hc_geom one{};
    one.nx = one.ny = one.nz = -1;  // ring box (n+2)^3 = 1 zone at storage (0,0,0)
    one.ghost = 1;
    G gg{-1, -1, -1, 1, 1, 1, 1};
    double idx = 1.0 / dx, idy = 1.0 / dy, idz = 1.0 / dz;
    if (modes == 5)
        k_predict<false><<<1, 32, 0, st>>>(d, gg, dt, idx, idy, idz, gamma, es.d);
    else
        k_predict<true><<<1, 32, 0, st>>>(d, gg, dt, idx, idy, idz, gamma, es.d);
    TRY(check_launch("k_predict(zone)"));
    TRY(d2h(zone_v, d, NV * modes * 8, st));
    (void)one;
    rc = es.finish();
    if (rc == HC_UNPHYSICAL) {  // predictor_ptwise throws without zone context
        char buf[512];
        hc_last_error(buf, sizeof buf);
        const char* m = strstr(buf, "): ");
        set_error(rc, m ? m + 3 : buf);
    }
    return rc;
}

int hc_rk_save_u0(const hc_geom* g, const double* skinny, double* stage_u0) {
    GEOM_OR_FAIL(g, 0);
    int rc = HC_OK;
    cudaStream_t st = host_stream(&rc);
    TRY(rc);
    PatchBufs b;
    TRY(patch_bufs(*g, 5, b));
    size_t ns = total_zones(*g) * NV;
    TRY(h2d(b.skinny, skinny, ns * 8, st));
    TRY(h2d(b.u0, stage_u0, ns * 8, st));
    k_rk_save<<<blocks_for(active_zones(*g)), TPB, 0, st>>>(b.skinny, b.u0, make_g(*g));
    TRY(check_launch("k_rk_save"));
    TRY(d2h(stage_u0, b.u0, ns * 8, st));
    return sync(st);
}

// stepper.cpp:100-143 on device buffers already uploaded
static int d_rk_stage(const hc_geom& g, const hc_params& p, PatchBufs& b, double dt, double a,
                      double bb, ErrBlock* eb, cudaStream_t st, StageEvents* ev = nullptr) {
    int modes = p.order == 2 ? 5 : 11;
    TRY(d_skinny_to_modal(g, modes, b.skinny, b.modal, st));
    if (ev) ev->mark(1, st);
    TRY(d_reconstruct(g, p.order, b.modal, to_lim(&p.lim), st));
    if (ev) ev->mark(2, st);
    k_zero_tm<<<blocks_for(total_zones(g) * NV), TPB, 0, st>>>(b.modal, total_zones(g), modes);
    TRY(check_launch("k_zero_tm"));
    if (ev) ev->mark(3, st);
    TRY(d_flux(g, modes, b.modal, 0, p.gamma, p.solver, b.fx, eb, st));
    TRY(d_flux(g, modes, b.modal, 1, p.gamma, p.solver, b.fy, eb, st));
    TRY(d_flux(g, modes, b.modal, 2, p.gamma, p.solver, b.fz, eb, st));
    if (ev) ev->mark(4, st);
    TRY(d_du_dt(g, b.fx, b.fy, b.fz, dt, b.rate, st));
    if (ev) ev->mark(5, st);
    k_rk_combine<<<blocks_for(active_zones(g)), TPB, 0, st>>>(b.modal, b.skinny, b.u0, b.rate,
                                                            make_g(g), modes, a, bb);
    if (ev) ev->mark(6, st);
    return check_launch("k_rk_combine");
}

static int upload_all(const hc_geom& g, int modes, PatchBufs& b, const double* modal,
                      const double* skinny, const double* fx, const double* fy,
                      const double* fz, const double* rate, const double* u0, cudaStream_t st) {
    TRY(h2d(b.modal, modal, total_zones(g) * NV * modes * 8, st));
    TRY(h2d(b.skinny, skinny, total_zones(g) * NV * 8, st));
    TRY(h2d(b.fx, fx, face_count(g, 0) * NV * 8, st));
    TRY(h2d(b.fy, fy, face_count(g, 1) * NV * 8, st));
    TRY(h2d(b.fz, fz, face_count(g, 2) * NV * 8, st));
    TRY(h2d(b.rate, rate, active_zones(g) * NV * 8, st));
    if (u0) TRY(h2d(b.u0, u0, total_zones(g) * NV * 8, st));
    return HC_OK;
}
static int download_all(const hc_geom& g, int modes, PatchBufs& b, double* modal,
                        double* skinny, double* fx, double* fy, double* fz, double* rate,
                        double* u0, cudaStream_t st) {
    TRY(d2h(modal, b.modal, total_zones(g) * NV * modes * 8, st));
    TRY(d2h(skinny, b.skinny, total_zones(g) * NV * 8, st));
    TRY(d2h(fx, b.fx, face_count(g, 0) * NV * 8, st));
    TRY(d2h(fy, b.fy, face_count(g, 1) * NV * 8, st));
    TRY(d2h(fz, b.fz, face_count(g, 2) * NV * 8, st));
    TRY(d2h(rate, b.rate, active_zones(g) * NV * 8, st));
    if (u0) TRY(d2h(u0, b.u0, total_zones(g) * NV * 8, st));
    return HC_OK;
}

int hc_rk_stage_timed(const hc_geom* g, const hc_params* p, double* modal, double* skinny,
                      double* fx, double* fy, double* fz, double* rate, const double* stage_u0,
                      double dt, double a, double b_, double* stage_seconds) {
    GEOM_OR_FAIL(g, p->order);
    int modes = p->order == 2 ? 5 : 11;
    int rc = HC_OK;
    cudaStream_t st = host_stream(&rc);
    TRY(rc);
    PatchBufs b;
    TRY(patch_bufs(*g, modes, b));
    StageEvents ev;
    ev.mark(0, st);
    TRY(upload_all(*g, modes, b, modal, skinny, fx, fy, fz, rate, stage_u0, st));
    ErrScope es(st);
    TRY(es.rc);
    TRY(d_rk_stage(*g, *p, b, dt, a, b_, es.d, st, &ev));
    TRY(download_all(*g, modes, b, modal, skinny, fx, fy, fz, rate, nullptr, st));
    ev.mark(7, st);
    rc = es.finish();
    if (stage_seconds && ev.ok) {  // rk_stage's StageTimer slots, stepper.cpp:100-143
        stage_seconds[0] = ev.ms(1, 2) * 1e-3;
        stage_seconds[1] = ev.ms(2, 3) * 1e-3;
        stage_seconds[2] = ev.ms(3, 4) * 1e-3;
        stage_seconds[3] = ev.ms(4, 5) * 1e-3;
        stage_seconds[4] = ev.ms(5, 6) * 1e-3;
        stage_seconds[5] = (ev.ms(0, 1) + ev.ms(6, 7)) * 1e-3;
    }
    return rc;
}

int hc_rk_stage(const hc_geom* g, const hc_params* p, double* modal, double* skinny,
                double* fx, double* fy, double* fz, double* rate, const double* stage_u0,
                double dt, double a, double b_) {
    return hc_rk_stage_timed(g, p, modal, skinny, fx, fy, fz, rate, stage_u0, dt, a, b_,
                             nullptr);
}

int hc_rk_step(const hc_geom* g, const hc_params* p, int nstages, double* modal,
               double* skinny, double* fx, double* fy, double* fz, double* rate,
               double* stage_u0, int bc, double dt, double cfl, double* dt_next) {
    GEOM_OR_FAIL(g, p->order);
    static const double heun[2][2] = {{0.0, 1.0}, {0.5, 0.5}};  // stepper.cpp:81-82
    static const double ssp3[3][2] = {{0.0, 1.0}, {0.75, 0.25}, {1.0 / 3.0, 2.0 / 3.0}};
    if (nstages != 2 && nstages != 3) {
        set_error(HC_INVALID, "rk_stages called for a non-RK integrator");
        return HC_INVALID;
    }
    int modes = p->order == 2 ? 5 : 11;
    int rc = HC_OK;
    cudaStream_t st = host_stream(&rc);
    TRY(rc);
    PatchBufs b;
    TRY(patch_bufs(*g, modes, b));
    TRY(upload_all(*g, modes, b, modal, skinny, fx, fy, fz, rate, stage_u0, st));
    ErrScope es(st);
    TRY(es.rc);
    k_rk_save<<<blocks_for(active_zones(*g)), TPB, 0, st>>>(b.skinny, b.u0, make_g(*g));
    TRY(check_launch("k_rk_save"));
    for (int s = 0; s < nstages; ++s) {
        const double* ab = nstages == 2 ? heun[s] : ssp3[s];
        TRY(d_fill(*g, b.skinny, bc, NV, 1, st));
        TRY(d_rk_stage(*g, *p, b, dt, ab[0], ab[1], es.d, st));
    }
    TRY(d_dt_next(*g, modes, b.modal, cfl, p->gamma, b.dtn, es.d, st));
    TRY(download_all(*g, modes, b, modal, skinny, fx, fy, fz, rate, stage_u0, st));
    TRY(d2h(dt_next, b.dtn, 8, st));
    return es.finish();
}

int hc_initial_dt(const hc_geom* g, const double* skinny, double gamma, double cfl,
                  double* dt) {
    GEOM_OR_FAIL(g, 0);
    int rc = HC_OK;
    cudaStream_t st = host_stream(&rc);
    TRY(rc);
    PatchBufs b;
    TRY(patch_bufs(*g, 5, b));
    TRY(h2d(b.skinny, skinny, total_zones(*g) * NV * 8, st));
    ErrScope es(st);
    TRY(es.rc);
    // the skinny layout is the modal layout with one mode
    TRY(d_dt_next(*g, 1, b.skinny, cfl, gamma, b.dtn, es.d, st));
    TRY(d2h(dt, b.dtn, 8, st));
    return es.finish();
}

// ---- device-buffer entry points

int hc_dev_skinny_to_modal(const hc_geom* g, int modes, const double* skinny, double* modal,
                           void* stream) {
    GEOM_OR_FAIL(g, 0);
    TRY(modes_ok(modes));
    return d_skinny_to_modal(*g, modes, skinny, modal, as_stream(stream));
}
int hc_dev_apply_boundary_skinny(const hc_geom* g, int kind, double* skinny, void* stream) {
    GEOM_OR_FAIL(g, 0);
    return d_fill(*g, skinny, kind, NV, 1, as_stream(stream));
}
int hc_dev_reconstruct(const hc_geom* g, int order, double* modal, const hc_limiter* lim,
                       void* stream) {
    GEOM_OR_FAIL(g, order);
    return d_reconstruct(*g, order, modal, to_lim(lim), as_stream(stream));
}
int hc_dev_predict_patch(const hc_geom* g, int modes, double* modal, double dt, double gamma,
                         void* stream) {
    GEOM_OR_FAIL(g, 0);
    TRY(modes_ok(modes));
    cudaStream_t st = as_stream(stream);
    ErrScope es(st);
    TRY(es.rc);
    TRY(d_predict(*g, modes, modal, dt, gamma, es.d, st));
    return es.finish();
}
int hc_dev_make_flux_axis(const hc_geom* g, int modes, const double* modal, int axis,
                          double gamma, int solver, double* out, void* stream) {
    GEOM_OR_FAIL(g, 0);
    TRY(modes_ok(modes));
    cudaStream_t st = as_stream(stream);
    ErrScope es(st);
    TRY(es.rc);
    TRY(d_flux(*g, modes, modal, axis, gamma, solver, out, es.d, st));
    return es.finish();
}
int hc_dev_make_du_dt(const hc_geom* g, const double* fx, const double* fy, const double* fz,
                      double dt, double* rate, void* stream) {
    GEOM_OR_FAIL(g, 0);
    return d_du_dt(*g, fx, fy, fz, dt, rate, as_stream(stream));
}
int hc_dev_update_u_timestep(const hc_geom* g, int modes, double* modal, double* skinny,
                             const double* rate, double cfl, double gamma, double* dt_next,
                             void* stream) {
    GEOM_OR_FAIL(g, 0);
    TRY(modes_ok(modes));
    cudaStream_t st = as_stream(stream);
    int rc = HC_OK;
    double* dtn = ws().get<double>("dev_dtn", 1, &rc);
    TRY(rc);
    ErrScope es(st);
    TRY(es.rc);
    TRY(d_update(*g, modes, modal, skinny, rate, cfl, gamma, dtn, es.d, st));
    TRY(d2h(dt_next, dtn, 8, st));
    return es.finish();
}

}  // extern "C"

// ---------------------------------------------------------------------------- self test
// The fused kernel's branch-free division/sqrt (pointwise.cuh div_fast/sqrt_fast) must equal
// IEEE a / b and sqrt(a) bit for bit whenever they report "no slow path needed".
namespace hc {
__global__ void k_fastmath(const double* a, const double* b, size_t n, double* q, int* qslow,
                           double* s, int* sslow) {
    size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    bool slow = false;
    q[i] = hc::div_fast(a[i], b[i], slow);
    qslow[i] = slow;
    slow = false;
    s[i] = hc::sqrt_fast(a[i], slow);
    sslow[i] = slow;
}
}  // namespace hc

extern "C" int hc_selftest_fastmath(const double* a, const double* b, size_t n, double* q,
                                    int* qslow, double* s, int* sslow) {
    double *da, *db, *dq, *ds;
    int *dqs, *dss;
    HC_CUDA(cudaMalloc(&da, n * 8));
    HC_CUDA(cudaMalloc(&db, n * 8));
    HC_CUDA(cudaMalloc(&dq, n * 8));
    HC_CUDA(cudaMalloc(&ds, n * 8));
    HC_CUDA(cudaMalloc(&dqs, n * 4));
    HC_CUDA(cudaMalloc(&dss, n * 4));
    HC_CUDA(cudaMemcpy(da, a, n * 8, cudaMemcpyHostToDevice));
    HC_CUDA(cudaMemcpy(db, b, n * 8, cudaMemcpyHostToDevice));
    k_fastmath<<<unsigned((n + 255) / 256), 256>>>(da, db, n, dq, dqs, ds, dss);
    HC_CUDA(cudaGetLastError());
    HC_CUDA(cudaMemcpy(q, dq, n * 8, cudaMemcpyDeviceToHost));
    HC_CUDA(cudaMemcpy(s, ds, n * 8, cudaMemcpyDeviceToHost));
    HC_CUDA(cudaMemcpy(qslow, dqs, n * 4, cudaMemcpyDeviceToHost));
    HC_CUDA(cudaMemcpy(sslow, dss, n * 4, cudaMemcpyDeviceToHost));
    cudaFree(da);
    cudaFree(db);
    cudaFree(dq);
    cudaFree(ds);
    cudaFree(dqs);
    cudaFree(dss);
    return HC_OK;
}
