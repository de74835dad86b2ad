// domain.cu -- the multi-GPU z-slab domain behind the C ABI (hc_domain_*).
//
// The reference splits a mesh into patches and steps them in one process: exchange_ghosts
// fills every patch's ghost shell by sequential x, y, z sweeps over its neighbours
// (transfer.cpp:87-150) and run_patch_step takes the global min of the patches' dt_next
// (transfer.cpp:177-215). Here the patches are z slabs, one per GPU (make_patch_set(global, 1,
// 1, world), transfer.cpp:17-47), each a device-resident fused stepper (stepper.cu):
//
//   per stage:  x/y ghosts of the slab's own planes on its device (the x and y sweeps; a slab
//               spans the whole x/y extent, so they are local)
//               z halos: whole (padded) planes, contiguous in [z][y][x][5], go straight from
//               the lowest / highest gh active planes into the neighbours' ghost planes --
//               ncclSend / ncclRecv in one group (no packing, no temporaries), or, for slabs of
//               one process, cudaMemcpyPeerAsync on the copy engines (the "peer" transport)
//               the fused step (or RK stage)
//   per step:   ncclAllReduce(MIN) of the 8-byte dt_next accumulator on the device, then the
//               device t/dt hand-off.
//
// Everything is enqueued on each slab's stream: n steps run without a host round trip. The
// z sweep copies whole planes, x/y ghosts included, which reproduces the reference's edge and
// corner ghosts, so the decomposed run is bit-identical to the single domain (acceptance
// criterion 8; tests/test_domain_gpu.py).
//
// Two ways in: hc_domain_create -- one process per GPU (rank / world, an NCCL unique id shared
// out of band, e.g. by torch.distributed or MPI) -- and hc_domain_create_local -- one process
// driving `ngpu` devices (ncclCommInitAll, or the peer transport). ngpu = 1 exchanges the
// periodic halos of the single slab with itself through the same NCCL calls (the N > 1 code
// path, runnable on one GPU). NCCL is opened at run time (dlopen "libnccl.so.2"), so the
// library loads without it; only the NCCL transport needs it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "hydro_cuda.h"

namespace hc {
namespace {

// ---- NCCL, resolved at run time
struct Nccl {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl n = [] {
        Nccl r;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            r.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return r;
        }
        auto sym = [&](const char* s) { return dlsym(h, s); };
        r.GetUniqueId = reinterpret_cast<decltype(r.GetUniqueId)>(sym("ncclGetUniqueId"));
        r.CommInitRank = reinterpret_cast<decltype(r.CommInitRank)>(sym("ncclCommInitRank"));
        r.CommInitAll = reinterpret_cast<decltype(r.CommInitAll)>(sym("ncclCommInitAll"));
        r.CommDestroy = reinterpret_cast<decltype(r.CommDestroy)>(sym("ncclCommDestroy"));
        r.GroupStart = reinterpret_cast<decltype(r.GroupStart)>(sym("ncclGroupStart"));
        r.GroupEnd = reinterpret_cast<decltype(r.GroupEnd)>(sym("ncclGroupEnd"));
        r.Send = reinterpret_cast<decltype(r.Send)>(sym("ncclSend"));
        r.Recv = reinterpret_cast<decltype(r.Recv)>(sym("ncclRecv"));
        r.AllReduce = reinterpret_cast<decltype(r.AllReduce)>(sym("ncclAllReduce"));
        r.GetErrorString = reinterpret_cast<decltype(r.GetErrorString)>(sym("ncclGetErrorString"));
        r.ok = r.GetUniqueId && r.CommInitRank && r.CommInitAll && r.CommDestroy &&
               r.GroupStart && r.GroupEnd && r.Send && r.Recv && r.AllReduce && r.GetErrorString;
        if (!r.ok) r.why = "libnccl.so.2 lacks a needed symbol";
        return r;
    }();
    return n;
}

int nccl_fail(ncclResult_t e, const char* where) {
    set_error(HC_CUDA, std::string("nccl error in ") + where + ": " + nccl().GetErrorString(e));
    return HC_CUDA;
}
#define HC_NCCL(call)                                            \
    do {                                                         \
        ncclResult_t e_ = (call);                                \
        if (e_ != ncclSuccess) return nccl_fail(e_, #call);      \
    } while (0)

struct Slab {
    int device = 0;
    int rank = 0;  // global slab index (z order)
    int z0 = 0;    // first global active plane
    hc_stepper* st = nullptr;
    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;
    double* buf[3] = {nullptr, nullptr, nullptr};
    int nbuf = 2;
    // overlap: the halo exchange runs on xstream while the interior planes are computed
    cudaStream_t xstream = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
};

}  // namespace
}  // namespace hc

using namespace hc;

struct hc_domain {
    hc_geom global{};
    hc_params p{};
    hc_domain_opts o{};
    int world = 1;       // slabs in the whole domain
    int nloc = 0;        // active planes per slab
    int gh = 0;
    size_t plane = 0;    // doubles per storage plane (my_pad * pitch)
    int my = 0, mx = 0;  // storage rows / columns per plane (ghosts included)
    int pitch = 0;
    std::vector<Slab> s;  // the slabs this process drives
    int cur = 0;          // host-tracked current buffer (the steppers flip it on the device)
    bool primed = false;  // (store transport) the z ghosts of the current state are in place
    bool nccl_owned = false;
    double** peer_accs = nullptr;  // (peer transport) device array of the slabs' dt accumulators
};

namespace hc_dom {  // (named: nvcc's stub generator trips over a second anonymous namespace)

int set_dev(int d) {
    HC_CUDA(cudaSetDevice(d));
    return HC_OK;
}

// storage plane k of buffer b of slab x
double* plane_ptr(const hc_domain* d, const Slab& x, int b, int k) {
    return x.buf[b] + size_t(k) * d->plane;
}

int check_args(const hc_geom* g, const hc_params* p, const hc_domain_opts* o, int world) {
    if (!g || !p || !o || world < 1) {
        set_error(HC_INVALID, "hc_domain: null argument or world < 1");
        return HC_INVALID;
    }
    if (g->nz % world) {  // transfer.cpp:19-22
        set_error(HC_INVALID, "patch split must divide the mesh evenly");
        return HC_INVALID;
    }
    if (g->nz / world < 4) {
        set_error(HC_INVALID, "patch must have at least 4 zones per axis");
        return HC_INVALID;
    }
    if (o->transport != HC_XCHG_NCCL && o->transport != HC_XCHG_PEER &&
        o->transport != HC_XCHG_STORE) {
        set_error(HC_INVALID, "hc_domain: unknown transport");
        return HC_INVALID;
    }
    return HC_OK;
}

// One slab: its stepper (z ghosts caller-filled) on its own stream.
int make_slab(hc_domain* d, Slab& x) {
    int rc;
    if ((rc = set_dev(x.device))) return rc;
    hc_geom g = d->global;
    g.nz = d->nloc;
    // the slab's origin and spacing set exactly (a re-derived dz could be one ulp off)
    g.origin[2] = d->global.origin[2] + double(x.z0) * d->global.dz;
    hc_stepper_opts so{};
    so.bc[0] = d->o.bc[0];
    so.bc[1] = d->o.bc[1];
    so.bc[2] = -1;
    so.exact = d->o.exact;
    so.device = x.device;
    so.integrator = d->o.integrator;
    if ((rc = hc_stepper_create(&g, &d->p, &so, &x.st))) return rc;
    HC_CUDA(cudaStreamCreateWithFlags(&x.stream, cudaStreamNonBlocking));
    if ((rc = hc_stepper_set_stream(x.st, x.stream))) return rc;
    if (d->o.overlap) {
        HC_CUDA(cudaStreamCreateWithFlags(&x.xstream, cudaStreamNonBlocking));
        HC_CUDA(cudaEventCreateWithFlags(&x.ev_ready, cudaEventDisableTiming));
        HC_CUDA(cudaEventCreateWithFlags(&x.ev_done, cudaEventDisableTiming));
    }
    if ((rc = hc_stepper_buffers(x.st, x.buf, &x.nbuf))) return rc;
    int my_pad = 0, pitch = 0, mz = 0;
    hc_stepper_layout(x.st, &my_pad, &pitch, &mz);
    d->plane = size_t(my_pad) * pitch;
    d->pitch = pitch;
    d->my = my_pad;
    d->mx = pitch / 5;
    return HC_OK;
}

int common_init(hc_domain* d, const hc_geom* g, const hc_params* p, const hc_domain_opts* o,
                int world) {
    d->global = *g;
    d->p = *p;
    d->o = *o;
    d->world = world;
    d->nloc = g->nz / world;
    d->gh = g->ghost;
    return HC_OK;
}

int outflow_ends(hc_domain* d, int b, bool xs);

// every slab's stream waits for the work enqueued so far on every other slab's stream
int barrier_all(hc_domain* d) {
    std::vector<cudaEvent_t> ev(d->s.size());
    for (size_t i = 0; i < d->s.size(); ++i) {
        HC_CUDA(cudaSetDevice(d->s[i].device));
        HC_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        HC_CUDA(cudaEventRecord(ev[i], d->s[i].stream));
    }
    for (size_t i = 0; i < d->s.size(); ++i) {
        HC_CUDA(cudaSetDevice(d->s[i].device));
        for (size_t j = 0; j < d->s.size(); ++j)
            if (j != i) HC_CUDA(cudaStreamWaitEvent(d->s[i].stream, ev[j], 0));
    }
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    return HC_OK;
}

// store transport: every slab's fused kernels write their boundary planes into the z
// neighbours' ghost planes (hc_stepper_set_zpeer); an outflow end has no neighbour
int setup_store(hc_domain* d) {
    const bool periodic = d->o.bc[2] == HC_PERIODIC;
    const int W = d->world;
    for (Slab& x : d->s) {
        const int lo = x.rank > 0 ? x.rank - 1 : (periodic ? W - 1 : -1);
        const int hi = x.rank < W - 1 ? x.rank + 1 : (periodic ? 0 : -1);
        const Slab* yl = lo >= 0 ? &d->s[size_t(lo)] : nullptr;
        const Slab* yh = hi >= 0 ? &d->s[size_t(hi)] : nullptr;
        int rc = hc_stepper_set_zpeer(x.st, yl ? yl->buf : nullptr, yh ? yh->buf : nullptr);
        if (rc) return rc;
    }
    return HC_OK;
}

// z halos of every local slab, buffer b: NCCL group (send down, receive from above, send up,
// receive from below -- the posting order that keeps the k-th send to a peer matched with
// that peer's k-th receive even when, at world 2, below == above), or peer copies. xs: on the
// slabs' exchange streams (overlap; the caller orders the compute streams after them).
int exchange(hc_domain* d, int b, bool xs) {
    auto S = [&](const Slab& x) { return xs ? x.xstream : x.stream; };
    const int gh = d->gh, nl = d->nloc, W = d->world;
    const bool periodic = d->o.bc[2] == HC_PERIODIC;
    const size_t cnt = size_t(gh) * d->plane;  // doubles per message
    const size_t bytes = cnt * sizeof(double);
    auto below = [&](int r) { return r > 0 ? r - 1 : (periodic ? W - 1 : -1); };
    auto above = [&](int r) { return r < W - 1 ? r + 1 : (periodic ? 0 : -1); };
    if (d->o.transport == HC_XCHG_NCCL) {
        const Nccl& N = nccl();
        HC_NCCL(N.GroupStart());
        for (Slab& x : d->s) {
            const int lo = below(x.rank), hi = above(x.rank);
            double* lo_act = plane_ptr(d, x, b, gh);
            double* hi_act = plane_ptr(d, x, b, nl);
            double* lo_gh = plane_ptr(d, x, b, 0);
            double* hi_gh = plane_ptr(d, x, b, gh + nl);
            if (lo >= 0) HC_NCCL(N.Send(lo_act, cnt, ncclFloat64, lo, x.comm, S(x)));
            if (hi >= 0) {
                HC_NCCL(N.Recv(hi_gh, cnt, ncclFloat64, hi, x.comm, S(x)));
                HC_NCCL(N.Send(hi_act, cnt, ncclFloat64, hi, x.comm, S(x)));
            }
            if (lo >= 0) HC_NCCL(N.Recv(lo_gh, cnt, ncclFloat64, lo, x.comm, S(x)));
        }
        HC_NCCL(N.GroupEnd());
    } else {  // peer copies: every slab in this process; each pulls its two halos
        // the neighbours' active planes must be final: order after their streams
        std::vector<cudaEvent_t> ev(d->s.size());
        for (size_t i = 0; i < d->s.size(); ++i) {
            HC_CUDA(cudaSetDevice(d->s[i].device));
            HC_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
            HC_CUDA(cudaEventRecord(ev[i], S(d->s[i])));
        }
        for (Slab& x : d->s) {
            HC_CUDA(cudaSetDevice(x.device));
            for (size_t i = 0; i < d->s.size(); ++i) HC_CUDA(cudaStreamWaitEvent(S(x), ev[i], 0));
            const int lo = below(x.rank), hi = above(x.rank);
            if (hi >= 0) {
                const Slab& y = d->s[size_t(hi)];
                HC_CUDA(cudaMemcpyPeerAsync(plane_ptr(d, x, b, gh + nl), x.device,
                                            plane_ptr(d, y, b, gh), y.device, bytes, S(x)));
            }
            if (lo >= 0) {
                const Slab& y = d->s[size_t(lo)];
                HC_CUDA(cudaMemcpyPeerAsync(plane_ptr(d, x, b, 0), x.device,
                                            plane_ptr(d, y, b, nl), y.device, bytes, S(x)));
            }
        }
        // the next stage overwrites the sources: order every slab after every copy (with
        // overlap the caller orders the compute streams after every exchange stream)
        if (!xs) {
            for (size_t i = 0; i < d->s.size(); ++i) {
                HC_CUDA(cudaSetDevice(d->s[i].device));
                HC_CUDA(cudaEventRecord(ev[i], d->s[i].stream));
            }
            for (Slab& x : d->s) {
                HC_CUDA(cudaSetDevice(x.device));
                for (size_t i = 0; i < d->s.size(); ++i)
                    HC_CUDA(cudaStreamWaitEvent(x.stream, ev[i], 0));
            }
        }
        for (size_t i = 0; i < d->s.size(); ++i) cudaEventDestroy(ev[i]);
    }
    return outflow_ends(d, b, xs);
}

// outflow ends: the ghost planes repeat the edge active plane (boundary.cpp map_index)
int outflow_ends(hc_domain* d, int b, bool xs) {
    auto S = [&](const Slab& x) { return xs ? x.xstream : x.stream; };
    const int gh = d->gh, nl = d->nloc, W = d->world;
    if (d->o.bc[2] != HC_PERIODIC) {
        for (Slab& x : d->s) {
            HC_CUDA(cudaSetDevice(x.device));
            for (int k = 0; k < gh; ++k) {
                if (x.rank == 0)
                    HC_CUDA(cudaMemcpyAsync(plane_ptr(d, x, b, k), plane_ptr(d, x, b, gh),
                                            d->plane * sizeof(double), cudaMemcpyDeviceToDevice,
                                            S(x)));
                if (x.rank == W - 1)
                    HC_CUDA(cudaMemcpyAsync(plane_ptr(d, x, b, gh + nl + k),
                                            plane_ptr(d, x, b, gh + nl - 1),
                                            d->plane * sizeof(double), cudaMemcpyDeviceToDevice,
                                            S(x)));
            }
        }
    }
    return HC_OK;
}

__global__ void k_peer_min(double* const* accs, int n) {
    double m = *accs[0];
    for (int i = 1; i < n; ++i) m = smin(m, *accs[i]);
    for (int i = 0; i < n; ++i) *accs[i] = m;
}

int peer_dt_min(hc_domain* d) {
    const size_t n = d->s.size();
    std::vector<double*> accs(n);
    for (size_t i = 0; i < n; ++i) hc_stepper_dt_ptrs(d->s[i].st, &accs[i], nullptr);
    if (!d->peer_accs) {
        HC_CUDA(cudaSetDevice(d->s[0].device));
        HC_CUDA(cudaMalloc(&d->peer_accs, n * sizeof(double*)));
        HC_CUDA(cudaMemcpy(d->peer_accs, accs.data(), n * sizeof(double*),
                           cudaMemcpyHostToDevice));
    }
    std::vector<cudaEvent_t> ev(n);
    for (size_t i = 0; i < n; ++i) {
        HC_CUDA(cudaSetDevice(d->s[i].device));
        HC_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        HC_CUDA(cudaEventRecord(ev[i], d->s[i].stream));
    }
    HC_CUDA(cudaSetDevice(d->s[0].device));
    for (size_t i = 1; i < n; ++i) HC_CUDA(cudaStreamWaitEvent(d->s[0].stream, ev[i], 0));
    k_peer_min<<<1, 1, 0, d->s[0].stream>>>(d->peer_accs, int(n));
    HC_CUDA(cudaGetLastError());
    HC_CUDA(cudaEventRecord(ev[0], d->s[0].stream));
    for (size_t i = 1; i < n; ++i) {
        HC_CUDA(cudaSetDevice(d->s[i].device));
        HC_CUDA(cudaStreamWaitEvent(d->s[i].stream, ev[0], 0));
    }
    for (size_t i = 0; i < n; ++i) cudaEventDestroy(ev[i]);
    return HC_OK;
}

int one_step(hc_domain* d) {
    int rc;
    const int ns = d->s.empty() ? 1 : hc_stepper_stages(d->s[0].st);
    const int nbuf = d->s.empty() ? 2 : d->s[0].nbuf;
    const bool store = d->o.transport == HC_XCHG_STORE;
    for (int k = 0; k < ns; ++k) {
        // store transport: the neighbours' previous stage (their stores into this slab's
        // ghost planes, their reads of the buffer this stage stores into) is complete
        if (store && d->s.size() > 1 && (rc = barrier_all(d))) return rc;
        for (Slab& x : d->s) {
            if ((rc = set_dev(x.device)) || (rc = hc_stepper_fill_ghosts(x.st))) return rc;
        }
        // the buffer this stage reads: cur (ADER, RK stage 0) or the previous stage's result
        const int b = (d->cur + (d->o.integrator ? k : 0)) % nbuf;
        if (store) {
            // the z ghosts arrived with the previous stage's compute; the first stage after a
            // scatter takes them by peer copies
            if ((rc = d->primed ? outflow_ends(d, b, false) : exchange(d, b, false))) return rc;
            d->primed = true;
            for (Slab& x : d->s) {
                if ((rc = set_dev(x.device)) || (rc = hc_stepper_compute(x.st))) return rc;
            }
            continue;
        }
        const int G = d->gh;  // planes whose stencils reach a z ghost plane, on each side
        if (!d->o.overlap || d->nloc <= 2 * G) {
            if ((rc = exchange(d, b, false))) return rc;
            for (Slab& x : d->s) {
                if ((rc = set_dev(x.device)) || (rc = hc_stepper_compute(x.st))) return rc;
            }
            continue;
        }
        // overlap: the exchange on the side streams while the interior planes [G, nloc - G)
        // -- whose stencils never reach a z ghost -- are updated, then the two boundary ranges
        for (Slab& x : d->s) {
            if ((rc = set_dev(x.device))) return rc;
            HC_CUDA(cudaEventRecord(x.ev_ready, x.stream));
            HC_CUDA(cudaStreamWaitEvent(x.xstream, x.ev_ready, 0));
        }
        if ((rc = exchange(d, b, true))) return rc;
        for (Slab& x : d->s) {
            if ((rc = set_dev(x.device))) return rc;
            HC_CUDA(cudaEventRecord(x.ev_done, x.xstream));
            if ((rc = hc_stepper_compute_range(x.st, G, d->nloc - G, 0))) return rc;
        }
        for (Slab& x : d->s) {
            if ((rc = set_dev(x.device))) return rc;
            for (Slab& y : d->s) HC_CUDA(cudaStreamWaitEvent(x.stream, y.ev_done, 0));
            if ((rc = hc_stepper_compute_range(x.st, 0, G, 0)) ||
                (rc = hc_stepper_compute_range(x.st, d->nloc - G, d->nloc, 1)))
                return rc;
        }
    }
    // global dt min (transfer.cpp:184): one 8-byte all-reduce on the device accumulators
    if (d->o.transport == HC_XCHG_NCCL) {
        const Nccl& N = nccl();
        HC_NCCL(N.GroupStart());
        for (Slab& x : d->s) {
            double* acc = nullptr;
            hc_stepper_dt_ptrs(x.st, &acc, nullptr);
            HC_NCCL(N.AllReduce(acc, acc, 1, ncclFloat64, ncclMin, x.comm, x.stream));
        }
        HC_NCCL(N.GroupEnd());
    } else if (d->s.size() > 1) {  // peer: one kernel on slab 0 takes the min over every
        // slab's accumulator through peer pointers and writes it back to all of them
        if ((rc = peer_dt_min(d))) return rc;
    }
    for (Slab& x : d->s) {
        if ((rc = set_dev(x.device)) || (rc = hc_stepper_advance(x.st))) return rc;
    }
    if (d->o.integrator == 0) d->cur = 1 - d->cur;  // ADER wrote the other buffer
    return HC_OK;
}

}  // namespace hc_dom

using namespace hc_dom;

extern "C" {

int hc_nccl_unique_id(unsigned char* id, size_t len) {
    const Nccl& N = nccl();
    if (!N.ok) {
        set_error(HC_CUDA, N.why);
        return HC_CUDA;
    }
    if (!id || len < sizeof(ncclUniqueId)) {
        set_error(HC_INVALID, "hc_nccl_unique_id: buffer shorter than NCCL_UNIQUE_ID_BYTES");
        return HC_INVALID;
    }
    ncclUniqueId u;
    HC_NCCL(N.GetUniqueId(&u));
    std::memcpy(id, &u, sizeof u);
    return HC_OK;
}

int hc_domain_create(const hc_geom* global, const hc_params* p, const hc_domain_opts* o,
                     int rank, int world, const unsigned char* nccl_id, hc_domain** out) {
    int rc = check_args(global, p, o, world);
    if (rc) return rc;
    if (rank < 0 || rank >= world || !out || (o->transport == HC_XCHG_NCCL && !nccl_id)) {
        set_error(HC_INVALID, "hc_domain_create: bad rank, world or NCCL id");
        return HC_INVALID;
    }
    if (o->transport != HC_XCHG_NCCL && world > 1) {
        set_error(HC_INVALID, "the peer and store transports need every slab in one process "
                              "(hc_domain_create_local)");
        return HC_INVALID;
    }
    auto* d = new hc_domain;
    common_init(d, global, p, o, world);
    Slab x;
    x.device = o->device;
    x.rank = rank;
    x.z0 = rank * d->nloc;
    d->s.push_back(x);
    if ((rc = make_slab(d, d->s[0]))) {
        hc_domain_destroy(d);
        return rc;
    }
    if (o->transport == HC_XCHG_NCCL) {
        const Nccl& N = nccl();
        if (!N.ok) {
            set_error(HC_CUDA, N.why);
            hc_domain_destroy(d);
            return HC_CUDA;
        }
        ncclUniqueId u;
        std::memcpy(&u, nccl_id, sizeof u);
        ncclResult_t e = N.CommInitRank(&d->s[0].comm, world, u, rank);
        if (e != ncclSuccess) {
            rc = nccl_fail(e, "ncclCommInitRank");
            hc_domain_destroy(d);
            return rc;
        }
        d->nccl_owned = true;
    }
    if (o->transport == HC_XCHG_STORE && (rc = setup_store(d))) {
        hc_domain_destroy(d);
        return rc;
    }
    *out = d;
    return HC_OK;
}

int hc_domain_create_local(const hc_geom* global, const hc_params* p, const hc_domain_opts* o,
                           int ngpu, const int* devices, hc_domain** out) {
    int rc = check_args(global, p, o, ngpu);
    if (rc) return rc;
    if (!out || !devices) {
        set_error(HC_INVALID, "hc_domain_create_local: null devices or out");
        return HC_INVALID;
    }
    auto* d = new hc_domain;
    common_init(d, global, p, o, ngpu);
    for (int r = 0; r < ngpu; ++r) {
        Slab x;
        x.device = devices[r];
        x.rank = r;
        x.z0 = r * d->nloc;
        d->s.push_back(x);
    }
    for (Slab& x : d->s)
        if ((rc = make_slab(d, x))) {
            hc_domain_destroy(d);
            return rc;
        }
    if (o->transport == HC_XCHG_NCCL) {
        const Nccl& N = nccl();
        if (!N.ok) {
            set_error(HC_CUDA, N.why);
            hc_domain_destroy(d);
            return HC_CUDA;
        }
        std::vector<ncclComm_t> comms(size_t(ngpu), nullptr);
        ncclResult_t e = N.CommInitAll(comms.data(), ngpu, devices);
        if (e != ncclSuccess) {
            rc = nccl_fail(e, "ncclCommInitAll");
            hc_domain_destroy(d);
            return rc;
        }
        for (int r = 0; r < ngpu; ++r) d->s[size_t(r)].comm = comms[size_t(r)];
        d->nccl_owned = true;
    } else {  // peer access between every pair of distinct devices that allows it
        for (Slab& x : d->s)
            for (Slab& y : d->s)
                if (x.device != y.device) {
                    int can = 0;
                    cudaDeviceCanAccessPeer(&can, x.device, y.device);
                    if (can) {
                        cudaSetDevice(x.device);
                        cudaError_t e = cudaDeviceEnablePeerAccess(y.device, 0);
                        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                    }
                }
        if (o->transport == HC_XCHG_STORE && (rc = setup_store(d))) {
            hc_domain_destroy(d);
            return rc;
        }
    }
    *out = d;
    return HC_OK;
}

int hc_domain_destroy(hc_domain* d) {
    if (!d) return HC_OK;
    if (d->peer_accs) {
        cudaSetDevice(d->s[0].device);
        cudaFree(d->peer_accs);
    }
    for (Slab& x : d->s) {
        cudaSetDevice(x.device);
        if (x.stream) cudaStreamSynchronize(x.stream);
        if (x.comm && d->nccl_owned) nccl().CommDestroy(x.comm);
        if (x.st) hc_stepper_destroy(x.st);
        if (x.stream) cudaStreamDestroy(x.stream);
        if (x.xstream) {
            cudaStreamSynchronize(x.xstream);
            cudaStreamDestroy(x.xstream);
        }
        if (x.ev_ready) cudaEventDestroy(x.ev_ready);
        if (x.ev_done) cudaEventDestroy(x.ev_done);
    }
    delete d;
    return HC_OK;
}

// The slabs this process drives, from / to a global HOST SkinnyState [mz][my][mx][5]
// (scatter_to_patches / gather_from_patches, transfer.cpp:50-76): active planes only, whole
// rows (the x/y ghosts travel along and are refilled on the device).
int hc_domain_scatter(hc_domain* d, const double* global_skinny) {
    int rc;
    d->primed = false;
    for (Slab& x : d->s) {
        if ((rc = set_dev(x.device))) return rc;
        const double* src = global_skinny + size_t(d->gh + x.z0) * d->plane;
        HC_CUDA(cudaMemcpyAsync(plane_ptr(d, x, d->cur, d->gh), src,
                                size_t(d->nloc) * d->plane * sizeof(double),
                                cudaMemcpyHostToDevice, x.stream));
        HC_CUDA(cudaStreamSynchronize(x.stream));
    }
    return HC_OK;
}

int hc_domain_gather(hc_domain* d, double* global_skinny) {
    int rc;
    if ((rc = hc_domain_sync(d, nullptr, nullptr, nullptr))) return rc;
    for (Slab& x : d->s) {
        if ((rc = set_dev(x.device))) return rc;
        double* dst = global_skinny + size_t(d->gh + x.z0) * d->plane;
        HC_CUDA(cudaMemcpyAsync(dst, plane_ptr(d, x, d->cur, d->gh),
                                size_t(d->nloc) * d->plane * sizeof(double),
                                cudaMemcpyDeviceToHost, x.stream));
        HC_CUDA(cudaStreamSynchronize(x.stream));
    }
    return HC_OK;
}

int hc_domain_set_time(hc_domain* d, double t, double dt, double cfl, double t_final) {
    int rc;
    for (Slab& x : d->s)
        if ((rc = set_dev(x.device)) || (rc = hc_stepper_set_time(x.st, t, dt, cfl, t_final)))
            return rc;
    return HC_OK;
}

// run_patch_step x n (transfer.cpp:152-216), enqueued without host synchronisation
int hc_domain_step(hc_domain* d, int n) {
    for (int i = 0; i < n; ++i) {
        int rc = one_step(d);
        if (rc) return rc;
    }
    return HC_OK;
}

int hc_domain_sync(hc_domain* d, double* t, double* dt, long* steps_done) {
    int rc = HC_OK;
    int first_err = HC_OK;
    for (size_t i = 0; i < d->s.size(); ++i) {
        Slab& x = d->s[i];
        if ((rc = set_dev(x.device))) return rc;
        double tt = 0.0, dd = 0.0;
        long n = 0;
        rc = hc_stepper_sync(x.st, &tt, &dd, &n);
        if (rc && !first_err) first_err = rc;
        if (i == 0) {
            if (t) *t = tt;
            if (dt) *dt = dd;
            if (steps_done) *steps_done = n;
        }
    }
    // the device decides which buffer is current (no-op steps after t_final do not flip)
    if (!d->s.empty()) {
        double* cur = nullptr;
        if ((rc = hc_stepper_state(d->s[0].st, &cur, nullptr))) return rc;
        d->cur = cur == d->s[0].buf[0] ? 0 : 1;
    }
    return first_err;
}

int hc_domain_info(hc_domain* d, int* nz_local, int* z0, int* nslabs, int* kernel) {
    if (!d) return HC_INVALID;
    if (nz_local) *nz_local = d->nloc;
    if (z0) *z0 = d->s.empty() ? 0 : d->s[0].z0;
    if (nslabs) *nslabs = int(d->s.size());
    if (kernel && !d->s.empty()) hc_stepper_info(d->s[0].st, kernel, nullptr);
    return HC_OK;
}

long hc_domain_launches(hc_domain* d) {
    long n = 0;
    for (Slab& x : d->s) n += hc_stepper_launches(x.st);
    return n;
}

}  // extern "C"
