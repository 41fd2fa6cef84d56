// dbp_api.cu -- the C ABI of include/dbp.h: validation, workspace layout,
// host-pointer staging, the per-call launch schedules and the NCCL consensus
// collective (one in-place ncclAllReduce of the N x N_sym x U partial sums per
// iteration, P311, P401, P513, P744-746).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dbp.h"
#include "dbp_internal.h"

using namespace dbp;

struct dbp_ctx {
    int device = 0, rank = 0, world = 1;
    ncclComm_t comm = nullptr;
    int* d_flag = nullptr;
    int64_t launches = 0;
    int64_t allreduce_calls = 0, allreduce_bytes = 0, consensus_rounds = 0;
    int force_split = 0;
    int no_fused = 0;
    int mode = 0;                // DBP_OPT_MODE: 0 paper rule (S < U -> S x S), 1 U x U, 2 S x S
    int cg_tc = 1;               // DBP_OPT_CG_TENSOR: world-1 CG-UL Gram on the tensor cores
    int pdl = 0;                 // DBP_OPT_OVERLAP_PREV: single-kernel solvers overlap the previous kernel
    // host allreduce hook (world > 1 without a communicator)
    dbp_allreduce_fn hook = nullptr;
    void* hook_user = nullptr;
    float* hbuf = nullptr;
    size_t hbuf_bytes = 0;
    // CUDA graphs of the multi-launch schedules (DBP_OPT_GRAPHS): key -> instantiated graph
    int graphs = 1;
    cudaStream_t cap = nullptr;
    struct GraphEnt {
        std::vector<uint64_t> key;
        cudaGraphExec_t exec;
        int64_t launches, ar_calls, ar_bytes, rounds;
        uint64_t used;
    };
    std::vector<GraphEnt> gcache;
    uint64_t gclock = 0;
    int64_t graph_replays = 0;
    // device-side consensus (DBP_OPT_DEVICE_CONSENSUS): symmetric buffer, peer mappings
    int xcons = 0;
    void* xbuf = nullptr;
    void* xpeer[8] = {nullptr};
    int xcap = 0;
    unsigned xround = 1;
    void* stage = nullptr;       // host-I/O staging (device)
    size_t stage_bytes = 0;
    void* iws = nullptr;         // internal workspace when ws == NULL
    size_t iws_bytes = 0;
    int max_smem = 0;
    // per-kernel event timing (DBP_OPT_KERNEL_TIMING)
    int timing = 0;
    struct Pending { int k; cudaEvent_t e0, e1; };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> pool;
    std::vector<std::string> knames;
    std::vector<int64_t> kcount;
    std::vector<double> kms;
};

static cudaEvent_t ev_get(dbp_ctx* c) {
    if (!c->pool.empty()) { cudaEvent_t e = c->pool.back(); c->pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

static int kname_id(dbp_ctx* c, const char* name) {
    for (size_t i = 0; i < c->knames.size(); ++i) if (c->knames[i] == name) return (int)i;
    c->knames.push_back(name);
    c->kcount.push_back(0);
    c->kms.push_back(0.0);
    return (int)c->knames.size() - 1;
}

static thread_local std::string g_err;

static dbp_status fail(dbp_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

#define CU(call)                                                                            \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess) return fail(DBP_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

#define NC(call)                                                                            \
    do {                                                                                    \
        ncclResult_t r_ = (call);                                                           \
        if (r_ != ncclSuccess) return fail(DBP_ERR_NCCL, "%s: %s", #call, ncclGetErrorString(r_)); \
    } while (0)

extern "C" const char* dbp_last_error(void) { return g_err.c_str(); }

static int pad_users(int U) { return U <= 4 ? 4 : U <= 8 ? 8 : U <= 16 ? 16 : 32; }
static size_t al(size_t b) { return (b + 255) & ~(size_t)255; }

extern "C" dbp_status dbp_get_unique_id(uint8_t id[128]) {
    if (!id) return fail(DBP_ERR_INVALID_ARG, "id is NULL");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId u;
    NC(ncclGetUniqueId(&u));
    memcpy(id, &u, 128);
    g_err.clear();
    return DBP_OK;
}

extern "C" dbp_status dbp_ctx_create(dbp_ctx** out, int device, int rank, int world, const uint8_t* id) {
    if (!out) return fail(DBP_ERR_INVALID_ARG, "ctx out-pointer is NULL");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return fail(DBP_ERR_INVALID_ARG, "bad rank %d / world %d", rank, world);
    int ndev = 0;
    CU(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(DBP_ERR_INVALID_ARG, "device %d of %d", device, ndev);
    CU(cudaSetDevice(device));
    dbp_ctx* c = new dbp_ctx();
    c->device = device;
    c->rank = rank;
    c->world = world;
    cudaError_t e = cudaMalloc(&c->d_flag, sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(c->d_flag, 0, sizeof(int));
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (e != cudaSuccess) {
        delete c;
        return fail(DBP_ERR_CUDA, "context setup: %s", cudaGetErrorString(e));
    }
    if (world > 1 && id) {
        ncclUniqueId u;
        memcpy(&u, id, 128);
        ncclResult_t r = ncclCommInitRank(&c->comm, world, u, rank);
        if (r != ncclSuccess) {
            cudaFree(c->d_flag);
            delete c;
            return fail(DBP_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
        }
    }
    *out = c;
    g_err.clear();
    return DBP_OK;
}

extern "C" dbp_status dbp_ctx_destroy(dbp_ctx* c) {
    if (!c) return DBP_OK;
    cudaSetDevice(c->device);
    for (int r = 0; r < 8; ++r)
        if (c->xpeer[r] && c->xpeer[r] != c->xbuf) cudaIpcCloseMemHandle(c->xpeer[r]);
    if (c->xbuf) cudaFree(c->xbuf);
    if (c->comm) ncclCommDestroy(c->comm);
    cudaFree(c->d_flag);
    if (c->stage) cudaFree(c->stage);
    if (c->iws) cudaFree(c->iws);
    if (c->hbuf) cudaFreeHost(c->hbuf);
    for (auto& g : c->gcache) cudaGraphExecDestroy(g.exec);
    if (c->cap) cudaStreamDestroy(c->cap);
    for (auto& p : c->pending) { cudaEventDestroy(p.e0); cudaEventDestroy(p.e1); }
    for (auto e : c->pool) cudaEventDestroy(e);
    delete c;
    return DBP_OK;
}

extern "C" dbp_status dbp_set_option(dbp_ctx* c, int option, int64_t value) {
    if (!c) return fail(DBP_ERR_INVALID_ARG, "ctx is NULL");
    if (option == DBP_OPT_FORCE_SPLIT) { c->force_split = value ? 1 : 0; return DBP_OK; }
    if (option == DBP_OPT_KERNEL_TIMING) { c->timing = value ? 1 : 0; return DBP_OK; }
    if (option == DBP_OPT_NO_FUSED) { c->no_fused = value ? 1 : 0; return DBP_OK; }
    if (option == DBP_OPT_GRAPHS) { c->graphs = value ? 1 : 0; return DBP_OK; }
    if (option == DBP_OPT_CG_TENSOR) { c->cg_tc = value ? 1 : 0; return DBP_OK; }
    if (option == DBP_OPT_OVERLAP_PREV) { c->pdl = value ? 1 : 0; return DBP_OK; }
    if (option == DBP_OPT_MODE) {
        if (value < 0 || value > 2) return fail(DBP_ERR_INVALID_ARG, "mode %lld (0 auto, 1 UxU, 2 SxS)", (long long)value);
        c->mode = (int)value;
        return DBP_OK;
    }
    if (option == DBP_OPT_DEVICE_CONSENSUS) {
        if (value < 0 || value > 2) return fail(DBP_ERR_INVALID_ARG, "device consensus mode %lld", (long long)value);
        if (value && c->world > 8) return fail(DBP_ERR_UNSUPPORTED, "device consensus supports world <= 8");
        c->xcons = (int)value;
        return DBP_OK;
    }
    return fail(DBP_ERR_INVALID_ARG, "unknown option %d", option);
}

extern "C" dbp_status dbp_get_stats(const dbp_ctx* c, dbp_stats* s) {
    if (!c || !s) return fail(DBP_ERR_INVALID_ARG, "NULL argument");
    s->allreduce_calls = c->allreduce_calls;
    s->allreduce_bytes = c->allreduce_bytes;
    s->kernel_launches = c->launches;
    s->consensus_rounds = c->consensus_rounds;
    s->graph_replays = c->graph_replays;
    return DBP_OK;
}

extern "C" dbp_status dbp_set_allreduce_hook(dbp_ctx* c, dbp_allreduce_fn fn, void* user) {
    if (!c) return fail(DBP_ERR_INVALID_ARG, "ctx is NULL");
    if (c->comm) return fail(DBP_ERR_INVALID_ARG, "the context has an NCCL communicator");
    c->hook = fn;
    c->hook_user = user;
    return DBP_OK;
}

extern "C" dbp_status dbp_get_comm_info(const dbp_ctx* c, int* nranks, int* rank) {
    if (!c || !nranks || !rank) return fail(DBP_ERR_INVALID_ARG, "NULL argument");
    if (!c->comm) {                       // world 1, or a host-hook context: the context's own view
        *nranks = c->world;
        *rank = c->rank;
        return DBP_OK;
    }
    NC(ncclCommCount(c->comm, nranks));
    NC(ncclCommUserRank(c->comm, rank));
    return DBP_OK;
}

// ----------------------------------------------------------------- shapes
struct Shape {
    int C, C_loc, S, U, UP, N, J;
    int ss, SP;                  // S x S form (DBP_OPT_MODE) and S padded to 4/8/16/32
    long pairs() const { return (long)C_loc * N; }
};

static dbp_status check_dims(const dbp_ctx* c, const dbp_dims* d, Shape* sh) {
    if (!c) return fail(DBP_ERR_INVALID_ARG, "ctx is NULL");
    if (!d) return fail(DBP_ERR_INVALID_ARG, "dims is NULL");
    // N = 0 is an empty frame (no subcarriers): valid, the solvers return DBP_OK with nothing enqueued.
    if (d->C < 1 || d->S < 1 || d->U < 1 || d->N < 0 || d->N_sym < 1)
        return fail(DBP_ERR_INVALID_ARG, "dims must be >= 1, N >= 0 (C=%d S=%d U=%d N=%d N_sym=%d)", d->C, d->S, d->U, d->N, d->N_sym);
    if (d->C % c->world) return fail(DBP_ERR_INVALID_ARG, "C=%d not divisible by world=%d (SPEC S107)", d->C, c->world);
    if (d->U > 32 || d->S > 64 || d->N_sym > 16)
        return fail(DBP_ERR_UNSUPPORTED, "v1 envelope: U<=32, S<=64, N_sym<=16 (got U=%d S=%d N_sym=%d)", d->U, d->S, d->N_sym);
    sh->C = d->C;
    sh->C_loc = d->C / c->world;
    sh->S = d->S;
    sh->U = d->U;
    sh->UP = pad_users(d->U);
    sh->N = d->N;
    sh->J = d->N_sym;
    sh->ss = c->mode == 2 || (c->mode == 0 && d->S < d->U);
    sh->SP = pad_users(d->S);
    if (sh->ss && d->S > 32) return fail(DBP_ERR_UNSUPPORTED, "the S x S form supports S <= 32 (got S=%d)", d->S);
    if ((long)sh->C_loc * sh->N > (1L << 31) - 1) return fail(DBP_ERR_UNSUPPORTED, "too many pairs");
    return DBP_OK;
}

// Workspace layout (256-byte aligned segments).
struct Layout {
    size_t off[8];
    size_t total;
};

static Layout layout(const Shape& sh, int algo) {
    // per-pair packed inverse: U x U, or the S x S form's A_c^{-1} (the larger of the two when forced)
    const size_t T = std::max((size_t)sh.UP * (sh.UP + 1) / 2, sh.ss ? (size_t)sh.SP * (sh.SP + 1) / 2 : (size_t)0);
    const size_t P = (size_t)sh.pairs();
    const size_t vecp = P * sh.J * sh.UP * 8;      // per pair per symbol vectors
    const size_t vecn = (size_t)sh.N * sh.J * sh.UP * 8;
    Layout L{};
    size_t sz[8] = {0};
    if (algo == DBP_ALGO_ADMM_UL) {
        sz[0] = P * T * 8;   // G, then G^{-1} in place (split path)
        sz[1] = vecp;        // matched filter H^H y
        sz[2] = vecp;        // yreg
        sz[3] = vecp;        // lam
        sz[4] = vecp;        // z
        sz[5] = vecn;        // wbuf
    } else if (algo == DBP_ALGO_CG_UL) {
        sz[0] = P * T * 8;                 // per-pair Gram
        sz[1] = vecp;                      // per-pair matched filter
        sz[2] = (size_t)sh.N * T * 8;      // G_loc
        sz[3] = vecn;                      // wbuf
        sz[4] = vecn;                      // x
        sz[5] = vecn;                      // r
        sz[6] = vecn;                      // p
        sz[7] = (size_t)sh.N * sh.J * 4;   // rr
    } else if (algo == DBP_ALGO_ADMM_DL) {
        sz[0] = P * T * 8;   // B, then B^{-1} in place (split path)
        sz[1] = vecp;        // m
        sz[2] = vecp;        // lam
        sz[3] = vecn;        // wbuf
    } else {                 // centralized MMSE-UL / ZF-DL
        sz[0] = P * T * 8;                               // per-pair Gram
        sz[1] = algo == DBP_ALGO_MMSE_UL ? vecp : 0;     // per-pair matched filter
        sz[2] = (size_t)sh.N * T * 8;                    // Gram sum (allreduced)
        sz[3] = vecn;                                    // y^MRC sum (UL) or r (DL)
    }
    size_t o = 0;
    for (int i = 0; i < 8; ++i) { L.off[i] = o; o += al(sz[i]); }
    L.total = o;
    return L;
}

extern "C" dbp_status dbp_workspace_bytes(const dbp_ctx* c, const dbp_dims* d, int algo, size_t* bytes) {
    if (!bytes) return fail(DBP_ERR_INVALID_ARG, "bytes is NULL");
    if (algo < 0 || algo > 4) return fail(DBP_ERR_INVALID_ARG, "algo %d", algo);
    Shape sh;
    dbp_status st = check_dims(c, d, &sh);
    if (st) return st;
    *bytes = layout(sh, algo).total;
    return DBP_OK;
}

// ------------------------------------------------------- pointer handling
static bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

struct Io {                     // one host<->device staged buffer
    const void* host_in;
    void* host_out;
    size_t bytes;
    void* dev;
};

static dbp_status ensure_stage(dbp_ctx* c, size_t bytes) {
    if (c->stage_bytes >= bytes) return DBP_OK;
    if (c->stage) cudaFree(c->stage);
    c->stage = nullptr;
    c->stage_bytes = 0;
    CU(cudaMalloc(&c->stage, bytes));
    c->stage_bytes = bytes;
    return DBP_OK;
}

static dbp_status ensure_iws(dbp_ctx* c, size_t bytes) {
    if (c->iws_bytes >= bytes) return DBP_OK;
    if (c->iws) cudaFree(c->iws);
    c->iws = nullptr;
    c->iws_bytes = 0;
    CU(cudaMalloc(&c->iws, bytes));
    c->iws_bytes = bytes;
    return DBP_OK;
}

// Resolve the device workspace and the host/device kind of the I/O pointers.
// In host mode, inputs are copied H2D into the staging buffer here.
struct Call {
    bool host = false;
    Io io[5];
    int nio = 0;
    char* ws = nullptr;
};

static dbp_status begin_call(dbp_ctx* c, Call& k, const Layout& L, void* ws, size_t ws_bytes, cudaStream_t st) {
    bool any_dev = false, any_host = false;
    for (int i = 0; i < k.nio; ++i) {
        const void* p = k.io[i].host_in ? k.io[i].host_in : k.io[i].host_out;
        if (!p) continue;
        (is_device_ptr(p) ? any_dev : any_host) = true;
    }
    if (any_dev && any_host) return fail(DBP_ERR_INVALID_ARG, "mixed host and device pointers in one call");
    k.host = any_host;
    if (ws) {
        if (ws_bytes < L.total) return fail(DBP_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, L.total);
        if (!is_device_ptr(ws)) return fail(DBP_ERR_INVALID_ARG, "workspace must be device memory");
        k.ws = static_cast<char*>(ws);
    } else if (L.total) {
        dbp_status s = ensure_iws(c, L.total);
        if (s) return s;
        k.ws = static_cast<char*>(c->iws);
    }
    if (!k.host) {
        for (int i = 0; i < k.nio; ++i) k.io[i].dev = k.io[i].host_in ? const_cast<void*>(k.io[i].host_in) : k.io[i].host_out;
        return DBP_OK;
    }
    size_t need = 0;
    for (int i = 0; i < k.nio; ++i) need += al(k.io[i].bytes);
    dbp_status s = ensure_stage(c, need);
    if (s) return s;
    size_t o = 0;
    for (int i = 0; i < k.nio; ++i) {
        k.io[i].dev = (k.io[i].host_in || k.io[i].host_out) ? static_cast<char*>(c->stage) + o : nullptr;
        o += al(k.io[i].bytes);
        if (k.io[i].host_in) CU(cudaMemcpyAsync(k.io[i].dev, k.io[i].host_in, k.io[i].bytes, cudaMemcpyHostToDevice, st));
    }
    return DBP_OK;
}

static dbp_status end_call(dbp_ctx*, Call& k, cudaStream_t st) {
    if (!k.host) return DBP_OK;
    for (int i = 0; i < k.nio; ++i)
        if (k.io[i].host_out) CU(cudaMemcpyAsync(k.io[i].host_out, k.io[i].dev, k.io[i].bytes, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return DBP_OK;
}

static dbp_status allreduce(dbp_ctx* c, float2* buf, size_t nfloat2, cudaStream_t st, bool round = true) {
    if (round) c->consensus_rounds += 1;
    if (c->world == 1) return DBP_OK;
    if (!c->comm) {
        // host hook (dbp_set_allreduce_hook): D2H, sum over ranks on the host, H2D
        if (!c->hook) return fail(DBP_ERR_NCCL, "world %d context without a communicator or allreduce hook", c->world);
        const size_t bytes = nfloat2 * 8;
        if (c->hbuf_bytes < bytes) {
            if (c->hbuf) cudaFreeHost(c->hbuf);
            c->hbuf = nullptr;
            c->hbuf_bytes = 0;
            CU(cudaMallocHost(&c->hbuf, bytes));
            c->hbuf_bytes = bytes;
        }
        CU(cudaMemcpyAsync(c->hbuf, buf, bytes, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (c->hook(c->hbuf, (int64_t)(nfloat2 * 2), c->hook_user) != 0)
            return fail(DBP_ERR_NCCL, "allreduce hook failed (rank %d)", c->rank);
        CU(cudaMemcpyAsync(buf, c->hbuf, bytes, cudaMemcpyHostToDevice, st));
        c->allreduce_calls += 1;
        c->allreduce_bytes += (int64_t)bytes;
        return DBP_OK;
    }
    NC(ncclAllReduce(buf, buf, nfloat2 * 2, ncclFloat32, ncclSum, c->comm, st));
    c->allreduce_calls += 1;
    c->allreduce_bytes += (int64_t)(nfloat2 * 8);
    return DBP_OK;
}

// Multi-launch schedules (preprocessing + per-round kernels + the NCCL allreduces between them)
// are captured once per (solver, shape, scalars, pointers) into a CUDA graph and replayed: one
// cudaGraphLaunch instead of T + 2 kernel launches and T collectives issued from the host
// (SURVEY 5 "capture the NCCL calls in a CUDA graph").  Capture runs on a library stream (the
// caller's may be the legacy default stream, which cannot be captured); the graph is launched
// on the caller's stream.  Not used for host-pointer calls (their staging is outside) or under
// DBP_OPT_KERNEL_TIMING (per-kernel events).  Counters (launches, allreduces, rounds) advance on
// every replay by the amounts the captured schedule issued.
template <class F>
static dbp_status graphed(dbp_ctx* c, bool host, cudaStream_t s, const std::vector<uint64_t>& key, F&& body) {
    if (!c->graphs || host || c->timing || (c->world > 1 && !c->comm)) return body(s);
    ++c->gclock;
    for (auto& g : c->gcache) {
        if (g.key != key) continue;
        g.used = c->gclock;
        CU(cudaGraphLaunch(g.exec, s));
        c->launches += g.launches;
        c->allreduce_calls += g.ar_calls;
        c->allreduce_bytes += g.ar_bytes;
        c->consensus_rounds += g.rounds;
        ++c->graph_replays;
        return DBP_OK;
    }
    if (!c->cap) CU(cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking));
    const int64_t l0 = c->launches, a0 = c->allreduce_calls, b0 = c->allreduce_bytes, r0 = c->consensus_rounds;
    CU(cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeRelaxed));
    dbp_status st = body(c->cap);
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(c->cap, &graph);
    cudaGraphExec_t exec = nullptr;
    cudaError_t ei = cudaErrorUnknown;
    if (!st && e == cudaSuccess) ei = cudaGraphInstantiate(&exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (st || e != cudaSuccess || ei != cudaSuccess) {
        // nothing ran during the capture: undo its bookkeeping, stop capturing on this context and
        // issue the schedule with plain launches (an argument error simply recurs there)
        cudaGetLastError();
        c->launches = l0;
        c->allreduce_calls = a0;
        c->allreduce_bytes = b0;
        c->consensus_rounds = r0;
        c->graphs = 0;
        return body(s);
    }
    if (c->gcache.size() >= 16) {                      // evict the least recently used
        size_t v = 0;
        for (size_t i = 1; i < c->gcache.size(); ++i)
            if (c->gcache[i].used < c->gcache[v].used) v = i;
        cudaGraphExecDestroy(c->gcache[v].exec);
        c->gcache.erase(c->gcache.begin() + (long)v);
    }
    c->gcache.push_back({key, exec, c->launches - l0, c->allreduce_calls - a0, c->allreduce_bytes - b0,
                         c->consensus_rounds - r0, c->gclock});
    CU(cudaGraphLaunch(exec, s));
    return DBP_OK;
}

static uint64_t fbits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static uint64_t pbits(const void* p) { return reinterpret_cast<uintptr_t>(p); }

#define KL(call)                                                                               \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) return fail(DBP_ERR_CUDA, "launch %s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

// Launch with optional per-kernel event timing on the launch stream.
#define KT(name, call)                                                                         \
    do {                                                                                       \
        cudaEvent_t e0_ = nullptr;                                                             \
        if (c->timing) { e0_ = ev_get(c); cudaEventRecord(e0_, s); }                            \
        KL(call);                                                                              \
        if (c->timing) {                                                                       \
            cudaEvent_t e1_ = ev_get(c);                                                       \
            cudaEventRecord(e1_, s);                                                           \
            c->pending.push_back({kname_id(c, name), e0_, e1_});                                \
        }                                                                                      \
    } while (0)

static Prox make_prox(int reg, int mod, int C, float rho, float N0, float Es) {
    Prox p;
    p.reg = reg;
    p.inv_c = (float)(1.0 / C);
    p.mmse_scale = (float)(1.0 / ((double)N0 / ((double)rho * Es) + C));
    p.r = modem_of(mod).radius;
    p.bpsk = mod == DBP_BPSK;
    return p;
}

static bool mod_ok(int mod) { return mod == DBP_BPSK || mod == DBP_QPSK || mod == DBP_QAM16 || mod == DBP_QAM64; }

// ------------------------------------------------ device-side consensus (NEXT-1)
// Symmetric per-rank buffer: part [2][8][cap][16] uint4 (layout in dbp_internal.h).
static size_t xbuf_bytes(int cap) { return (size_t)2 * 8 * cap * 16 * 16; }

// Collective when world > 1 (every rank calls it with the same N): allocate the buffer and map
// every rank's buffer through CUDA IPC handles exchanged by one ncclAllGather.
static dbp_status xbuf_ensure(dbp_ctx* c, int N, cudaStream_t s) {
    if (c->xbuf && c->xcap >= N) return DBP_OK;
    CU(cudaStreamSynchronize(s));
    for (int r = 0; r < 8; ++r) {
        if (c->xpeer[r] && c->xpeer[r] != c->xbuf) cudaIpcCloseMemHandle(c->xpeer[r]);
        c->xpeer[r] = nullptr;
    }
    if (c->xbuf) cudaFree(c->xbuf);
    c->xbuf = nullptr;
    const int cap = std::max(N, 64);
    CU(cudaMalloc(&c->xbuf, xbuf_bytes(cap)));
    CU(cudaMemset(c->xbuf, 0, xbuf_bytes(cap)));
    c->xcap = cap;
    c->xround = 1;
    c->xpeer[c->rank] = c->xbuf;
    if (c->world > 1) {
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
        cudaIpcMemHandle_t h;
        CU(cudaIpcGetMemHandle(&h, c->xbuf));
        uint8_t* dh = nullptr;
        CU(cudaMalloc(&dh, (size_t)64 * (c->world + 1)));
        CU(cudaMemcpyAsync(dh + (size_t)64 * c->world, &h, 64, cudaMemcpyHostToDevice, s));
        NC(ncclAllGather(dh + (size_t)64 * c->world, dh, 64, ncclUint8, c->comm, s));
        std::vector<cudaIpcMemHandle_t> all(c->world);
        CU(cudaMemcpyAsync(all.data(), dh, (size_t)64 * c->world, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        cudaFree(dh);
        for (int r = 0; r < c->world; ++r) {
            if (r == c->rank) continue;
            CU(cudaIpcOpenMemHandle(&c->xpeer[r], all[r], cudaIpcMemLazyEnablePeerAccess));
        }
    }
    return DBP_OK;
}

// Consensus-exchange arguments for one call with `rounds` rounds (nullptr: not in use).
static bool xcons_active(const dbp_ctx* c) {
    return c->xcons == 2 || (c->xcons == 1 && c->world > 1 && c->comm);
}

static XArgs xargs_for(dbp_ctx* c, int rounds) {
    XArgs x{};
    x.on = 1;
    x.world = c->world;
    x.rank = c->rank;
    x.cap = c->xcap;
    for (int r = 0; r < c->world; ++r) x.part[r] = static_cast<uint4*>(c->xpeer[r]);
    // This call's rounds use ids base + 1 .. base + rounds; the next call continues at
    // base + rounds + 1, so consecutive rounds -- also across calls -- alternate buffer parity
    // (the two-buffer argument of DESIGN.md section 7 needs consecutive ids).
    x.base = c->xround;
    c->xround += (unsigned)rounds;
    return x;
}

// Device consensus preconditions that can differ between ranks (checked before any rank-local
// launch decision, so a rank never silently leaves the protocol its peers are spinning in).
static dbp_status xc_check(const void* a, const void* b) {
    if ((reinterpret_cast<uintptr_t>(a) & 15) || (reinterpret_cast<uintptr_t>(b) & 15))
        return fail(DBP_ERR_UNSUPPORTED, "device consensus needs 16-byte aligned H / y (TMA); peers will time out");
    return DBP_OK;
}

// ============================================================ Algorithm 1
extern "C" dbp_status dbp_detect_admm(dbp_ctx* c, const dbp_dims* d, const dbp_cf32* H, const dbp_cf32* y,
                                      float rho, float gamma, float N0, float Es, int reg, int mod, int32_t T,
                                      dbp_cf32* s_hat, uint8_t* hard, void* ws, size_t ws_bytes, void* stream) {
    Shape sh;
    dbp_status st = check_dims(c, d, &sh);
    if (st) return st;
    if (sh.N > 0 && (!H || !y || !s_hat)) return fail(DBP_ERR_INVALID_ARG, "H, y and s_hat are required");
    if (!(rho > 0.f) || !std::isfinite(rho)) return fail(DBP_ERR_INVALID_ARG, "rho must be > 0 (SPEC S54)");
    if (!(gamma > 0.f) || !std::isfinite(gamma)) return fail(DBP_ERR_INVALID_ARG, "gamma must be > 0");
    if (!(Es > 0.f) || !(N0 >= 0.f) || !std::isfinite(N0) || !std::isfinite(Es)) return fail(DBP_ERR_INVALID_ARG, "need N0 >= 0, Es > 0");
    if (reg < 0 || reg > 2) return fail(DBP_ERR_INVALID_ARG, "reg %d", reg);
    if (!mod_ok(mod)) return fail(DBP_ERR_INVALID_ARG, "mod %d", mod);
    if (T < 1) return fail(DBP_ERR_INVALID_ARG, "T must be >= 1");
    if (prelr_smem(sh.UP, sh.S, sh.U, sh.J, true) > (size_t)c->max_smem) return fail(DBP_ERR_UNSUPPORTED, "S too large for the preprocessing tile");
    if (sh.N == 0) return DBP_OK;                 // empty frame: nothing to compute or exchange
    CU(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const Layout Lw = layout(sh, DBP_ALGO_ADMM_UL);
    Call k;
    k.io[0] = {H, nullptr, (size_t)sh.pairs() * sh.S * sh.U * 8, nullptr};
    k.io[1] = {y, nullptr, (size_t)sh.pairs() * sh.J * sh.S * 8, nullptr};
    k.io[2] = {nullptr, s_hat, (size_t)sh.N * sh.J * sh.U * 8, nullptr};
    k.io[3] = {nullptr, hard, hard ? (size_t)sh.N * sh.J * sh.U : 0, nullptr};
    k.nio = 4;
    if ((st = begin_call(c, k, Lw, ws, ws_bytes, s))) return st;
    const float2* dH = static_cast<const float2*>(k.io[0].dev);
    const float2* dy = static_cast<const float2*>(k.io[1].dev);
    float2* G = reinterpret_cast<float2*>(k.ws + Lw.off[0]);
    float2* mf = reinterpret_cast<float2*>(k.ws + Lw.off[1]);
    LaunchCtx L{s, c->d_flag, &c->launches};

    if (sh.ss) {
        // S x S form (Alg. 1 lines 3-5, 13; eq. (4)): A_c^{-1}, y^reg = H^H A^{-1} y, then one launch
        // per round with the allreduce in between (T rounds), s_hat = prox of the last sum
        SsArgs a{};
        a.H = dH; a.y = dy;
        a.Ainv = G;
        a.yreg = reinterpret_cast<float2*>(k.ws + Lw.off[2]);
        a.lam = reinterpret_cast<float2*>(k.ws + Lw.off[3]);
        a.st = reinterpret_cast<float2*>(k.ws + Lw.off[4]);
        a.wbuf = reinterpret_cast<float2*>(k.ws + Lw.off[5]);
        a.flag = c->d_flag;
        a.C_loc = sh.C_loc; a.N = sh.N; a.J = sh.J; a.S = sh.S; a.U = sh.U; a.UPW = sh.UP; a.T = T;
        a.delta = rho; a.rho = rho; a.gamma = gamma;
        a.px = make_prox(reg, mod, sh.C, rho, N0, Es);
        const std::vector<uint64_t> key{10, (uint64_t)sh.C, (uint64_t)sh.S, (uint64_t)sh.U, (uint64_t)sh.N, (uint64_t)sh.J, (uint64_t)T, (uint64_t)sh.ss, (uint64_t)c->force_split, (uint64_t)c->no_fused, (uint64_t)reg, (uint64_t)mod, fbits(rho), fbits(gamma),
                                        fbits(N0), fbits(Es), pbits(dH), pbits(dy), pbits(k.io[2].dev),
                                        pbits(k.io[3].dev), pbits(k.ws)};
        st = graphed(c, k.host, s, key, [&](cudaStream_t s) -> dbp_status {
            LaunchCtx L{s, c->d_flag, &c->launches};
            dbp_status st;
            KT("pre_ss_ul", launch_ss_pre(L, false, a));
            const size_t nw = (size_t)sh.N * sh.J * sh.UP;
            for (int t = 1; t <= T; ++t) {
                a.step = t;
                KT("ss_ul_step", launch_ss_it(L, false, a));                      // lines 12-17 (t = 1: 10)
                if ((st = allreduce(c, a.wbuf, nw, s))) return st;              // line 18 consensus
            }
            KT("prox_out", launch_prox_out(L, sh.UP, a.wbuf, sh.N, sh.J, sh.U, a.px, modem_of(mod),
                                           static_cast<float2*>(k.io[2].dev), static_cast<uint8_t*>(k.io[3].dev)));
            return DBP_OK;
        });
        if (st) return st;
        return end_call(c, k, s);
    }
    if (c->world == 1 && !c->force_split && !c->no_fused && sh.J > 1 && gamma == 1.f) {
        // N_sym > 1 in one per-subcarrier kernel (the Gram and B_c^{-1} serve all symbols, P706-709)
        bool launched = false;
        KT("fused_ulj", (launched = launch_fused_ulj(L, sh.UP, false, dH, dy, sh.C_loc, sh.N, sh.S, sh.U, sh.J, T, rho,
                                                     make_prox(reg, mod, sh.C, rho, N0, Es), modem_of(mod),
                                                     static_cast<float2*>(k.io[2].dev),
                                                     static_cast<uint8_t*>(k.io[3].dev)),
                         cudaGetLastError()));
        if (launched) {
            c->consensus_rounds += T;
            return end_call(c, k, s);
        }
    }
    const bool xc_on = xcons_active(c) && T < 250;
    if ((c->world == 1 || xc_on) && !c->force_split && !c->no_fused &&
        fused_ok(sh.UP, sh.C_loc, sh.N, sh.J, sh.S, sh.U)) {
        // a1-a8 in one per-subcarrier kernel (world == 1, or world > 1 with device-side consensus)
        XArgs xa{};
        if (xc_on) {
            if ((st = xc_check(dH, dy))) return st;
            if ((st = xbuf_ensure(c, sh.N, s))) return st;
            xa = xargs_for(c, T);
        }
        bool launched = false;
        L.pdl = c->pdl && !xc_on;
        KT("fused_ul", (launched = launch_fused_ul(L, sh.UP, false, dH, dy, sh.C_loc, sh.N, sh.S, sh.U, T, rho, gamma,
                                                   make_prox(reg, mod, sh.C, rho, N0, Es), modem_of(mod),
                                                   static_cast<float2*>(k.io[2].dev),
                                                   static_cast<uint8_t*>(k.io[3].dev), xc_on ? &xa : nullptr),
                        cudaGetLastError()));
        if (launched) {
            c->consensus_rounds += T;
            return end_call(c, k, s);
        }
        if (xc_on) return fail(DBP_ERR_CUDA, "fused ADMM-UL launch with device consensus failed (rank %d)", c->rank);
    }
    float2* yreg = reinterpret_cast<float2*>(k.ws + Lw.off[2]);
    const std::vector<uint64_t> key{11, (uint64_t)sh.C, (uint64_t)sh.S, (uint64_t)sh.U, (uint64_t)sh.N, (uint64_t)sh.J, (uint64_t)T, (uint64_t)sh.ss, (uint64_t)c->force_split, (uint64_t)c->no_fused, (uint64_t)reg, (uint64_t)mod, fbits(rho), fbits(gamma), fbits(N0),
                                    fbits(Es), pbits(dH), pbits(dy), pbits(k.io[2].dev), pbits(k.io[3].dev),
                                    pbits(k.ws)};
    st = graphed(c, k.host, s, key, [&](cudaStream_t s) -> dbp_status {
    LaunchCtx L{s, c->d_flag, &c->launches};
    dbp_status st;
    // a1-a3: G_c = H_c^H H_c + rho I, B_c^{-1} and y^reg = B_c^{-1} H_c^H y_c (Alg. 1 lines 7-8)
    KT("pre_ul", launch_prelr(L, sh.UP, 1, dH, dy, sh.S, sh.U, sh.J, sh.pairs(), rho, G, yreg));

    UlArgs a{};
    a.G = G; a.mf = mf; a.Ginv = G;
    a.yreg = yreg;
    a.lam = reinterpret_cast<float2*>(k.ws + Lw.off[3]);
    a.z = reinterpret_cast<float2*>(k.ws + Lw.off[4]);
    a.wbuf = reinterpret_cast<float2*>(k.ws + Lw.off[5]);
    a.s_hat = static_cast<float2*>(k.io[2].dev);
    a.hard = static_cast<uint8_t*>(k.io[3].dev);
    a.flag = c->d_flag;
    a.C_loc = sh.C_loc; a.N = sh.N; a.J = sh.J; a.U = sh.U; a.T = T;
    a.rho = rho; a.gamma = gamma;
    a.wonly = gamma == 1.f;                 // split rounds: w-only state (5504 -> 4992 B per pair at UP = 32)
    a.px = make_prox(reg, mod, sh.C, rho, N0, Es);
    a.md = modem_of(mod);
    int NT, CCH;
    if (c->world == 1 && !c->force_split && iter_cfg(sh.UP, sh.C_loc, sh.N, c->max_smem, &NT)) {
        // a4-a8 fused: all T iterations on chip (world == 1)
        a.NT = NT;
        KT("admm_fused", launch_admm_gj(L, sh.UP, a));
        c->consensus_rounds += T;
    } else {
        split_cfg(sh.UP, sh.C_loc, sh.N, sh.J, &NT, &CCH);
        a.NT = NT;
        const size_t nw = (size_t)sh.N * sh.J * sh.UP;
        for (int t = 1; t <= T; ++t) {
            a.init = (t == 1);
            KT("admm_step", launch_admm_it(L, sh.UP, a, CCH));              // lines 12-17 (t = 1: line 10)
            if ((st = allreduce(c, a.wbuf, nw, s))) return st;              // line 18 consensus
        }
        KT("prox_out", launch_prox_out(L, sh.UP, a.wbuf, sh.N, sh.J, sh.U, a.px, a.md, a.s_hat, a.hard));  // line 19
    }
    return DBP_OK;
    });
    if (st) return st;
    return end_call(c, k, s);
}

// ============================================================ Algorithm 2
extern "C" dbp_status dbp_detect_cg(dbp_ctx* c, const dbp_dims* d, const dbp_cf32* H, const dbp_cf32* y, float rho,
                                    int mod, int32_t T, dbp_cf32* x_hat, uint8_t* hard, void* ws, size_t ws_bytes,
                                    void* stream) {
    Shape sh;
    dbp_status st = check_dims(c, d, &sh);
    if (st) return st;
    if (sh.N > 0 && (!H || !y || !x_hat)) return fail(DBP_ERR_INVALID_ARG, "H, y and x_hat are required");
    if (!(rho >= 0.f) || !std::isfinite(rho)) return fail(DBP_ERR_INVALID_ARG, "rho must be >= 0 (P376)");
    if (!mod_ok(mod)) return fail(DBP_ERR_INVALID_ARG, "mod %d", mod);
    if (T < 1) return fail(DBP_ERR_INVALID_ARG, "T must be >= 1");
    if (prelr_smem(sh.UP, sh.S, sh.U, sh.J, true) > (size_t)c->max_smem) return fail(DBP_ERR_UNSUPPORTED, "S too large for the preprocessing tile");
    if (sh.N == 0) return DBP_OK;                 // empty frame: nothing to compute or exchange
    CU(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const Layout Lw = layout(sh, DBP_ALGO_CG_UL);
    Call k;
    k.io[0] = {H, nullptr, (size_t)sh.pairs() * sh.S * sh.U * 8, nullptr};
    k.io[1] = {y, nullptr, (size_t)sh.pairs() * sh.J * sh.S * 8, nullptr};
    k.io[2] = {nullptr, x_hat, (size_t)sh.N * sh.J * sh.U * 8, nullptr};
    k.io[3] = {nullptr, hard, hard ? (size_t)sh.N * sh.J * sh.U : 0, nullptr};
    k.nio = 4;
    if ((st = begin_call(c, k, Lw, ws, ws_bytes, s))) return st;
    LaunchCtx L{s, c->d_flag, &c->launches};
    float2* Gp = reinterpret_cast<float2*>(k.ws + Lw.off[0]);
    float2* mf = reinterpret_cast<float2*>(k.ws + Lw.off[1]);
    CgArgs a{};
    a.Gloc = reinterpret_cast<float2*>(k.ws + Lw.off[2]);
    a.wbuf = reinterpret_cast<float2*>(k.ws + Lw.off[3]);
    a.x = reinterpret_cast<float2*>(k.ws + Lw.off[4]);
    a.r = reinterpret_cast<float2*>(k.ws + Lw.off[5]);
    a.p = reinterpret_cast<float2*>(k.ws + Lw.off[6]);
    a.rr = reinterpret_cast<float*>(k.ws + Lw.off[7]);
    a.x_hat = static_cast<float2*>(k.io[2].dev);
    a.hard = static_cast<uint8_t*>(k.io[3].dev);
    a.N = sh.N; a.J = sh.J; a.U = sh.U; a.T = T; a.rho = rho;
    a.md = modem_of(mod);

    if (c->cg_tc && c->world == 1 && !c->force_split && !c->no_fused && !xcons_active(c) &&
        cg_tc_ok(sh.UP, sh.J, sh.N, sh.C_loc, sh.S)) {
        // b1-b5 with the cluster-summed Gram on the tensor cores (long K = C * S): one kernel
        bool launched = false;
        L.pdl = c->pdl;
        KT("cg_tc", (launched = launch_cg_tc(L, sh.UP, static_cast<const float2*>(k.io[0].dev),
                                             static_cast<const float2*>(k.io[1].dev), sh.C_loc, sh.N, sh.S, sh.U,
                                             sh.J, T, rho, modem_of(mod), a.x_hat, a.hard), cudaGetLastError()));
        if (launched) {
            c->consensus_rounds += T + 1;
            return end_call(c, k, s);
        }
    }
    if (c->world == 1 && !c->force_split && !c->no_fused && sh.J > 1) {
        // N_sym > 1 in one per-subcarrier kernel (G and the J matched filters summed once, J CG solves)
        bool launched = false;
        KT("fused_cgj", (launched = launch_fused_ulj(L, sh.UP, true, static_cast<const float2*>(k.io[0].dev),
                                                     static_cast<const float2*>(k.io[1].dev), sh.C_loc, sh.N, sh.S,
                                                     sh.U, sh.J, T, rho, Prox{}, modem_of(mod), a.x_hat, a.hard),
                         cudaGetLastError()));
        if (launched) {
            c->consensus_rounds += T + 1;
            return end_call(c, k, s);
        }
    }
    const bool xc_on = xcons_active(c) && T < 250;
    if ((c->world == 1 || xc_on) && !c->force_split && !c->no_fused &&
        fused_ok(sh.UP, sh.C_loc, sh.N, sh.J, sh.S, sh.U)) {
        // b1-b5 in one per-subcarrier kernel (world == 1, or world > 1 with device-side consensus)
        XArgs xa{};
        if (xc_on) {
            if ((st = xc_check(k.io[0].dev, k.io[1].dev))) return st;
            if ((st = xbuf_ensure(c, sh.N, s))) return st;
            xa = xargs_for(c, T + 1);
        }
        bool launched = false;
        L.pdl = c->pdl && !xc_on;
        KT("fused_cg", (launched = launch_fused_ul(L, sh.UP, true, static_cast<const float2*>(k.io[0].dev),
                                                   static_cast<const float2*>(k.io[1].dev), sh.C_loc, sh.N, sh.S,
                                                   sh.U, T, rho, 1.f, Prox{}, modem_of(mod), a.x_hat, a.hard,
                                                   xc_on ? &xa : nullptr),
                        cudaGetLastError()));
        if (launched) {
            c->consensus_rounds += T + 1;
            return end_call(c, k, s);
        }
        if (xc_on) return fail(DBP_ERR_CUDA, "fused CG launch with device consensus failed (rank %d)", c->rank);
    }
    const std::vector<uint64_t> key{12, (uint64_t)sh.C, (uint64_t)sh.S, (uint64_t)sh.U, (uint64_t)sh.N, (uint64_t)sh.J, (uint64_t)T, (uint64_t)sh.ss, (uint64_t)c->force_split, (uint64_t)c->no_fused, (uint64_t)c->cg_tc, (uint64_t)mod, fbits(rho), pbits(k.io[0].dev), pbits(k.io[1].dev),
                                    pbits(k.io[2].dev), pbits(k.io[3].dev), pbits(k.ws)};
    st = graphed(c, k.host, s, key, [&](cudaStream_t s) -> dbp_status {
    LaunchCtx L{s, c->d_flag, &c->launches};
    dbp_status st;
    // b1: the per-GPU sums G_loc = sum_c H_c^H H_c and local y^MRC -- one tensor-core pass over H
    // (k_cgg_tc), else per-pair Grams and matched filters summed in fixed cluster order.
    bool gtc = false;
    if (c->cg_tc && cgg_tc_ok(sh.UP, sh.J, sh.N, sh.C_loc, sh.S, sh.U))
        KT("cgg_tc", (gtc = launch_cgg_tc(L, sh.UP, static_cast<const float2*>(k.io[0].dev),
                                          static_cast<const float2*>(k.io[1].dev), sh.C_loc, sh.N, sh.S, sh.U,
                                          const_cast<float2*>(a.Gloc), a.wbuf),
                      cudaGetLastError()));
    if (!gtc) {
        KT("pre_cg", launch_prelr(L, sh.UP, 0, static_cast<const float2*>(k.io[0].dev),
                                  static_cast<const float2*>(k.io[1].dev), sh.S, sh.U, sh.J, sh.pairs(), 0.f, Gp, mf));
        KT("cg_gsum", launch_cg_gsum(L, sh.UP, Gp, mf, sh.C_loc, sh.N, sh.J, const_cast<float2*>(a.Gloc), a.wbuf));
    }
    const size_t nw = (size_t)sh.N * sh.J * sh.UP;
    if ((st = allreduce(c, a.wbuf, nw, s))) return st;              // line 4: y^MRC consensus
    if (c->world == 1 && !c->force_split) {
        KT("cg_fused", launch_cg_it(L, sh.UP, true, a));                          // lines 6-18, all T iterations
        c->consensus_rounds += T;
    } else {
        for (int t = 0; t <= T; ++t) {
            a.step = t;
            KT("cg_step", launch_cg_it(L, sh.UP, false, a));
            if (t < T && (st = allreduce(c, a.wbuf, nw, s))) return st;   // line 11 consensus
        }
    }
    return DBP_OK;
    });
    if (st) return st;
    return end_call(c, k, s);
}

// ============================================================ Algorithm 3
extern "C" dbp_status dbp_beamform_admm(dbp_ctx* c, const dbp_dims* d, const dbp_cf32* Hd, const dbp_cf32* sv,
                                        float rho, float gamma, float eps, int32_t T, dbp_cf32* x, void* ws,
                                        size_t ws_bytes, void* stream) {
    Shape sh;
    dbp_status st = check_dims(c, d, &sh);
    if (st) return st;
    if (sh.N > 0 && (!Hd || !sv || !x)) return fail(DBP_ERR_INVALID_ARG, "Hd, s and x are required");
    if (!(rho > 0.f) || !std::isfinite(rho)) return fail(DBP_ERR_INVALID_ARG, "rho must be > 0");
    if (!(gamma > 0.f) || !std::isfinite(gamma)) return fail(DBP_ERR_INVALID_ARG, "gamma must be > 0");
    if (!(eps >= 0.f)) return fail(DBP_ERR_INVALID_ARG, "eps must be >= 0");
    if (!std::isfinite(eps)) return fail(DBP_ERR_INVALID_ARG, "eps must be finite");
    if (T < 1) return fail(DBP_ERR_INVALID_ARG, "T must be >= 1");
    if (prelr_smem(sh.UP, sh.S, sh.U, sh.J, false) > (size_t)c->max_smem) return fail(DBP_ERR_UNSUPPORTED, "S too large for the preprocessing tile");
    if (sh.N == 0) return DBP_OK;                 // empty frame: nothing to compute or exchange
    CU(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const Layout Lw = layout(sh, DBP_ALGO_ADMM_DL);
    Call k;
    k.io[0] = {Hd, nullptr, (size_t)sh.pairs() * sh.S * sh.U * 8, nullptr};
    k.io[1] = {sv, nullptr, (size_t)sh.N * sh.J * sh.U * 8, nullptr};
    k.io[2] = {nullptr, x, (size_t)sh.pairs() * sh.J * sh.S * 8, nullptr};
    k.nio = 3;
    if ((st = begin_call(c, k, Lw, ws, ws_bytes, s))) return st;
    LaunchCtx L{s, c->d_flag, &c->launches};
    DlArgs a{};
    a.Hd = static_cast<const float2*>(k.io[0].dev);
    a.s = static_cast<const float2*>(k.io[1].dev);
    float2* G = reinterpret_cast<float2*>(k.ws + Lw.off[0]);
    a.G = G; a.Binv = G;
    a.m = reinterpret_cast<float2*>(k.ws + Lw.off[1]);
    a.lam = reinterpret_cast<float2*>(k.ws + Lw.off[2]);
    a.wbuf = reinterpret_cast<float2*>(k.ws + Lw.off[3]);
    a.x = static_cast<float2*>(k.io[2].dev);
    a.flag = c->d_flag;
    a.C_loc = sh.C_loc; a.C = sh.C; a.N = sh.N; a.J = sh.J; a.U = sh.U; a.S = sh.S; a.T = T;
    a.rho_inv = (float)(1.0 / rho);
    a.gamma = gamma;
    a.a0 = (float)std::max((double)sh.U / ((double)sh.C * sh.S), 1.0 / sh.C);   // Alg. 3 line 8 (P507)
    a.inv_c = (float)(1.0 / sh.C);
    a.eps = eps;

    if (sh.ss) {
        // S x S form (Alg. 3 lines 3-4, 9, 17): A_c^{-1} = (H_c^H H_c + rho^{-1} I_S)^{-1}; one launch per
        // round, T - 1 allreduces (the first iteration is local, P811)
        SsArgs b{};
        b.H = a.Hd; b.s = a.s; b.x = a.x;
        b.Ainv = G;
        b.st = a.m; b.lam = a.lam; b.wbuf = a.wbuf;
        b.flag = c->d_flag;
        b.C_loc = sh.C_loc; b.N = sh.N; b.J = sh.J; b.S = sh.S; b.U = sh.U; b.UPW = sh.UP; b.T = T;
        b.delta = a.rho_inv; b.gamma = gamma; b.a0 = a.a0; b.inv_c = a.inv_c; b.eps = eps;
        const std::vector<uint64_t> key{13, (uint64_t)sh.C, (uint64_t)sh.S, (uint64_t)sh.U, (uint64_t)sh.N, (uint64_t)sh.J, (uint64_t)T, (uint64_t)sh.ss, (uint64_t)c->force_split, (uint64_t)c->no_fused, fbits(rho), fbits(gamma), fbits(eps), pbits(a.Hd), pbits(a.s),
                                        pbits(a.x), pbits(k.ws)};
        st = graphed(c, k.host, s, key, [&](cudaStream_t s) -> dbp_status {
            LaunchCtx L{s, c->d_flag, &c->launches};
            dbp_status st;
            KT("pre_ss_dl", launch_ss_pre(L, true, b));
            const size_t nw = (size_t)sh.N * sh.J * sh.UP;
            b.step = 0;
            KT("ss_dl_step", launch_ss_it(L, true, b));                            // lines 8-9 (+ 11-12)
            if (T > 1 && (st = allreduce(c, b.wbuf, nw, s))) return st;
            for (int t = 2; t <= T; ++t) {
                b.step = t;
                KT("ss_dl_step", launch_ss_it(L, true, b));                        // lines 14-17 (+ 11-12)
                if (t < T && (st = allreduce(c, b.wbuf, nw, s))) return st;      // line 13 consensus
            }
            return DBP_OK;
        });
        if (st) return st;
        return end_call(c, k, s);
    }
    const bool xc_on = xcons_active(c) && T < 250;
    if ((c->world == 1 || xc_on) && !c->force_split && !c->no_fused &&
        fused_ok(sh.UP, sh.C_loc, sh.N, sh.J, sh.S, sh.U)) {
        // c1-c4 in one per-subcarrier kernel (world == 1, or world > 1 with device-side consensus)
        XArgs xa{};
        if (xc_on) {
            if ((st = xc_check(a.Hd, a.s))) return st;
            if ((st = xbuf_ensure(c, sh.N, s))) return st;
            xa = xargs_for(c, T - 1);               // Alg. 3: T - 1 consensus rounds (P811)
        }
        bool launched = false;
        L.pdl = c->pdl && !xc_on;
        KT("fused_dl", (launched = launch_fused_dl(L, sh.UP, a.Hd, a.s, sh.C_loc, sh.C, sh.N, sh.S, sh.U, T, rho,
                                                   gamma, a.a0, eps, a.x, xc_on ? &xa : nullptr),
                        cudaGetLastError()));
        if (launched) {
            c->consensus_rounds += T - 1;
            return end_call(c, k, s);
        }
        if (xc_on) return fail(DBP_ERR_CUDA, "fused ADMM-DL launch with device consensus failed (rank %d)", c->rank);
    }
    const std::vector<uint64_t> key{14, (uint64_t)sh.C, (uint64_t)sh.S, (uint64_t)sh.U, (uint64_t)sh.N, (uint64_t)sh.J, (uint64_t)T, (uint64_t)sh.ss, (uint64_t)c->force_split, (uint64_t)c->no_fused, fbits(rho), fbits(gamma), fbits(eps), pbits(a.Hd), pbits(a.s),
                                    pbits(a.x), pbits(k.ws)};
    st = graphed(c, k.host, s, key, [&](cudaStream_t s) -> dbp_status {
    LaunchCtx L{s, c->d_flag, &c->launches};
    dbp_status st;
    // c1: B_c = H_c H_c^H + rho^{-1} I_U and its inverse (Alg. 3 lines 5-6)
    KT("pre_dl", launch_prelr(L, sh.UP, 2, a.Hd, nullptr, sh.S, sh.U, sh.J, sh.pairs(), a.rho_inv, G, nullptr));
    int NT, CCH;
    if (c->world == 1 && !c->force_split && iter_cfg(sh.UP, sh.C_loc, sh.N, c->max_smem, &NT)) {
        a.NT = NT;
        KT("bf_fused", launch_bf_gj(L, sh.UP, a));                         // c2-c4
        c->consensus_rounds += T - 1;
    } else {
        split_cfg(sh.UP, sh.C_loc, sh.N, sh.J, &NT, &CCH);
        a.NT = NT;
        const size_t nw = (size_t)sh.N * sh.J * sh.UP;
        for (int t = 2; t <= T; ++t) {
            a.step = t;
            KT("bf_step", launch_bf_it(L, sh.UP, a, CCH));                 // lines 11-12 (+14-15 of t-1)
            if ((st = allreduce(c, a.wbuf, nw, s))) return st;             // line 13 consensus
        }
        a.step = T + 1;
        KT("bf_final", launch_bf_it(L, sh.UP, a, CCH));                    // output x_c^(T) (P525)
    }
    return DBP_OK;
    });
    if (st) return st;
    return end_call(c, k, s);
}

// ============================================================ centralized baselines
extern "C" dbp_status dbp_detect_mmse(dbp_ctx* c, const dbp_dims* d, const dbp_cf32* H, const dbp_cf32* y, float N0,
                                      float Es, int mod, dbp_cf32* x_hat, uint8_t* hard, void* ws, size_t ws_bytes,
                                      void* stream) {
    Shape sh;
    dbp_status st = check_dims(c, d, &sh);
    if (st) return st;
    if (sh.N > 0 && (!H || !y || !x_hat)) return fail(DBP_ERR_INVALID_ARG, "H, y and x_hat are required");
    if (!(N0 >= 0.f) || !std::isfinite(N0) || !(Es > 0.f) || !std::isfinite(Es))
        return fail(DBP_ERR_INVALID_ARG, "need N0 >= 0, Es > 0");
    if (!mod_ok(mod)) return fail(DBP_ERR_INVALID_ARG, "mod %d", mod);
    if (prelr_smem(sh.UP, sh.S, sh.U, sh.J, true) > (size_t)c->max_smem) return fail(DBP_ERR_UNSUPPORTED, "S too large for the preprocessing tile");
    if (sh.N == 0) return DBP_OK;                 // empty frame: nothing to compute or exchange
    CU(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const Layout Lw = layout(sh, DBP_ALGO_MMSE_UL);
    Call k;
    k.io[0] = {H, nullptr, (size_t)sh.pairs() * sh.S * sh.U * 8, nullptr};
    k.io[1] = {y, nullptr, (size_t)sh.pairs() * sh.J * sh.S * 8, nullptr};
    k.io[2] = {nullptr, x_hat, (size_t)sh.N * sh.J * sh.U * 8, nullptr};
    k.io[3] = {nullptr, hard, hard ? (size_t)sh.N * sh.J * sh.U : 0, nullptr};
    k.nio = 4;
    if ((st = begin_call(c, k, Lw, ws, ws_bytes, s))) return st;
    LaunchCtx L{s, c->d_flag, &c->launches};
    const float2* dH = static_cast<const float2*>(k.io[0].dev);
    const float2* dy = static_cast<const float2*>(k.io[1].dev);
    float2* xo = static_cast<float2*>(k.io[2].dev);
    uint8_t* ho = static_cast<uint8_t*>(k.io[3].dev);
    const float reg = N0 / Es;
    if (c->world == 1 && !c->force_split && !c->no_fused && fused_ok(sh.UP, sh.C, sh.N, sh.J, sh.S, sh.U)) {
        bool launched = false;
        KT("fused_mmse", (launched = launch_fused_central(L, sh.UP, false, dH, dy, sh.C, sh.N, sh.S, sh.U, reg,
                                                          modem_of(mod), xo, ho), cudaGetLastError()));
        if (launched) return end_call(c, k, s);
    }
    float2* Gp = reinterpret_cast<float2*>(k.ws + Lw.off[0]);
    float2* mf = reinterpret_cast<float2*>(k.ws + Lw.off[1]);
    float2* Gloc = reinterpret_cast<float2*>(k.ws + Lw.off[2]);
    float2* b = reinterpret_cast<float2*>(k.ws + Lw.off[3]);
    // G = sum_c H_c^H H_c and H^H y over the rank's clusters: one tensor-core pass over H (k_cgg_tc,
    // the CG preprocessing), else per-pair Grams summed in fixed cluster order
    bool gtc = false;
    if (c->cg_tc && cgg_tc_ok(sh.UP, sh.J, sh.N, sh.C_loc, sh.S, sh.U))
        KT("cgg_tc", (gtc = launch_cgg_tc(L, sh.UP, dH, dy, sh.C_loc, sh.N, sh.S, sh.U, Gloc, b), cudaGetLastError()));
    if (!gtc) {
        KT("pre_cg", launch_prelr(L, sh.UP, 0, dH, dy, sh.S, sh.U, sh.J, sh.pairs(), 0.f, Gp, mf));
        KT("cg_gsum", launch_cg_gsum(L, sh.UP, Gp, mf, sh.C_loc, sh.N, sh.J, Gloc, b));
    }
    const size_t ng = (size_t)sh.N * sh.UP * (sh.UP + 1) / 2, nb = (size_t)sh.N * sh.J * sh.UP;
    if ((st = allreduce(c, Gloc, ng, s, false))) return st;             // gather the whole array's Gram
    if ((st = allreduce(c, b, nb, s, false))) return st;                // and matched filter
    KT("central_solve", launch_central_solve(L, sh.UP, false, Gloc, b, reg, sh.N, sh.J, sh.U, xo, ho, modem_of(mod)));
    return end_call(c, k, s);
}

extern "C" dbp_status dbp_precode_zf(dbp_ctx* c, const dbp_dims* d, const dbp_cf32* Hd, const dbp_cf32* sv,
                                     dbp_cf32* x, void* ws, size_t ws_bytes, void* stream) {
    Shape sh;
    dbp_status st = check_dims(c, d, &sh);
    if (st) return st;
    if (sh.N > 0 && (!Hd || !sv || !x)) return fail(DBP_ERR_INVALID_ARG, "Hd, s and x are required");
    if (prelr_smem(sh.UP, sh.S, sh.U, sh.J, false) > (size_t)c->max_smem) return fail(DBP_ERR_UNSUPPORTED, "S too large for the preprocessing tile");
    if (sh.N == 0) return DBP_OK;                 // empty frame: nothing to compute or exchange
    CU(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const Layout Lw = layout(sh, DBP_ALGO_ZF_DL);
    Call k;
    k.io[0] = {Hd, nullptr, (size_t)sh.pairs() * sh.S * sh.U * 8, nullptr};
    k.io[1] = {sv, nullptr, (size_t)sh.N * sh.J * sh.U * 8, nullptr};
    k.io[2] = {nullptr, x, (size_t)sh.pairs() * sh.J * sh.S * 8, nullptr};
    k.nio = 3;
    if ((st = begin_call(c, k, Lw, ws, ws_bytes, s))) return st;
    LaunchCtx L{s, c->d_flag, &c->launches};
    const float2* dH = static_cast<const float2*>(k.io[0].dev);
    const float2* ds = static_cast<const float2*>(k.io[1].dev);
    float2* xo = static_cast<float2*>(k.io[2].dev);
    if (c->world == 1 && !c->force_split && !c->no_fused && fused_ok(sh.UP, sh.C, sh.N, sh.J, sh.S, sh.U)) {
        bool launched = false;
        KT("fused_zf", (launched = launch_fused_central(L, sh.UP, true, dH, ds, sh.C, sh.N, sh.S, sh.U, 0.f,
                                                        modem_of(DBP_QPSK), xo, nullptr), cudaGetLastError()));
        if (launched) return end_call(c, k, s);
    }
    float2* Gp = reinterpret_cast<float2*>(k.ws + Lw.off[0]);
    float2* Gloc = reinterpret_cast<float2*>(k.ws + Lw.off[2]);
    float2* r = reinterpret_cast<float2*>(k.ws + Lw.off[3]);
    KT("pre_dl", launch_prelr(L, sh.UP, 3, dH, nullptr, sh.S, sh.U, sh.J, sh.pairs(), 0.f, Gp, nullptr));
    KT("cg_gsum", launch_cg_gsum(L, sh.UP, Gp, nullptr, sh.C_loc, sh.N, 0, Gloc, nullptr));
    if ((st = allreduce(c, Gloc, (size_t)sh.N * sh.UP * (sh.UP + 1) / 2, s, false))) return st;
    KT("central_solve", launch_central_solve(L, sh.UP, true, Gloc, ds, 0.f, sh.N, sh.J, sh.U, r, nullptr,
                                             modem_of(DBP_QPSK)));
    KT("zf_out", launch_zf_out(L, sh.UP, dH, r, sh.N, sh.J, sh.U, sh.S, sh.pairs(), xo));
    return end_call(c, k, s);
}

// ============================================================ utilities
extern "C" dbp_status dbp_slice(dbp_ctx* c, int mod, int64_t count, const dbp_cf32* x, uint8_t* bits, void* stream) {
    if (!c) return fail(DBP_ERR_INVALID_ARG, "ctx is NULL");
    if (!mod_ok(mod)) return fail(DBP_ERR_INVALID_ARG, "mod %d", mod);
    if (count < 0 || (count > 0 && (!x || !bits))) return fail(DBP_ERR_INVALID_ARG, "bad count/pointers");
    if (count == 0) return DBP_OK;
    CU(cudaSetDevice(c->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Call k;
    k.io[0] = {x, nullptr, (size_t)count * 8, nullptr};
    k.io[1] = {nullptr, bits, (size_t)count, nullptr};
    k.nio = 2;
    Layout Lw{};
    dbp_status st = begin_call(c, k, Lw, nullptr, 0, s);
    if (st) return st;
    LaunchCtx L{s, c->d_flag, &c->launches};
    KT("slice", launch_slice(L, static_cast<const float2*>(k.io[0].dev), count, modem_of(mod), static_cast<uint8_t*>(k.io[1].dev)));
    return end_call(c, k, s);
}

extern "C" dbp_status dbp_get_kernel_times(dbp_ctx* c, dbp_kernel_time* out, int max_entries, int* n_entries,
                                           int reset) {
    if (!c || !n_entries || max_entries < 0 || (max_entries > 0 && !out)) return fail(DBP_ERR_INVALID_ARG, "bad arguments");
    CU(cudaSetDevice(c->device));
    for (auto& p : c->pending) {
        CU(cudaEventSynchronize(p.e1));
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, p.e0, p.e1));
        c->kms[p.k] += ms;
        c->kcount[p.k] += 1;
        c->pool.push_back(p.e0);
        c->pool.push_back(p.e1);
    }
    c->pending.clear();
    int n = 0;
    for (size_t i = 0; i < c->knames.size() && n < max_entries; ++i) {
        if (!c->kcount[i]) continue;
        memset(out[n].name, 0, sizeof out[n].name);
        strncpy(out[n].name, c->knames[i].c_str(), sizeof out[n].name - 1);
        out[n].launches = c->kcount[i];
        out[n].total_ms = c->kms[i];
        ++n;
    }
    *n_entries = n;
    if (reset)
        for (size_t i = 0; i < c->knames.size(); ++i) { c->kcount[i] = 0; c->kms[i] = 0.0; }
    return DBP_OK;
}

extern "C" dbp_status dbp_sync(dbp_ctx* c, void* stream) {
    if (!c) return fail(DBP_ERR_INVALID_ARG, "ctx is NULL");
    CU(cudaSetDevice(c->device));
    CU(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    int flag = 0;
    CU(cudaMemcpy(&flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost));
    if (flag) {
        CU(cudaMemset(c->d_flag, 0, sizeof(int)));
        if (flag & DBP_FLAG_XC_TIMEOUT)
            return fail(DBP_ERR_CUDA, "device consensus timed out waiting for a peer rank's round (outputs undefined)");
        return fail(DBP_ERR_NOT_HPD, "a Cholesky pivot was not positive/finite (non-HPD or non-finite input)");
    }
    CU(cudaGetLastError());
    return DBP_OK;
}
