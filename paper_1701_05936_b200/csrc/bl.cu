// bl.cu -- host orchestrator and C ABI (include/bl.h) of the B200-native
// lasso / elastic-net path (biglasso, arXiv 1701.05936).
//
// The host side only sequences kernels and keeps the small sorted index sets
// (working set W, strong/violator lists) -- every arithmetic step of the path
// runs in the sm_100a kernels of bl_kernels.cuh.  One device->host status copy
// per KKT round decides whether to re-solve ("post-convergence check").
#include "bl.h"
#include "bl_kernels.cuh"
#include "bl_tc.cuh"

#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

using namespace bl;

namespace {

thread_local std::string g_err;

// ---- block cache for device and pinned-host allocations (process-wide)
// bl_free and workspace growth return blocks here instead of cudaFree / cudaFreeHost
// (which synchronise the device and unmap); a later allocation of a similar size
// (need <= size <= 2 need) reuses one, so repeated design loads and fits skip the
// driver's allocation path.  Callers return a block only after synchronising the
// stream that used it (as they did before cudaFree).  At most kCacheCapDev / kCacheCapHost bytes stay
// cached per device (larger or surplus blocks go back to the driver), and a failed
// allocation releases every cached block and retries.
namespace cache {
// freed blocks kept for reuse (a failed allocation flushes the cache and retries): up to 8 GB of
// device memory -- a cfg3 / cfg4-sized design reloaded in a loop reuses its buffer instead of a
// cudaMalloc + cudaFree of 4 GB per load -- and 2 GB of pinned host memory
constexpr size_t kCacheCapDev = (size_t)8 << 30, kCacheCapHost = (size_t)2 << 30;
struct Pool {
    std::mutex mu;
    std::multimap<size_t, void *> freeb;
    std::map<void *, size_t> live;
    size_t cached = 0;
};
Pool &pool(bool host) {
    static std::mutex mu;
    static std::map<int, std::unique_ptr<Pool>> pools;
    int dev = -1;
    if (!host) cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto &pp = pools[dev];
    if (!pp) pp = std::make_unique<Pool>();
    return *pp;
}
cudaError_t raw_alloc(void **p, size_t b, bool host) { return host ? cudaMallocHost(p, b) : cudaMalloc(p, b); }
void raw_free(void *p, bool host) { if (host) cudaFreeHost(p); else cudaFree(p); }
cudaError_t alloc(void **p, size_t bytes, bool host) {
    Pool &P = pool(host);
    {
        std::lock_guard<std::mutex> lk(P.mu);
        auto it = P.freeb.lower_bound(bytes);
        if (it != P.freeb.end() && it->first <= 2 * bytes) {
            *p = it->second;
            P.live[*p] = it->first;
            P.cached -= it->first;
            P.freeb.erase(it);
            return cudaSuccess;
        }
    }
    cudaError_t e = raw_alloc(p, bytes, host);
    if (e != cudaSuccess) {                          // release the cache and retry once
        cudaGetLastError();
        std::lock_guard<std::mutex> lk(P.mu);
        for (auto &kv : P.freeb) raw_free(kv.second, host);
        P.freeb.clear();
        P.cached = 0;
        e = raw_alloc(p, bytes, host);
    }
    if (e == cudaSuccess) {
        std::lock_guard<std::mutex> lk(P.mu);
        P.live[*p] = bytes;
    }
    return e;
}
void release(void *p, bool host) {
    if (!p) return;
    Pool &P = pool(host);
    std::lock_guard<std::mutex> lk(P.mu);
    auto it = P.live.find(p);
    if (it == P.live.end()) { raw_free(p, host); return; }
    const size_t b = it->second;
    P.live.erase(it);
    if (P.cached + b > (host ? kCacheCapHost : kCacheCapDev)) { raw_free(p, host); return; }
    P.freeb.emplace(b, p);
    P.cached += b;
}
// every cached block of this process back to the driver (bl_trim)
void trim() {
    for (bool host : {false, true}) {
        Pool &P = pool(host);
        std::lock_guard<std::mutex> lk(P.mu);
        for (auto &kv : P.freeb) raw_free(kv.second, host);
        P.freeb.clear();
        P.cached = 0;
    }
}
cudaError_t dmalloc(void **p, size_t bytes) { return alloc(p, bytes, false); }
cudaError_t hmalloc(void **p, size_t bytes) { return alloc(p, bytes, true); }
void dfree(void *p) { release(p, false); }
void hfree(void *p) { release(p, true); }
}  // namespace cache

enum Magic : uint32_t { MAGIC_DESIGN = 0xB1DE5160u, MAGIC_PATH = 0xB1BA7400u, MAGIC_CV = 0xB1C0FF00u,
                        MAGIC_PREP = 0xB1B4E900u, MAGIC_DEAD = 0xDEADDEADu };

struct Err {
    bl_status code;
};

[[noreturn]] void raise(bl_status code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    throw Err{code};
}

#define CK(call)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess) {                                                                  \
            cudaGetLastError(); /* do not leak a recoverable error into later checks */          \
            raise(BL_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
        }                                                                                         \
    } while (0)
#define CKL()                                                                                     \
    do {                                                                                          \
        cudaError_t e_ = cudaGetLastError();                                                      \
        if (e_ != cudaSuccess) raise(BL_ERR_CUDA, "kernel launch: %s (%s:%d)",                    \
                                     cudaGetErrorString(e_), __FILE__, __LINE__);                 \
    } while (0)
#define CKN(call)                                                                                 \
    do {                                                                                          \
        ncclResult_t r_ = (call);                                                                 \
        if (r_ != ncclSuccess) raise(BL_ERR_NCCL, "%s: %s", #call, ncclGetErrorString(r_));       \
    } while (0)

constexpr int kListPrefix = 2048;   // list entries copied back with each round's status
int itemsize(int dt) { return dt == DT_F64 ? 8 : dt == DT_F32 ? 4 : 1; }
int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

}  // namespace

// ------------------------------------------------------------ communicators
// Collectives of the sharded path.  Every call is collective and
// ENQUEUED on stream `st` (the result is valid for later work on st); wait(st) blocks the
// host until st is done -- with NCCL it also polls the communicator's asynchronous error
// and aborts it after the timeout.  group_begin/end batch the calls between them into one
// launch (NCCL groups).  Payloads are small except the broadcast of the columns entering
// the working set.
struct Comm {
    int rank = 0, world = 1;
    virtual ~Comm() {}
    virtual void allgather(const void *send, void *recv, size_t bytes, cudaStream_t st) = 0;   // recv: world * bytes
    virtual void bcast(void *buf, size_t bytes, int root, cudaStream_t st) = 0;
    virtual void allreduce_sum(double *buf, size_t count, cudaStream_t st) = 0;
    virtual void group_begin() {}
    virtual void group_end() {}
    virtual void wait(cudaStream_t st) { CK(cudaStreamSynchronize(st)); }
};

struct NcclComm : Comm {
    ncclComm_t c = nullptr;
    int timeout_ms = 600000;
    ~NcclComm() override { if (c) ncclCommDestroy(c); }
    ncclComm_t live() {
        if (!c) raise(BL_ERR_NCCL, "the NCCL communicator was aborted by an earlier error or timeout");
        return c;
    }
    void allgather(const void *send, void *recv, size_t bytes, cudaStream_t st) override {
        CKN(ncclAllGather(send, recv, bytes, ncclUint8, live(), st));
    }
    void bcast(void *buf, size_t bytes, int root, cudaStream_t st) override {
        CKN(ncclBroadcast(buf, buf, bytes, ncclUint8, root, live(), st));
    }
    void allreduce_sum(double *buf, size_t count, cudaStream_t st) override {
        CKN(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, live(), st));
    }
    void group_begin() override { CKN(ncclGroupStart()); }
    void group_end() override { CKN(ncclGroupEnd()); }
    void wait(cudaStream_t st) override {
        const auto t0 = std::chrono::steady_clock::now();
        for (int spin = 0;; spin++) {
            const cudaError_t e = cudaStreamQuery(st);
            if (e == cudaSuccess) return;
            if (e != cudaErrorNotReady) {
                cudaGetLastError();
                raise(BL_ERR_CUDA, "stream of a collective: %s", cudaGetErrorString(e));
            }
            ncclResult_t ae = ncclSuccess;
            if (c && ncclCommGetAsyncError(c, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress) {
                ncclCommAbort(c);
                c = nullptr;
                raise(BL_ERR_NCCL, "NCCL asynchronous error: %s (communicator aborted)", ncclGetErrorString(ae));
            }
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (ms > timeout_ms) {
                if (c) ncclCommAbort(c);
                c = nullptr;
                raise(BL_ERR_NCCL, "a collective did not complete within %d ms (peer lost?); communicator aborted", timeout_ms);
            }
            if (spin > 256) std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
    }
};

// Caller-supplied host collectives (bl_dist.backend = 2, e.g. gloo or MPI between processes):
// each payload is staged through host memory around the caller's function.
struct HostComm : Comm {
    bl_host_coll hc{};
    std::vector<char> a, b;
    void stage_in(const void *dev, size_t bytes, cudaStream_t st) {
        a.resize(std::max<size_t>(bytes, 1));
        if (bytes) CK(cudaMemcpyAsync(a.data(), dev, bytes, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    void stage_out(void *dev, const void *host, size_t bytes, cudaStream_t st) {
        if (bytes) CK(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));                  // the staging buffers are reused by the next call
    }
    void allgather(const void *send, void *recv, size_t bytes, cudaStream_t st) override {
        stage_in(send, bytes, st);
        b.resize(std::max<size_t>(bytes * world, 1));
        if (hc.allgather(hc.ctx, a.data(), b.data(), (int64_t)bytes) != 0) raise(BL_ERR_NCCL, "host allgather failed");
        stage_out(recv, b.data(), bytes * world, st);
    }
    void bcast(void *buf, size_t bytes, int root, cudaStream_t st) override {
        if (rank == root) stage_in(buf, bytes, st);
        else a.resize(std::max<size_t>(bytes, 1));
        if (hc.bcast(hc.ctx, a.data(), (int64_t)bytes, root) != 0) raise(BL_ERR_NCCL, "host broadcast failed");
        if (rank != root) stage_out(buf, a.data(), bytes, st);
    }
    void allreduce_sum(double *buf, size_t count, cudaStream_t st) override {
        stage_in(buf, 8 * count, st);
        if (hc.allreduce_sum_f64(hc.ctx, reinterpret_cast<double *>(a.data()), (int64_t)count) != 0)
            raise(BL_ERR_NCCL, "host allreduce failed");
        stage_out(buf, a.data(), 8 * count, st);
    }
};

// In-process loopback (testing): the ranks are host threads sharing one device;
// data is staged through host memory between two group barriers.
struct LoopGroup {
    std::mutex mu;
    std::condition_variable cv;
    int world = 0, arrived = 0, members = 0;
    long gen = 0;
    std::vector<std::vector<char>> stage;
};
std::mutex g_loop_mu;
std::map<std::string, std::shared_ptr<LoopGroup>> g_loop_groups;

struct LoopComm : Comm {
    std::shared_ptr<LoopGroup> g;
    std::string key;
    ~LoopComm() override {
        if (!g) return;
        std::lock_guard<std::mutex> lk(g_loop_mu);
        if (--g->members == 0) g_loop_groups.erase(key);
    }
    void barrier() {
        std::unique_lock<std::mutex> lk(g->mu);
        const long my = g->gen;
        if (++g->arrived == world) {
            g->arrived = 0;
            g->gen++;
            g->cv.notify_all();
        } else {
            g->cv.wait(lk, [&] { return g->gen != my; });
        }
    }
    void put(const void *dev, size_t bytes, cudaStream_t st) {
        g->stage[rank].resize(bytes);
        if (bytes) CK(cudaMemcpyAsync(g->stage[rank].data(), dev, bytes, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    void allgather(const void *send, void *recv, size_t bytes, cudaStream_t st) override {
        put(send, bytes, st);
        barrier();
        for (int r = 0; r < world; r++)
            if (bytes) CK(cudaMemcpyAsync((char *)recv + (size_t)r * bytes, g->stage[r].data(), bytes, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
        barrier();
    }
    void bcast(void *buf, size_t bytes, int root, cudaStream_t st) override {
        if (rank == root) put(buf, bytes, st);
        barrier();
        if (rank != root && bytes) CK(cudaMemcpyAsync(buf, g->stage[root].data(), bytes, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
        barrier();
    }
    void allreduce_sum(double *buf, size_t count, cudaStream_t st) override {
        put(buf, 8 * count, st);
        barrier();
        std::vector<double> acc(count, 0.0);
        for (int r = 0; r < world; r++) {
            const double *v = (const double *)g->stage[r].data();
            for (size_t i = 0; i < count; i++) acc[i] += v[i];
        }
        if (count) CK(cudaMemcpyAsync(buf, acc.data(), 8 * count, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
        barrier();
    }
};

// ------------------------------------------------------------------ handles

struct bl_design {
    uint32_t magic;
    std::mutex pool_mu;
    std::vector<bl_prep *> pool;     // idle fit workspaces, reused by later fits
    void *X;          // device
    bool owned;
    int dt;
    int64_t n, p, ld;
    int64_t col_offset, p_global;
    int device, nsm;
    int rank, world;
    Comm *comm;                      // world > 1 only
    bool sharded;                    // columns split over the ranks (p_global > p_local)
    bool hostres = false;            // NEXT-4: X stays in (mapped, pinned) host memory, read over PCIe
    bool wstore = false;             // CD reads its columns from the working-set store (sharded || hostres)
    void *host_reg = nullptr;        // host range this design registered (unregistered by bl_free)
    std::vector<int64_t> shard_off;  // world + 1 global column offsets of the shards (rank order)
    std::mutex comm_mu;
    std::atomic<int> busy{0};        // world > 1: one call at a time (collective order, bl.h)
    float *xsc = nullptr;            // fp32: 2^-E_j per column (k_xscale), the tensor-core scan's digit scale
};

struct bl_path {
    uint32_t magic;
    int n_lambda, n_converged;
    std::vector<double> lambda, a0, obj;
    std::vector<int64_t> col_ptr, feat;
    std::vector<double> beta_std, beta_orig;
    std::vector<int32_t> passes, kkt_rounds;
    std::vector<int64_t> cols_scanned;
    std::vector<int64_t> n_safe, n_strong, n_working;   // screening diagnostics per lambda (Fig 1 analog)
    std::vector<int32_t> outer;                          // logistic path: IRLS iterations (last solve) per lambda
    int family = 0;
    bl_perf perf;
    int64_t cd_visits = 0, cd_updates = 0, cd_cycles = 0, cd_prof[4] = {0, 0, 0, 0}, cd_cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0},
            cd_dbg[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};

struct bl_cvres {
    uint32_t magic;
    int n_lambda, K, lmin;
    int64_t n;
    std::vector<double> cve, cvse, E;
    std::vector<int32_t> fold_id;
    bl_path *full;
    bl_perf perf;            // summed over every fit of the CV (folds + full data)
    std::mutex perf_mu;
};

// Per-(y, row mask) device workspace: one arena allocation carved into the
// vectors the path needs.
constexpr int kXPre = 1024;   // list entries a round exchange carries per rank (C3)
struct RoundX {               // one KKT round of a sharded fit, combined over the ranks (C3)
    std::vector<int64_t> nviol, nstrong;        // per rank
    int64_t nscope = 0, nsafe = 0;
    std::vector<int> viol, strong;              // sorted GLOBAL indices (when *_ok)
    bool viol_ok = false, strong_ok = false;    // every rank's list fit in the exchange
};

struct bl_prep {
    uint32_t magic;
    bl_design *d;
    cudaStream_t stream;
    bool own_stream;
    double alpha;
    int64_t p, ld, vlen;
    int limb_ld;
    int has_mask;
    double nt;
    // arena
    char *arena;
    size_t arena_bytes;
    double *c, *s, *a, *b, *z, *beta;
    uint8_t *flags, *wflag, *mask;
    int *scope, *viol, *strong, *W;
    int64_t Wcap;
    double *betaW, *yt, *rfull, *rscan, *vtmp;
    double *yraw;             // y as given (the logistic path's 0/1 response)
    double *LG = nullptr;     // logistic covariance CD: weighted Gram ((|W|+1)^2, ld ldLG)
    int64_t ldLG = 0;
    double *lgbuf = nullptr;  // logistic covariance CD: slot coefficients, weights, partial sums
    size_t lgcap = 0;
    // NEXT-4 host-resident designs: double-buffered column chunks for the streamed scans
    char *sbuf[2] = {nullptr, nullptr};
    int64_t scols = 0;        // columns per chunk
    cudaStream_t cstream = nullptr;
    cudaEvent_t copied[2] = {nullptr, nullptr}, used[2] = {nullptr, nullptr};
    int8_t *limbs;
    double *limb_scale, *limb_sum;
    PrepScalars *ps;
    RoundStatus *st;
    double *amax_v;
    long long *amax_i;
    int *nlive;
    int amax_blocks;
    // host mirrors
    PrepScalars hps;
    RoundStatus *hst;       // pinned
    int *hlist;             // pinned read-back buffer (grows)
    int *hpre;              // pinned: prefixes of the violator and strong lists, copied with each round's status
    int *hup;               // pinned upload staging (grows)
    double *hbw;            // pinned, 3*|W| entries (beta, c, s of W) (grows)
    size_t hlist_cap, hup_cap, hbw_cap;
    char *warena;           // device W buffers (grow): W sorted, Wst, ord (int32); betaW (3 x fp64), dbeta
    int *Wst_d, *ord_d;     // Gram CD: storage slots (append order) and cyclic order
    double *dbeta;          // Gram CD: coefficient change per slot over one solve
    double *G;              // Gram CD: ldG x ldG, row-major by storage slot (HBM / L2)
    double *GA;             // Gram CD workspace: G_AA (ldG x ldG) followed by the block inverses (32 ldG)
    int64_t ldG;
    int nG;                 // slots whose G row/column is computed
    double *rpart;          // per-block partials of the residual refresh
    double *rbuf;           // residual refresh: per-chunk row partials (grows)
    size_t rbuf_cap;
    // sharded designs: device scratch of the collectives, and the working-set column
    // store (every rank holds the W columns, broadcast by their owners, in slot order)
    void *cbuf;
    size_t cbuf_cap;
    void *Xw;               // ld x ws_cap, raw dtype
    double *cw, *sw, *bw, *zw;   // per slot: c, s, beta, gradient
    int *widx;              // identity 0..ws_cap-1 (slot -> column of the store)
    int64_t ws_cap;
    int star_root;          // rank owning x_* (sharded)
    RoundX xr;              // sharded: the last round exchange
    double batch_bytes;     // lockstep CV: X bytes read by the batched scans this fit timed
    int batch_passes;       // ... batched launches of the current round
    int cd_mode;            // 0 auto (Gram when |W| <= 4096), 1 residual, 2 Gram
    int cd_cluster;         // CTAs per Gram-CD cluster (4, 8, 16)
    int cd_cluster_auto;    // the caller left cd_cluster at 0 (the library picks per solve kind)
    int cd_newton;          // Newton (CG) steps on settled active sets in the Gram CD
    int fault_strong_drop;  // TEST ONLY (bl_opts): admit no strong-rule candidate in advance
    size_t chunk_bytes;     // out-of-core: bytes per streamed chunk (the buffers are sized for it)
    cudaStream_t own;       // library stream (used when the caller passes none)
    // profiling
    int profile;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_scan, ev_cd, ev_prep;
    std::vector<cudaEvent_t> evpool;   // timing events of finished profiled fits, reused (no create per launch)
    std::vector<int64_t> scan_full;   // per timed scan launch: its local columns if it covered every live column, else -1
    int scan_rev = 0;                 // direction of the next KKT scan (alternates, see ScanArgs::rev)
    double prep_bytes;
    int64_t launches;
};

namespace {

void check_device() {
    int cnt = 0;
    cudaError_t e = cudaGetDeviceCount(&cnt);
    if (e != cudaSuccess || cnt == 0)
        raise(BL_ERR_CUDA, "no CUDA device available (%s); libbl has no CPU path",
              e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
    int dev = 0;
    CK(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10)
        raise(BL_ERR_CUDA, "device %d is sm_%d%d; libbl is built for sm_100a only", dev, prop.major, prop.minor);
}

// A multi-rank design accepts one call at a time (include/bl.h): two concurrent calls
// could issue their collectives in different orders on different ranks.
struct BusyGuard {
    bl_design *d;
    bool held = false;
    explicit BusyGuard(bl_design *d_) : d(d_) {
        if (d->world <= 1) return;
        int expect = 0;
        if (!d->busy.compare_exchange_strong(expect, 1))
            raise(BL_ERR_ARG, "a multi-rank design accepts one call at a time (collectives must run in the same order on every rank)");
        held = true;
    }
    ~BusyGuard() { if (held) d->busy.store(0); }
};

template <typename F>
bl_status guard(F &&f) {
    cudaGetLastError();   // a stale error from an earlier call must not be reported here
    try {
        f();
        return BL_OK;
    } catch (const Err &e) {
        return e.code;
    } catch (const std::bad_alloc &) {
        g_err = "host allocation failed";
        return BL_ERR_OOM;
    }
}

cudaEvent_t ev_get(bl_prep *pp) {
    cudaEvent_t e;
    if (!pp->evpool.empty()) {
        e = pp->evpool.back();
        pp->evpool.pop_back();
    } else {
        CK(cudaEventCreate(&e));
    }
    return e;
}

struct EvPair {
    bl_prep *pp;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> *vec;
    cudaEvent_t e1 = nullptr;
    EvPair(bl_prep *pp_, std::vector<std::pair<cudaEvent_t, cudaEvent_t>> *v) : pp(pp_), vec(v) {
        if (!pp->profile) return;
        cudaEvent_t e0 = ev_get(pp);
        e1 = ev_get(pp);
        CK(cudaEventRecord(e0, pp->stream));
        vec->push_back({e0, e1});
    }
    ~EvPair() {
        if (pp->profile && e1) cudaEventRecord(e1, pp->stream);
    }
};

struct EvPairOpt {
    bl_prep *pp;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> *vec;
    cudaEvent_t e1 = nullptr;
    EvPairOpt(bl_prep *pp_, std::vector<std::pair<cudaEvent_t, cudaEvent_t>> *v) : pp(pp_), vec(v) {
        if (!pp->profile || !vec) return;
        cudaEvent_t e0 = ev_get(pp);
        e1 = ev_get(pp);
        CK(cudaEventRecord(e0, pp->stream));
        vec->push_back({e0, e1});
    }
    ~EvPairOpt() {
        if (pp->profile && vec && e1) cudaEventRecord(e1, pp->stream);
    }
};

double sum_events(std::vector<std::pair<cudaEvent_t, cudaEvent_t>> &v, const std::vector<int64_t> *sel = nullptr,
                  double *sel_ms = nullptr, std::vector<cudaEvent_t> *pool = nullptr) {
    double tot = 0.0;
    for (size_t i = 0; i < v.size(); i++) {
        auto &pr = v[i];
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) {
            tot += ms;
            if (sel && sel_ms && i < sel->size() && (*sel)[i] >= 0) *sel_ms += ms;
        }
        if (pool) {
            pool->push_back(pr.first);
            pool->push_back(pr.second);
        } else {
            cudaEventDestroy(pr.first);
            cudaEventDestroy(pr.second);
        }
    }
    v.clear();
    return tot;
}

int grid_for(const void *kern, int threads, size_t smem, int nsm) {
    static std::mutex mu;
    struct Key { const void *k; int t; size_t s; int occ; };
    static std::vector<Key> cache;
    {
        std::lock_guard<std::mutex> lk(mu);
        for (auto &e : cache)
            if (e.k == kern && e.t == threads && e.s == smem) return e.occ * nsm;
    }
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
    {
        std::lock_guard<std::mutex> lk(mu);
        cache.push_back({kern, threads, smem, occ});
    }
    if (occ < 1) raise(BL_ERR_OOM, "kernel does not fit on an SM (smem %zu B)", smem);
    return occ * nsm;
}

// Opt a kernel into the largest dynamic shared memory the device allows
// (opt-in limit minus the kernel's static shared memory); returns that limit.
size_t allow_dyn_smem(const void *kern) {
    static std::mutex mu;
    static std::vector<std::pair<const void *, size_t>> done;
    std::lock_guard<std::mutex> lk(mu);
    for (auto &pr : done)
        if (pr.first == kern) return pr.second;
    int dev = 0, optin = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, kern));
    size_t lim = (size_t)optin - fa.sharedSizeBytes;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lim));
    done.push_back({kern, lim});
    return lim;
}

// ------------------------------------------------------------ scan launcher
// Raw-dot + identity epilogue over `list` (or all columns); v = fp64 vector
// (fp32/fp64 designs) -- for int8 designs v is quantised to limbs first.
// `cols`: another column source with the design's layout (the sharded working-set
// store) and its c, s; nullptr => the design.
// NEXT-4: a dense scan of a host-resident design streams X through two device chunk
// buffers: the copy engine fills chunk i+1 (cudaMemcpyAsync on its own stream) while
// the scan kernel reads chunk i from HBM; events order buffer reuse.  The kernel sees
// a "virtual base" X - j0 * ld, so column indices, outputs and lists stay global.
constexpr size_t kStreamChunkBytes = (size_t)256 << 20;
void ensure_stream_bufs(bl_prep *pp) {
    if (pp->sbuf[0]) return;
    bl_design *d = pp->d;
    const size_t colb = (size_t)d->ld * itemsize(d->dt);
    pp->scols = std::max<int64_t>(1, std::min<int64_t>(d->p, (int64_t)(pp->chunk_bytes / colb)));
    for (int u = 0; u < 2; u++) {
        cudaError_t e = cache::dmalloc((void **)&pp->sbuf[u], colb * pp->scols);
        if (e != cudaSuccess) { cudaGetLastError(); raise(BL_ERR_OOM, "cudaMalloc for the streamed-scan buffers: %s", cudaGetErrorString(e)); }
        if (!pp->copied[u]) CK(cudaEventCreateWithFlags(&pp->copied[u], cudaEventDisableTiming));
        if (!pp->used[u]) CK(cudaEventCreateWithFlags(&pp->used[u], cudaEventDisableTiming));
    }
    if (!pp->cstream) CK(cudaStreamCreateWithFlags(&pp->cstream, cudaStreamNonBlocking));
}

template <typename F>
void stream_chunks(bl_prep *pp, ScanArgs &a, F launch) {
    bl_design *d = pp->d;
    ensure_stream_bufs(pp);
    const size_t colb = (size_t)d->ld * itemsize(d->dt);
    const char *Xh = (const char *)d->X;
    CK(cudaEventRecord(pp->used[0], pp->stream));       // the buffers are free once prior work on the fit stream is
    CK(cudaEventRecord(pp->used[1], pp->stream));
    int u = 0;
    for (int64_t c0 = 0; c0 < d->p; c0 += pp->scols, u ^= 1) {
        const int64_t k = std::min<int64_t>(pp->scols, d->p - c0);
        CK(cudaStreamWaitEvent(pp->cstream, pp->used[u], 0));
        CK(cudaMemcpyAsync(pp->sbuf[u], Xh + (size_t)c0 * colb, (size_t)k * colb, cudaMemcpyDefault, pp->cstream));
        CK(cudaEventRecord(pp->copied[u], pp->cstream));
        CK(cudaStreamWaitEvent(pp->stream, pp->copied[u], 0));
        a.X = pp->sbuf[u] - (ptrdiff_t)((size_t)c0 * colb);     // virtual base: column j at X + j * ld
        a.j0 = c0;
        a.p = c0 + k;
        launch();
        CK(cudaEventRecord(pp->used[u], pp->stream));
    }
}

void launch_scan(bl_prep *pp, ScanArgs a, const double *v_dev, bool timed, bool events = true,
                 const void *cols = nullptr, const double *cc = nullptr, const double *cs = nullptr) {
    bl_design *d = pp->d;
    a.X = cols ? cols : d->X;
    a.ld = d->ld;
    a.n = (int)d->n;
    a.p = d->p;
    a.c = cols ? cc : pp->c;
    a.s = cols ? cs : pp->s;
    // host-resident design, scan over the design: stream it densely when the scope covers
    // at least half of the columns (columns outside the scope are gated off by their flags);
    // a short scope list is read in place (zero-copy)
    bool streamed = false;
    if (d->hostres && !cols) {
        int64_t m = a.list ? (a.nlist ? -1 : (int64_t)a.nlist_host) : d->p;
        if (m < 0) {
            int h = 0;
            CK(cudaMemcpyAsync(&h, a.nlist, sizeof h, cudaMemcpyDeviceToHost, pp->stream));
            CK(cudaStreamSynchronize(pp->stream));
            m = h;
        }
        if (2 * m >= d->p && (!a.list || a.flags)) {
            streamed = true;
            a.list = nullptr;
            a.rev = 0;
        }
    }
    if (d->dt == DT_I8) {
        k_limbs<<<1, 1024, 0, pp->stream>>>(v_dev, (int)d->n, pp->limb_ld, pp->limbs, pp->limb_scale,
                                            pp->limb_sum);
        CKL();
        pp->launches++;
        a.limbs = pp->limbs;
        a.limb_ld = pp->limb_ld;
        a.limb_scale = pp->limb_scale;
        a.K1 = pp->limb_sum;      // sum of the quantised vector: identity holds exactly for it
        size_t smem = (size_t)8 * pp->limb_ld;
        allow_dyn_smem((const void *)k_scan_i8);
        int grid = grid_for((const void *)k_scan_i8, kScanThreads, smem, d->nsm);
        EvPairOpt ev(pp, events ? (timed ? &pp->ev_scan : &pp->ev_prep) : nullptr);
        if (streamed) {
            stream_chunks(pp, a, [&] {
                k_scan_i8<<<grid, kScanThreads, smem, pp->stream>>>(a);
                CKL();
            });
        } else {
            k_scan_i8<<<grid, kScanThreads, smem, pp->stream>>>(a);
            CKL();
        }
    } else {
        a.v = v_dev;
        int V = 16 / itemsize(d->dt);
        size_t smem = (size_t)8 * round_up(d->n, 32 * V);
        // 4 columns per warp iteration (16-byte loads, four columns' loads in flight per lane)
        const void *kern = d->dt == DT_F32 ? (const void *)k_scan_fp<float, 4> : (const void *)k_scan_fp<double, 4>;
        allow_dyn_smem(kern);
        int grid = grid_for(kern, kScanThreads, smem, d->nsm);
        EvPairOpt ev(pp, events ? (timed ? &pp->ev_scan : &pp->ev_prep) : nullptr);
        void *args[] = {&a};
        if (streamed) {
            stream_chunks(pp, a, [&] { CK(cudaLaunchKernel(kern, dim3(grid), dim3(kScanThreads), args, smem, pp->stream)); });
        } else {
            CK(cudaLaunchKernel(kern, dim3(grid), dim3(kScanThreads), args, smem, pp->stream));
        }
    }
    pp->launches++;
}

template <typename T>
void launch_colstats(bl_prep *pp, int i0) {
    bl_design *d = pp->d;
    int grid = d->nsm * 8;
    if (pp->has_mask)
        k_colstats<T, true><<<grid, 256, 0, pp->stream>>>((const T *)d->X, d->ld, (int)d->n, d->p, pp->mask, i0,
                                                           pp->nt, pp->c, pp->s);
    else
        k_colstats<T, false><<<grid, 256, 0, pp->stream>>>((const T *)d->X, d->ld, (int)d->n, d->p, nullptr, i0,
                                                            pp->nt, pp->c, pp->s);
    CKL();
    pp->launches++;
}

template <typename T>
void launch_xstar(bl_prep *pp) {
    bl_design *d = pp->d;
    k_xstar<T><<<1, 1024, 0, pp->stream>>>((const T *)d->X, d->ld, (int)d->n, (int)pp->vlen,
                                           pp->has_mask ? pp->mask : nullptr, pp->ps, pp->vtmp);
    CKL();
    pp->launches++;
}

void free_prep(bl_prep *pp) {
    if (!pp) return;
    if (pp->stream) cudaStreamSynchronize(pp->stream);
    sum_events(pp->ev_scan);
    sum_events(pp->ev_cd);
    sum_events(pp->ev_prep);
    for (cudaEvent_t e : pp->evpool) cudaEventDestroy(e);
    pp->evpool.clear();
    if (pp->arena) cache::dfree(pp->arena);
    if (pp->hst) cache::hfree(pp->hst);
    if (pp->hlist) cache::hfree(pp->hlist);
    if (pp->hpre) cache::hfree(pp->hpre);
    if (pp->hbw) cache::hfree(pp->hbw);
    if (pp->hup) cache::hfree(pp->hup);
    if (pp->warena) cache::dfree(pp->warena);
    if (pp->G) cache::dfree(pp->G);
    if (pp->GA) cache::dfree(pp->GA);
    if (pp->cbuf) cache::dfree(pp->cbuf);
    if (pp->rbuf) cache::dfree(pp->rbuf);
    if (pp->Xw) cache::dfree(pp->Xw);
    if (pp->cw) cache::dfree(pp->cw);
    if (pp->LG) cache::dfree(pp->LG);
    if (pp->lgbuf) cache::dfree(pp->lgbuf);
    for (int u = 0; u < 2; u++) {
        if (pp->sbuf[u]) cache::dfree(pp->sbuf[u]);
        if (pp->copied[u]) cudaEventDestroy(pp->copied[u]);
        if (pp->used[u]) cudaEventDestroy(pp->used[u]);
    }
    if (pp->cstream) cudaStreamDestroy(pp->cstream);
    if (pp->own) cudaStreamDestroy(pp->own);
    pp->magic = MAGIC_DEAD;
    delete pp;
}

struct PrepGuard {
    bl_prep *pp;
    ~PrepGuard() { free_prep(pp); }
};

// Return a fit workspace to its design's pool (or free it).
void release_prep(bl_prep *pp) {
    if (!pp) return;
    if (pp->stream) cudaStreamSynchronize(pp->stream);
    sum_events(pp->ev_scan, nullptr, nullptr, &pp->evpool);
    sum_events(pp->ev_cd, nullptr, nullptr, &pp->evpool);
    sum_events(pp->ev_prep, nullptr, nullptr, &pp->evpool);
    pp->stream = pp->own;          // never keep a caller's stream beyond the call
    std::lock_guard<std::mutex> lk(pp->d->pool_mu);
    if (pp->d->pool.size() < 4) pp->d->pool.push_back(pp);
    else free_prep(pp);
}

struct PoolGuard {
    bl_prep *pp;
    ~PoolGuard() { release_prep(pp); }
};

template <typename Tp>
void ensure_host(Tp *&ptr, size_t &cap, size_t need) {
    if (need <= cap) return;
    size_t nc = std::max<size_t>(need, 2 * cap);
    nc = std::max<size_t>(nc, 1024);
    if (ptr) cache::hfree(ptr);
    ptr = nullptr;
    CK(cache::hmalloc((void **)&ptr, nc * sizeof(Tp)));
    cap = nc;
}

// Device W buffers grow geometrically (contents are re-uploaded / rewritten each round).
void ensure_W(bl_prep *pp, int64_t need) {
    if (need <= pp->Wcap && pp->warena) return;
    int64_t nc = std::max<int64_t>(std::max<int64_t>(need, 2 * pp->Wcap), 1024);
    nc = std::min<int64_t>(std::max<int64_t>(nc, need), std::max<int64_t>(pp->d->sharded ? pp->d->p_global : pp->p, 1));
    CK(cudaStreamSynchronize(pp->stream));
    if (pp->warena) cache::dfree(pp->warena);
    pp->warena = nullptr;
    size_t ib = (size_t)round_up(4 * nc, 256);
    size_t bytes = 3 * ib + (size_t)32 * nc;
    cudaError_t e = cache::dmalloc((void **)&pp->warena, bytes);
    if (e != cudaSuccess) { cudaGetLastError(); raise(BL_ERR_OOM, "cudaMalloc(%zu) for W: %s", bytes, cudaGetErrorString(e)); }
    pp->W = (int *)pp->warena;
    pp->Wst_d = (int *)(pp->warena + ib);
    pp->ord_d = (int *)(pp->warena + 2 * ib);
    pp->betaW = (double *)(pp->warena + 3 * ib);
    pp->dbeta = pp->betaW + 3 * nc;
    pp->Wcap = nc;
}

double *ensure_rbuf(bl_prep *pp, size_t count) {
    if (count <= pp->rbuf_cap) return pp->rbuf;
    CK(cudaStreamSynchronize(pp->stream));
    if (pp->rbuf) cache::dfree(pp->rbuf);
    pp->rbuf = nullptr;
    const size_t nc = std::max<size_t>(count, 2 * pp->rbuf_cap);
    cudaError_t e = cache::dmalloc((void **)&pp->rbuf, 8 * nc);
    if (e != cudaSuccess) { cudaGetLastError(); pp->rbuf_cap = 0; raise(BL_ERR_OOM, "cudaMalloc(%zu) for the residual refresh: %s", 8 * nc, cudaGetErrorString(e)); }
    pp->rbuf_cap = nc;
    return pp->rbuf;
}

void *ensure_cbuf(bl_prep *pp, size_t bytes) {
    if (bytes <= pp->cbuf_cap) return pp->cbuf;
    CK(cudaStreamSynchronize(pp->stream));
    if (pp->cbuf) cache::dfree(pp->cbuf);
    pp->cbuf = nullptr;
    size_t nb = std::max<size_t>(std::max<size_t>(bytes, 2 * pp->cbuf_cap), 4096);
    cudaError_t e = cache::dmalloc((void **)&pp->cbuf, nb);
    if (e != cudaSuccess) { cudaGetLastError(); pp->cbuf_cap = 0; raise(BL_ERR_OOM, "cudaMalloc(%zu) for collectives: %s", nb, cudaGetErrorString(e)); }
    pp->cbuf_cap = nb;
    return pp->cbuf;
}

// Sharded: the working-set column store grows geometrically, keeping its contents.
void ensure_Ws(bl_prep *pp, int64_t need, int64_t have) {
    if (need <= pp->ws_cap) return;
    bl_design *d = pp->d;
    const size_t isz = itemsize(d->dt);
    const int64_t nc = std::max<int64_t>(std::max<int64_t>(need, 2 * pp->ws_cap), 256);
    void *X2 = nullptr;
    double *v2 = nullptr;
    cudaError_t e = cache::dmalloc((void **)&X2, (size_t)d->ld * nc * isz);
    if (e == cudaSuccess) e = cache::dmalloc((void **)&v2, (size_t)8 * 4 * nc + (size_t)4 * nc);
    if (e != cudaSuccess) {
        cudaGetLastError();
        if (X2) cache::dfree(X2);
        raise(BL_ERR_OOM, "cudaMalloc for the working-set column store (%lld columns): %s", (long long)nc, cudaGetErrorString(e));
    }
    cudaStream_t st = pp->stream;
    double *c2 = v2, *s2 = v2 + nc, *b2 = v2 + 2 * nc, *z2 = v2 + 3 * nc;
    int *w2 = (int *)(v2 + 4 * nc);
    if (have > 0) {
        CK(cudaMemcpyAsync(X2, pp->Xw, (size_t)d->ld * have * isz, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(c2, pp->cw, 8 * (size_t)have, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(s2, pp->sw, 8 * (size_t)have, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(b2, pp->bw, 8 * (size_t)have, cudaMemcpyDeviceToDevice, st));
    }
    k_iota<<<(unsigned)((nc + 255) / 256), 256, 0, st>>>(w2, (int)nc);
    CKL();
    CK(cudaStreamSynchronize(st));
    if (pp->Xw) cache::dfree(pp->Xw);
    if (pp->cw) cache::dfree(pp->cw);
    pp->Xw = X2;
    pp->cw = c2; pp->sw = s2; pp->bw = b2; pp->zw = z2;
    pp->widx = w2;
    pp->ws_cap = nc;
}

// Columns of the coordinate-descent side: the design itself (single GPU /
// replicated), or the working-set column store (sharded; slot j = store column j).
struct CdView {
    const void *X;
    const double *c, *s;
    double *beta, *z;
    const int *Wst;          // slot -> column of the view
    const int *Wsorted;      // W in ascending global order -> columns of the view
};
CdView cd_view(bl_prep *pp) {
    if (!pp->d->wstore) return CdView{pp->d->X, pp->c, pp->s, pp->beta, pp->z, pp->Wst_d, pp->W};
    return CdView{pp->Xw, pp->cw, pp->sw, pp->bw, pp->zw, pp->widx, pp->ord_d};
}

// ---- collectives of the sharded path
// per-rank int64 records (k entries each) -> world x k on the host
std::vector<int64_t> gather_i64(bl_prep *pp, const int64_t *mine, int k) {
    bl_design *d = pp->d;
    int64_t *buf = (int64_t *)ensure_cbuf(pp, (size_t)8 * k * (d->world + 1));
    CK(cudaMemcpyAsync(buf, mine, 8 * (size_t)k, cudaMemcpyHostToDevice, pp->stream));
    d->comm->allgather(buf, buf + k, 8 * (size_t)k, pp->stream);
    std::vector<int64_t> all((size_t)k * d->world);
    CK(cudaMemcpyAsync(all.data(), buf + k, 8 * (size_t)k * d->world, cudaMemcpyDeviceToHost, pp->stream));
    d->comm->wait(pp->stream);
    return all;
}
// every rank's local index list (device, counts[r] entries on rank r) -> sorted GLOBAL indices
std::vector<int> gather_list(bl_prep *pp, const int *dev, const std::vector<int64_t> &counts) {
    bl_design *d = pp->d;
    int64_t mx = 0, tot = 0;
    for (int64_t c : counts) { mx = std::max(mx, c); tot += c; }
    std::vector<int> out;
    if (mx == 0) return out;
    int *buf = (int *)ensure_cbuf(pp, (size_t)4 * mx * (d->world + 1));
    const int64_t mine = counts[d->rank];
    if (mine) CK(cudaMemcpyAsync(buf, dev, 4 * (size_t)mine, cudaMemcpyDeviceToDevice, pp->stream));
    d->comm->allgather(buf, buf + mx, 4 * (size_t)mx, pp->stream);
    ensure_host(pp->hlist, pp->hlist_cap, (size_t)mx * d->world);
    CK(cudaMemcpyAsync(pp->hlist, buf + mx, 4 * (size_t)mx * d->world, cudaMemcpyDeviceToHost, pp->stream));
    d->comm->wait(pp->stream);
    out.reserve(tot);
    for (int r = 0; r < d->world; r++)
        for (int64_t q = 0; q < counts[r]; q++) out.push_back(pp->hlist[(size_t)r * mx + q] + (int)d->shard_off[r]);
    std::sort(out.begin(), out.end());
    return out;
}

// One-time preprocessing for (y, optional training mask).
// Preprocessing of one fit (a2-a4), in stages so that bl_cv's lockstep fits can
// share the two store-mode scans (a_j and b_j) as fold-batched passes (make_prep runs them per fit):
// prep_begin (workspace, y~, column statistics), the a_j scan, prep_mid (lambda_max, j*, x~_*),
// the b_j scan, prep_end (the solve's start, the one host round trip, degenerate-input checks).
bl_prep *prep_begin(bl_design *d, const double *y, const uint8_t *train, double alpha, const bl_opts *opts,
                    bool skip_colstats = false) {
    if (!y) raise(BL_ERR_ARG, "y is NULL");
    if (!(alpha > 0.0 && alpha <= 1.0)) raise(BL_ERR_ARG, "alpha must be in (0, 1], got %g", alpha);
    CK(cudaSetDevice(d->device));
    bl_prep *pp = nullptr;
    {
        std::lock_guard<std::mutex> lk(d->pool_mu);
        if (!d->pool.empty()) { pp = d->pool.back(); d->pool.pop_back(); }
    }
    bool reused = pp != nullptr;
    if (!pp) pp = new bl_prep();
    PrepGuard guard{pp};
    pp->magic = MAGIC_PREP;
    pp->d = d;
    pp->alpha = alpha;
    pp->p = d->p;
    pp->ld = d->ld;
    pp->profile = opts ? opts->profile : 0;
    pp->cd_mode = opts ? opts->cd_mode : 0;
    {
        const int cc = opts ? opts->cd_cluster : 0;
        if (cc != 0 && cc != 4 && cc != 8 && cc != 16) raise(BL_ERR_ARG, "cd_cluster must be 0, 4, 8 or 16 (got %d)", cc);
        pp->cd_cluster = cc == 0 ? 16 : cc;   // one fit: 16 SMs (bl_cv's concurrent fits default to 8)
        pp->cd_cluster_auto = cc == 0;
        if (opts && opts->stream_chunk_bytes < 0) raise(BL_ERR_ARG, "stream_chunk_bytes must be >= 0");
        const size_t cb = opts && opts->stream_chunk_bytes > 0 ? (size_t)opts->stream_chunk_bytes : kStreamChunkBytes;
        if (cb != pp->chunk_bytes && pp->sbuf[0]) {          // a reused workspace with other chunk buffers
            for (int u = 0; u < 2; u++) { cache::dfree(pp->sbuf[u]); pp->sbuf[u] = nullptr; }
        }
        pp->chunk_bytes = cb;
        pp->fault_strong_drop = opts ? opts->fault_strong_drop : 0;
        pp->cd_newton = opts ? opts->cd_accel == 0 : 1;
    }
    pp->nG = 0;
    pp->launches = 0;
    pp->scan_full.clear();
    if (!pp->own) CK(cudaStreamCreateWithFlags(&pp->own, cudaStreamNonBlocking));
    pp->stream = (opts && opts->stream) ? (cudaStream_t)opts->stream : pp->own;
    pp->own_stream = false;
    const int64_t n = d->n, p = d->p;
    int64_t nt = n, i0 = 0;
    if (train) {
        nt = 0;
        i0 = -1;
        for (int64_t i = 0; i < n; i++)
            if (train[i]) { nt++; if (i0 < 0) i0 = i; }
    }
    if (nt < 2) raise(BL_ERR_ARG, "need at least 2 rows, got %lld", (long long)nt);
    pp->nt = (double)nt;
    pp->has_mask = train != nullptr;
    pp->vlen = round_up(std::max<int64_t>(d->ld, 1024), 128);
    pp->limb_ld = (int)(round_up(d->ld, 128) + 64);
    pp->amax_blocks = d->nsm * 4;
    if (!reused) {
        // arena layout (sizes depend only on the design)
        size_t off = 0;
        auto take = [&](size_t bytes) { size_t o = off; off = round_up(off + bytes, 256); return o; };
        size_t o_c = take(8 * p), o_s = take(8 * p), o_a = take(8 * p), o_b = take(8 * p), o_z = take(8 * p),
               o_beta = take(8 * p), o_flags = take(p), o_wflag = take(p), o_mask = take(pp->vlen),
               o_scope = take(4 * p), o_viol = take(4 * p), o_strong = take(4 * p), o_yt = take(8 * pp->vlen),
               o_rf = take(8 * pp->vlen), o_rs = take(8 * pp->vlen), o_vt = take(8 * pp->vlen),
               o_limbs = take((size_t)8 * pp->limb_ld), o_lsc = take(32), o_ps = take(sizeof(PrepScalars)),
               o_st = take(sizeof(RoundStatus)), o_av = take(8 * pp->amax_blocks), o_ai = take(8 * pp->amax_blocks),
               o_nl = take(16), o_rp = take(16 * (pp->vlen / 256 + 1)), o_yr = take(8 * pp->vlen);
        pp->arena_bytes = off;
        cudaError_t e = cache::dmalloc((void **)&pp->arena, off);
        if (e != cudaSuccess) { cudaGetLastError(); raise(BL_ERR_OOM, "cudaMalloc(%zu) failed: %s", off, cudaGetErrorString(e)); }
        char *A = pp->arena;
        pp->c = (double *)(A + o_c); pp->s = (double *)(A + o_s); pp->a = (double *)(A + o_a);
        pp->b = (double *)(A + o_b); pp->z = (double *)(A + o_z); pp->beta = (double *)(A + o_beta);
        pp->flags = (uint8_t *)(A + o_flags); pp->wflag = (uint8_t *)(A + o_wflag); pp->mask = (uint8_t *)(A + o_mask);
        pp->scope = (int *)(A + o_scope); pp->viol = (int *)(A + o_viol); pp->strong = (int *)(A + o_strong);
        pp->yt = (double *)(A + o_yt);
        pp->rfull = (double *)(A + o_rf); pp->rscan = (double *)(A + o_rs); pp->vtmp = (double *)(A + o_vt);
        pp->limbs = (int8_t *)(A + o_limbs); pp->limb_scale = (double *)(A + o_lsc); pp->limb_sum = pp->limb_scale + 1;
        pp->ps = (PrepScalars *)(A + o_ps); pp->st = (RoundStatus *)(A + o_st);
        pp->amax_v = (double *)(A + o_av); pp->amax_i = (long long *)(A + o_ai); pp->nlive = (int *)(A + o_nl);
        pp->rpart = (double *)(A + o_rp);
        pp->yraw = (double *)(A + o_yr);
        pp->Wcap = 0;
        ensure_W(pp, std::min<int64_t>(p, 4096));
    }
    if (!pp->hst) CK(cache::hmalloc((void **)&pp->hst, sizeof(RoundStatus)));
    if (!pp->hpre) CK(cache::hmalloc((void **)&pp->hpre, sizeof(int) * 2 * kListPrefix));
    cudaStream_t st = pp->stream;
    CK(cudaMemsetAsync(pp->beta, 0, 8 * p, st));
    CK(cudaMemsetAsync(pp->wflag, 0, p, st));
    CK(cudaMemsetAsync(pp->st, 0, sizeof(RoundStatus), st));
    CK(cudaMemsetAsync(pp->nlive, 0, 16, st));
    CK(cudaMemsetAsync(pp->limbs, 0, (size_t)8 * pp->limb_ld, st));
    if (train) {
        std::vector<uint8_t> m(pp->vlen, 0);
        for (int64_t i = 0; i < n; i++) m[i] = train[i] ? 1 : 0;
        CK(cudaMemcpyAsync(pp->mask, m.data(), pp->vlen, cudaMemcpyHostToDevice, st));
    }
    // y -> device (staged through the rfull buffer, then centred in place into yt / rfull)
    CK(cudaMemcpyAsync(pp->vtmp, y, 8 * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(pp->yraw, pp->vtmp, 8 * n, cudaMemcpyDeviceToDevice, st));
    {
        EvPair ev(pp, &pp->ev_prep);
        k_center_y<<<1, 1024, 0, st>>>(pp->vtmp, (int)n, (int)pp->vlen, train ? pp->mask : nullptr, pp->nt,
                                       pp->yt, pp->rfull, pp->ps);
        CKL();
        pp->launches++;
        if (skip_colstats) {                            // (bl_cv: all fits' statistics in one pass)
        } else if (d->dt == DT_F64) launch_colstats<double>(pp, (int)i0);
        else if (d->dt == DT_F32) launch_colstats<float>(pp, (int)i0);
        else launch_colstats<int8_t>(pp, (int)i0);
    }
    guard.pp = nullptr;
    return pp;
}

void prep_a_scan(bl_prep *pp) {
    // a_j = x~_j' y~  (identity (2))
    {
        ScanArgs sa{};
        sa.K1 = &pp->ps->sum_yt;
        sa.K2 = nullptr;
        sa.K2v = 1.0;
        sa.out = pp->a;
        sa.jfix = nullptr;
        launch_scan(pp, sa, pp->yt, false);
    }
}

void prep_mid(bl_prep *pp, double alpha) {
    bl_design *d = pp->d;
    const int64_t p = d->p;
    cudaStream_t st = pp->stream;
    // lambda_max, j*
    k_argmax1<<<pp->amax_blocks, 256, 0, st>>>(pp->a, pp->s, p, pp->amax_v, pp->amax_i, pp->nlive);
    CKL();
    k_argmax2<<<1, 256, 0, st>>>(pp->amax_v, pp->amax_i, pp->amax_blocks, pp->a, pp->c, pp->s, alpha, pp->nlive,
                                pp->ps);
    CKL();
    pp->launches += 2;
    if (d->sharded) {
        // C1: the shards' best |a_j| -> global lambda_max, j* (lowest global index on ties)
        PrepScalars h;
        CK(cudaMemcpyAsync(&h, pp->ps, sizeof h, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        double rec[6] = {h.A, (double)(h.jstar >= 0 ? h.jstar + d->col_offset : -1), h.sigma, h.c_star, h.s_star,
                         (double)h.n_live};
        int64_t mine[6];
        std::memcpy(mine, rec, sizeof rec);
        std::vector<int64_t> all = gather_i64(pp, mine, 6);
        int win = -1;
        double best = -1.0, bj = -1.0, live = 0.0;
        for (int r = 0; r < d->world; r++) {
            double v[6];
            std::memcpy(v, &all[6 * (size_t)r], sizeof v);
            live += v[5];
            if (v[1] < 0.0) continue;
            if (v[0] > best || (v[0] == best && v[1] < bj)) { best = v[0]; bj = v[1]; win = r; }
        }
        pp->star_root = win;
        h.n_live = (int)live;
        if (win >= 0) {
            double v[6];
            std::memcpy(v, &all[6 * (size_t)win], sizeof v);
            h.A = v[0];
            h.lmax = h.A / alpha;
            h.sigma = v[2];
            h.c_star = v[3];
            h.s_star = v[4];
            h.inv_s_star = v[4] > 0.0 ? 1.0 / v[4] : 0.0;
            h.jstar = win == d->rank ? (long long)(bj - (double)d->col_offset) : -1;
        } else {
            h.A = 0.0; h.lmax = 0.0; h.sigma = 1.0; h.c_star = 0.0; h.s_star = 0.0; h.inv_s_star = 0.0; h.jstar = -1;
        }
        CK(cudaMemcpyAsync(pp->ps, &h, sizeof h, cudaMemcpyHostToDevice, st));
    }
    // b_j = x~_j' x~_*  (identity (1)); b_j* = n exactly
    if (d->dt == DT_F64) launch_xstar<double>(pp);
    else if (d->dt == DT_F32) launch_xstar<float>(pp);
    else launch_xstar<int8_t>(pp);
    if (d->sharded && pp->star_root >= 0) {      // C2: x_* - c_* (and its sum) from its owner
        d->comm->group_begin();
        d->comm->bcast(pp->vtmp, 8 * (size_t)pp->vlen, pp->star_root, st);
        d->comm->bcast(&pp->ps->sum_v, 8, pp->star_root, st);
        d->comm->group_end();
    }
}

void prep_b_scan(bl_prep *pp) {
    {
        ScanArgs sa{};
        sa.K1 = &pp->ps->sum_v;
        sa.K2 = &pp->ps->inv_s_star;
        sa.out = pp->b;
        sa.jfix = &pp->ps->jstar;
        sa.fixval = &pp->ps->nt;
        launch_scan(pp, sa, pp->vtmp, false);
    }
}

void prep_end(bl_prep *pp) {
    bl_design *d = pp->d;
    cudaStream_t st = pp->stream;
    // the solve starts from r = y~: r_scan <- y~ (used rows), sum r <- sum y~
    CK(cudaMemcpyAsync(pp->rscan, pp->yt, 8 * pp->vlen, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(&pp->st->sumr, &pp->ps->sum_yt, sizeof(double), cudaMemcpyDeviceToDevice, st));
    // the one host round trip of preprocessing: the scalars the lambda loop branches on
    CK(cudaMemcpyAsync(&pp->hps, pp->ps, sizeof(PrepScalars), cudaMemcpyDeviceToHost, st));
    if (d->world > 1) d->comm->wait(st);                 // (collectives above: error / timeout aware)
    else CK(cudaStreamSynchronize(st));
    pp->prep_bytes = 3.0 * (double)d->n * itemsize(d->dt) * (double)d->p;
    if (!(pp->hps.Y2 > 0.0)) raise(BL_ERR_DEGENERATE, "y is constant on the used rows (y~ == 0)");
    if (pp->hps.n_live == 0 && (d->world == 1 || d->sharded)) raise(BL_ERR_DEGENERATE, "every column has zero variance");
    if (!(pp->hps.A > 0.0) && (d->world == 1 || d->sharded)) raise(BL_ERR_DEGENERATE, "lambda_max == 0: y~ orthogonal to every column");
}

bl_prep *make_prep(bl_design *d, const double *y, const uint8_t *train, double alpha, const bl_opts *opts) {
    bl_prep *pp = prep_begin(d, y, train, alpha, opts);
    PrepGuard guard{pp};
    prep_a_scan(pp);
    prep_mid(pp, alpha);
    prep_b_scan(pp);
    prep_end(pp);
    guard.pp = nullptr;
    return pp;
}

// ------------------------------------------------------------------ the path

// The working set W (a7): `sorted` = ascending local columns (the cyclic CD
// order); `slots` = append order (stable storage slots of the Gram matrix).
struct WorkingSet {
    std::vector<int> sorted, slots;
    std::vector<int> ord;          // ord[q] = the storage slot of sorted[q] (the cyclic order over slots)
    // add candidates; returns the columns that were not yet in W (sorted, unique)
    std::vector<int> add(std::vector<int> cand) {
        std::sort(cand.begin(), cand.end());
        cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
        std::vector<int> fresh;
        std::set_difference(cand.begin(), cand.end(), sorted.begin(), sorted.end(), std::back_inserter(fresh));
        if (fresh.empty()) return fresh;
        // merge the sorted columns and their slots in one pass: fresh[i] takes slot |W| + i
        const int base = (int)sorted.size();
        std::vector<int> out, ord2;
        out.reserve(sorted.size() + fresh.size());
        ord2.reserve(sorted.size() + fresh.size());
        size_t a = 0, b = 0;
        while (a < sorted.size() || b < fresh.size()) {
            if (b == fresh.size() || (a < sorted.size() && sorted[a] < fresh[b])) {
                out.push_back(sorted[a]);
                ord2.push_back(ord[a++]);
            } else {
                out.push_back(fresh[b]);
                ord2.push_back(base + (int)b++);
            }
        }
        sorted.swap(out);
        ord.swap(ord2);
        slots.insert(slots.end(), fresh.begin(), fresh.end());
        return fresh;
    }
    int size() const { return (int)sorted.size(); }
};

// W holds GLOBAL column indices (= local ones unless the design is sharded).
void upload_W(bl_prep *pp, const WorkingSet &ws, const std::vector<int> &added) {
    bl_design *d = pp->d;
    const size_t nW = ws.sorted.size();
    const int off = (int)d->col_offset;
    ensure_W(pp, (int64_t)nW);
    ensure_host(pp->hup, pp->hup_cap, 3 * nW + added.size() + 1);
    cudaStream_t st = pp->stream;
    // nothing new: W, its slots and order are on the device already (W only grows within a path)
    if (added.empty()) return;
    const std::vector<int> &ord = ws.ord;   // cyclic order over storage slots: slots sorted by column
    // this shard's new columns (local indices) -> the "in W" flags of the scans
    std::vector<int> mine;
    for (int g : added)
        if (g >= off && g < off + d->p) mine.push_back(g - off);
    // pinned staging: the previous round ended with a stream sync, so hup is free
    int *h = pp->hup;
    for (size_t q = 0; q < nW; q++) { h[q] = ws.sorted[q] - off; h[nW + q] = ws.slots[q] - off; }
    std::memcpy(h + 2 * nW, ord.data(), 4 * nW);
    std::memcpy(h + 3 * nW, mine.data(), 4 * mine.size());
    if (nW || !mine.empty()) {                 // one launch reads the staging in place (zero-copy)
        const int total = (int)std::max(nW, mine.size());
        k_upload_W<<<(unsigned)std::min(64, (total + 255) / 256), 256, 0, st>>>(
            h, (int)nW, (int)mine.size(), d->sharded ? 0 : 1, pp->W, pp->Wst_d, pp->ord_d, pp->viol, pp->wflag);
        CKL();
        pp->launches++;
    }
    if (d->wstore && !added.empty()) {
        // C4: each new column is broadcast by its owner into every rank's store (slots
        // nW - |added| ..; a shard's columns are contiguous in that order).  A host-resident
        // design (NEXT-4) packs its new columns over PCIe into the device store the same way.
        const int64_t slot0 = (int64_t)nW - (int64_t)added.size();
        ensure_Ws(pp, (int64_t)nW, slot0);
        const size_t isz = itemsize(d->dt), colb = (size_t)d->ld * isz;
        CK(cudaMemsetAsync(pp->bw + slot0, 0, 8 * added.size(), st));
        size_t q = 0;
        // the pack kernel of this rank's columns first, then ONE group of broadcasts (every owner's
        // columns, c and s): a single launch per round, nothing waited for on the host
        const int nsh = (int)d->shard_off.size() - 1;      // shards (1 for a replicated design)
        const int mine_r = d->sharded ? d->rank : 0;
        for (int r = 0; r < nsh; r++) {
            const size_t q0 = q;
            while (q < added.size() && added[q] < d->shard_off[r + 1]) q++;
            const int k = (int)(q - q0);
            if (k == 0 || r != mine_r) continue;
            k_pack_cols<<<k, 256, 0, st>>>((const char *)d->X, (int64_t)colb, pp->viol, k, pp->c, pp->s,
                                           (char *)pp->Xw, pp->cw, pp->sw, pp->bw, (int)(slot0 + q0));
            CKL();
            pp->launches++;
        }
        if (!d->sharded) return;
        q = 0;
        d->comm->group_begin();
        for (int r = 0; r < nsh; r++) {
            const size_t q0 = q;
            while (q < added.size() && added[q] < d->shard_off[r + 1]) q++;
            const int k = (int)(q - q0);
            if (k == 0) continue;
            d->comm->bcast((char *)pp->Xw + (size_t)(slot0 + q0) * colb, colb * k, r, st);
            d->comm->bcast(pp->cw + slot0 + q0, 8 * (size_t)k, r, st);
            d->comm->bcast(pp->sw + slot0 + q0, 8 * (size_t)k, r, st);
        }
        d->comm->group_end();
    }
}

// The round's status and the first kListPrefix entries of both index lists in
// ONE device->host round trip (the lists are short except in rare rounds).
int list_prefix(const bl_prep *pp) { return (int)std::min<int64_t>(kListPrefix, pp->p); }   // the lists hold p entries
void copy_round(bl_prep *pp, cudaStream_t st) {
    k_round_out<<<1, 256, 0, st>>>(pp->st, pp->viol, pp->strong, list_prefix(pp), pp->hst, pp->hpre, kListPrefix);
    CKL();
    pp->launches++;
}
std::vector<int> read_list(bl_prep *pp, const int *dev, int count);
// list `which` (0 violators, 1 strong) of the round copied by copy_round
std::vector<int> round_list(bl_prep *pp, int which, int count) {
    if (count > list_prefix(pp)) return read_list(pp, which ? pp->strong : pp->viol, count);
    std::vector<int> v(pp->hpre + which * kListPrefix, pp->hpre + which * kListPrefix + count);
    std::sort(v.begin(), v.end());
    return v;
}

std::vector<int> read_list(bl_prep *pp, const int *dev, int count) {
    std::vector<int> v(count);
    if (count > 0) {
        ensure_host(pp->hlist, pp->hlist_cap, (size_t)count);
        CK(cudaMemcpyAsync(pp->hlist, dev, 4 * (size_t)count, cudaMemcpyDeviceToHost, pp->stream));
        CK(cudaStreamSynchronize(pp->stream));
        std::memcpy(v.data(), pp->hlist, 4 * (size_t)count);
        std::sort(v.begin(), v.end());
    }
    return v;
}

// A device list of local column indices -> sorted GLOBAL indices (all-gathered
// over the shards of a sharded design: C3).
std::vector<int> global_list(bl_prep *pp, const int *dev, int count) {
    if (!pp->d->sharded) return read_list(pp, dev, count);
    const int64_t c = count;
    return gather_list(pp, dev, gather_i64(pp, &c, 1));
}

// C3 for several fits in ONE collective: every rank's round counts (nviol, nstrong, nscope,
// nsafe -- the first four ints of RoundStatus) and the first kXPre entries of both of its
// lists, for every fit, all-gathered on stream st (where the rounds' results were written).
// A list longer than kXPre on some rank is gathered in full afterwards (gather_list).
void exchange_rounds(bl_design *d, const std::vector<bl_prep *> &fits, cudaStream_t st) {
    const size_t F = fits.size(), rec = 4 + 2 * (size_t)kXPre;
    if (F == 0) return;
    bl_prep *p0 = fits[0];
    int *buf = (int *)ensure_cbuf(p0, 4 * rec * F * (d->world + 1));
    CK(cudaStreamSynchronize(p0->stream));               // ensure_cbuf may have swapped the buffer on p0's stream
    for (size_t u = 0; u < F; u++) {
        bl_prep *pp = fits[u];
        const size_t m = (size_t)std::min<int64_t>(kXPre, pp->p);
        int *r0 = buf + u * rec;
        CK(cudaMemcpyAsync(r0, pp->st, 4 * sizeof(int), cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(r0 + 4, pp->viol, 4 * m, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(r0 + 4 + kXPre, pp->strong, 4 * m, cudaMemcpyDeviceToDevice, st));
    }
    d->comm->allgather(buf, buf + rec * F, 4 * rec * F, st);
    ensure_host(p0->hlist, p0->hlist_cap, rec * F * d->world);
    CK(cudaMemcpyAsync(p0->hlist, buf + rec * F, 4 * rec * F * d->world, cudaMemcpyDeviceToHost, st));
    d->comm->wait(st);
    const int *h = p0->hlist;
    for (size_t u = 0; u < F; u++) {
        RoundX &x = fits[u]->xr;
        x.nviol.assign(d->world, 0);
        x.nstrong.assign(d->world, 0);
        x.nscope = x.nsafe = 0;
        x.viol.clear();
        x.strong.clear();
        x.viol_ok = x.strong_ok = true;
        for (int r = 0; r < d->world; r++) {
            const int *q = h + ((size_t)r * F + u) * rec;
            x.nviol[r] = q[0];
            x.nstrong[r] = q[1];
            x.nscope += q[2];
            x.nsafe += q[3];
            const int off = (int)d->shard_off[r];
            if (q[0] > kXPre) x.viol_ok = false;
            else for (int e = 0; e < q[0]; e++) x.viol.push_back(q[4 + e] + off);
            if (q[1] > kXPre) x.strong_ok = false;
            else for (int e = 0; e < q[1]; e++) x.strong.push_back(q[4 + kXPre + e] + off);
        }
        std::sort(x.viol.begin(), x.viol.end());
        std::sort(x.strong.begin(), x.strong.end());
    }
}

// CD block shape: rows per thread R <= RM in {4, 8, 16}; RM <= 8 kernels are
// compiled for <= 512 threads (128 registers), RM = 16 for 1024 threads.
int cd_threads(int64_t n) {
    int64_t rm = n <= 2048 ? 4 : n <= 4096 ? 8 : 16;
    int64_t t = round_up(std::max<int64_t>((n + rm - 1) / rm, 64), 32);
    return (int)std::min<int64_t>(t, rm >= 16 ? 1024 : 512);
}

template <typename T, bool M>
const void *cd_kernel_rm(int R) {
    if (R <= 4) return (const void *)k_cd<T, M, 4>;
    if (R <= 8) return (const void *)k_cd<T, M, 8>;
    return (const void *)k_cd<T, M, 16>;   // R <= 16 by construction (n <= 16384)
}

const void *cd_kernel(int dt, bool mask, int R) {
    if (dt == DT_F64) return mask ? cd_kernel_rm<double, true>(R) : cd_kernel_rm<double, false>(R);
    if (dt == DT_F32) return mask ? cd_kernel_rm<float, true>(R) : cd_kernel_rm<float, false>(R);
    return mask ? cd_kernel_rm<int8_t, true>(R) : cd_kernel_rm<int8_t, false>(R);
}

void launch_cd(bl_prep *pp, int nW, double lam, double alpha, double tol, int max_iter) {
    bl_design *d = pp->d;
    const CdView v = cd_view(pp);
    CdArgs ca{};
    ca.X = v.X;
    ca.ld = d->ld;
    ca.n = (int)d->n;
    ca.W = v.Wsorted;
    ca.nW = nW;
    ca.c = v.c;
    ca.s = v.s;
    ca.beta = v.beta;
    ca.r = pp->rfull;
    ca.r_scan = pp->rscan;
    ca.mask = pp->has_mask ? pp->mask : nullptr;
    ca.lam_alpha = lam * alpha;
    ca.inv_den = 1.0 / (1.0 + lam * (1.0 - alpha));
    ca.inv_n = 1.0 / pp->nt;
    ca.tol = tol;
    ca.floor_ = 1e-13 * (alpha * lam + std::sqrt(pp->hps.Y2 / pp->nt));   // Q6 noise floor
    ca.max_iter = max_iter;
    ca.betaW_out = pp->betaW;
    ca.st = pp->st;
    int T = cd_threads(d->n);
    int R = (int)((d->n + T - 1) / T);
    size_t smem = (size_t)kCdSlotBytes * nW + 16;
    const void *kern = cd_kernel(d->dt, pp->has_mask != 0, R);
    size_t lim = allow_dyn_smem(kern);
    if (smem > lim)
        raise(BL_ERR_OOM, "working set of %d columns does not fit the CD kernel's shared memory (n=%lld)", nW,
              (long long)d->n);
    EvPair ev(pp, &pp->ev_cd);
    void *args[] = {&ca};
    CK(cudaLaunchKernel(kern, dim3(1), dim3(T), args, smem, pp->stream));
    pp->launches++;
}

// ---- NEXT-3 logistic path: IRLS + weighted CD, one CTA per fit (k_cd_logit)
template <typename T, bool M>
const void *logit_kernel_rm(int R) {
    if (R <= 4) return (const void *)k_cd_logit<T, M, 4>;
    if (R <= 8) return (const void *)k_cd_logit<T, M, 8>;
    return (const void *)k_cd_logit<T, M, 16>;
}
const void *logit_kernel(int dt, bool mask, int R) {
    if (dt == DT_F64) return mask ? logit_kernel_rm<double, true>(R) : logit_kernel_rm<double, false>(R);
    if (dt == DT_F32) return mask ? logit_kernel_rm<float, true>(R) : logit_kernel_rm<float, false>(R);
    return mask ? logit_kernel_rm<int8_t, true>(R) : logit_kernel_rm<int8_t, false>(R);
}

void launch_cd_logit(bl_prep *pp, int nW, double lam, double alpha, double tol, int max_iter) {
    bl_design *d = pp->d;
    const CdView v = cd_view(pp);
    CdLogitArgs ca{};
    ca.X = v.X;
    ca.ld = d->ld;
    ca.n = (int)d->n;
    ca.W = v.Wsorted;
    ca.nW = nW;
    ca.c = v.c;
    ca.s = v.s;
    ca.beta = v.beta;
    ca.eta = pp->rfull;                 // the logistic path keeps eta where the linear one keeps r
    ca.y = pp->yraw;
    ca.r_scan = pp->rscan;
    ca.mask = pp->has_mask ? pp->mask : nullptr;
    ca.lam_alpha = lam * alpha;
    ca.lam_l2 = lam * (1.0 - alpha);
    ca.inv_n = 1.0 / pp->nt;
    ca.tol = tol;
    ca.floor_ = 1e-13 * (alpha * lam + 1.0);   // Q6 noise floor (QL6)
    ca.max_iter = max_iter;
    ca.betaW_out = pp->betaW;
    ca.st = pp->st;
    const int T = cd_threads(d->n);
    const int R = (int)((d->n + T - 1) / T);
    const size_t smem = (size_t)kCdLogitSlotBytes * nW + (size_t)4 * round_up(d->n, 2) + 16;
    const void *kern = logit_kernel(d->dt, pp->has_mask != 0, R);
    const size_t lim = allow_dyn_smem(kern);
    if (smem > lim)
        raise(BL_ERR_OOM, "working set of %d columns does not fit the logistic CD kernel's shared memory (n=%lld)",
              nW, (long long)d->n);
    EvPair ev(pp, &pp->ev_cd);
    void *args[] = {&ca};
    CK(cudaLaunchKernel(kern, dim3(1), dim3(T), args, smem, pp->stream));
    pp->launches++;
}

// covariance form (|W| + 1 <= kLogitGramMax): one IRLS iteration = k_logit_eta (eta, weights,
// v = y - pi) -> k_gram_w (weighted Gram incl. the intercept) -> k_cd_logit_gram; the host reads
// the status once per iteration.  The final k_logit_eta leaves r_scan = y - pi for the KKT scan.
template <typename T, bool M>
void solve_logit_gram_t(bl_prep *pp, int nW, double lam, double alpha, double tol, int max_iter) {
    bl_design *d = pp->d;
    cudaStream_t st = pp->stream;
    const CdView v = cd_view(pp);
    const int m = nW + 1;
    const int64_t ld = d->ld;
    const int nblk = (int)((ld + kLogitEtaThreads - 1) / kLogitEtaThreads);
    if (m > pp->ldLG) {
        int64_t nl = round_up(std::max<int64_t>(m, std::min<int64_t>(2 * pp->ldLG, kLogitGramMax)), 32);
        if (pp->LG) cache::dfree(pp->LG);
        pp->LG = nullptr;
        cudaError_t e = cache::dmalloc((void **)&pp->LG, (size_t)8 * nl * nl);
        if (e != cudaSuccess) { cudaGetLastError(); pp->ldLG = 0; raise(BL_ERR_OOM, "cudaMalloc for the weighted Gram: %s", cudaGetErrorString(e)); }
        pp->ldLG = nl;
    }
    const size_t need = (size_t)8 * (kLogitGramMax + ld + 3 * (size_t)nblk);
    if (need > pp->lgcap) {
        if (pp->lgbuf) cache::dfree(pp->lgbuf);
        pp->lgbuf = nullptr;
        cudaError_t e = cache::dmalloc((void **)&pp->lgbuf, need);
        if (e != cudaSuccess) { cudaGetLastError(); pp->lgcap = 0; raise(BL_ERR_OOM, "cudaMalloc for the logistic workspace: %s", cudaGetErrorString(e)); }
        pp->lgcap = need;
    }
    double *bS = pp->lgbuf, *w = bS + kLogitGramMax, *part = w + ld;
    const T *X = reinterpret_cast<const T *>(v.X);
    const uint8_t *mask = M ? pp->mask : nullptr;
    EvPair ev(pp, &pp->ev_cd);
    k_logit_gather<<<(m + 255) / 256, 256, 0, st>>>(bS, v.beta, v.Wst, nW, pp->st);
    CKL();
    pp->launches++;
    CdLogitGramArgs ga{};
    ga.X = v.X; ga.ld = ld; ga.n = (int)d->n; ga.Wst = v.Wst; ga.nW = nW; ga.c = v.c; ga.s = v.s;
    ga.G = pp->LG; ga.ldG = (int)pp->ldLG; ga.gz = v.z; ga.bS = bS;
    ga.beta = v.beta; ga.lam_alpha = lam * alpha; ga.lam_l2 = lam * (1.0 - alpha); ga.inv_n = 1.0 / pp->nt;
    ga.tol = tol; ga.floor_ = 1e-13 * (alpha * lam + 1.0); ga.max_iter = max_iter; ga.st = pp->st;
    const size_t smem = (size_t)40 * m + (size_t)8 * (m + 1) + 16;   // gb, dv (16 B), bo (8 B), two sequences
    const void *kcd = m <= kLGThreads ? (const void *)k_cd_logit_gram<T, 1>
                    : m <= 2 * kLGThreads ? (const void *)k_cd_logit_gram<T, 2>
                    : m <= 4 * kLGThreads ? (const void *)k_cd_logit_gram<T, 4>
                    : m <= 8 * kLGThreads ? (const void *)k_cd_logit_gram<T, 8>
                                          : (const void *)k_cd_logit_gram<T, 16>;
    const size_t lim = allow_dyn_smem(kcd);
    if (smem > lim) raise(BL_ERR_OOM, "logistic covariance CD shared memory %zu > %zu", smem, lim);
    const void *kgw = (const void *)k_gram_w<T, M>;
    allow_dyn_smem(kgw);
    for (int it = 0;; it++) {
        k_logit_eta<T, M><<<nblk, kLogitEtaThreads, 0, st>>>(X, ld, (int)d->n, v.Wst, nW, v.c, v.s, bS, pp->yraw,
                                                             mask, pp->rfull, w, pp->rscan, part, pp->st, it == 0);
        CKL();
        k_gram_w<T, M><<<dim3(m, (m + 31) / 32), 256, (size_t)8 * d->n, st>>>(X, ld, (int)d->n, v.Wst, nW,
                                                                             (int)pp->ldLG, v.c, v.s, w,
                                                                             1.0 / pp->nt, pp->LG, part, nblk,
                                                                             pp->st);
        CKL();
        {                                      // g_W = x~_W' (y - pi) / n (identity (3) with K1 = sum(y - pi))
            ScanArgs sa{};
            sa.list = v.Wst;
            sa.nlist = nullptr;
            sa.nlist_host = nW;
            sa.K1 = &pp->st->sumr;
            sa.K2v = 1.0 / pp->nt;
            sa.out = v.z;
            launch_scan(pp, sa, pp->rscan, false, false, d->wstore ? pp->Xw : nullptr, v.c, v.s);
        }
        void *args[] = {&ga};
        CK(cudaLaunchKernel(kcd, dim3(1), dim3(kLGThreads), args, smem, st));
        pp->launches += 3;
        CK(cudaMemcpyAsync(pp->hst, pp->st, sizeof(RoundStatus), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (pp->hst->cd_status || pp->hst->irls_done) break;
    }
    k_logit_eta<T, M><<<nblk, kLogitEtaThreads, 0, st>>>(X, ld, (int)d->n, v.Wst, nW, v.c, v.s, bS, pp->yraw, mask,
                                                         pp->rfull, w, pp->rscan, part, pp->st, 0);
    CKL();
    k_logit_finish<<<1, 256, 0, st>>>(part, nblk, bS, nW, v.Wst, pp->ord_d, v.c, v.s, pp->betaW, pp->st);
    CKL();
    pp->launches += 2;
}


__global__ void k_logit_init(double *eta, int ld, const PrepScalars *ps, RoundStatus *st) {
    const double yb = ps->ybar, b0 = log(yb / (1.0 - yb));     // the null model (QL2)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ld; i += gridDim.x * blockDim.x) eta[i] = b0;
    if (blockIdx.x == 0 && threadIdx.x == 0) st->b0 = b0;
}

// ---- NEXT-2 Gram CD (covariance updates) -------------------------------------
// Workspace after G: G_AA (ldG^2), block inverses (32 ldG), then the cluster
// kernel's global state: gradients, catch-up deltas (fp64), active list, catch-up
// rows (int32), membership flags (bytes).
size_t gram_ws_bytes(int64_t nl) { return (size_t)8 * nl * nl + (size_t)8 * 32 * nl + (size_t)8 * 7 * nl + (size_t)4 * 2 * nl + (size_t)nl + 64; }
G7Work gram_ws(bl_prep *pp) {
    const int64_t nl = pp->ldG;
    double *base = pp->GA + nl * nl + 32 * nl;
    G7Work w;
    w.g = base;
    w.dl = base + nl;
    w.cg = base + 2 * nl;                                  // 5 nl: the Newton step's vectors (>= 4 (nW + 1))
    w.act = reinterpret_cast<int *>(base + 7 * nl);
    w.rl = w.act + nl;
    w.inA = reinterpret_cast<uint8_t *>(w.rl + nl);
    return w;
}

const void *gram7_kernel(bool enet, int R) {
    static std::once_flag once;
    std::call_once(once, [] {       // 16-CTA clusters are a non-portable size
        cudaFuncSetAttribute((const void *)k_cd_gram7<false, 16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute((const void *)k_cd_gram7<true, 16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    });
    if (R == 4) return enet ? (const void *)k_cd_gram7<true, 4> : (const void *)k_cd_gram7<false, 4>;
    if (R == 16) return enet ? (const void *)k_cd_gram7<true, 16> : (const void *)k_cd_gram7<false, 16>;
    return enet ? (const void *)k_cd_gram7<true, 8> : (const void *)k_cd_gram7<false, 8>;
}
void ensure_G(bl_prep *pp, int64_t need) {
    if (need <= pp->ldG) return;
    int64_t nl = std::max<int64_t>(std::max<int64_t>(need, 2 * pp->ldG), 256);
    nl = round_up(nl, 32);
    double *G2 = nullptr;
    cudaError_t e = cache::dmalloc((void **)&G2, (size_t)8 * nl * nl);
    if (e != cudaSuccess) { cudaGetLastError(); raise(BL_ERR_OOM, "cudaMalloc for the %lld^2 Gram matrix: %s", (long long)nl, cudaGetErrorString(e)); }
    CK(cudaMemsetAsync(G2, 0, (size_t)8 * nl * nl, pp->stream));   // rows/columns past |W| are read (x 0) by bulk copies
    if (pp->G && pp->nG > 0)
        CK(cudaMemcpy2DAsync(G2, 8 * nl, pp->G, 8 * pp->ldG, 8 * (size_t)pp->nG, pp->nG, cudaMemcpyDeviceToDevice,
                             pp->stream));
    if (pp->G) { CK(cudaStreamSynchronize(pp->stream)); cache::dfree(pp->G); }
    pp->G = G2;
    pp->ldG = nl;
    // CD workspaces (contents need not survive): compact G_AA (ldG x ldG) + per-block inverses
    if (pp->GA) cache::dfree(pp->GA);
    pp->GA = nullptr;
    e = cache::dmalloc((void **)&pp->GA, gram_ws_bytes(nl));
    if (e != cudaSuccess) { cudaGetLastError(); pp->GA = nullptr; raise(BL_ERR_OOM, "cudaMalloc for the %lld^2 G_AA workspace: %s", (long long)nl, cudaGetErrorString(e)); }
    CK(cudaMemsetAsync(pp->GA, 0, gram_ws_bytes(nl), pp->stream));
}

template <typename T, bool M>
void launch_gram_t(bl_prep *pp, int nW) {
    bl_design *d = pp->d;
    const void *kern = (const void *)k_gram<T, M>;
    allow_dyn_smem(kern);
    dim3 grid(nW - pp->nG, (nW + 31) / 32);
    const CdView v = cd_view(pp);
    k_gram<T, M><<<grid, 256, 8 * d->n, pp->stream>>>((const T *)v.X, d->ld, (int)d->n, v.Wst, nW, pp->nG,
                                                       (int)pp->ldG, v.c, v.s, M ? pp->mask : nullptr,
                                                       1.0 / pp->nt, pp->G);
    CKL();
    pp->launches++;
}

template <typename T, bool M>
void launch_resid_t(bl_prep *pp, int nW) {
    bl_design *d = pp->d;
    const int nb = (int)((d->ld + 255) / 256);
    const int nch = (nW + kResidChunk - 1) / kResidChunk;
    const CdView v = cd_view(pp);
    double *part = ensure_rbuf(pp, (size_t)nch * d->ld);
    k_resid_part<T, M><<<dim3(nb, nch), 256, 0, pp->stream>>>((const T *)v.X, d->ld, (int)d->n, v.Wst, nW, pp->dbeta,
                                                              v.c, v.s, part);
    CKL();
    k_resid_apply<M><<<nb, 256, 0, pp->stream>>>(part, nch, d->ld, (int)d->n, M ? pp->mask : nullptr, pp->rfull,
                                                pp->rscan, pp->rpart, pp->st);
    CKL();
    pp->launches += 2;
}

bool use_gram(bl_prep *pp, int nW) {
    if (pp->cd_mode == 1) return false;
    if (nW > 4096) {
        if (pp->cd_mode == 2) raise(BL_ERR_OOM, "Gram CD supports |W| <= 4096 (got %d)", nW);
        return false;
    }
    return true;
}

// One CD solve at lambda on the current W (a8), either flavour.
// NEXT-3: the IRLS iteration's quadratic model solved by the cluster Gram CD (k_cd_gram7) in
// intercept-eliminated, unit-curvature coordinates (k_logit_g7_* kernels; per-slot thresholds and,
// for alpha < 1, per-slot ridge denominators).
template <typename T, bool M>
void solve_logit_g7_t(bl_prep *pp, int nW, double lam, double alpha, double tol, int max_iter) {
    bl_design *d = pp->d;
    cudaStream_t st = pp->stream;
    const CdView v = cd_view(pp);
    const int m = nW + 1;
    const int64_t ld = d->ld;
    const int nblk = (int)((ld + kLogitEtaThreads - 1) / kLogitEtaThreads);
    if (m > pp->ldLG) {
        int64_t nl = round_up(std::max<int64_t>(m, std::min<int64_t>(2 * pp->ldLG, kLogitGramMax)), 32);
        if (pp->LG) cache::dfree(pp->LG);
        pp->LG = nullptr;
        cudaError_t e = cache::dmalloc((void **)&pp->LG, (size_t)8 * nl * nl);
        if (e != cudaSuccess) { cudaGetLastError(); pp->ldLG = 0; raise(BL_ERR_OOM, "cudaMalloc for the weighted Gram: %s", cudaGetErrorString(e)); }
        pp->ldLG = nl;
    }
    const size_t need = (size_t)8 * (kLogitGramMax + ld + 3 * (size_t)nblk + 4 * (size_t)kLogitGramMax + 8);
    if (need > pp->lgcap) {
        if (pp->lgbuf) cache::dfree(pp->lgbuf);
        pp->lgbuf = nullptr;
        cudaError_t e = cache::dmalloc((void **)&pp->lgbuf, need);
        if (e != cudaSuccess) { cudaGetLastError(); pp->lgcap = 0; raise(BL_ERR_OOM, "cudaMalloc for the logistic workspace: %s", cudaGetErrorString(e)); }
        pp->lgcap = need;
    }
    ensure_G(pp, nW);
    double *bS = pp->lgbuf, *w = bS + kLogitGramMax, *part = w + ld, *ws = part + 3 * (size_t)nblk;
    long long *acc = reinterpret_cast<long long *>(ws + 4 * (size_t)kLogitGramMax);
    const T *X = reinterpret_cast<const T *>(v.X);
    const uint8_t *mask = M ? pp->mask : nullptr;
    const double inv_n = 1.0 / pp->nt, floor_ = 1e-13 * (alpha * lam + 1.0);
    EvPair ev(pp, &pp->ev_cd);
    k_logit_gather<<<(m + 255) / 256, 256, 0, st>>>(bS, v.beta, v.Wst, nW, pp->st);
    CKL();
    CK(cudaMemsetAsync(acc, 0, 8 * sizeof(long long), st));
    CdGramArgs ga{};
    ga.Wst = v.Wst;
    ga.ord = pp->ord_d;
    ga.nW = nW;
    ga.ldG = (int)pp->ldG;
    ga.G = pp->G;
    ga.GA = pp->GA;
    ga.MA = pp->GA + pp->ldG * pp->ldG;
    ga.z = v.z;
    ga.beta = v.beta;
    ga.dbeta = pp->dbeta;
    ga.lam_alpha = lam * alpha;
    ga.inv_den = 1.0;
    ga.tol = tol;
    ga.floor_ = floor_;
    ga.max_iter = max_iter;
    ga.betaW_out = pp->betaW;
    ga.c = v.c;
    ga.s = v.s;
    ga.st = pp->st;
    ga.tau = ws + nW;
    ga.idv = alpha < 1.0 ? ws + 3 * (size_t)nW : nullptr;
    ga.nu = 0.0;
    ga.newton = 0;                             // per-slot thresholds / curvatures: plain sweeps
    // CTA 0 leads, 1..R-1 own the gradients.  IRLS runs ~2 short solves per lambda: 8-CTA clusters
    // are faster there than 16 (logit bench 124.2 -> 118.7 ms, scripts/cluster_sweep.py) when |W| fits
    int R = pp->cd_cluster;
    if (pp->cd_cluster_auto && gram7_smem(nW, 8) <= allow_dyn_smem(gram7_kernel(alpha < 1.0, 8))) R = 8;
    const void *kern = gram7_kernel(alpha < 1.0, R);
    const size_t smem = gram7_smem(nW, R);
    const size_t lim = allow_dyn_smem(kern);
    if (smem > lim) raise(BL_ERR_OOM, "Gram CD shared memory %zu > %zu (|W| = %d)", smem, lim, nW);
    const void *kgw = (const void *)k_gram_w<T, M>;
    allow_dyn_smem(kgw);
    for (int it = 0;; it++) {
        k_logit_eta<T, M><<<nblk, kLogitEtaThreads, 0, st>>>(X, ld, (int)d->n, v.Wst, nW, v.c, v.s, bS, pp->yraw,
                                                             mask, pp->rfull, w, pp->rscan, part, pp->st, it == 0);
        CKL();
        k_gram_w<T, M><<<dim3(m, (m + 31) / 32), 256, (size_t)8 * d->n, st>>>(X, ld, (int)d->n, v.Wst, nW,
                                                                             (int)pp->ldLG, v.c, v.s, w, inv_n,
                                                                             pp->LG, part, nblk, pp->st);
        CKL();
        {                                      // g_W = x~_W' (y - pi) / n
            ScanArgs sa{};
            sa.list = v.Wst;
            sa.nlist = nullptr;
            sa.nlist_host = nW;
            sa.K1 = &pp->st->sumr;
            sa.K2v = inv_n;
            sa.out = v.z;
            launch_scan(pp, sa, pp->rscan, false, false, d->wstore ? pp->Xw : nullptr, v.c, v.s);
        }
        k_logit_g7_slots<<<(nW + 255) / 256, 256, 0, st>>>(nW, pp->LG, (int)pp->ldLG, v.Wst, bS, v.z, v.beta, ws,
                                                            lam * alpha, lam * (1.0 - alpha), inv_n, pp->st);
        CKL();
        k_logit_g7_schur<<<dim3(nW, (nW + 255) / 256), 256, 0, st>>>(nW, pp->LG, (int)pp->ldLG, ws, pp->G,
                                                                     (int)pp->ldG);
        CKL();
        G7Work wk = gram_ws(pp);
        void *args[] = {&ga, &wk};
        CK(cudaLaunchKernel(kern, dim3(R), dim3(kG7Threads), args, smem, st));
        k_logit_g7_post<<<1, 256, 0, st>>>(nW, pp->LG, (int)pp->ldLG, v.Wst, v.beta, bS, ws, inv_n, tol, floor_,
                                           max_iter, pp->st, acc);
        CKL();
        pp->launches += 6;
        CK(cudaMemcpyAsync(pp->hst, pp->st, sizeof(RoundStatus), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (pp->hst->cd_status || pp->hst->irls_done) break;
    }
    pp->nG = 0;                                // G now holds this model, not the linear Gram
    k_logit_eta<T, M><<<nblk, kLogitEtaThreads, 0, st>>>(X, ld, (int)d->n, v.Wst, nW, v.c, v.s, bS, pp->yraw, mask,
                                                         pp->rfull, w, pp->rscan, part, pp->st, 0);
    CKL();
    k_logit_finish<<<1, 256, 0, st>>>(part, nblk, bS, nW, v.Wst, pp->ord_d, v.c, v.s, pp->betaW, pp->st);
    CKL();
    k_logit_g7_counters<<<1, 1, 0, st>>>(pp->st, acc);
    CKL();
    pp->launches += 3;
}

void solve_logit(bl_prep *pp, int nW, double lam, double alpha, double tol, int max_iter) {
    bl_design *d = pp->d;
    if (nW + 1 > kLogitGramMax || pp->cd_mode == 1) {       // residual form (or requested)
        launch_cd_logit(pp, nW, lam, alpha, tol, max_iter);
        return;
    }
    const bool M = pp->has_mask != 0;
    if (nW >= 1) {                                           // the cluster Gram CD
        if (d->dt == DT_F64) M ? solve_logit_g7_t<double, true>(pp, nW, lam, alpha, tol, max_iter)
                               : solve_logit_g7_t<double, false>(pp, nW, lam, alpha, tol, max_iter);
        else if (d->dt == DT_F32) M ? solve_logit_g7_t<float, true>(pp, nW, lam, alpha, tol, max_iter)
                                    : solve_logit_g7_t<float, false>(pp, nW, lam, alpha, tol, max_iter);
        else M ? solve_logit_g7_t<int8_t, true>(pp, nW, lam, alpha, tol, max_iter)
               : solve_logit_g7_t<int8_t, false>(pp, nW, lam, alpha, tol, max_iter);
        return;
    }
    if (d->dt == DT_F64) M ? solve_logit_gram_t<double, true>(pp, nW, lam, alpha, tol, max_iter)
                           : solve_logit_gram_t<double, false>(pp, nW, lam, alpha, tol, max_iter);
    else if (d->dt == DT_F32) M ? solve_logit_gram_t<float, true>(pp, nW, lam, alpha, tol, max_iter)
                                : solve_logit_gram_t<float, false>(pp, nW, lam, alpha, tol, max_iter);
    else M ? solve_logit_gram_t<int8_t, true>(pp, nW, lam, alpha, tol, max_iter)
           : solve_logit_gram_t<int8_t, false>(pp, nW, lam, alpha, tol, max_iter);
}


void solve_cd(bl_prep *pp, int nW, double lam, double alpha, double tol, int max_iter) {
    if (nW == 0 || !use_gram(pp, nW)) {        // (an empty W -- possible under fault injection -- is a no-op solve)
        launch_cd(pp, nW, lam, alpha, tol, max_iter);
        return;
    }
    bl_design *d = pp->d;
    const bool M = pp->has_mask != 0;
    EvPairOpt ev(pp, &pp->ev_cd);
    if (nW > pp->nG) {                        // G rows/columns of the slots added since the last solve
        ensure_G(pp, nW);
        if (d->dt == DT_F64) M ? launch_gram_t<double, true>(pp, nW) : launch_gram_t<double, false>(pp, nW);
        else if (d->dt == DT_F32) M ? launch_gram_t<float, true>(pp, nW) : launch_gram_t<float, false>(pp, nW);
        else M ? launch_gram_t<int8_t, true>(pp, nW) : launch_gram_t<int8_t, false>(pp, nW);
        pp->nG = nW;
    }
    const CdView v = cd_view(pp);
    {                                          // g_W = x~_W' r / n at the solve's starting residual
        ScanArgs sa{};
        sa.list = v.Wst;
        sa.nlist = nullptr;
        sa.nlist_host = nW;
        sa.K1 = &pp->st->sumr;
        sa.K2v = 1.0 / pp->nt;
        sa.out = v.z;
        launch_scan(pp, sa, pp->rscan, false, false, d->wstore ? pp->Xw : nullptr, v.c, v.s);
    }
    CdGramArgs ga{};
    ga.Wst = v.Wst;
    ga.ord = pp->ord_d;
    ga.nW = nW;
    ga.ldG = (int)pp->ldG;
    ga.G = pp->G;
    ga.GA = pp->GA;
    ga.MA = pp->GA + pp->ldG * pp->ldG;
    ga.z = v.z;
    ga.beta = v.beta;
    ga.dbeta = pp->dbeta;
    ga.lam_alpha = lam * alpha;
    ga.inv_den = 1.0 / (1.0 + lam * (1.0 - alpha));
    ga.tol = tol;
    ga.floor_ = 1e-13 * (alpha * lam + std::sqrt(pp->hps.Y2 / pp->nt));   // Q6 noise floor
    ga.max_iter = max_iter;
    ga.betaW_out = pp->betaW;
    ga.c = v.c;
    ga.s = v.s;
    ga.st = pp->st;
    ga.tau = nullptr;
    ga.idv = nullptr;
    ga.nu = lam * (1.0 - alpha);
    ga.newton = pp->cd_newton;
    // cluster Gram CD: R CTAs of 256 threads (CTA 0 leads, 1..R-1 own the gradients)
    const int R = pp->cd_cluster;   // CTA 0 leads, 1..R-1 own the gradients
    const void *kern = gram7_kernel(alpha < 1.0, R);
    const size_t need = gram7_smem(nW, R);
    const size_t lim = allow_dyn_smem(kern);
    if (need > lim) raise(BL_ERR_OOM, "Gram CD shared memory %zu > %zu (|W| = %d)", need, lim, nW);
    // one CTA per SM either way (255 registers x 256 threads): take all of the SM's shared memory,
    // the Newton steps keep G_AA rows in it
    const size_t smem = lim;
    ga.smem_bytes = (int)smem;
    G7Work wk = gram_ws(pp);
    void *args[] = {&ga, &wk};
    CK(cudaLaunchKernel(kern, dim3(R), dim3(kG7Threads), args, smem, pp->stream));
    pp->launches++;
    if (d->dt == DT_F64) M ? launch_resid_t<double, true>(pp, nW) : launch_resid_t<double, false>(pp, nW);
    else if (d->dt == DT_F32) M ? launch_resid_t<float, true>(pp, nW) : launch_resid_t<float, false>(pp, nW);
    else M ? launch_resid_t<int8_t, true>(pp, nW) : launch_resid_t<int8_t, false>(pp, nW);
}

// One full path as a per-fit state machine, so that one fit (run_path)
// and the K+1 fits of a lockstep cross-validation (run_cv_lockstep) share every
// step.  Per lambda: start() -> [solve() -> fused scan -> after_scan()]* -> record().
struct PathRun {
    bl_prep *pp;
    const double *lambda;
    int K;
    double alpha, tol;
    int max_iter, screen, max_rounds;
    bl_path *out;
    double *heldout;              // device, n_lambda x n, or nullptr
    int family = 0;               // 0 gaussian, 1 binomial (NEXT-3)
    WorkingSet W;
    bool first = true;
    double lam_prev = 0.0, lam = 0.0, lam_next = -1.0, snap = 0.0;
    std::vector<int> strong_next;
    bl_status status = BL_OK;
    int bgrid = 1, use_bedpp = 0;
    // once every live column is safe (BEDPP keeps all below ~0.5 lambda_max; it only keeps more
    // as lambda falls), the flags are constant: one k_bedpp pass without the rule sets them and
    // later lambdas skip the kernel (keeping extra columns is always safe: the KKT check covers them)
    int flags_const = 0;          // 1: flags hold "safe now and next" for every live column
    bool bedpp_skipped = false;
    int k = -1, rounds = 0, passes = 0;
    int64_t scanned = 0, nstrong_k = 0, nsafe_k = 0;

    void begin() {
        bl_design *d = pp->d;
        cudaStream_t st = pp->stream;
        out->n_lambda = K;
        out->n_converged = 0;
        out->lambda.assign(lambda, lambda + K);
        out->a0.assign(K, 0.0);
        out->obj.assign(K, 0.0);
        out->passes.assign(K, 0);
        out->kkt_rounds.assign(K, 0);
        out->cols_scanned.assign(K, 0);
        out->n_safe.assign(K, 0);
        out->n_strong.assign(K, 0);
        out->n_working.assign(K, 0);
        out->outer.assign(K, 0);
        out->family = family;
        out->col_ptr.assign(K + 1, 0);
        const int bthreads = 256;
        bgrid = (int)std::min<int64_t>((d->p + 4 * bthreads - 1) / (4 * bthreads), (int64_t)d->nsm * 8);   // k_bedpp: 1024 cols/block-step
        use_bedpp = screen == BL_SCREEN_HYBRID && family == 0;   // QL3: BEDPP is a linear-model rule
        lam_prev = pp->hps.lmax;
        if (family == 1) {
            k_logit_init<<<(unsigned)((d->ld + 255) / 256), 256, 0, st>>>(pp->rfull, (int)d->ld, pp->ps, pp->st);
            CKL();
            pp->launches++;
        }
        snap = pp->hps.lmax * (1.0 - 1e-12);                   // Q25
        if (screen == BL_SCREEN_NONE) {
            // W = every non-constant column; no screening, no scans (SPEC "policy none")
            CK(cudaMemsetAsync(pp->st, 0, 4 * sizeof(int), st));
            k_bedpp<<<bgrid, 256, 0, st>>>(d->p, pp->s, pp->a, pp->b, pp->ps, alpha, pp->hps.lmax, -1.0, 0,
                                           pp->flags, pp->scope, pp->st);
            CKL();
            pp->launches++;
            CK(cudaMemcpyAsync(pp->hst, pp->st, sizeof(RoundStatus), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            std::vector<int> all = global_list(pp, pp->scope, pp->hst->nscope);
            upload_W(pp, W, W.add(all));
        }
    }
    void heldout_errors() {
        if (!heldout) return;
        bl_design *d = pp->d;
        k_heldout<<<(unsigned)((d->n + 255) / 256), 256, 0, pp->stream>>>(pp->rfull, pp->mask, (int)d->n,
                                                                          heldout + (size_t)k * d->n);
        CKL();
        pp->launches++;
    }
    // lambda_k: false if it is the null solution (recorded here)
    bool start(int kk) {
        bl_design *d = pp->d;
        cudaStream_t st = pp->stream;
        k = kk;
        lam = lambda[k];
        rounds = 0;
        passes = 0;
        scanned = 0;
        nstrong_k = 0;
        nsafe_k = screen == BL_SCREEN_NONE ? pp->hps.n_live : 0;
        if (lam >= snap) {          // null solution, exactly (Q25)
            flush();
            if (family == 1) {          // null logistic model: b0 = logit(ybar), Q = binary entropy of ybar
                const double yb = pp->hps.ybar;
                out->a0[k] = std::log(yb / (1.0 - yb));
                out->obj[k] = -(yb * std::log(yb) + (1.0 - yb) * std::log1p(-yb));
            } else {
                out->a0[k] = pp->hps.ybar;
                out->obj[k] = pp->hps.Y2 / (2.0 * pp->nt);
            }
            out->col_ptr[k + 1] = out->col_ptr[k];
            out->n_converged = k + 1;
            heldout_errors();       // null model: rfull = y_i - ybar_train
            return false;
        }
        lam_next = k + 1 < K ? lambda[k + 1] : -1.0;
        if (screen != BL_SCREEN_NONE) {
            CK(cudaMemsetAsync(pp->st, 0, 4 * sizeof(int), st));   // counters only: sum r / rss persist
            bedpp_skipped = !use_bedpp && flags_const && !first;
            if (!bedpp_skipped) {
                k_bedpp<<<bgrid, 256, 0, st>>>(d->p, pp->s, pp->a, pp->b, pp->ps, alpha, lam, lam_next, use_bedpp,
                                               pp->flags, use_bedpp ? pp->scope : nullptr, pp->st);
                CKL();
                pp->launches++;
                if (!use_bedpp && lam_next > 0.0) flags_const = 1;
            }
            if (first) {
                // strong set at the first solved lambda from the null solution z = a/n (a6)
                const double lp = std::min(lam_prev, pp->hps.lmax);
                const double thr = alpha * (2.0 * lam - lp);
                k_ssr_init<<<bgrid, 256, 0, st>>>(d->p, pp->a, pp->s, pp->flags, pp->wflag, pp->ps,
                                                  thr < 0.0 ? 0.0 : thr, pp->z, pp->strong, &pp->st->nstrong);
                CKL();
                pp->launches++;
                CK(cudaMemcpyAsync(pp->hst, pp->st, sizeof(RoundStatus), cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                strong_next = global_list(pp, pp->strong, pp->hst->nstrong);
                first = false;
            }
            if (pp->fault_strong_drop) strong_next.clear();   // TEST ONLY: the KKT check must find them
            nstrong_k = (int64_t)strong_next.size();
            upload_W(pp, W, W.add(strong_next));
            strong_next.clear();
        }
        return true;
    }
    void solve() {
        if (family == 1) solve_logit(pp, W.size(), lam, alpha, tol, max_iter);
        else solve_cd(pp, W.size(), lam, alpha, tol, max_iter);
        if (screen != BL_SCREEN_NONE) CK(cudaMemsetAsync(&pp->st->nviol, 0, 2 * sizeof(int), pp->stream));
    }
    // the fused KKT + strong-rule scan of this round (a9)
    ScanArgs scan_args() const {
        ScanArgs sa{};
        sa.list = use_bedpp ? pp->scope : nullptr;
        sa.nlist = &pp->st->nscope;
        sa.K1 = &pp->st->sumr;
        sa.K2v = 1.0 / pp->nt;
        sa.out = pp->z;
        sa.jfix = nullptr;
        sa.scan = 1;
        sa.flags = pp->flags;
        sa.wflag = pp->wflag;
        sa.thr_viol = alpha * lam;
        sa.thr_strong = lam_next > 0.0 ? alpha * (2.0 * lam_next - lam) : -1.0;
        if (sa.thr_strong < 0.0 && lam_next > 0.0) sa.thr_strong = 0.0;
        sa.viol = pp->viol;
        sa.nviol = &pp->st->nviol;
        sa.strong = pp->strong;
        sa.nstrong = &pp->st->nstrong;
        sa.rev = pp->scan_rev;
        pp->scan_rev ^= 1;
        return sa;
    }
    void count_cd() {
        passes += pp->hst->cd_passes;
        out->cd_visits += pp->hst->cd_visits;
        out->cd_updates += pp->hst->cd_updates;
        out->cd_cycles += pp->hst->cd_cycles;
        for (int u = 0; u < 4; u++) out->cd_prof[u] += pp->hst->cd_prof[u];
        for (int u = 0; u < 8; u++) out->cd_cnt[u] += pp->hst->cd_cnt[u];
        for (int u = 0; u < 8; u++) out->cd_dbg[u] += pp->hst->cd_dbg[u];
    }
    // after the round's status reached pp->hst: 0 = lambda done, 1 = re-solve, -1 = error (status set).
    // `batched`: the round's scan was a fold-batched launch shared with other fits (its columns --
    // the union scope -- are in RoundStatus.nscope; it is timed on the batch's first fit only).
    int after_scan(bool batched = false) {
        bl_design *d = pp->d;
        count_cd();
        if (screen == BL_SCREEN_NONE) {
            if (pp->hst->cd_status) { status = BL_ERR_CONVERGENCE; return -1; }
            return 0;
        }
        // the round's counts over all shards (C3, exchanged by exchange_rounds before this call):
        // violators, strong candidates, columns scanned
        int64_t nviol = 0, nscope = 0, nsafe = 0;
        std::vector<int64_t> cv, cs;
        if (d->sharded) {
            const RoundX &x = pp->xr;
            cv = x.nviol;
            cs = x.nstrong;
            for (int64_t v : cv) nviol += v;
            nscope = x.nscope;
            nsafe = x.nsafe;
        } else {
            nviol = pp->hst->nviol;
            nscope = pp->hst->nscope;
            nsafe = pp->hst->nsafe;
        }
        nsafe_k = bedpp_skipped ? (int64_t)pp->hps.n_live : nsafe;
        const int64_t round_cols = use_bedpp ? nscope : pp->hps.n_live;
        scanned += round_cols;
        if (!batched && pp->scan_full.size() < pp->ev_scan.size())   // classify the timed scan launch of this round
            pp->scan_full.push_back(round_cols == pp->hps.n_live ? (use_bedpp ? (int64_t)pp->hst->nscope : pp->p) : -1);
        if (use_bedpp && nsafe == pp->hps.n_live) use_bedpp = 0;   // BEDPP keeps everything from here on
        if (pp->hst->cd_status) { status = BL_ERR_CONVERGENCE; return -1; }
        if (nviol > 0) {
            if (++rounds >= max_rounds) {             // R_k = rounds + 1 would exceed the cap
                g_err = "more than max KKT rounds at one lambda";
                status = BL_ERR_CONVERGENCE;
                return -1;
            }
            std::vector<int> v = !d->sharded ? round_list(pp, 0, pp->hst->nviol)
                                 : pp->xr.viol_ok ? pp->xr.viol : gather_list(pp, pp->viol, cv);
            upload_W(pp, W, W.add(v));
            return 1;
        }
        strong_next = !d->sharded ? round_list(pp, 1, pp->hst->nstrong)
                      : pp->xr.strong_ok ? pp->xr.strong : gather_list(pp, pp->strong, cs);
        return 0;
    }
    void fail() {
        if (g_err.empty() || pp->hst->cd_status)
            g_err = "coordinate descent did not converge within max_iter passes at lambda index " + std::to_string(k);
    }
    // record lambda_k (a11).  The coefficients are copied device -> pinned host without
    // waiting; they are unstandardised in order when the buffer is full or the path ends.
    struct Pending {
        int k, nW, passes, rounds;
        size_t off;
        std::vector<int> sorted;
        double lam;
        RoundStatus rs;
        int64_t scanned, nsafe, nstrong;
    };
    std::vector<Pending> pend;
    size_t hoff = 0;
    void emit(const Pending &r, const double *hb) {
        // unstandardise (Q4): beta_orig = beta/s_j, a0 = ybar - sum beta_orig c_j
        double shift = 0.0;
        for (int q = 0; q < r.nW; q++) {
            const double bq = hb[q];
            if (bq == 0.0) continue;
            const double cq = hb[r.nW + q], sq = hb[2 * r.nW + q];
            out->feat.push_back(r.sorted[q]);
            out->beta_std.push_back(bq);
            out->beta_orig.push_back(bq / sq);
            shift += bq * cq / sq;
        }
        out->col_ptr[r.k + 1] = (int64_t)out->feat.size();
        const double pen = r.lam * (alpha * r.rs.l1 + 0.5 * (1.0 - alpha) * r.rs.l2);
        if (family == 1) {              // QL1: intercept b0 on the standardised scale; loss sum in rs.rss
            out->a0[r.k] = r.rs.b0 - shift;
            out->obj[r.k] = r.rs.rss / pp->nt + pen;
            out->outer[r.k] = r.rs.outer;
        } else {
            out->a0[r.k] = pp->hps.ybar - shift;
            out->obj[r.k] = r.rs.rss / (2.0 * pp->nt) + pen;
        }
        out->passes[r.k] = r.passes;
        out->kkt_rounds[r.k] = r.rounds;
        out->cols_scanned[r.k] = r.scanned;
        out->n_safe[r.k] = r.nsafe;
        out->n_strong[r.k] = r.nstrong;
        out->n_working[r.k] = r.nW;
        out->n_converged = r.k + 1;
    }
    void flush() {
        if (pend.empty()) return;
        CK(cudaStreamSynchronize(pp->stream));
        for (const Pending &r : pend) emit(r, pp->hbw + r.off);
        pend.clear();
        hoff = 0;
    }
    void record() {
        const int nW = (int)W.size();
        if (hoff + 3 * (size_t)nW > pp->hbw_cap) {
            flush();
            ensure_host(pp->hbw, pp->hbw_cap, std::max<size_t>(3 * (size_t)nW, (size_t)1 << 18));
        }
        if (nW > 0)
            CK(cudaMemcpyAsync(pp->hbw + hoff, pp->betaW, 24 * (size_t)nW, cudaMemcpyDeviceToHost, pp->stream));
        pend.push_back(Pending{k, nW, passes, rounds + (screen == BL_SCREEN_NONE ? 0 : 1), hoff, W.sorted, lam,
                               *pp->hst, scanned, nsafe_k, nstrong_k});
        hoff += 3 * (size_t)nW;
        heldout_errors();
        lam_prev = lam;
    }
};

bl_status run_path(bl_prep *pp, const double *lambda, int K, double alpha, double tol, int max_iter, int screen,
                   int max_rounds, bl_path *out, double *heldout /* device, n_lambda x n, or nullptr */,
                   int family = 0) {
    PathRun pr{pp, lambda, K, alpha, tol, max_iter, screen, max_rounds, out, heldout, family};
    pr.begin();
    cudaStream_t st = pp->stream;
    for (int k = 0; k < K; k++) {
        if (!pr.start(k)) continue;
        int res;
        do {
            pr.solve();
            if (screen != BL_SCREEN_NONE) launch_scan(pp, pr.scan_args(), pp->rscan, true);
            copy_round(pp, st);
            CK(cudaStreamSynchronize(st));
            if (pp->d->sharded && screen != BL_SCREEN_NONE) exchange_rounds(pp->d, {pp}, st);
            res = pr.after_scan();
        } while (res == 1);
        if (res < 0) { pr.fail(); break; }
        pr.record();
    }
    pr.flush();
    CK(cudaStreamSynchronize(st));
    return pr.status;
}

void validate_grid(const double *lambda, int K) {
    if (!lambda || K < 1) raise(BL_ERR_ARG, "need at least one lambda");
    for (int k = 0; k < K; k++) {
        if (!(lambda[k] > 0.0) || !std::isfinite(lambda[k])) raise(BL_ERR_ARG, "lambda[%d] = %g must be > 0", k, lambda[k]);
        if (k > 0 && !(lambda[k] < lambda[k - 1])) raise(BL_ERR_ARG, "lambda must be strictly decreasing (index %d)", k);
    }
}

void finish_perf(bl_prep *pp, bl_path *out, double wall_ms) {
    CK(cudaStreamSynchronize(pp->stream));
    bl_perf &pf = out->perf;
    std::memset(&pf, 0, sizeof pf);
    pf.scan_launches = (int64_t)pp->ev_scan.size();
    pf.cd_launches = (int64_t)pp->ev_cd.size();
    double full_ms = 0.0;
    for (size_t i = 0; i < pp->scan_full.size() && i < pp->ev_scan.size(); i++)
        if (pp->scan_full[i] >= 0) {
            pf.full_scan_launches++;
            pf.full_scan_bytes += (double)pp->scan_full[i] * (double)pp->d->n * itemsize(pp->d->dt);
        }
    pf.scan_ms = sum_events(pp->ev_scan, &pp->scan_full, &full_ms, &pp->evpool);
    pf.full_scan_ms = full_ms;
    pp->scan_full.clear();
    pf.cd_ms = sum_events(pp->ev_cd, nullptr, nullptr, &pp->evpool);
    pf.prep_ms = sum_events(pp->ev_prep, nullptr, nullptr, &pp->evpool);
    int64_t cols = 0;
    for (int k = 0; k < out->n_converged; k++) cols += out->cols_scanned[k];
    pf.scan_bytes = (double)cols * (double)pp->d->n * itemsize(pp->d->dt);
    pf.prep_bytes = pp->prep_bytes;
    pf.kernel_launches = pp->launches;
    pf.cd_visits = out->cd_visits;
    pf.cd_updates = out->cd_updates;
    pf.cd_kernel_cycles = out->cd_cycles;
    for (int u = 0; u < 4; u++) pf.cd_prof[u] = out->cd_prof[u];
    for (int u = 0; u < 8; u++) pf.cd_events[u] = out->cd_cnt[u];
    for (int u = 0; u < 8; u++) pf.cd_sub[u] = out->cd_dbg[u];
    pf.wall_ms = wall_ms;
}

// ---- NEXT-1: lockstep cross-validation with fold-batched scans
// All fits of this rank (folds, and the full-data fit: fold index -1) advance
// lambda by lambda.  Their CD solves run concurrently on their own streams; each
// KKT round's fused scans of every fit still solving at that lambda are ONE pass
// over X (k_scan_batch; int8 designs scan per fit).  Results are the same paths
// as independent fits: every fit's arithmetic is unchanged, only the scan kernel
// that evaluates the (identical) identity-(3) epilogue differs.
struct LockFit {
    bl_prep *pp = nullptr;
    bl_path *out = nullptr;
    std::unique_ptr<PathRun> run;
    bool alive = true;
    bl_status st = BL_OK;
    std::string err;
    cudaEvent_t solved = nullptr;
};

template <int NF>
const void *batch_kernel_n(bool f64, int nb) {
    if constexpr (NF > 1) {
        if (nb < NF) return batch_kernel_n<NF - 1>(f64, nb);
    }
    return f64 ? (const void *)k_scan_batch<double, NF> : (const void *)k_scan_batch<float, NF>;
}
const void *batch_kernel(bool f64, int nb) { return batch_kernel_n<kBatchMax>(f64, nb); }
template <int NF>
const void *batch_i8_kernel_n(int nb) {
    if constexpr (NF > 1) {
        if (nb < NF) return batch_i8_kernel_n<NF - 1>(nb);
    }
    return (const void *)k_scan_batch_i8<NF>;
}
template <int NF>
const void *batch_mma_kernel_n(bool f64, int nb) {
    if constexpr (NF > 1) {
        if (nb < NF) return batch_mma_kernel_n<NF - 1>(f64, nb);
    }
    return f64 ? (const void *)k_scan_batch_mma<double, NF> : (const void *)k_scan_batch_mma<float, NF>;
}
// fold-batched scan kernels (bl_opts.cv_mode): BK_TC the integer tensor cores (tcgen05, fp32 designs),
// BK_DMMA the fp64 tensor cores (fp64 designs, or on request), BK_FMA fp64 FMAs; int8 designs: IMMA
enum BatchKind { BK_TC = 0, BK_FMA = 1, BK_DMMA = 3 };
template <int NF>
const void *batch_tc_kernel_n(int nb) {
    if constexpr (NF > 1) {
        if (nb < NF) return batch_tc_kernel_n<NF - 1>(nb);
    }
    return (const void *)k_scan_batch_tc<NF>;
}
// the per-column digit scale of an fp32 design (one pass over X, once per design)
const float *design_xscale(bl_design *d, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(d->pool_mu);
    if (!d->xsc) {
        float *x = nullptr;
        CK(cache::dmalloc((void **)&x, sizeof(float) * (size_t)std::max<int64_t>(d->p, 1)));
        const int grid = (int)std::min<int64_t>((d->p + 7) / 8, (int64_t)d->nsm * 8);
        k_xscale<<<grid, 256, 0, st>>>((const float *)d->X, d->ld, (int)d->n, d->p, x);
        CKL();
        CK(cudaStreamSynchronize(st));
        d->xsc = x;
    }
    return d->xsc;
}
struct TcScratch {
    int8_t *img = nullptr;           // residual digit tiles of one pass (stages x tc_bbytes(kTcMaxFits))
    double *rsc = nullptr;           // 2^-S_f per fit
    int *dsum = nullptr;             // digit sums per (fit, digit)
    ~TcScratch() {
        if (img) cache::dfree(img);
        if (rsc) cache::dfree(rsc);
        if (dsum) cache::dfree(dsum);
    }
};
// the batched kernels' view of one fit (its ScanArgs plus the residual and column statistics)
FitScan fitscan_of(const bl_design *d, bl_prep *pp, const ScanArgs &sa) {
    FitScan F{};
    F.r = pp->rscan;
    F.K1 = sa.K1;
    F.K2 = sa.K2v;
    F.c = pp->c;
    F.s = pp->s;
    F.out = sa.out;
    F.flags = sa.flags;
    F.wflag = sa.wflag;
    F.thr_viol = sa.thr_viol;
    F.thr_strong = sa.thr_strong;
    F.viol = sa.viol;
    F.nviol = sa.nviol;
    F.strong = sa.strong;
    F.nstrong = sa.nstrong;
    F.limbs = nullptr;
    F.limb_scale = nullptr;
    if (d->dt == DT_I8) {                           // the quantised residual (k_limbs, launched by the caller)
        F.limbs = pp->limbs;
        F.limb_scale = pp->limb_scale;
        F.K1 = pp->limb_sum;                        // identity (3) holds exactly for the quantised vector
    }
    return F;
}
// One fold-batched pass for the nf fits whose FitScan entries are in hfs (host); int8 designs
// need the fits' digit planes (k_limbs) already launched on sst.  limb_ld: the fits' plane stride.
void launch_scan_batch_fs(bl_design *d, size_t nf, int limb_ld, cudaStream_t sst, FitScan *dfs, FitScan *hfs,
                          bl_prep *timer, int bk, const int *list, const int *lctl, TcScratch *tcs, bool prep = false) {
    CK(cudaMemcpyAsync(dfs, hfs, sizeof(FitScan) * nf, cudaMemcpyHostToDevice, sst));
    const bool f64 = d->dt == DT_F64;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timer->profile) {
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, sst));
    }
    // (the integer accumulators are exact for n <= 27,000 -- bl_tc.cuh; designs hold n <= 16,384)
    const bool tc = bk == BK_TC && d->dt == DT_F32 && d->n <= 27000;
    const bool mma = bk == BK_DMMA || (bk == BK_TC && !tc);     // fp64 designs (and any the tc path declines)
    const int nst = (int)((d->n + kTcRows - 1) / kTcRows);
    const float *xsc = tc ? design_xscale(d, sst) : nullptr;
    if (tc && !tcs->img) {
        CK(cache::dmalloc((void **)&tcs->img, (size_t)nst * tc_bbytes(kTcMaxFits)));
        CK(cache::dmalloc((void **)&tcs->rsc, sizeof(double) * kTcMaxFits));
        CK(cache::dmalloc((void **)&tcs->dsum, sizeof(int) * kTcRL * kTcMaxFits));
    }
    for (size_t u0 = 0; u0 < nf; u0 += (tc ? kTcMaxFits : kBatchMax)) {
        int nb = (int)std::min<size_t>(tc ? kTcMaxFits : kBatchMax, nf - u0);
        const bool i8 = d->dt == DT_I8;
        if (tc) {                                    // residual digits, then the tensor-core pass
            FitScan *fp = dfs + u0;
            CK(cudaMemsetAsync(tcs->img, 0, (size_t)nst * tc_bbytes(nb), sst));
            k_rimg<<<nb, 1024, 0, sst>>>(fp, (int)d->n, tc_n(nb) / 2, tcs->img, tcs->rsc, tcs->dsum);
            CKL();
            const void *kern = batch_tc_kernel_n<kTcMaxFits>(nb);
            const size_t smem = tc_smem(nb);
            allow_dyn_smem(kern);
            // CTA pairs (cluster dims 2), one CTA per SM, persistent over 256-column tiles
            const int pairs = (int)std::max<int64_t>(1, std::min<int64_t>((d->p + 2 * kTcCols - 1) / (2 * kTcCols),
                                                                          (int64_t)d->nsm / 2));
            const float *X = (const float *)d->X;
            int64_t ld = d->ld, p = d->p;
            int n = (int)d->n;
            const int8_t *img = tcs->img;
            const double *rsc = tcs->rsc;
            const int *dsum = tcs->dsum;
            void *args[] = {&X, &ld, &n, &p, &fp, &xsc, &img, &rsc, &dsum, &list, &lctl};
            CK(cudaLaunchKernel(kern, dim3(2 * pairs), dim3(kTcThreads), args, smem, sst));
            timer->launches += 2;
            if (!prep) timer->batch_passes++;
            continue;
        }
        const void *kern = i8 ? batch_i8_kernel_n<kBatchMax>(nb)
                         : mma ? batch_mma_kernel_n<kBatchMax>(f64, nb) : batch_kernel(f64, nb);
        const size_t smem = i8 ? batch_i8_smem(nb) : mma ? batch_mma_smem(nb) : batch_smem(nb, itemsize(d->dt));
        const int threads = i8 ? kScanThreads : mma ? kBMThreads : kBatchThreads;
        allow_dyn_smem(kern);
        const int grid = grid_for(kern, threads, smem, d->nsm);
        const void *X = d->X;
        int64_t ld = d->ld, p = d->p;
        int n = (int)d->n;
        FitScan *fp = dfs + u0;
        void *args[] = {&X, &ld, &n, &p, &fp, &nb, &list, &lctl};
        void *args_i8[] = {&X, &ld, &n, &p, &fp, &limb_ld, &list, &lctl};
        if (i8) {
            CK(cudaLaunchKernel(kern, dim3(grid), dim3(threads), args_i8, smem, sst));
            timer->launches++;
            if (!prep) timer->batch_passes++;
            continue;
        }
        CK(cudaLaunchKernel(kern, dim3(grid), dim3(threads), args, smem, sst));
        timer->launches++;
        if (!prep) timer->batch_passes++;                           // X bytes: accounted once the union size is known
    }
    if (timer->profile) {
        CK(cudaEventRecord(e1, sst));
        (prep ? timer->ev_prep : timer->ev_scan).push_back({e0, e1});
    }
}

void launch_scan_batch(bl_design *d, const std::vector<LockFit *> &fits, cudaStream_t sst, FitScan *dfs,
                       FitScan *hfs, bl_prep *timer, int bk, const int *list, const int *lctl, TcScratch *tcs) {
    for (size_t u = 0; u < fits.size(); u++) hfs[u] = fitscan_of(d, fits[u]->pp, fits[u]->run->scan_args());
    launch_scan_batch_fs(d, fits.size(), fits.empty() ? 0 : fits[0]->pp->limb_ld, sst, dfs, hfs, timer, bk, list, lctl,
                         tcs);
}

// fit_ids: fold index per fit (-1 = full data).  Paths (prefix on failure) and
// statuses per fit; held-out errors of the folds go to dE (n_lambda x n).
void cv_lockstep(bl_design *d, const double *y, const std::vector<int32_t> &fold, const std::vector<int> &fit_ids,
                 const double *lambda, int K, double alpha, double tol, int max_iter, const bl_opts *opts,
                 double *dE, std::vector<bl_path *> &paths, std::vector<bl_status> &sts, std::vector<std::string> &errs) {
    const int64_t n = d->n;
    const size_t F = fit_ids.size();
    bl_opts fo{};
    if (opts) fo = *opts;
    fo.stream = nullptr;                                   // every fit on its own library stream
    if (fo.cd_cluster == 0) fo.cd_cluster = 8;             // K + 1 concurrent CD clusters share the SMs
    const int rounds = opts && opts->max_kkt_rounds > 0 ? opts->max_kkt_rounds : 10;
    std::vector<LockFit> fits(F);
    cudaStream_t sst = nullptr;
    FitScan *dfs = nullptr, *hfs = nullptr;
    int *uni = nullptr;                                    // [count, use_list, list (p)]: the union BEDPP scope
    void **dptr = nullptr, **hptr = nullptr;               // per pending fit: flags, nlive, RoundStatus pointers
    int *hctl = nullptr;                                   // pinned: the round's [count, use_list]
    const bool batched = true;                           // every round is one fold-batched pass (int8: IMMA)
    const int bk = opts ? opts->cv_mode : BK_TC;           // fold-batched scan kernel (BatchKind)
    TcScratch tcs;
    auto t0 = std::chrono::steady_clock::now();
    auto cleanup = [&]() {
        if (sst) cudaStreamSynchronize(sst);
        for (auto &lf : fits) {
            if (lf.solved) cudaEventDestroy(lf.solved);
            if (lf.pp) release_prep(lf.pp);
            lf.pp = nullptr;
        }
        if (dfs) cache::dfree(dfs);
        if (hfs) cache::hfree(hfs);
        if (uni) cache::dfree(uni);
        if (dptr) cache::dfree(dptr);
        if (hptr) cache::hfree(hptr);
        if (hctl) cache::hfree(hctl);
        if (sst) cudaStreamDestroy(sst);
    };
    try {
        CK(cudaStreamCreateWithFlags(&sst, cudaStreamNonBlocking));
        CK(cache::dmalloc((void **)&dfs, sizeof(FitScan) * std::max<size_t>(F, 1)));
        CK(cache::dmalloc((void **)&uni, sizeof(int) * (size_t)(d->p + 2)));
        CK(cache::dmalloc((void **)&dptr, 3 * sizeof(void *) * std::max<size_t>(F, 1)));
        CK(cache::hmalloc((void **)&hptr, 3 * sizeof(void *) * std::max<size_t>(F, 1)));
        CK(cache::hmalloc((void **)&hctl, 2 * sizeof(int)));
        CK(cache::hmalloc((void **)&hfs, sizeof(FitScan) * std::max<size_t>(F, 1)));
        // Preprocessing in stages (a2-a4): every fit's a_j and b_j store-mode scans run as two
        // fold-batched passes over X instead of 2 (K + 1) -- NEXT-1 applied to the preprocessing
        // (one X serves every fold); column statistics stay per fit.  A fit whose
        // preprocessing fails (e.g. y constant on its training rows) drops out, as in the threaded mode.
        auto drop = [&](LockFit &lf, const Err &er) {
            lf.alive = false;
            lf.st = er.code;
            lf.err = g_err;
            g_err.clear();
            if (lf.pp) { release_prep(lf.pp); lf.pp = nullptr; }
        };
        auto prep_batch = [&](int which) {             // 0: a_j = x~'y~, 1: b_j = x~'x~_* (b_j* = n)
            std::vector<LockFit *> live;
            for (auto &lf : fits)
                if (lf.alive && lf.pp) live.push_back(&lf);
            if (live.empty()) return;
            std::vector<PrepScalars> hs(live.size());
            for (size_t u = 0; u < live.size(); u++) {
                bl_prep *pp = live[u]->pp;
                if (which == 1) {                          // 1 / s_* and j* of every fit on the host
                    CK(cudaMemcpyAsync(&hs[u], pp->ps, sizeof(PrepScalars), cudaMemcpyDeviceToHost, pp->stream));
                    CK(cudaStreamSynchronize(pp->stream));
                }
                cudaEvent_t ev;
                CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                CK(cudaEventRecord(ev, pp->stream));
                CK(cudaStreamWaitEvent(sst, ev, 0));
                CK(cudaEventDestroy(ev));
            }
            for (size_t u = 0; u < live.size(); u++) {
                bl_prep *pp = live[u]->pp;
                const double *v = which ? pp->vtmp : pp->yt;
                if (d->dt == DT_I8) {                      // the vector's digit planes (Q27)
                    k_limbs<<<1, 1024, 0, sst>>>(v, (int)d->n, pp->limb_ld, pp->limbs, pp->limb_scale, pp->limb_sum);
                    CKL();
                }
                ScanArgs sa{};
                sa.K1 = which ? &pp->ps->sum_v : &pp->ps->sum_yt;
                sa.K2v = which ? hs[u].inv_s_star : 1.0;
                sa.out = which ? pp->b : pp->a;
                sa.flags = pp->flags;
                sa.wflag = pp->wflag;
                sa.thr_viol = HUGE_VAL;                    // store mode: no tests, no lists
                sa.thr_strong = -1.0;
                sa.viol = pp->viol;
                sa.nviol = &pp->st->nviol;
                sa.strong = pp->strong;
                sa.nstrong = &pp->st->nstrong;
                hfs[u] = fitscan_of(d, pp, sa);
                hfs[u].r = v;
            }
            // the fp64 tensor-core (or FMA) kernel: a_j and b_j feed lambda_max and BEDPP, kept fp64
            launch_scan_batch_fs(d, live.size(), live[0]->pp->limb_ld, sst, dfs, hfs, live[0]->pp,
                                 bk == BK_FMA ? BK_FMA : BK_DMMA, nullptr, nullptr, &tcs, true);
            if (which == 1)
                for (size_t u = 0; u < live.size(); u++)
                    if (hs[u].jstar >= 0)                  // b_j* = n exactly (identity (1))
                        CK(cudaMemcpyAsync(live[u]->pp->b + hs[u].jstar, &live[u]->pp->ps->nt, sizeof(double),
                                           cudaMemcpyDeviceToDevice, sst));
            cudaEvent_t ev;
            CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            CK(cudaEventRecord(ev, sst));
            for (LockFit *lf : live) CK(cudaStreamWaitEvent(lf->pp->stream, ev, 0));
            CK(cudaEventDestroy(ev));
            CK(cudaStreamSynchronize(sst));                // (hfs is rewritten by the next pass)
        };
        // column statistics of every fit in one pass (k_colstats_folds): folds partition the rows
        int kfold = 0;
        for (int64_t i = 0; i < n; i++) kfold = std::max(kfold, (int)fold[i] + 1);
        const bool fold_stats = F <= 32 && kfold <= 32;
        std::vector<std::vector<uint8_t>> trains(F);
        for (size_t u = 0; u < F; u++) {
            LockFit &lf = fits[u];
            if (fit_ids[u] >= 0) {
                trains[u].resize(n);
                for (int64_t i = 0; i < n; i++) trains[u][i] = fold[i] != fit_ids[u];
            }
            lf.out = new bl_path();
            lf.out->magic = MAGIC_PATH;
            try {
                lf.pp = prep_begin(d, y, trains[u].empty() ? nullptr : trains[u].data(), alpha, &fo, fold_stats);
            } catch (const Err &er) {
                if (d->sharded) throw;                     // (a sharded fit is collective: every rank fails it)
                drop(lf, er);
            }
        }
        if (fold_stats) {
            std::vector<LockFit *> live;
            std::vector<int> ff;
            std::vector<double> nts;
            std::vector<double *> ptrs;
            for (size_t u = 0; u < F; u++)
                if (fits[u].alive && fits[u].pp) {
                    live.push_back(&fits[u]);
                    ff.push_back(fit_ids[u]);
                    nts.push_back(fits[u].pp->nt);
                    ptrs.push_back(fits[u].pp->c);
                    ptrs.push_back(fits[u].pp->s);
                }
            if (!live.empty()) {
                const size_t nl = live.size();
                std::vector<int8_t> fh(n);
                for (int64_t i = 0; i < n; i++) fh[i] = (int8_t)fold[i];
                char *buf = nullptr;                       // [fold ids (n, padded)][fit folds][nt][c, s pointers]
                const size_t o_ff = round_up((size_t)n, 16), o_nt = o_ff + round_up(4 * nl, 16),
                             o_p = o_nt + 8 * nl, tot = o_p + 16 * nl;
                CK(cache::dmalloc((void **)&buf, tot));
                CK(cudaMemcpyAsync(buf, fh.data(), n, cudaMemcpyHostToDevice, sst));
                CK(cudaMemcpyAsync(buf + o_ff, ff.data(), 4 * nl, cudaMemcpyHostToDevice, sst));
                CK(cudaMemcpyAsync(buf + o_nt, nts.data(), 8 * nl, cudaMemcpyHostToDevice, sst));
                CK(cudaMemcpyAsync(buf + o_p, ptrs.data(), 16 * nl, cudaMemcpyHostToDevice, sst));
                const void *kern = d->dt == DT_F64 ? (const void *)k_colstats_folds<double>
                                 : d->dt == DT_F32 ? (const void *)k_colstats_folds<float>
                                                   : (const void *)k_colstats_folds<int8_t>;
                const size_t smem = (size_t)8 * kfold * 64 * 8 + round_up((size_t)n, 16);
                allow_dyn_smem(kern);
                const int grid = grid_for(kern, 256, smem, d->nsm);
                const void *Xp = d->X;
                int64_t ld = d->ld, p = d->p;
                int nn = (int)n, K_ = kfold, nfl = (int)nl;
                const int8_t *fd = (const int8_t *)buf;
                const int *ffd = (const int *)(buf + o_ff);
                const double *ntd = (const double *)(buf + o_nt);
                double *const *csd = (double *const *)(buf + o_p);
                void *args[] = {&Xp, &ld, &nn, &p, &fd, &K_, &ffd, &nfl, &ntd, &csd};
                CK(cudaLaunchKernel(kern, dim3(grid), dim3(256), args, smem, sst));
                live[0]->pp->launches++;
                CK(cudaStreamSynchronize(sst));            // (host vectors above; a one-time pass)
                cache::dfree(buf);
            }
        }
        prep_batch(0);
        for (auto &lf : fits) {
            if (!lf.alive || !lf.pp) continue;
            try { prep_mid(lf.pp, alpha); } catch (const Err &er) { if (d->sharded) throw; drop(lf, er); }
        }
        prep_batch(1);
        for (auto &lf : fits) {
            if (!lf.alive || !lf.pp) continue;
            try { prep_end(lf.pp); } catch (const Err &er) { if (d->sharded) throw; drop(lf, er); }
        }
        for (size_t u = 0; u < F; u++) {
            LockFit &lf = fits[u];
            if (!lf.alive || !lf.pp) continue;
            lf.pp->batch_bytes = 0.0;
            lf.run.reset(new PathRun{lf.pp, lambda, K, alpha, tol, max_iter, BL_SCREEN_HYBRID, rounds, lf.out,
                                     fit_ids[u] >= 0 ? dE : nullptr});
            lf.run->begin();
            CK(cudaEventCreateWithFlags(&lf.solved, cudaEventDisableTiming));
        }
        bl_prep *timer = nullptr;
        for (auto &lf : fits)
            if (lf.pp) { timer = lf.pp; break; }
        for (int k = 0; k < K; k++) {
            std::vector<LockFit *> pending;
            for (auto &lf : fits)
                if (lf.alive && lf.run->start(k)) pending.push_back(&lf);
            std::vector<LockFit *> active = pending;
            while (!pending.empty()) {
                for (LockFit *lf : pending) {
                    lf->run->solve();
                    CK(cudaEventRecord(lf->solved, lf->pp->stream));
                }
                {
                    for (LockFit *lf : pending) CK(cudaStreamWaitEvent(sst, lf->solved, 0));
                    // the union of the pending fits' BEDPP scopes: near lambda_max BEDPP
                    // discards most columns for every fit, and only the union is read
                    const size_t np_ = pending.size();
                    for (size_t u = 0; u < np_; u++) {
                        hptr[u] = pending[u]->pp->flags;
                        hptr[np_ + u] = pending[u]->pp->nlive;
                        hptr[2 * np_ + u] = pending[u]->pp->st;
                    }
                    CK(cudaMemcpyAsync(dptr, hptr, 3 * sizeof(void *) * np_, cudaMemcpyHostToDevice, sst));
                    CK(cudaMemsetAsync(uni, 0, 2 * sizeof(int), sst));
                    if (d->dt == DT_I8)                     // every fit's residual -> 8 digit planes (Q27)
                        for (LockFit *lf : pending) {
                            bl_prep *q = lf->pp;
                            k_limbs<<<1, 1024, 0, sst>>>(q->rscan, (int)d->n, q->limb_ld, q->limbs, q->limb_scale,
                                                         q->limb_sum);
                            CKL();
                            timer->launches++;
                        }
                    {
                        const int ug = (int)std::min<int64_t>((d->p + 255) / 256, (int64_t)d->nsm * 8);
                        k_scope_union<<<ug, 256, 0, sst>>>(d->p, (const uint8_t *const *)dptr, (int)np_, uni + 2, uni);
                        CKL();
                        k_scope_finish<<<1, 32, 0, sst>>>(d->p, uni, (const int *const *)(dptr + np_), (int)np_,
                                                          (RoundStatus *const *)(dptr + 2 * np_), uni + 1);
                        CKL();
                        timer->launches += 2;
                    }
                    timer->batch_passes = 0;
                    launch_scan_batch(d, pending, sst, dfs, hfs, timer, bk, uni + 2, uni, &tcs);
                    for (LockFit *lf : pending) copy_round(lf->pp, sst);
                    CK(cudaMemcpyAsync(hctl, uni, 2 * sizeof(int), cudaMemcpyDeviceToHost, sst));
                    CK(cudaStreamSynchronize(sst));
                    const int64_t cols = hctl[1] ? hctl[0] : d->p;
                    timer->batch_bytes += (double)timer->batch_passes * (double)d->n * itemsize(d->dt) * (double)cols;
                }
                if (d->sharded) {                           // C3 for every pending fit in one collective
                    std::vector<bl_prep *> pps;
                    for (LockFit *lf : pending) pps.push_back(lf->pp);
                    exchange_rounds(d, pps, sst);
                }
                std::vector<LockFit *> again;
                for (LockFit *lf : pending) {
                    const int res = lf->run->after_scan(batched);
                    if (res == 1) again.push_back(lf);
                    else if (res < 0) {
                        lf->run->fail();
                        lf->alive = false;
                        lf->st = lf->run->status;
                        lf->err = g_err;
                        g_err.clear();
                    }
                }
                pending.swap(again);
            }
            for (LockFit *lf : active)
                if (lf->alive) lf->run->record();
        }
        for (auto &lf : fits)
            if (lf.run) lf.run->flush();
        const double wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        paths.assign(F, nullptr);
        sts.assign(F, BL_OK);
        errs.assign(F, std::string());
        for (size_t u = 0; u < F; u++) {
            LockFit &lf = fits[u];
            if (lf.pp) finish_perf(lf.pp, lf.out, wall);
            if (batched && lf.pp) {                         // the batched passes: charged once, to the timer fit
                lf.out->perf.scan_bytes = lf.pp == timer ? lf.pp->batch_bytes : 0.0;
                if (lf.pp != timer) { lf.out->perf.scan_ms = 0.0; lf.out->perf.scan_launches = 0; }
            }
            paths[u] = lf.out;
            lf.out = nullptr;
            sts[u] = lf.st;
            errs[u] = lf.err;
        }
    } catch (...) {
        for (auto &lf : fits) delete lf.out;
        cleanup();
        throw;
    }
    cleanup();
}

bl_path *fit_impl(bl_design *d, const double *y, const uint8_t *train, const double *lambda, int K, double alpha,
                  double tol, int max_iter, int screen, const bl_opts *opts, bl_status *st_out,
                  double *heldout = nullptr, int family = 0) {
    auto t0 = std::chrono::steady_clock::now();
    validate_grid(lambda, K);
    if (!(tol > 0.0)) raise(BL_ERR_ARG, "tol must be > 0");
    if (max_iter < 1) raise(BL_ERR_ARG, "max_iter must be >= 1");
    if (screen < 0 || screen > 2) raise(BL_ERR_ARG, "screen must be 0, 1 or 2");
    bl_prep *pp = make_prep(d, y, train, alpha, opts);
    PoolGuard g{pp};
    bl_path *out = new bl_path();
    out->magic = MAGIC_PATH;
    int rounds = opts && opts->max_kkt_rounds > 0 ? opts->max_kkt_rounds : 10;
    std::string saved;
    bl_status s;
    try {
        s = run_path(pp, lambda, K, alpha, tol, max_iter, screen, rounds, out, heldout, family);
    } catch (...) {
        delete out;
        throw;
    }
    saved = g_err;
    double wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    finish_perf(pp, out, wall);
    g_err = saved;
    *st_out = s;
    return out;
}

void add_perf(bl_cvres *cv, const bl_perf &p) {
    std::lock_guard<std::mutex> lk(cv->perf_mu);
    bl_perf &q = cv->perf;
    q.scan_ms += p.scan_ms; q.scan_bytes += p.scan_bytes; q.scan_launches += p.scan_launches;
    q.cd_ms += p.cd_ms; q.cd_launches += p.cd_launches; q.prep_ms += p.prep_ms; q.prep_bytes += p.prep_bytes;
    q.kernel_launches += p.kernel_launches; q.wall_ms = std::max(q.wall_ms, p.wall_ms);
    q.cd_visits += p.cd_visits; q.cd_updates += p.cd_updates; q.cd_kernel_cycles += p.cd_kernel_cycles;
    for (int u = 0; u < 4; u++) q.cd_prof[u] += p.cd_prof[u];
    for (int u = 0; u < 8; u++) q.cd_events[u] += p.cd_events[u];
    for (int u = 0; u < 8; u++) q.cd_sub[u] += p.cd_sub[u];
}

uint64_t splitmix64(uint64_t &state) {
    uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

}  // namespace

// ================================================================== C ABI

extern "C" {

const char *bl_last_error(void) { return g_err.c_str(); }

void bl_trim(void) {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cache::trim();
    cudaGetLastError();
}

bl_status bl_nccl_unique_id(void *out128) {
    return guard([&] {
        if (!out128) raise(BL_ERR_ARG, "out is NULL");
        ncclUniqueId id;
        CKN(ncclGetUniqueId(&id));
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
        std::memcpy(out128, &id, 128);
    });
}

bl_status bl_load_design(const void *X, bl_dtype dt, int64_t n, int64_t p_local, int64_t ld, int x_is_device_ptr,
                         const bl_dist *dist, bl_design **out) {
    return guard([&] {
        if (!out) raise(BL_ERR_ARG, "out is NULL");
        *out = nullptr;
        if (!X) raise(BL_ERR_ARG, "X is NULL");
        if (dt < BL_F64 || dt > BL_I8) raise(BL_ERR_ARG, "bad dtype %d", (int)dt);
        if (n < 2) raise(BL_ERR_ARG, "n must be >= 2 (got %lld)", (long long)n);
        if (n > (int64_t)kCdRmax * 1024) raise(BL_ERR_ARG, "n = %lld exceeds 16384 (r must fit one SM)", (long long)n);
        if (p_local < 1) raise(BL_ERR_ARG, "p must be >= 1");
        if (ld < n) raise(BL_ERR_ARG, "ld < n");
        if (p_local > INT32_MAX) raise(BL_ERR_ARG, "p_local too large");
        if (x_is_device_ptr < 0 || x_is_device_ptr > 2) raise(BL_ERR_ARG, "x_is_device_ptr must be 0, 1 or 2");
        check_device();
        bl_design *d = new bl_design();
        d->magic = MAGIC_DESIGN;
        d->dt = (int)dt;
        d->n = n;
        d->p = p_local;
        d->rank = 0;
        d->world = 1;
        d->comm = nullptr;
        d->sharded = false;
        d->col_offset = 0;
        d->p_global = p_local;
        CK(cudaGetDevice(&d->device));
        if (dist) {
            if (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world) { delete d; raise(BL_ERR_ARG, "bad bl_dist"); }
            d->rank = dist->rank;
            d->world = dist->world;
            d->col_offset = dist->col_offset;
            d->p_global = dist->p_global;
            if (dist->device >= 0) d->device = dist->device;
            CK(cudaSetDevice(d->device));
        }
        CK(cudaDeviceGetAttribute(&d->nsm, cudaDevAttrMultiProcessorCount, d->device));
        int isz = itemsize(dt);
        if (x_is_device_ptr == 2) {
            // NEXT-4: out-of-core.  X stays in host memory (borrowed), page-locked and mapped
            // into the device address space; every full pass over X (stats, scans) streams it
            // over PCIe, the working-set columns are copied once into a device store.
            if (((uintptr_t)X % 16) != 0 || (ld * isz) % 16 != 0) {
                delete d;
                raise(BL_ERR_ARG, "host-resident X needs a 16-byte aligned base and ld*itemsize %% 16 == 0");
            }
            const size_t bytes = (size_t)ld * p_local * isz;
            cudaPointerAttributes pa{};
            const bool pinned = cudaPointerGetAttributes(&pa, X) == cudaSuccess && pa.type == cudaMemoryTypeHost;
            cudaGetLastError();
            cudaError_t e = pinned ? cudaSuccess
                                   : cudaHostRegister(const_cast<void *>(X), bytes, cudaHostRegisterMapped | cudaHostRegisterReadOnly);
            if (pinned || e == cudaErrorHostMemoryAlreadyRegistered) {
                cudaGetLastError();              // the caller pinned it: map without taking ownership
            } else if (e != cudaSuccess) {
                cudaGetLastError();
                delete d;
                raise(BL_ERR_OOM, "cudaHostRegister(%zu bytes): %s", bytes, cudaGetErrorString(e));
            } else {
                d->host_reg = const_cast<void *>(X);
            }
            void *dp = nullptr;
            e = cudaHostGetDevicePointer(&dp, const_cast<void *>(X), 0);
            if (e != cudaSuccess) {
                cudaGetLastError();
                if (d->host_reg) cudaHostUnregister(d->host_reg);
                delete d;
                raise(BL_ERR_CUDA, "cudaHostGetDevicePointer: %s", cudaGetErrorString(e));
            }
            d->X = dp;
            d->owned = false;
            d->ld = ld;
            d->hostres = true;
        } else if (x_is_device_ptr == 1) {
            if (((uintptr_t)X % 16) != 0 || (ld * isz) % 16 != 0) {
                delete d;
                raise(BL_ERR_ARG, "device X needs a 16-byte aligned base and ld*itemsize %% 16 == 0");
            }
            d->X = const_cast<void *>(X);
            d->owned = false;
            d->ld = ld;
        } else {
            int64_t ldp = round_up(n, 16 / isz);
            size_t bytes = (size_t)ldp * p_local * isz;
            cudaError_t e = cache::dmalloc((void **)&d->X, bytes);
            if (e != cudaSuccess) { delete d; raise(BL_ERR_OOM, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e)); }
            d->owned = true;
            d->ld = ldp;
            if (ld == ldp) CK(cudaMemcpy(d->X, X, (size_t)ld * p_local * isz, cudaMemcpyHostToDevice));
            else CK(cudaMemcpy2D(d->X, ldp * isz, X, ld * isz, n * isz, p_local, cudaMemcpyHostToDevice));
            if (ldp > n)                               // padding rows are zero (whatever the caller's held)
                CK(cudaMemset2D((char *)d->X + n * isz, ldp * isz, 0, (ldp - n) * isz, p_local));
        }
        d->sharded = false;
        d->wstore = d->hostres;
        d->shard_off.assign(2, 0);
        d->shard_off[1] = p_local;
        if (d->world > 1) {
            try {
                if (!dist->nccl_unique_id && dist->backend != 2)
                    raise(BL_ERR_ARG, "nccl_unique_id (or loopback group key) required for world > 1");
                if (dist->backend == 1) {
                    auto *lc = new LoopComm();
                    d->comm = lc;
                    lc->rank = d->rank;
                    lc->world = d->world;
                    lc->key.assign((const char *)dist->nccl_unique_id, 128);
                    std::lock_guard<std::mutex> lk(g_loop_mu);
                    auto &g = g_loop_groups[lc->key];
                    if (!g) {
                        g = std::make_shared<LoopGroup>();
                        g->world = d->world;
                        g->stage.resize(d->world);
                    }
                    if (g->world != d->world) raise(BL_ERR_ARG, "loopback group world mismatch");
                    g->members++;
                    lc->g = g;
                } else if (dist->backend == 0) {
                    auto *nc = new NcclComm();
                    d->comm = nc;
                    nc->rank = d->rank;
                    nc->world = d->world;
                    ncclUniqueId id;
                    std::memcpy(&id, dist->nccl_unique_id, sizeof id);
                    nc->timeout_ms = dist->timeout_ms > 0 ? dist->timeout_ms : 600000;
                    CKN(ncclCommInitRank(&nc->c, d->world, id, d->rank));
                } else if (dist->backend == 2) {
                    if (!dist->host_coll || !dist->host_coll->allgather || !dist->host_coll->bcast ||
                        !dist->host_coll->allreduce_sum_f64)
                        raise(BL_ERR_ARG, "backend 2 needs host_coll with allgather, bcast and allreduce_sum_f64");
                    auto *hc = new HostComm();
                    d->comm = hc;
                    hc->rank = d->rank;
                    hc->world = d->world;
                    hc->hc = *dist->host_coll;
                } else {
                    raise(BL_ERR_ARG, "bad bl_dist backend %d", dist->backend);
                }
                // shard table (C0): every rank's (col_offset, p_local), in rank order
                int64_t *dbuf = nullptr;
                CK(cache::dmalloc((void **)&dbuf, 16 * (size_t)(d->world + 1)));
                const int64_t mine[2] = {d->col_offset, p_local};
                CK(cudaMemcpy(dbuf, mine, 16, cudaMemcpyHostToDevice));
                std::vector<int64_t> all(2 * (size_t)d->world);
                d->comm->allgather(dbuf, dbuf + 2, 16, 0);
                d->comm->wait(0);
                CK(cudaMemcpy(all.data(), dbuf + 2, 16 * (size_t)d->world, cudaMemcpyDeviceToHost));
                cache::dfree(dbuf);
                d->shard_off.assign(d->world + 1, 0);
                for (int r = 0; r < d->world; r++) {
                    if (all[2 * r] != d->shard_off[r]) raise(BL_ERR_ARG, "shards must be contiguous in rank order (rank %d col_offset %lld)", r, (long long)all[2 * r]);
                    d->shard_off[r + 1] = d->shard_off[r] + all[2 * r + 1];
                }
                d->sharded = d->world > 1 && d->p_global != p_local;
                d->wstore = d->sharded || d->hostres;
                if (d->sharded && d->shard_off[d->world] != d->p_global) raise(BL_ERR_ARG, "shards cover %lld columns, p_global = %lld", (long long)d->shard_off[d->world], (long long)d->p_global);
                if (!d->sharded) {
                    for (int r = 0; r < d->world; r++)
                        if (all[2 * r] != 0 || all[2 * r + 1] != p_local) raise(BL_ERR_ARG, "replicated design: every rank must hold all columns");
                    d->shard_off.assign(2, 0);
                    d->shard_off[1] = p_local;
                }
            } catch (...) {
                delete d->comm;
                if (d->owned) cache::dfree(d->X);
                if (d->host_reg) cudaHostUnregister(d->host_reg);
                delete d;
                throw;
            }
        }
        *out = d;
    });
}

bl_status bl_prepare(bl_design *d, const double *y, const uint8_t *train, double alpha, bl_prep **out) {
    return guard([&] {
        if (!d || d->magic != MAGIC_DESIGN) raise(BL_ERR_ARG, "bad design handle");
        if (!out) raise(BL_ERR_ARG, "out is NULL");
        BusyGuard bg(d);
        *out = make_prep(d, y, train, alpha, nullptr);
    });
}

bl_status bl_lambda_max(bl_design *d, const double *y, double alpha, double *out) {
    return guard([&] {
        if (!d || d->magic != MAGIC_DESIGN) raise(BL_ERR_ARG, "bad design handle");
        if (!out) raise(BL_ERR_ARG, "out is NULL");
        BusyGuard bg(d);
        bl_prep *pp = make_prep(d, y, nullptr, alpha, nullptr);
        *out = pp->hps.lmax;
        free_prep(pp);
    });
}

bl_status bl_prep_copy(const bl_prep *pp, double *c, double *s, double *a, double *b, int64_t *jstar_global,
                       double *lambda_max) {
    return guard([&] {
        if (!pp || pp->magic != MAGIC_PREP) raise(BL_ERR_ARG, "bad prep handle");
        int64_t p = pp->p;
        if (c) CK(cudaMemcpy(c, pp->c, 8 * p, cudaMemcpyDeviceToHost));
        if (s) CK(cudaMemcpy(s, pp->s, 8 * p, cudaMemcpyDeviceToHost));
        if (a) CK(cudaMemcpy(a, pp->a, 8 * p, cudaMemcpyDeviceToHost));
        if (b) CK(cudaMemcpy(b, pp->b, 8 * p, cudaMemcpyDeviceToHost));
        if (jstar_global) *jstar_global = pp->hps.jstar >= 0 ? pp->hps.jstar + pp->d->col_offset : -1;
        if (lambda_max) *lambda_max = pp->hps.lmax;
    });
}

bl_status bl_bedpp(bl_prep *pp, double lambda, uint8_t *keep, int64_t *n_keep) {
    return guard([&] {
        if (!pp || pp->magic != MAGIC_PREP) raise(BL_ERR_ARG, "bad prep handle");
        if (!(lambda > 0.0)) raise(BL_ERR_ARG, "lambda must be > 0");
        bl_design *d = pp->d;
        CK(cudaSetDevice(d->device));
        cudaStream_t st = pp->stream;
        CK(cudaMemsetAsync(pp->st, 0, sizeof(RoundStatus), st));
        int grid = (int)std::min<int64_t>((d->p + 1023) / 1024, (int64_t)d->nsm * 8);
        k_bedpp<<<grid, 256, 0, st>>>(d->p, pp->s, pp->a, pp->b, pp->ps, pp->alpha, lambda, -1.0, 1, pp->flags,
                                      pp->scope, pp->st);
        CKL();
        std::vector<uint8_t> f(d->p);
        CK(cudaMemcpyAsync(f.data(), pp->flags, d->p, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(pp->hst, pp->st, sizeof(RoundStatus), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int64_t j = 0; j < d->p; j++)
            if (keep) keep[j] = f[j] & 1;
        if (n_keep) *n_keep = pp->hst->nsafe;
    });
}

bl_status bl_scan(bl_prep *pp, const double *r, double lam, double lam_next, const uint8_t *in_w, double *z,
                  int32_t *viol, int64_t *n_viol, int32_t *strong, int64_t *n_strong) {
    return guard([&] {
        if (!pp || pp->magic != MAGIC_PREP) raise(BL_ERR_ARG, "bad prep handle");
        if (!r) raise(BL_ERR_ARG, "r is NULL");
        bl_design *d = pp->d;
        CK(cudaSetDevice(d->device));
        cudaStream_t st = pp->stream;
        std::vector<double> rv(pp->vlen, 0.0);
        std::memcpy(rv.data(), r, 8 * d->n);
        CK(cudaMemcpyAsync(pp->rscan, rv.data(), 8 * pp->vlen, cudaMemcpyHostToDevice, st));
        std::vector<uint8_t> w(d->p, 0);
        if (in_w) std::memcpy(w.data(), in_w, d->p);
        CK(cudaMemcpyAsync(pp->wflag, w.data(), d->p, cudaMemcpyHostToDevice, st));
        CK(cudaMemsetAsync(pp->st, 0, sizeof(RoundStatus), st));
        int grid = (int)std::min<int64_t>((d->p + 1023) / 1024, (int64_t)d->nsm * 8);
        k_bedpp<<<grid, 256, 0, st>>>(d->p, pp->s, pp->a, pp->b, pp->ps, pp->alpha, lam, lam_next > 0 ? lam_next : -1.0,
                                      0, pp->flags, nullptr, pp->st);
        CKL();
        k_vsum<<<1, 1024, 0, st>>>(pp->rscan, (int)d->n, pp->limb_scale + 2);
        CKL();
        ScanArgs sa{};
        sa.K1 = pp->limb_scale + 2;    // sum_i r_i (identity (3))
        sa.K2v = 1.0 / pp->nt;
        sa.out = pp->z;
        sa.jfix = nullptr;
        sa.scan = 1;
        sa.flags = pp->flags;
        sa.wflag = pp->wflag;
        sa.thr_viol = pp->alpha * lam;
        sa.thr_strong = lam_next > 0.0 ? std::max(0.0, pp->alpha * (2.0 * lam_next - lam)) : -1.0;
        sa.viol = pp->viol;
        sa.nviol = &pp->st->nviol;
        sa.strong = pp->strong;
        sa.nstrong = &pp->st->nstrong;
        launch_scan(pp, sa, pp->rscan, false);
        CK(cudaMemcpyAsync(pp->hst, pp->st, sizeof(RoundStatus), cudaMemcpyDeviceToHost, st));
        if (z) CK(cudaMemcpyAsync(z, pp->z, 8 * d->p, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        std::vector<int> v = read_list(pp, pp->viol, pp->hst->nviol);
        std::vector<int> sv = read_list(pp, pp->strong, pp->hst->nstrong);
        if (viol) std::copy(v.begin(), v.end(), viol);
        if (strong) std::copy(sv.begin(), sv.end(), strong);
        if (n_viol) *n_viol = (int64_t)v.size();
        if (n_strong) *n_strong = (int64_t)sv.size();
    });
}

bl_status bl_scan_batch(bl_prep *const *pps, int nf, const double *const *r, double lam, double lam_next, int cv_mode,
                        double *z, int64_t *n_viol, int64_t *n_strong) {
    return guard([&] {
        if (!pps || nf < 1) raise(BL_ERR_ARG, "need nf >= 1 preps");
        if (!r) raise(BL_ERR_ARG, "r is NULL");
        if (cv_mode != 0 && cv_mode != 1 && cv_mode != 3) raise(BL_ERR_ARG, "cv_mode must be 0, 1 or 3 (got %d)", cv_mode);
        bl_design *d = nullptr;
        for (int u = 0; u < nf; u++) {
            if (!pps[u] || pps[u]->magic != MAGIC_PREP) raise(BL_ERR_ARG, "bad prep handle %d", u);
            if (!r[u]) raise(BL_ERR_ARG, "r[%d] is NULL", u);
            if (u == 0) d = pps[0]->d;
            else if (pps[u]->d != d) raise(BL_ERR_ARG, "preps of different designs");
            for (int v = 0; v < u; v++)
                if (pps[v] == pps[u]) raise(BL_ERR_ARG, "prep %d repeated", u);
        }
        CK(cudaSetDevice(d->device));
        cudaStream_t st = pps[0]->stream;
        std::vector<FitScan> hfs(nf);
        for (int u = 0; u < nf; u++) {                 // each fit's round inputs, as bl_scan sets them up
            bl_prep *pp = pps[u];
            if (pp->stream != st) {                    // (preps made by bl_prepare have their own streams)
                cudaEvent_t ev;
                CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                CK(cudaEventRecord(ev, pp->stream));
                CK(cudaStreamWaitEvent(st, ev, 0));
                CK(cudaEventDestroy(ev));
            }
            std::vector<double> rv(pp->vlen, 0.0);
            std::memcpy(rv.data(), r[u], 8 * d->n);
            CK(cudaMemcpyAsync(pp->rscan, rv.data(), 8 * pp->vlen, cudaMemcpyHostToDevice, st));
            CK(cudaMemsetAsync(pp->wflag, 0, d->p, st));
            CK(cudaMemsetAsync(pp->st, 0, sizeof(RoundStatus), st));
            const int grid = (int)std::min<int64_t>((d->p + 1023) / 1024, (int64_t)d->nsm * 8);
            k_bedpp<<<grid, 256, 0, st>>>(d->p, pp->s, pp->a, pp->b, pp->ps, pp->alpha, lam,
                                          lam_next > 0 ? lam_next : -1.0, 0, pp->flags, nullptr, pp->st);
            CKL();
            k_vsum<<<1, 1024, 0, st>>>(pp->rscan, (int)d->n, pp->limb_scale + 2);
            CKL();
            if (d->dt == DT_I8) {
                k_limbs<<<1, 1024, 0, st>>>(pp->rscan, (int)d->n, pp->limb_ld, pp->limbs, pp->limb_scale, pp->limb_sum);
                CKL();
            }
            ScanArgs sa{};
            sa.K1 = pp->limb_scale + 2;
            sa.K2v = 1.0 / pp->nt;
            sa.out = pp->z;
            sa.flags = pp->flags;
            sa.wflag = pp->wflag;
            sa.thr_viol = pp->alpha * lam;
            sa.thr_strong = lam_next > 0.0 ? std::max(0.0, pp->alpha * (2.0 * lam_next - lam)) : -1.0;
            sa.viol = pp->viol;
            sa.nviol = &pp->st->nviol;
            sa.strong = pp->strong;
            sa.nstrong = &pp->st->nstrong;
            hfs[u] = fitscan_of(d, pp, sa);
        }
        FitScan *dfs = nullptr;
        CK(cache::dmalloc((void **)&dfs, sizeof(FitScan) * nf));
        TcScratch tcs;
        try {
            launch_scan_batch_fs(d, (size_t)nf, pps[0]->limb_ld, st, dfs, hfs.data(), pps[0], cv_mode, nullptr, nullptr,
                                 &tcs);
            for (int u = 0; u < nf; u++) {
                if (z) CK(cudaMemcpyAsync(z + (size_t)u * d->p, pps[u]->z, 8 * d->p, cudaMemcpyDeviceToHost, st));
                CK(cudaMemcpyAsync(pps[u]->hst, pps[u]->st, sizeof(RoundStatus), cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                if (n_viol) n_viol[u] = pps[u]->hst->nviol;
                if (n_strong) n_strong[u] = pps[u]->hst->nstrong;
            }
        } catch (...) {
            cudaStreamSynchronize(st);
            cache::dfree(dfs);
            throw;
        }
        CK(cudaStreamSynchronize(st));
        cache::dfree(dfs);
    });
}

bl_status bl_fit_path(bl_design *d, const double *y, const double *lambda, int n_lambda, double alpha, double tol,
                      int max_iter, int screen, const bl_opts *opts, bl_path **out) {
    bl_status s = BL_OK;
    bl_status g = guard([&] {
        if (!d || d->magic != MAGIC_DESIGN) raise(BL_ERR_ARG, "bad design handle");
        if (!out) raise(BL_ERR_ARG, "out is NULL");
        *out = nullptr;
        BusyGuard bg(d);
        *out = fit_impl(d, y, nullptr, lambda, n_lambda, alpha, tol, max_iter, screen, opts, &s);
    });
    return g != BL_OK ? g : s;
}

bl_status bl_fit_path_binomial(bl_design *d, const double *y, const double *lambda, int n_lambda, double alpha,
                               double tol, int max_iter, int screen, const bl_opts *opts, bl_path **out) {
    bl_status s = BL_OK;
    bl_status g = guard([&] {
        if (!d || d->magic != MAGIC_DESIGN) raise(BL_ERR_ARG, "bad design handle");
        if (!out) raise(BL_ERR_ARG, "out is NULL");
        if (!y) raise(BL_ERR_ARG, "y is NULL");
        *out = nullptr;
        int64_t n1 = 0;
        for (int64_t i = 0; i < d->n; i++) {
            if (!(y[i] == 0.0 || y[i] == 1.0)) raise(BL_ERR_ARG, "binomial y[%lld] = %g is not 0 or 1", (long long)i, y[i]);
            n1 += y[i] == 1.0;
        }
        if (n1 == 0 || n1 == d->n) raise(BL_ERR_DEGENERATE, "binomial y has a single class (S:311)");
        BusyGuard bg(d);
        *out = fit_impl(d, y, nullptr, lambda, n_lambda, alpha, tol, max_iter, screen, opts, &s, nullptr, 1);
    });
    return g != BL_OK ? g : s;
}

bl_status bl_cv(bl_design *d, const double *y, const double *lambda, int n_lambda, double alpha, double tol,
                int max_iter, int n_folds, const int32_t *fold_id, uint64_t seed, const bl_opts *opts,
                bl_cvres **out) {
    bl_status s = BL_OK;
    bl_status g = guard([&] {
        if (!d || d->magic != MAGIC_DESIGN) raise(BL_ERR_ARG, "bad design handle");
        if (!out) raise(BL_ERR_ARG, "out is NULL");
        *out = nullptr;
        const int64_t n = d->n;
        if (n_folds < 2 || n_folds > n) raise(BL_ERR_ARG, "need 2 <= K <= n (K = %d, n = %lld)", n_folds, (long long)n);
        validate_grid(lambda, n_lambda);
        if (!(tol > 0.0)) raise(BL_ERR_ARG, "tol must be > 0");
        if (max_iter < 1) raise(BL_ERR_ARG, "max_iter must be >= 1");
        const int cv_mode = opts ? opts->cv_mode : 0;
        if (cv_mode < 0 || cv_mode > 3) raise(BL_ERR_ARG, "cv_mode must be 0, 1, 2 or 3 (got %d)", cv_mode);
        BusyGuard bg(d);
        std::vector<int32_t> f(n);
        if (fold_id) {
            for (int64_t i = 0; i < n; i++) {
                if (fold_id[i] < 0 || fold_id[i] >= n_folds) raise(BL_ERR_ARG, "fold_id[%lld] out of range", (long long)i);
                f[i] = fold_id[i];
            }
        } else {   // Q18
            std::vector<int64_t> perm(n);
            for (int64_t i = 0; i < n; i++) perm[i] = i;
            uint64_t stt = seed;
            for (int64_t i = n - 1; i >= 1; i--) {
                int64_t jj = (int64_t)(splitmix64(stt) % (uint64_t)(i + 1));
                std::swap(perm[i], perm[jj]);
            }
            for (int64_t i = 0; i < n; i++) f[perm[i]] = (int32_t)(i % n_folds);
        }
        std::vector<int64_t> cnt(n_folds, 0);
        for (int64_t i = 0; i < n; i++) cnt[f[i]]++;
        for (int k = 0; k < n_folds; k++)
            if (cnt[k] == 0) raise(BL_ERR_ARG, "fold %d is empty", k);
        struct CvOwner {                                // the result is the caller's only on success
            bl_cvres *p;
            ~CvOwner() {
                if (!p) return;
                if (p->full) { p->full->magic = MAGIC_DEAD; delete p->full; }
                delete p;
            }
        } cvo{new bl_cvres()};
        bl_cvres *cv = cvo.p;
        cv->magic = MAGIC_CV;
        cv->n_lambda = n_lambda;
        cv->K = n_folds;
        cv->n = n;
        cv->fold_id = f;
        cv->E.assign((size_t)n_lambda * n, 0.0);
        cv->full = nullptr;
        std::memset(&cv->perf, 0, sizeof cv->perf);
        CK(cudaSetDevice(d->device));
        // device E (n_lambda x n): fold fits write disjoint held-out rows, so they run concurrently
        double *dE = nullptr, *dcv = nullptr;
        cudaError_t e = cache::dmalloc((void **)&dE, 8 * (size_t)n_lambda * n + 16 * (size_t)n_lambda);
        if (e != cudaSuccess) { cudaGetLastError(); raise(BL_ERR_OOM, "cudaMalloc for CV errors: %s", cudaGetErrorString(e)); }
        dcv = dE + (size_t)n_lambda * n;
        struct Free { double *p; ~Free() { if (p) cache::dfree(p); } } fr{dE};
        CK(cudaMemset(dE, 0, 8 * (size_t)n_lambda * n));
        // fold-parallel.  With world > 1 ranks and a replicated design, fold f
        // runs on rank f mod world and E is summed; a sharded design runs every fit on every
        // rank (each fit's collectives span the shards).
        std::vector<int> mine;
        for (int fo = 0; fo < n_folds; fo++)
            if (d->sharded || fo % d->world == d->rank) mine.push_back(fo);
        std::vector<bl_status> fst(mine.size() + 1, BL_OK);
        std::vector<std::string> ferr(mine.size() + 1);
        std::vector<bl_path *> full(1, nullptr);
        bl_opts fo_opts{};
        if (opts) fo_opts = *opts;
        fo_opts.stream = nullptr;                       // each fold on its own library stream
        if (fo_opts.cd_cluster == 0) fo_opts.cd_cluster = 8;   // K + 1 concurrent CD clusters share the SMs
        auto run_fold = [&](size_t idx) {
            try {
                CK(cudaSetDevice(d->device));
                if (idx < mine.size()) {
                    std::vector<uint8_t> train(n);
                    for (int64_t i = 0; i < n; i++) train[i] = f[i] != mine[idx];
                    bl_status fs = BL_OK;
                    bl_path *pth = fit_impl(d, y, train.data(), lambda, n_lambda, alpha, tol, max_iter,
                                            BL_SCREEN_HYBRID, &fo_opts, &fs, dE);
                    add_perf(cv, pth->perf);
                    delete pth;
                    fst[idx] = fs;
                    if (fs != BL_OK) ferr[idx] = g_err;
                } else {
                    bl_status fs = BL_OK;
                    full[0] = fit_impl(d, y, nullptr, lambda, n_lambda, alpha, tol, max_iter, BL_SCREEN_HYBRID,
                                       &fo_opts, &fs);
                    add_perf(cv, full[0]->perf);
                    fst[idx] = fs;
                    if (fs != BL_OK) ferr[idx] = g_err;
                }
            } catch (const Err &er) {
                fst[idx] = er.code;
                ferr[idx] = g_err;
            } catch (const std::bad_alloc &) {
                fst[idx] = BL_ERR_OOM;
                ferr[idx] = "host allocation failed";
            }
        };
        if (cv_mode != 2) {                             // NEXT-1: one pass over X per round for all fits
            std::vector<int> ids(mine.begin(), mine.end());
            ids.push_back(-1);
            std::vector<bl_path *> paths;
            std::vector<bl_status> sts;
            std::vector<std::string> errs;
            cv_lockstep(d, y, f, ids, lambda, n_lambda, alpha, tol, max_iter, opts, dE, paths, sts, errs);
            for (size_t u = 0; u < ids.size(); u++) {
                add_perf(cv, paths[u]->perf);
                fst[u] = sts[u];
                ferr[u] = errs[u];
                if (ids[u] >= 0) delete paths[u];
                else full[0] = paths[u];
            }
        } else if (d->sharded) {                        // collectives must be issued in the same order
            for (size_t idx = 0; idx <= mine.size(); idx++) run_fold(idx);
        } else {                                        // independent fits, one host thread + stream each
            std::vector<std::thread> th;
            for (size_t idx = 0; idx <= mine.size(); idx++) th.emplace_back(run_fold, idx);
            for (auto &t : th) t.join();
        }
        cv->full = full[0];
        for (size_t idx = 0; idx < fst.size(); idx++)
            if (fst[idx] != BL_OK && s == BL_OK) { s = fst[idx]; g_err = ferr[idx]; }
        CK(cudaDeviceSynchronize());
        if (d->world > 1 && !d->sharded) {            // replicated: each rank ran its own folds
            std::lock_guard<std::mutex> lk(d->comm_mu);
            d->comm->allreduce_sum(dE, (size_t)n_lambda * n, 0);
            d->comm->wait(0);
        }
        k_cv_reduce<<<n_lambda, 256>>>(dE, (int)n, dcv, dcv + n_lambda);
        CKL();
        cv->cve.assign(n_lambda, 0.0);
        cv->cvse.assign(n_lambda, 0.0);
        CK(cudaMemcpy(cv->E.data(), dE, 8 * (size_t)n_lambda * n, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(cv->cve.data(), dcv, 8 * (size_t)n_lambda, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(cv->cvse.data(), dcv + n_lambda, 8 * (size_t)n_lambda, cudaMemcpyDeviceToHost));
        int best = 0;                                   // lambda_min: lowest index on ties
        for (int k = 1; k < n_lambda; k++)
            if (cv->cve[k] < cv->cve[best]) best = k;
        cv->lmin = best;
        *out = cv;
        cvo.p = nullptr;
    });
    return g != BL_OK ? g : s;
}

bl_status bl_path_info(const bl_path *p, int *n_lambda, int64_t *nnz_total, int *n_converged) {
    return guard([&] {
        if (!p || p->magic != MAGIC_PATH) raise(BL_ERR_ARG, "bad path handle");
        if (n_lambda) *n_lambda = p->n_lambda;
        if (nnz_total) *nnz_total = (int64_t)p->feat.size();
        if (n_converged) *n_converged = p->n_converged;
    });
}

bl_status bl_path_copy(const bl_path *p, double *lambda, double *a0, double *objective, int64_t *col_ptr,
                       int64_t *feat_idx, double *beta_std, double *beta_orig, int32_t *passes, int32_t *kkt_rounds,
                       int64_t *cols_scanned) {
    return guard([&] {
        if (!p || p->magic != MAGIC_PATH) raise(BL_ERR_ARG, "bad path handle");
        int K = p->n_lambda;
        if (lambda) std::copy(p->lambda.begin(), p->lambda.end(), lambda);
        if (a0) std::copy(p->a0.begin(), p->a0.end(), a0);
        if (objective) std::copy(p->obj.begin(), p->obj.end(), objective);
        if (col_ptr) std::copy(p->col_ptr.begin(), p->col_ptr.begin() + K + 1, col_ptr);
        if (feat_idx) std::copy(p->feat.begin(), p->feat.end(), feat_idx);
        if (beta_std) std::copy(p->beta_std.begin(), p->beta_std.end(), beta_std);
        if (beta_orig) std::copy(p->beta_orig.begin(), p->beta_orig.end(), beta_orig);
        if (passes) std::copy(p->passes.begin(), p->passes.end(), passes);
        if (kkt_rounds) std::copy(p->kkt_rounds.begin(), p->kkt_rounds.end(), kkt_rounds);
        if (cols_scanned) std::copy(p->cols_scanned.begin(), p->cols_scanned.end(), cols_scanned);
    });
}

bl_status bl_path_screen(const bl_path *p, int64_t *n_safe, int64_t *n_strong, int64_t *n_working) {
    return guard([&] {
        if (!p || p->magic != MAGIC_PATH) raise(BL_ERR_ARG, "bad path handle");
        const size_t K = (size_t)p->n_lambda;
        if (n_safe) std::copy(p->n_safe.begin(), p->n_safe.begin() + std::min(K, p->n_safe.size()), n_safe);
        if (n_strong) std::copy(p->n_strong.begin(), p->n_strong.begin() + std::min(K, p->n_strong.size()), n_strong);
        if (n_working) std::copy(p->n_working.begin(), p->n_working.begin() + std::min(K, p->n_working.size()), n_working);
    });
}

bl_status bl_path_irls(const bl_path *p, int32_t *outer) {
    return guard([&] {
        if (!p || p->magic != MAGIC_PATH) raise(BL_ERR_ARG, "bad path handle");
        if (p->family != 1) raise(BL_ERR_ARG, "not a logistic path");
        if (outer) std::copy(p->outer.begin(), p->outer.end(), outer);
    });
}

bl_status bl_path_perf(const bl_path *p, bl_perf *out) {
    return guard([&] {
        if (!p || p->magic != MAGIC_PATH) raise(BL_ERR_ARG, "bad path handle");
        if (!out) raise(BL_ERR_ARG, "out is NULL");
        *out = p->perf;
    });
}

bl_status bl_cv_copy(const bl_cvres *cv, double *cve, double *cvse, int *lambda_min_index, int32_t *fold_id_out,
                     const bl_path **full_fit) {
    return guard([&] {
        if (!cv || cv->magic != MAGIC_CV) raise(BL_ERR_ARG, "bad cv handle");
        if (cve) std::copy(cv->cve.begin(), cv->cve.end(), cve);
        if (cvse) std::copy(cv->cvse.begin(), cv->cvse.end(), cvse);
        if (lambda_min_index) *lambda_min_index = cv->lmin;
        if (fold_id_out) std::copy(cv->fold_id.begin(), cv->fold_id.end(), fold_id_out);
        if (full_fit) *full_fit = cv->full;
    });
}

bl_status bl_cv_perf(const bl_cvres *cv, bl_perf *out) {
    return guard([&] {
        if (!cv || cv->magic != MAGIC_CV) raise(BL_ERR_ARG, "bad cv handle");
        if (!out) raise(BL_ERR_ARG, "out is NULL");
        *out = cv->perf;
    });
}

bl_status bl_cv_errors(const bl_cvres *cv, double *E) {
    return guard([&] {
        if (!cv || cv->magic != MAGIC_CV) raise(BL_ERR_ARG, "bad cv handle");
        if (E) std::copy(cv->E.begin(), cv->E.end(), E);
    });
}

void bl_free(void *handle) {
    if (!handle) return;
    uint32_t magic = *(uint32_t *)handle;
    if (magic == MAGIC_DESIGN) {
        bl_design *d = (bl_design *)handle;
        for (bl_prep *pp : d->pool) free_prep(pp);
        d->pool.clear();
        delete d->comm;
        if (d->owned && d->X) cache::dfree(d->X);
        if (d->xsc) cache::dfree(d->xsc);
        if (d->host_reg) cudaHostUnregister(d->host_reg);
        d->magic = MAGIC_DEAD;
        delete d;
    } else if (magic == MAGIC_PATH) {
        bl_path *p = (bl_path *)handle;
        p->magic = MAGIC_DEAD;
        delete p;
    } else if (magic == MAGIC_CV) {
        bl_cvres *c = (bl_cvres *)handle;
        if (c->full) { c->full->magic = MAGIC_DEAD; delete c->full; }
        c->magic = MAGIC_DEAD;
        delete c;
    } else if (magic == MAGIC_PREP) {
        free_prep((bl_prep *)handle);
    }
}

}  // extern "C"
