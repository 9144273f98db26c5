// engine.cu -- device contexts, receiver tiling, the beam-group pipeline and the
// extern "C" ABI.
//
// The ABI (include/bf_gbs.h) is the drop-in boundary for the reference's
// kernels.gbs_accumulate (kernels.py:352-399) and its neighbours; this file
// owns everything between that boundary and the kernels: argument checks that
// mirror the reference's contracts, per-device streams and grow-only
// workspaces, the Hilbert receiver tiling used by the fp32 kernel, and the
// pipeline that sums a call's beams in GROUPS of whole beam ranges:
//
//   per group (a slot of device buffers, its own stream):  compact rows (packed on the
//   device from the padded bundle, or packed on host threads into pinned staging and
//   copied) -> tile work list -> scan -> unit queue order ->
//   compaction -> summation kernels;  then, on the call's stream, in group order:
//   fold of the group's range partials into acc.
//
// The range size depends only on the call's beam count and frequency count, groups are
// whole ranges and the folds add the ranges in ascending order, so the result bits do
// not depend on the grouping (memory budget), on host vs device inputs, or on the number
// of ranks.  Nothing in a call waits on the host: work-list buffers are sized from an
// upper bound, the wide-patch kernel is always launched, and statistics are copied back
// asynchronously and only waited for when bf_last_stats asks.
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <atomic>
#include <functional>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"
#include "hostpool.h"

namespace bf {

namespace {
thread_local char g_err[512] = "";
std::atomic<uint64_t> g_launches{0};
}  // namespace

int fail(int status, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return status;
}

void note_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

int check_cuda(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return BF_OK;
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return fail(BF_ENOMEM, "%s: %s", what, cudaGetErrorString(e));
    }
    return fail(BF_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

namespace {

// Bumped whenever a workspace (device or pinned) is reallocated or the statistics events
// are recreated: a captured call graph (GraphCache) is only replayed while it is unchanged.
std::atomic<uint64_t> g_pool_gen{0};

// Grow-only device buffer.
struct Buf {
    void *p = nullptr;
    size_t cap = 0;
    int get(size_t bytes, void **out) {
        if (bytes > cap) {
            g_pool_gen.fetch_add(1);
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            size_t want = bytes + bytes / 4 + 256;
            BF_TRY_CUDA(cudaMalloc(&p, want));
            cap = want;
        }
        *out = p;
        return BF_OK;
    }
};

// Grow-only pinned host buffer.
struct PinBuf {
    void *p = nullptr;
    size_t cap = 0;
    int get(size_t bytes, void **out) {
        if (bytes > cap) {
            g_pool_gen.fetch_add(1);
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            size_t want = bytes + bytes / 4 + 256;
            BF_TRY_CUDA(cudaHostAlloc(&p, want, cudaHostAllocPortable));
            cap = want;
        }
        *out = p;
        return BF_OK;
    }
};

// Call-level device workspaces.
enum BufId {
    B_ORIGIN, B_DIR, B_E1, B_E2, B_LEN, B_S0, B_REFL, B_NSEGS, B_W, B_OBS, B_ACC, B_EVALS,
    B_KEYS, B_KEYS2, B_VALS, B_VALS2, B_CUB, B_RLOC, B_CENTRE, B_BBOX, B_TBOX, B_STATS, B_CAND,
    B_QOBS, B_QBEAM, B_QOUT, B_PRL, B_POS64, B_PCEN, B_PBOX, B_CBOX, B_WLBITS, B_WLTIGHT, B_COUNT
};

// Per-slot device workspaces of one beam group.
enum SlotBufId {
    S_START, S_P0, S_P1, S_AMP, S_WLBITS, S_WLTIGHT, S_WLCNT, S_WLOFF, S_WLITEMS,
    S_UKEYS, S_UKEYS2, S_UVALS, S_UVALS2, S_PART, S_PARTEV, S_UCTR, S_CUB, S_F64, S_COUNT
};
// Per-slot pinned staging (host-buffer ABI).
enum SlotPinId { P_START, P_P0, P_P1, P_AMP, P_F64, P_COUNT };
// Call-level pinned staging (host-buffer ABI).
enum CallPinId { H_OBS, H_ACC, H_EV, H_COUNT };

constexpr int NSLOT = 3;  // beam groups in flight

struct Slot {
    cudaStream_t ss = nullptr, sw = nullptr;  // the group's stream, its wide-kernel stream
    cudaEvent_t fork = nullptr, join = nullptr, kdone = nullptr, freed = nullptr,
                h2d = nullptr, qfork = nullptr, qjoin = nullptr;
    bool freed_valid = false, h2d_valid = false;
    Buf buf[S_COUNT];
    PinBuf pin[P_COUNT];
    template <typename T>
    int get(SlotBufId id, size_t n, T **out) {
        void *p;
        BF_TRY(buf[id].get(n * sizeof(T) + 16, &p));
        *out = (T *)p;
        return BF_OK;
    }
    template <typename T>
    int pinned(SlotPinId id, size_t n, T **out) {
        void *p;
        BF_TRY(pin[id].get(n * sizeof(T) + 16, &p));
        *out = (T *)p;
        return BF_OK;
    }
};

struct DeviceCtx {
    int dev = -1;
    int sms = 0;
    size_t total_mem = 0;
    cudaStream_t stream = nullptr;
    // Completion of the last call that used this context's workspaces.  Calls may come
    // on different caller streams and return before their kernels finish; each call
    // orders itself after the previous one (StreamOrder) so no workspace is reused early.
    cudaEvent_t done = nullptr;
    bool done_valid = false;
    cudaEvent_t pro = nullptr;  // end of a call's prologue (tiling) on its stream
    cudaEvent_t entry = nullptr;  // start of an fp32 call on its stream (beam-side work)
    cudaEvent_t zdone = nullptr;  // an fp32 call's counters zeroed (beside the tiling)
    cudaEvent_t fin = nullptr, fout = nullptr;  // CallStream fences (legacy stream handles)
    // statistics read-back (stats_copy) on a side stream, off the caller's critical path;
    // the next call waits for it (StreamOrder) before zeroing the counters again
    cudaStream_t side = nullptr;
    cudaEvent_t kend = nullptr, sdone = nullptr;
    bool sdone_valid = false;
    cudaEvent_t piece[2] = {};  // staged copy-out pieces landed (d2h_out)
    int64_t budget = 0;         // group-workspace budget in bytes (0: automatic)
    // Small fp32 device calls repeated with identical arguments replay a captured graph
    // of the whole call (tiling .. fold): one launch instead of ~30.  The first call with
    // a key runs eagerly, the second is captured, later ones replay while no workspace has
    // been reallocated since (g_pool_gen).
    struct GraphCache {
        std::vector<double> key;
        bool seen = false;
        cudaGraphExec_t exec = nullptr;
        uint64_t gen = 0;
        int sb = -1;        // statistics buffer the graph writes
        int launches = 0;   // library kernels in the graph
        const void *d_stats = nullptr, *d_cand = nullptr;  // its counters (stats_copy)
        int64_t n_tiles = 0;
    } gc;
    std::mutex mu;
    Buf buf[B_COUNT];
    PinBuf hpin[H_COUNT];
    Slot slot[NSLOT];
    template <typename T>
    int get(BufId id, size_t n, T **out) {
        void *p;
        BF_TRY(buf[id].get(n * sizeof(T) + 16, &p));
        *out = (T *)p;
        return BF_OK;
    }
    template <typename T>
    int pinned(CallPinId id, size_t n, T **out) {
        void *p;
        BF_TRY(hpin[id].get(n * sizeof(T) + 16, &p));
        *out = (T *)p;
        return BF_OK;
    }
};

// Held (with ctx->mu) for the duration of an ABI call that uses the context's workspaces:
// the call's stream waits for the previous such call, and records completion on exit.
struct StreamOrder {
    DeviceCtx *c;
    cudaStream_t st;
    StreamOrder(DeviceCtx *c_, cudaStream_t st_) : c(c_), st(st_) {
        if (c->done_valid) cudaStreamWaitEvent(st, c->done, 0);
        if (c->sdone_valid) cudaStreamWaitEvent(st, c->sdone, 0);
    }
    ~StreamOrder() {
        if (cudaEventRecord(c->done, st) == cudaSuccess) c->done_valid = true;
    }
};

// The stream a summation call's work goes on.  NULL: the context's stream, and the call
// returns after the work.  cudaStreamLegacy / cudaStreamPerThread (what torch's default
// stream is passed as): work on those cannot be captured into a CUDA graph, so the call
// runs on the context's stream between two event fences -- ordered after the caller's
// earlier work and before its later work, without a host wait.  Any other handle: that
// stream itself.
struct CallStream {
    DeviceCtx *c;
    cudaStream_t user, st;
    bool fenced;
    CallStream(DeviceCtx *c_, void *stream) : c(c_), user((cudaStream_t)stream) {
        fenced = user == cudaStreamLegacy || user == cudaStreamPerThread;
        st = (user && !fenced) ? user : c->stream;
    }
    int enter() {
        if (fenced) {
            BF_TRY_CUDA(cudaEventRecord(c->fin, user));
            BF_TRY_CUDA(cudaStreamWaitEvent(st, c->fin, 0));
        }
        return BF_OK;
    }
    int leave() {
        if (fenced) {
            BF_TRY_CUDA(cudaEventRecord(c->fout, st));
            BF_TRY_CUDA(cudaStreamWaitEvent(user, c->fout, 0));
        } else if (!user) {
            BF_TRY_CUDA(cudaStreamSynchronize(st));
        }
        return BF_OK;
    }
};

std::mutex g_ctx_mu;
std::vector<DeviceCtx *> g_ctx;

int get_ctx(int device, DeviceCtx **out) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(BF_ENODEV, "no CUDA device available (%s)",
                    e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
    }
    if (device < 0 || device >= n) return fail(BF_EINVAL, "device %d out of range [0,%d)", device, n);
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    if ((int)g_ctx.size() < n) g_ctx.resize(n, nullptr);
    if (!g_ctx[device]) {
        BF_TRY_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop;
        BF_TRY_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10)
            return fail(BF_ENODEV, "device %d is sm_%d%d; this library is built for sm_100a",
                        device, prop.major, prop.minor);
        DeviceCtx *c = new DeviceCtx();
        c->dev = device;
        c->sms = prop.multiProcessorCount;
        c->total_mem = prop.totalGlobalMem;
        const unsigned fl = cudaEventDisableTiming;
        BF_TRY_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        BF_TRY_CUDA(cudaEventCreateWithFlags(&c->done, fl));
        BF_TRY_CUDA(cudaEventCreateWithFlags(&c->pro, fl));
        BF_TRY_CUDA(cudaEventCreateWithFlags(&c->entry, fl));
        BF_TRY_CUDA(cudaEventCreateWithFlags(&c->zdone, fl));
        BF_TRY_CUDA(cudaEventCreateWithFlags(&c->fin, fl));
        BF_TRY_CUDA(cudaEventCreateWithFlags(&c->fout, fl));
        BF_TRY_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
        BF_TRY_CUDA(cudaEventCreateWithFlags(&c->kend, fl));
        BF_TRY_CUDA(cudaEventCreateWithFlags(&c->sdone, fl));
        for (Slot &s : c->slot) {
            BF_TRY_CUDA(cudaStreamCreateWithFlags(&s.ss, cudaStreamNonBlocking));
            BF_TRY_CUDA(cudaStreamCreateWithFlags(&s.sw, cudaStreamNonBlocking));
            BF_TRY_CUDA(cudaEventCreateWithFlags(&s.fork, fl));
            BF_TRY_CUDA(cudaEventCreateWithFlags(&s.join, fl));
            BF_TRY_CUDA(cudaEventCreateWithFlags(&s.kdone, fl));
            BF_TRY_CUDA(cudaEventCreateWithFlags(&s.freed, fl));
            BF_TRY_CUDA(cudaEventCreateWithFlags(&s.h2d, fl));
            BF_TRY_CUDA(cudaEventCreateWithFlags(&s.qfork, fl));
            BF_TRY_CUDA(cudaEventCreateWithFlags(&s.qjoin, fl));
        }
        g_ctx[device] = c;
    }
    *out = g_ctx[device];
    return BF_OK;
}

// ---------------------------------------------------- deferred statistics ----

// Statistics of the last fp32 call on this thread: the device counters are copied into
// pinned memory at the end of the call (stream-ordered) and reduced only when asked.
// Two buffers alternate, so a call never waits for the one right before it.
struct StatsBuf {
    cudaEvent_t ready = nullptr, t0 = nullptr, t1 = nullptr;
    bool inflight = false;
    GbsStats *h_stats = nullptr;
    unsigned long long *h_cand = nullptr;
    size_t cand_cap = 0;
    int64_t n_tiles = 0, tile = 0, n_obs = 0;
    bool timed = false;  // t0/t1 recorded by the call (bf_set_kernel_timing)
};
struct PendingStats {
    int dev = -1;
    StatsBuf buf[2];
    int cur = 0;           // buffer of the last call
    bool pending = false;  // buf[cur] holds an unread call
    GbsStats last = {};
    int64_t last_total_pairs = 0, last_tiles = 0;
};
thread_local PendingStats g_ps;

// While a call is being captured into a graph (GraphCache) the statistics events are
// recorded as external event nodes, so every replay records them for real.
thread_local bool g_capturing = false;
// Kernel timing of fp32 calls (bf_last_stats kernel_ms): two event records around the
// summation, ~10 us per call of graph-node latency on small calls, so off by default.
std::atomic<int> g_kernel_timing{0};
cudaError_t rec_ext(cudaEvent_t e, cudaStream_t s) {
    return g_capturing ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
                       : cudaEventRecord(e, s);
}

int stats_events(int dev) {
    if (g_ps.dev == dev && g_ps.buf[0].ready) return BF_OK;
    g_pool_gen.fetch_add(1);
    for (StatsBuf &b : g_ps.buf) {
        if (b.ready) {
            cudaEventSynchronize(b.ready);
            cudaEventDestroy(b.ready);
            cudaEventDestroy(b.t0);
            cudaEventDestroy(b.t1);
        }
        b.inflight = false;
        BF_TRY_CUDA(cudaEventCreateWithFlags(&b.ready, cudaEventDisableTiming));
        BF_TRY_CUDA(cudaEventCreate(&b.t0));
        BF_TRY_CUDA(cudaEventCreate(&b.t1));
    }
    g_ps.pending = false;
    g_ps.dev = dev;
    return BF_OK;
}

void materialize_stats() {
    if (!g_ps.pending) return;
    g_ps.pending = false;
    StatsBuf &b = g_ps.buf[g_ps.cur];
    b.inflight = false;
    if (cudaEventSynchronize(b.ready) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    GbsStats h = *b.h_stats;
    float ms = 0.f;
    if (b.timed && cudaEventElapsedTime(&ms, b.t0, b.t1) != cudaSuccess) {
        cudaGetLastError();
        ms = 0.f;
    }
    h.kernel_ms = ms;
    unsigned long long cp = 0, cs = 0, tp = 0, ts = 0;
    const int64_t nt = b.n_tiles;
    for (int64_t i = 0; i < nt; ++i) {
        const unsigned long long in_tile =
            (unsigned long long)((i + 1 < nt) ? b.tile : b.n_obs - i * b.tile);
        cp += b.h_cand[(size_t)i] * in_tile;
        cs += b.h_cand[(size_t)(nt + i)] * in_tile;
        tp += b.h_cand[(size_t)(2 * nt + i)] * in_tile;
        ts += b.h_cand[(size_t)(3 * nt + i)] * in_tile;
    }
    h.candidate_pairs = cp;
    h.cand_pair_segs = cs;
    h.tight_pairs = tp;
    h.tight_pair_segs = ts;
    g_ps.last = h;
    g_ps.last_tiles = nt;
    if (getenv("BF_DEBUG_STATS"))
        fprintf(stderr, "bf stats: items culled %llu single %llu wedge %llu multi %llu ties %llu\n",
                h.paths[0], h.paths[1], h.paths[2], h.paths[3], h.tie_pairs);
}

// Starts a call's statistics (forgets the previous call's).
void stats_begin(int64_t total_pairs) {
    g_ps.pending = false;
    g_ps.last = GbsStats{};
    g_ps.last_tiles = 0;
    g_ps.last_total_pairs = total_pairs;
}

// The buffer the current fp32 call writes: the one not used by the previous call, after
// its copy from two calls back has landed.
int stats_next(StatsBuf **out) {
    const int i = g_ps.cur ^ 1;
    StatsBuf &b = g_ps.buf[i];
    if (b.inflight) BF_TRY_CUDA(cudaEventSynchronize(b.ready));
    b.inflight = false;
    g_ps.cur = i;
    *out = &b;
    return BF_OK;
}

// ------------------------------------------------------------ tiling ----

// Bounding box of n observers: grid-stride partial boxes per block (pass 1, out =
// 6 x gridDim doubles), then one block reduces the partials (pass 2).
__global__ void bbox_kernel(const double *obs, int64_t n, int stride3, double *out) {
    __shared__ double smin[3][256], smax[3][256];
    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        for (int d = 0; d < 3; ++d) {
            const double lo = obs[stride3 ? 3 * i + d : d * n + i];
            const double hi = stride3 ? lo : obs[3 * n + d * n + i];
            mn[d] = fmin(mn[d], lo);
            mx[d] = fmax(mx[d], hi);
        }
    for (int d = 0; d < 3; ++d) {
        smin[d][threadIdx.x] = mn[d];
        smax[d][threadIdx.x] = mx[d];
    }
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s)
            for (int d = 0; d < 3; ++d) {
                smin[d][threadIdx.x] = fmin(smin[d][threadIdx.x], smin[d][threadIdx.x + s]);
                smax[d][threadIdx.x] = fmax(smax[d][threadIdx.x], smax[d][threadIdx.x + s]);
            }
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int d = 0; d < 3; ++d) {
            out[d * gridDim.x + blockIdx.x] = smin[d][0];
            out[3 * gridDim.x + d * gridDim.x + blockIdx.x] = smax[d][0];
        }
}

__device__ __forceinline__ uint64_t spread3(uint64_t x) {
    x &= 0x1fffff;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}

// Hilbert index of a receiver (the tiling order: consecutive receivers are spatial
// neighbours with no jumps, so 128-receiver patches and 1024-receiver tiles are compact).
// A planar set (third extent < 1/64 of the largest) is cut along its longest axis into
// square blocks of the second extent, each traversed by the 2-D curve (which enters a
// block at its lower-left and leaves at its lower-right corner, so consecutive blocks
// join up); key = block << 42 | 2-D index.  Otherwise the 3-D curve over the isotropic
// bounding cube.  21 bits per axis within a block / the cube.
__device__ __forceinline__ uint64_t hilbert2(uint64_t x, uint64_t y) {
    const uint64_t n = 1ull << 21;
    uint64_t d = 0;
    for (uint64_t s = n >> 1; s > 0; s >>= 1) {
        const uint64_t rx = (x & s) ? 1 : 0, ry = (y & s) ? 1 : 0;
        d += s * s * ((3 * rx) ^ ry);
        if (ry == 0) {  // rotate the quadrant
            if (rx == 1) {
                x = n - 1 - x;
                y = n - 1 - y;
            }
            const uint64_t t = x;
            x = y;
            y = t;
        }
    }
    return d;
}

// 3-D curve: axes -> transposed Hilbert index (Skilling's construction), bit-interleaved.
__device__ __forceinline__ uint64_t hilbert3(uint64_t x0, uint64_t x1, uint64_t x2) {
    uint64_t X[3] = {x0, x1, x2};
    for (uint64_t Q = 1ull << 20; Q > 1; Q >>= 1) {
        const uint64_t P = Q - 1;
        for (int i = 0; i < 3; ++i) {
            if (X[i] & Q) {
                X[0] ^= P;
            } else {
                const uint64_t t = (X[0] ^ X[i]) & P;
                X[0] ^= t;
                X[i] ^= t;
            }
        }
    }
    X[1] ^= X[0];
    X[2] ^= X[1];
    uint64_t t = 0;
    for (uint64_t Q = 1ull << 20; Q > 1; Q >>= 1)
        if (X[2] & Q) t ^= Q - 1;
    for (int i = 0; i < 3; ++i) X[i] ^= t;
    return spread3(X[2]) | (spread3(X[1]) << 1) | (spread3(X[0]) << 2);
}

__global__ void order_key_kernel(const double *obs, int64_t n, const double *bbox,
                                 uint64_t *keys, int32_t *vals) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double ext[3], emax = 0.0;
    for (int d = 0; d < 3; ++d) {
        ext[d] = bbox[3 + d] - bbox[d];
        emax = fmax(emax, ext[d]);
    }
    uint64_t q[3];
    for (int d = 0; d < 3; ++d) {
        double u = emax > 0 ? (obs[3 * i + d] - bbox[d]) / emax : 0.0;
        u = fmin(fmax(u, 0.0), 1.0);
        q[d] = (uint64_t)(u * 2097151.0);
    }
    // axes by decreasing extent (ties: lower axis first)
    int a0 = 0, a1 = 1, a2 = 2;
    if (ext[a1] > ext[a0]) { const int t = a0; a0 = a1; a1 = t; }
    if (ext[a2] > ext[a1]) { const int t = a1; a1 = a2; a2 = t; }
    if (ext[a1] > ext[a0]) { const int t = a0; a0 = a1; a1 = t; }
    if (ext[a2] * 64.0 < emax) {
        const double L = fmax(ext[a1], ext[a0] * 0x1p-20);  // block side, <= 2^20 blocks
        if (!(L > 0.0)) {
            keys[i] = 0;
        } else {
            const double nbl = ceil(ext[a0] / L);
            const double u0 = (obs[3 * i + a0] - bbox[a0]) / L;
            const double blk = fmin(floor(u0), fmax(nbl - 1.0, 0.0));
            const double f0 = fmin(fmax(u0 - blk, 0.0), 1.0);
            const double f1 = fmin(fmax((obs[3 * i + a1] - bbox[a1]) / L, 0.0), 1.0);
            keys[i] = ((uint64_t)blk << 42) |
                      hilbert2((uint64_t)(f0 * 2097151.0), (uint64_t)(f1 * 2097151.0));
        }
    } else {
        keys[i] = hilbert3(q[a0], q[a1], q[a2]);
    }
    vals[i] = (int32_t)i;
}

// One block per tile: centre and half extents of the tile's bounding box, patch-local fp32
// offsets, and the tile radius.  The six extrema reduce together (warp shuffles, one
// shared-memory round; min/max are exact, so any order gives the same bits).  perm_in ==
// nullptr: receivers already in tile order, the identity permutation is written to perm_out.
template <int T>
__global__ void __launch_bounds__(T)
    tile_kernel(const double *obs, int64_t n, const int32_t *perm_in, int32_t *perm_out,
                float4 *rloc, double4 *centre, double4 *tbox) {
    constexpr int NW = T / 32;
    __shared__ double s_red[6][NW];
    __shared__ double s_c[3], s_h[3];
    __shared__ float s_r;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t si = (int64_t)blockIdx.x * T + threadIdx.x;
    const bool valid = si < n;
    double p[3] = {0, 0, 0};
    if (valid) {
        int64_t oi = si;
        if (perm_in)
            oi = perm_in[si];
        else
            perm_out[si] = (int32_t)si;
        for (int d = 0; d < 3; ++d) p[d] = obs[3 * oi + d];
    }
    // v[d] -> min p_d, v[3 + d] -> min -p_d = -max p_d
    double v[6];
    for (int d = 0; d < 3; ++d) {
        v[d] = valid ? p[d] : INFINITY;
        v[3 + d] = valid ? -p[d] : INFINITY;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1)
#pragma unroll
        for (int k = 0; k < 6; ++k) v[k] = fmin(v[k], __shfl_xor_sync(0xffffffffu, v[k], o));
    if (lane == 0)
        for (int k = 0; k < 6; ++k) s_red[k][wid] = v[k];
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int k = 0; k < 6; ++k) v[k] = lane < NW ? s_red[k][lane] : INFINITY;
#pragma unroll
        for (int o = 16; o; o >>= 1)
#pragma unroll
            for (int k = 0; k < 6; ++k) v[k] = fmin(v[k], __shfl_xor_sync(0xffffffffu, v[k], o));
        if (lane == 0)
            for (int d = 0; d < 3; ++d) {
                const double mn = v[d], mx = -v[3 + d];
                s_c[d] = 0.5 * (mn + mx);
                s_h[d] = 0.5 * (mx - mn);
            }
    }
    __syncthreads();
    // the tile radius bounds |p - c| from above: fp64 offsets, rounded up to fp32 (the
    // work-list cut tests use it as a conservative bound)
    double rad = 0.0;
    if (valid) {
        const double dx = p[0] - s_c[0], dy = p[1] - s_c[1], dz = p[2] - s_c[2];
        rloc[si] = make_float4((float)dx, (float)dy, (float)dz, 0.f);
        rad = sqrt(dx * dx + dy * dy + dz * dz) * (1.0 + 1e-15);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) rad = fmax(rad, __shfl_xor_sync(0xffffffffu, rad, o));
    if (lane == 0) s_red[0][wid] = rad;
    __syncthreads();
    if (wid == 0) {
        rad = lane < NW ? s_red[0][lane] : 0.0;
#pragma unroll
        for (int o = 16; o; o >>= 1) rad = fmax(rad, __shfl_xor_sync(0xffffffffu, rad, o));
        if (lane == 0) {
            s_r = __double2float_ru(rad);
            centre[blockIdx.x] = make_double4(s_c[0], s_c[1], s_c[2], (double)s_r);
            tbox[blockIdx.x] = make_double4(s_h[0], s_h[1], s_h[2], (double)s_r);
        }
    }
}


// Hilbert order of n observers into *perm (a workspace buffer).
int hilbert_order(DeviceCtx *c, const double *obs, int64_t n, cudaStream_t st,
                 const int32_t **perm) {
    double *bbox;
    uint64_t *k1, *k2;
    int32_t *v1, *v2;
    BF_TRY(c->get(B_BBOX, 6 + 6 * 256, &bbox));
    BF_TRY(c->get(B_KEYS, n, &k1));
    BF_TRY(c->get(B_KEYS2, n, &k2));
    BF_TRY(c->get(B_VALS, n, &v1));
    BF_TRY(c->get(B_VALS2, n, &v2));
    // pass 1: 256 partial boxes (min block-major in bbox[6..], max after); pass 2: final
    bbox_kernel<<<256, 256, 0, st>>>(obs, n, 1, bbox + 6);
    bbox_kernel<<<1, 256, 0, st>>>(bbox + 6, 256, 0, bbox);
    order_key_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(obs, n, bbox, k1, v1);
    note_launch(3);
    BF_TRY_CUDA(cudaGetLastError());
    cub::DoubleBuffer<uint64_t> dk(k1, k2);
    cub::DoubleBuffer<int32_t> dv(v1, v2);
    size_t tmp_bytes = 0;
    BF_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dk, dv, (int)n, 0, 63, st));
    void *tmp;
    BF_TRY(c->buf[B_CUB].get(tmp_bytes + 16, &tmp));
    BF_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, dk, dv, (int)n, 0, 63, st));
    note_launch(4);
    *perm = dv.Current();
    return BF_OK;
}

int build_tiling(DeviceCtx *c, const double *obs, int64_t n, bool presorted, cudaStream_t st,
                 Tiling *out) {
    const int T = gbs_fp32_tile();
    out->n = n;
    out->tile = T;
    out->n_tiles = (n + T - 1) / T;
    if (n <= 0) return BF_OK;
    if (n > INT32_MAX) return fail(BF_EINVAL, "observer range too large (%lld)", (long long)n);
    float4 *rloc;
    double4 *cen, *box;
    BF_TRY(c->get(B_RLOC, n, &rloc));
    BF_TRY(c->get(B_CENTRE, out->n_tiles, &cen));
    BF_TRY(c->get(B_TBOX, out->n_tiles, &box));
    const int32_t *perm, *perm_in = nullptr;
    int32_t *perm_out = nullptr;
    if (presorted) {  // identity order, written by tile_kernel
        BF_TRY(c->get(B_VALS, n, &perm_out));
        perm = perm_out;
    } else {
        BF_TRY(hilbert_order(c, obs, n, st, &perm));
        perm_in = perm;
    }
    if (T == 512)
        tile_kernel<512><<<(unsigned)out->n_tiles, 512, 0, st>>>(obs, n, perm_in, perm_out, rloc,
                                                                 cen, box);
    else if (T == 256)
        tile_kernel<256><<<(unsigned)out->n_tiles, 256, 0, st>>>(obs, n, perm_in, perm_out, rloc,
                                                                 cen, box);
    else if (T == 1024)
        tile_kernel<1024><<<(unsigned)out->n_tiles, 1024, 0, st>>>(obs, n, perm_in, perm_out,
                                                                   rloc, cen, box);
    else
        return fail(BF_EINVAL, "unsupported tile size %d", T);
    note_launch();
    BF_TRY_CUDA(cudaGetLastError());
    out->perm = perm;
    out->rloc = rloc;
    out->centre = cen;
    out->tbox = box;
    return BF_OK;
}


int validate(int64_t n_beams, int64_t max_seg, int64_t n_obs, int64_t nf, int64_t obs_lo,
             int64_t obs_hi, int64_t beam_lo, int64_t beam_hi, int precision) {
    if (max_seg < 1) return fail(BF_EINVAL, "max_seg must be >= 1");
    if (nf < 0) return fail(BF_EINVAL, "negative frequency count %lld", (long long)nf);
    if (obs_lo < 0 || obs_hi < obs_lo || obs_hi > n_obs)
        return fail(BF_EINVAL, "observer range [%lld,%lld) outside [0,%lld)", (long long)obs_lo,
                    (long long)obs_hi, (long long)n_obs);
    if (beam_lo < 0 || beam_hi < beam_lo || beam_hi > n_beams)
        return fail(BF_EINVAL, "beam range [%lld,%lld) outside [0,%lld)", (long long)beam_lo,
                    (long long)beam_hi, (long long)n_beams);
    if (precision != BF_PRECISION_FP32 && precision != BF_PRECISION_FP64)
        return fail(BF_EINVAL, "unknown precision %d", precision);
    if (precision == BF_PRECISION_FP32 && max_seg > BF_FP32_MAX_SEG)
        return fail(BF_EINVAL,
                    "fp32 mode supports max_seg <= %d (r_max <= %d), got %lld; use fp64 mode",
                    BF_FP32_MAX_SEG, BF_FP32_MAX_SEG - 1, (long long)max_seg);
    if (obs_hi - obs_lo > INT32_MAX)
        return fail(BF_EINVAL, "observer range too large (%lld); split the call",
                    (long long)(obs_hi - obs_lo));
    if (precision == BF_PRECISION_FP32 && beam_hi - beam_lo >= ((int64_t)1 << 27))
        return fail(BF_EINVAL, "more than 2^27 beams in one fp32 call; split the beam range");
    return BF_OK;
}

// Group-workspace budget: the caller's (bf_set_memory_budget) or 1/8 of device memory,
// at most 24 GiB.  Only the grouping depends on it, never the result bits.
int64_t group_budget(DeviceCtx *c) {
    if (c->budget > 0) return c->budget;
    return std::min<int64_t>((int64_t)(c->total_mem / 8), (int64_t)24 << 30);
}

struct GroupPlan {
    int64_t range_beams = 0, n_ranges = 0;
    std::vector<std::pair<int64_t, int64_t>> groups;  // [q0, q1) in ranges
};

// Beam groups of whole ranges sized so that NSLOT groups' workspaces fit the budget.
// The host-buffer path ramps the group size up from one range (1, 4, 16, ...) so the
// first group's packing and copy are short and the later ones hide behind the summation
// (few groups: each group's kernel ends in a tail of long units near the source).
void plan_groups(DeviceCtx *c, int64_t nb, int64_t max_seg, int nf, int64_t n_tiles,
                 int64_t n_patches, int64_t n_pad, bool host, GroupPlan *g) {
    g->range_beams = gbs_fp32_range_beams(nb, nf);
    const int64_t rb = g->range_beams;
    g->n_ranges = (nb + rb - 1) / rb;
    const int64_t per_range = n_pad * (16 * nf + 4) + n_patches * 24 + n_tiles * 16;
    const int64_t per_beam = n_tiles / 4 + 1 + n_tiles * 4 + max_seg * (68 + 8 * nf) + 8;
    const int64_t per_r = per_range + rb * per_beam;
    const int64_t budget = group_budget(c);
    int64_t max_r;
    if (!host && per_r * g->n_ranges <= budget)
        max_r = g->n_ranges;  // everything in one group
    else
        max_r = std::max<int64_t>(1, budget / NSLOT / std::max<int64_t>(per_r, 1));
    max_r = std::min(max_r, std::max<int64_t>(1, (((int64_t)1 << 27) - 1) / (rb * max_seg)));
    max_r = std::min(max_r, std::max<int64_t>(1, (((int64_t)1 << 31) - 1) / std::max<int64_t>(n_patches, 1)));
    max_r = std::min(max_r, g->n_ranges);
    g->groups.clear();
#ifndef BF_HOST_FIRST
#define BF_HOST_FIRST 1
#endif
#ifndef BF_HOST_RAMP
#define BF_HOST_RAMP 4  // measured on config 3: 8 -> 447.6 ms, 4 -> 444.9, 3 -> 444.7, uniform groups worse
#endif
    int64_t q = 0, step = host ? std::min<int64_t>(BF_HOST_FIRST, max_r) : max_r;
    while (q < g->n_ranges) {
        const int64_t n = std::min(step, g->n_ranges - q);
        g->groups.emplace_back(q, q + n);
        q += n;
        step = std::min(max_r, step * BF_HOST_RAMP);
    }
}

// Host -> device of `bytes` from host memory that may be pageable: pinned sources are
// copied directly, pageable ones through pinned staging filled on the host threads.
int h2d(void *dst, const void *src, size_t bytes, PinBuf &stage, cudaStream_t st) {
    if (bytes == 0) return BF_OK;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost) {
        BF_TRY_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        return BF_OK;
    }
    cudaGetLastError();
    void *p;
    BF_TRY(stage.get(bytes, &p));
    parallel_copy(p, src, bytes);
    BF_TRY_CUDA(cudaMemcpyAsync(dst, p, bytes, cudaMemcpyHostToDevice, st));
    return BF_OK;
}

// The host call's results (acc, then evals) back into memory that may be pageable, then
// synchronise st.  Pageable targets: all DMAs into pinned staging are enqueued first (acc
// in two halves, each followed by an event), and the host threads copy each piece out as
// soon as it has landed while the next ones are still in flight.
int d2h_out(DeviceCtx *c, void *acc_dst, const void *acc_src, size_t acc_bytes,
            void *ev_dst, const void *ev_src, size_t ev_bytes, cudaStream_t st) {
    cudaPointerAttributes at;
    const bool pa = cudaPointerGetAttributes(&at, acc_dst) == cudaSuccess &&
                    at.type == cudaMemoryTypeHost;
    cudaGetLastError();
    const bool pe = cudaPointerGetAttributes(&at, ev_dst) == cudaSuccess &&
                    at.type == cudaMemoryTypeHost;
    cudaGetLastError();
    for (auto &e : c->piece)
        if (!e) BF_TRY_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    char *sa = nullptr, *se = nullptr;
    const size_t h0 = acc_bytes / 2 / 16 * 16, h1 = acc_bytes - h0;
    if (pa) {
        if (acc_bytes) BF_TRY_CUDA(cudaMemcpyAsync(acc_dst, acc_src, acc_bytes, cudaMemcpyDeviceToHost, st));
    } else if (acc_bytes) {
        void *p;
        BF_TRY(c->hpin[H_ACC].get(acc_bytes, &p));
        sa = (char *)p;
        BF_TRY_CUDA(cudaMemcpyAsync(sa, acc_src, h0, cudaMemcpyDeviceToHost, st));
        BF_TRY_CUDA(cudaEventRecord(c->piece[0], st));
        BF_TRY_CUDA(cudaMemcpyAsync(sa + h0, (const char *)acc_src + h0, h1,
                                    cudaMemcpyDeviceToHost, st));
        BF_TRY_CUDA(cudaEventRecord(c->piece[1], st));
    }
    if (pe) {
        if (ev_bytes) BF_TRY_CUDA(cudaMemcpyAsync(ev_dst, ev_src, ev_bytes, cudaMemcpyDeviceToHost, st));
    } else if (ev_bytes) {
        void *p;
        BF_TRY(c->hpin[H_EV].get(ev_bytes, &p));
        se = (char *)p;
        BF_TRY_CUDA(cudaMemcpyAsync(se, ev_src, ev_bytes, cudaMemcpyDeviceToHost, st));
    }
    if (sa) {
        BF_TRY_CUDA(cudaEventSynchronize(c->piece[0]));
        parallel_copy(acc_dst, sa, h0);
        BF_TRY_CUDA(cudaEventSynchronize(c->piece[1]));
        parallel_copy((char *)acc_dst + h0, sa + h0, h1);
    }
    BF_TRY_CUDA(cudaStreamSynchronize(st));
    if (se) parallel_copy(ev_dst, se, ev_bytes);
    return BF_OK;
}

// Compact rows of host beams [b0, b0 + nb) (local indices of h) packed on the host
// threads into the slot's pinned staging and copied to its device buffers on s.ss.
int rows_from_host(const GbsArgs &h, int64_t b0, int64_t nb, Slot &s, Rows *out,
                   int64_t *n_rows) {
    if (s.h2d_valid) BF_TRY_CUDA(cudaEventSynchronize(s.h2d));  // staging reused
    int64_t *hs;
    BF_TRY(s.pinned(P_START, (size_t)(nb + 1), &hs));
    const int64_t S = h.max_seg;
    hs[0] = 0;
    for (int64_t i = 0; i < nb; ++i) {
        int64_t n = h.n_segs[b0 + i];
        n = n < 0 ? 0 : (n > S ? S : n);
        hs[i + 1] = hs[i] + n;
    }
    const int64_t rows = hs[nb];
    double4 *hp0, *hp1;
    float *ha;
    BF_TRY(s.pinned(P_P0, (size_t)rows, &hp0));
    BF_TRY(s.pinned(P_P1, (size_t)rows, &hp1));
    BF_TRY(s.pinned(P_AMP, (size_t)rows, &ha));
    const double amp_scale = h.phi_amp * sqrt(h.c) / (2.0 * 3.141592653589793 * h.c);
    parallel_for(nb, 4096, [&](int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi; ++i) {
            const int64_t b = b0 + i, dst0 = hs[i], n = hs[i + 1] - hs[i];
            const double wb = h.weights[b];
            for (int64_t k = 0; k < n; ++k) {
                const int64_t row = b * S + k, d = dst0 + k;
                const double *o = h.seg_origin + 3 * row, *dd = h.seg_dir + 3 * row;
                hp0[d] = make_double4(o[0], o[1], o[2], h.seg_len[row]);
                hp1[d] = make_double4(dd[0], dd[1], dd[2], h.seg_s0[row]);
                // same operations as rows_pack_kernel: (amp_scale * refl) * w_b, one rounding
                ha[d] = (float)(amp_scale * h.seg_refl[row] * wb);
            }
        }
    });
    int64_t *ds;
    double4 *dp0, *dp1;
    float *da;
    BF_TRY(s.get(S_START, (size_t)(nb + 1), &ds));
    BF_TRY(s.get(S_P0, (size_t)std::max<int64_t>(rows, 1), &dp0));
    BF_TRY(s.get(S_P1, (size_t)std::max<int64_t>(rows, 1), &dp1));
    BF_TRY(s.get(S_AMP, (size_t)std::max<int64_t>(rows, 1), &da));
    const auto H2D = cudaMemcpyHostToDevice;
    BF_TRY_CUDA(cudaMemcpyAsync(ds, hs, 8 * (size_t)(nb + 1), H2D, s.ss));
    BF_TRY_CUDA(cudaMemcpyAsync(dp0, hp0, 32 * (size_t)rows, H2D, s.ss));
    BF_TRY_CUDA(cudaMemcpyAsync(dp1, hp1, 32 * (size_t)rows, H2D, s.ss));
    BF_TRY_CUDA(cudaMemcpyAsync(da, ha, 4 * (size_t)rows, H2D, s.ss));
    BF_TRY_CUDA(cudaEventRecord(s.h2d, s.ss));
    s.h2d_valid = true;
    *out = Rows{ds, dp0, dp1, da, nb, S};
    *n_rows = rows;
    return BF_OK;
}

// Single-CTA scans for small arrays (small calls): one launch instead of a count kernel
// plus cub's init and scan kernels.  Thread t sums a contiguous run of the input, a block
// scan offsets the runs; integer sums, so the result equals cub's.
constexpr int SCAN1_T = 1024;
constexpr int64_t SCAN1_MAX = (int64_t)SCAN1_T * 64;

// start[0] = 0, start[b + 1] = sum over k <= b of n_segs[k] clamped to [0, max_seg]
// (= rows_count_kernel + an inclusive scan of n_beams + 1 entries)
__global__ void __launch_bounds__(SCAN1_T)
    rows_scan1_kernel(const int32_t *n_segs, int64_t n_beams, int64_t max_seg, int64_t *start) {
    using BS = cub::BlockScan<int64_t, SCAN1_T>;
    __shared__ typename BS::TempStorage tmp;
    const int64_t per = (n_beams + SCAN1_T - 1) / SCAN1_T;
    const int64_t b0 = threadIdx.x * per, b1 = min(n_beams, b0 + per);
    auto cnt = [&](int64_t b) {
        const int64_t n = n_segs[b];
        return n < 0 ? (int64_t)0 : (n > max_seg ? max_seg : n);
    };
    int64_t loc = 0;
    for (int64_t b = b0; b < b1; ++b) loc += cnt(b);
    int64_t pre;
    BS(tmp).ExclusiveSum(loc, pre);
    if (threadIdx.x == 0) start[0] = 0;
    for (int64_t b = b0; b < b1; ++b) {
        pre += cnt(b);
        start[b + 1] = pre;
    }
}

// out[i] = sum over k < i of in[k] for i < n (= cub::DeviceScan::ExclusiveSum)
__global__ void __launch_bounds__(SCAN1_T)
    exscan1_kernel(const int64_t *in, int64_t *out, int64_t n) {
    using BS = cub::BlockScan<int64_t, SCAN1_T>;
    __shared__ typename BS::TempStorage tmp;
    const int64_t per = (n + SCAN1_T - 1) / SCAN1_T;
    const int64_t i0 = threadIdx.x * per, i1 = min(n, i0 + per);
    int64_t loc = 0;
    for (int64_t i = i0; i < i1; ++i) loc += in[i];
    int64_t pre;
    BS(tmp).ExclusiveSum(loc, pre);
    for (int64_t i = i0; i < i1; ++i) {
        const int64_t v = in[i];
        out[i] = pre;
        pre += v;
    }
}

// Compact rows of device beams [b0, b0 + nb) of the padded bundle in g (local indices),
// packed on s.ss.  The row count stays on the device; rows_bound = nb * max_seg.
int rows_from_device(const GbsArgs &g, Slot &s, Rows *out) {
    const int64_t nb = g.n_beams, S = g.max_seg;
    int64_t *ds;
    double4 *dp0, *dp1;
    float *da;
    BF_TRY(s.get(S_START, (size_t)(nb + 1), &ds));
    BF_TRY(s.get(S_P0, (size_t)std::max<int64_t>(nb * S, 1), &dp0));
    BF_TRY(s.get(S_P1, (size_t)std::max<int64_t>(nb * S, 1), &dp1));
    BF_TRY(s.get(S_AMP, (size_t)std::max<int64_t>(nb * S, 1), &da));
    if (nb + 1 <= SCAN1_MAX) {
        rows_scan1_kernel<<<1, SCAN1_T, 0, s.ss>>>(g.n_segs, nb, S, ds);
        note_launch();
        BF_TRY_CUDA(cudaGetLastError());
    } else {
        BF_TRY(launch_rows_count(g.n_segs, nb, S, 0, ds, s.ss));
        size_t tb = 0;
        BF_TRY_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, ds, ds, (int)(nb + 1), s.ss));
        void *tmp;
        BF_TRY(s.buf[S_CUB].get(tb + 16, &tmp));
        BF_TRY_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, ds, ds, (int)(nb + 1), s.ss));
        note_launch();
    }
    BF_TRY(launch_rows_pack(g, ds, dp0, dp1, da, s.ss));
    *out = Rows{ds, dp0, dp1, da, nb, S};
    return BF_OK;
}

}  // namespace
}  // namespace bf

// Compact segment rows resident on one device (bf_rows_*): appended chunk by chunk,
// summed in one call.
struct bf_rows {
    int device = 0;
    int64_t n_beams = 0, n_rows = 0;     // exact totals
    int64_t cap_beams = 0, cap_rows = 0;  // allocated
    int64_t max_seg = 0;                  // largest padded row count appended
    double c = 0.0, phi_amp = 0.0;
    int64_t *start = nullptr;             // n_beams + 1
    double4 *p0 = nullptr, *p1 = nullptr;
    float *amp = nullptr;
    bf::Rows view() const { return bf::Rows{start, p0, p1, amp, n_beams, max_seg}; }
};

namespace bf {
namespace {

// Beams [b0, b0 + nb) of resident rows copied into the slot's own rows (start at 0).
int rows_from_resident(const bf_rows &R, int64_t b0, int64_t nb, Slot &s, Rows *out) {
    const int64_t S = R.max_seg;
    int64_t *ds;
    double4 *dp0, *dp1;
    float *da;
    BF_TRY(s.get(S_START, (size_t)(nb + 1), &ds));
    BF_TRY(s.get(S_P0, (size_t)std::max<int64_t>(nb * S, 1), &dp0));
    BF_TRY(s.get(S_P1, (size_t)std::max<int64_t>(nb * S, 1), &dp1));
    BF_TRY(s.get(S_AMP, (size_t)std::max<int64_t>(nb * S, 1), &da));
    BF_TRY(launch_rows_slice(R.view(), b0, nb, ds, dp0, dp1, da, s.ss));
    *out = Rows{ds, dp0, dp1, da, nb, S};
    return BF_OK;
}

// Zeroes two word arrays in one launch (the call's counters: one graph node instead of
// two memset nodes).
__global__ void zero2_kernel(unsigned long long *a, int64_t na, unsigned long long *b,
                             int64_t nb) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na + nb;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i < na) a[i] = 0ull;
        else b[i - na] = 0ull;
    }
}

thread_local struct {
    const void *d_stats, *d_cand;
    int64_t n_tiles;
} g_stats_src;  // the counters of the call being captured (run_fp32_graph copies them back)

// The call's statistics back into sb's pinned buffers on the context's side stream after
// everything enqueued on st so far: the caller's stream does not wait for the copies.
int stats_copy(DeviceCtx *c, StatsBuf *sb, const void *d_stats, const void *d_cand,
               int64_t n_tiles, cudaStream_t st) {
    if (!sb->h_stats) {
        g_pool_gen.fetch_add(1);
        BF_TRY_CUDA(cudaHostAlloc(&sb->h_stats, sizeof(GbsStats), cudaHostAllocPortable));
    }
    if (sb->cand_cap < (size_t)(4 * n_tiles)) {
        g_pool_gen.fetch_add(1);
        if (sb->h_cand) cudaFreeHost(sb->h_cand);
        sb->h_cand = nullptr;
        sb->cand_cap = 0;
        BF_TRY_CUDA(cudaHostAlloc(&sb->h_cand, 4 * sizeof(unsigned long long) * n_tiles,
                                  cudaHostAllocPortable));
        sb->cand_cap = (size_t)(4 * n_tiles);
    }
    BF_TRY_CUDA(cudaEventRecord(c->kend, st));
    BF_TRY_CUDA(cudaStreamWaitEvent(c->side, c->kend, 0));
    BF_TRY_CUDA(cudaMemcpyAsync(sb->h_stats, d_stats, sizeof(GbsStats), cudaMemcpyDeviceToHost,
                                c->side));
    BF_TRY_CUDA(cudaMemcpyAsync(sb->h_cand, d_cand, 4 * sizeof(unsigned long long) * n_tiles,
                                cudaMemcpyDeviceToHost, c->side));
    BF_TRY_CUDA(cudaEventRecord(sb->ready, c->side));
    BF_TRY_CUDA(cudaEventRecord(c->sdone, c->side));
    c->sdone_valid = true;
    sb->inflight = true;
    return BF_OK;
}

// The fp32 operator on LOCAL ranges: base.obs/acc/evals are device pointers (offset to
// obs_lo, acc rows of base.acc_stride complex values); base.seg_*/n_segs/weights are the
// padded bundle from beam_lo, on the device or (host_rows) in host memory.
// first_fold (may be null) runs on the host right before the first fold is enqueued on st
// (the host-buffer path stages and uploads the caller's acc/evals there, overlapping the
// first group's kernels).
// resident (may be null): the beams are rows [beam_off, beam_off + base.n_beams) of these
// resident compact rows instead of base.seg_*.
int run_fp32(DeviceCtx *c, const GbsArgs &base, const double *omegas, int64_t nf,
             bool host_rows, int flags, cudaStream_t st,
             const std::function<int()> *first_fold = nullptr,
             const bf_rows *resident = nullptr, int64_t beam_off = 0) {
    stats_begin(base.n_obs * base.n_beams);
    if (base.n_obs <= 0 || base.n_beams <= 0 || nf <= 0) return BF_OK;
    // the beam side of each group (compact rows) depends only on the call's inputs: the
    // slot streams start from the call's entry and overlap the receiver tiling below;
    // each group's work list waits for the tiling (c->pro)
    BF_TRY_CUDA(cudaEventRecord(c->entry, st));
    for (Slot &s : c->slot) BF_TRY_CUDA(cudaStreamWaitEvent(s.ss, c->entry, 0));
    // ---- prologue on the call's stream: receiver tiling, patches, zeroed counters
    Tiling t;
    BF_TRY(build_tiling(c, base.obs, base.n_obs, (flags & BF_FLAG_OBS_PRESORTED) != 0, st, &t));
    Fp32Work w0{};
    const int P = gbs_fp32_patch();
    w0.n_patches = (base.n_obs + P - 1) / P;
    w0.n_pad = w0.n_patches * P;
    BF_TRY(c->get(B_PRL, (size_t)base.n_obs, &w0.prl));
    BF_TRY(c->get(B_POS64, (size_t)base.n_obs, &w0.pos64));
    BF_TRY(c->get(B_PCEN, (size_t)w0.n_patches, &w0.pcen));
    BF_TRY(c->get(B_PBOX, (size_t)w0.n_patches, &w0.pbox));
    BF_TRY(launch_fp32_patches(base, t, w0, st));
    GbsStats *d_stats;
    unsigned long long *d_cand;  // per tile: a9 beams, a9 segments, tight beams, tight segments
    BF_TRY(c->get(B_STATS, 1, &d_stats));
    BF_TRY(c->get(B_CAND, (size_t)(4 * t.n_tiles), &d_cand));
    {   // zeroed on slot 0's stream (started at the call's entry), beside the tiling
        const int64_t na = sizeof(GbsStats) / 8, nb = 4 * t.n_tiles;
        const cudaStream_t zs = c->slot[0].ss;
        zero2_kernel<<<(unsigned)std::min<int64_t>((na + nb + 255) / 256, 1024), 256, 0, zs>>>(
            reinterpret_cast<unsigned long long *>(d_stats), na, d_cand, nb);
        note_launch();
        BF_TRY_CUDA(cudaGetLastError());
        BF_TRY_CUDA(cudaEventRecord(c->zdone, zs));
        BF_TRY_CUDA(cudaStreamWaitEvent(st, c->zdone, 0));
    }
    BF_TRY_CUDA(cudaEventRecord(c->pro, st));
    BF_TRY(stats_events(c->dev));
    StatsBuf *sb;
    BF_TRY(stats_next(&sb));
    sb->timed = g_kernel_timing.load() != 0;
    bool timed = false;
    int64_t gi = 0;
    // ---- frequency groups of <= BF_MAXF (acc columns are independent)
    for (int64_t f0 = 0; f0 < nf; f0 += BF_MAXF) {
        GbsArgs ag = base;
        ag.nf = (int)std::min<int64_t>(BF_MAXF, nf - f0);
        for (int f = 0; f < BF_MAXF; ++f) ag.omegas[f] = f < ag.nf ? omegas[f0 + f] : 0.0;
        ag.acc = base.acc + 2 * f0;
        Fp32Work wf = w0;
        {   // wide patches (fp64 tail, see unit_keys_kernel): kappa_max RW > 16 turns or
            // omega_max RW^2 / (2 c b) > 200 (the fp32 error of r.d and q^2 grows with RW;
            // at these bounds it stays ~5x below the 0.01 dB gate at 50 dB below the maximum)
            double wmax = 0.0;
            for (int f = 0; f < ag.nf; ++f) wmax = ag.omegas[f] > wmax ? ag.omegas[f] : wmax;
            wf.wide_k = (float)(wmax / (2.0 * 3.141592653589793 * ag.c) / 16.0);
            wf.wide_q = (float)(wmax / (2.0 * ag.c * ag.width_b) / 200.0);
        }
        double wmin = INFINITY;
        for (int f = 0; f < ag.nf; ++f) wmin = ag.omegas[f] < wmin ? ag.omegas[f] : wmin;
        GroupPlan plan;
        plan_groups(c, ag.n_beams, ag.max_seg, ag.nf, t.n_tiles, w0.n_patches, w0.n_pad,
                    host_rows, &plan);
        const int64_t rb = plan.range_beams;
        for (const auto &grp : plan.groups) {
            Slot &s = c->slot[gi++ % NSLOT];
            if (s.freed_valid) BF_TRY_CUDA(cudaStreamWaitEvent(s.ss, s.freed, 0));
            const int64_t b0 = grp.first * rb, b1 = std::min(grp.second * rb, ag.n_beams);
            GbsArgs gg = ag;
            gg.n_beams = b1 - b0;
            const int64_t r0 = b0 * ag.max_seg;
            gg.seg_origin = ag.seg_origin + 3 * r0;
            gg.seg_dir = ag.seg_dir + 3 * r0;
            gg.seg_e1 = gg.seg_e2 = nullptr;
            gg.seg_len = ag.seg_len + r0;
            gg.seg_s0 = ag.seg_s0 + r0;
            gg.seg_refl = ag.seg_refl + r0;
            gg.n_segs = ag.n_segs + b0;
            gg.weights = ag.weights + b0;
            // ---- compact rows of the group
            Rows rv;
            int64_t rows_bound;
            if (resident) {
                BF_TRY(rows_from_resident(*resident, beam_off + b0, gg.n_beams, s, &rv));
                rows_bound = gg.n_beams * resident->max_seg;
                gg.max_seg = resident->max_seg;
            } else if (host_rows) {
                BF_TRY(rows_from_host(ag, b0, gg.n_beams, s, &rv, &rows_bound));
            } else {
                BF_TRY(rows_from_device(gg, s, &rv));
                rows_bound = gg.n_beams * gg.max_seg;
            }
            (void)rows_bound;
            Fp32Work w = wf;
            w.start = rv.start;
            w.p0 = rv.p0;
            w.p1 = rv.p1;
            w.amp = rv.amp;
            w.range_beams = rb;
            w.n_ranges = grp.second - grp.first;
            // ---- tight work list of the group: bitmasks + counts per (tile, range)
            const int64_t n_words = (gg.n_beams + 31) / 32;
            uint32_t *bits, *tbits;
            BF_TRY(s.get(S_WLBITS, (size_t)(t.n_tiles * n_words), &bits));
            BF_TRY(s.get(S_WLTIGHT, (size_t)(t.n_tiles * n_words), &tbits));
            const int64_t nu_wl = t.n_tiles * w.n_ranges;
            int64_t *cnt;
            BF_TRY(s.get(S_WLCNT, (size_t)(nu_wl + 1), &cnt));
            BF_TRY(s.get(S_WLOFF, (size_t)(nu_wl + 1), &w.wl_off));
            BF_TRY_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (nu_wl + 1), s.ss));
            BF_TRY_CUDA(cudaStreamWaitEvent(s.ss, c->pro, 0));  // the tiling and counters
            BF_TRY(launch_worklist(gg, rv, t.centre, t.tbox, t.n_tiles, wmin, bits, tbits, rb,
                                   w.n_ranges, reinterpret_cast<unsigned long long *>(cnt),
                                   d_cand, s.ss));
            Tiling tg = t;
            tg.wl_bits = bits;
            tg.wl_tight = tbits;
            tg.wl_words = n_words;
            BF_TRY(s.get(S_WLITEMS, (size_t)(t.n_tiles * gg.n_beams + 1), &w.wl_items));
            BF_TRY(s.get(S_UCTR, 3, &w.unit_ctr));
            w.n_wide = w.unit_ctr + 2;
            const int64_t nu = w.n_patches * w.n_ranges;
            int32_t *v1;
            BF_TRY(s.get(S_UVALS2, (size_t)nu, &v1));
            if (nu <= SMALL_QUEUE_N && nu_wl + 1 <= SCAN1_MAX) {
                // small calls: the unit queue (one CTA; it needs only the counts) on the
                // wide-kernel stream, concurrent with the offsets scan and the compaction
                BF_TRY_CUDA(cudaEventRecord(s.qfork, s.ss));
                BF_TRY_CUDA(cudaStreamWaitEvent(s.sw, s.qfork, 0));
                BF_TRY(launch_fp32_small_queue(w, cnt, v1, s.sw));
                BF_TRY_CUDA(cudaEventRecord(s.qjoin, s.sw));
                w.unit_order = v1;
                exscan1_kernel<<<1, SCAN1_T, 0, s.ss>>>(cnt, w.wl_off, nu_wl + 1);
                note_launch();
                BF_TRY_CUDA(cudaGetLastError());
                BF_TRY(launch_fp32_wl_compact(tg, w, s.ss));
            } else {
                if (nu_wl + 1 <= SCAN1_MAX) {
                    exscan1_kernel<<<1, SCAN1_T, 0, s.ss>>>(cnt, w.wl_off, nu_wl + 1);
                    note_launch();
                    BF_TRY_CUDA(cudaGetLastError());
                } else {
                    size_t tb = 0;
                    BF_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, w.wl_off,
                                                              (int)(nu_wl + 1), s.ss));
                    void *tmp;
                    BF_TRY(s.buf[S_CUB].get(tb + 16, &tmp));
                    BF_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, w.wl_off,
                                                              (int)(nu_wl + 1), s.ss));
                    note_launch();
                }
                // ---- compacted work list (on the wide-kernel stream, concurrent with the queue
                //      order below): sized by its bound (tiles x beams), no host sync
                BF_TRY_CUDA(cudaEventRecord(s.qfork, s.ss));
                BF_TRY_CUDA(cudaStreamWaitEvent(s.sw, s.qfork, 0));
                BF_TRY(launch_fp32_wl_compact(tg, w, s.sw));
                BF_TRY_CUDA(cudaEventRecord(s.qjoin, s.sw));
                // ---- unit queue order (wide patches last; longest-first buckets, range-major
                //      inside a bucket) from the counts and the patch radii
                {
                    if (nu <= SMALL_QUEUE_N) {  // one CTA, one launch (small calls; it also
                                                // sets the queue heads and the wide count)
                        BF_TRY(launch_fp32_small_queue(w, cnt, v1, s.ss));
                        w.unit_order = v1;
                    } else {
                        BF_TRY_CUDA(cudaMemsetAsync(w.unit_ctr, 0, 3 * sizeof(unsigned), s.ss));
                        uint64_t *k0, *k1;
                        int32_t *v0;
                        BF_TRY(s.get(S_UKEYS, (size_t)nu, &k0));
                        BF_TRY(s.get(S_UKEYS2, (size_t)nu, &k1));
                        BF_TRY(s.get(S_UVALS, (size_t)nu, &v0));
                        BF_TRY(launch_fp32_unit_keys(tg, w, cnt, k0, v0, s.ss));
                        const int end_bit = 14;  // wide << 13 | bucket (7 bits) << 6 | range (< 64)
                        cub::DoubleBuffer<uint64_t> dk(k0, k1);
                        cub::DoubleBuffer<int32_t> dv(v0, v1);
                        size_t tb = 0;
                        BF_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)nu, 0,
                                                                    end_bit, s.ss));
                        void *tmp;
                        BF_TRY(s.buf[S_CUB].get(tb + 16, &tmp));
                        BF_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, (int)nu, 0,
                                                                    end_bit, s.ss));
                        note_launch();
                        w.unit_order = dv.Current();
                    }
                }
            }
            BF_TRY_CUDA(cudaStreamWaitEvent(s.ss, s.qjoin, 0));
            BF_TRY(s.get(S_PART, (size_t)(w.n_ranges * w.n_pad * ag.nf), &w.part));
            BF_TRY(s.get(S_PARTEV, (size_t)(w.n_ranges * w.n_pad), &w.part_ev));
            if (!timed) {
                if (sb->timed) BF_TRY_CUDA(rec_ext(sb->t0, s.ss));
                timed = true;
            }
            BF_TRY(launch_gbs_fp32(gg, tg, w, d_stats, StreamPair{s.ss, s.sw, s.fork, s.join}));
            BF_TRY_CUDA(cudaEventRecord(s.kdone, s.ss));
            // ---- fold on the call's stream, groups in order
            if (first_fold) {
                BF_TRY((*first_fold)());
                first_fold = nullptr;
            }
            BF_TRY_CUDA(cudaStreamWaitEvent(st, s.kdone, 0));
            BF_TRY(launch_fp32_fold(gg, tg, w, st));
            BF_TRY_CUDA(cudaEventRecord(s.freed, st));
            s.freed_valid = true;
        }
    }
    if (sb->timed) BF_TRY_CUDA(rec_ext(sb->t1, st));
    // ---- statistics: copied back asynchronously, reduced on request (bf_last_stats); a
    //      call being captured leaves the copies to run_fp32_graph (after the graph)
    sb->n_tiles = t.n_tiles;
    sb->tile = t.tile;
    sb->n_obs = base.n_obs;
    g_ps.pending = true;
    if (g_capturing) {
        g_stats_src = {d_stats, d_cand, t.n_tiles};
        sb->inflight = true;
        return BF_OK;
    }
    return stats_copy(c, sb, d_stats, d_cand, t.n_tiles, st);
}

// Small device calls (see DeviceCtx::GraphCache): identical repeated calls replay a graph
// captured from the second one.  The graph reads the caller's buffers at replay time, so
// only the arguments (pointers, sizes, scalars, frequencies, flags, stream) form the key.
#ifndef BF_GRAPHS
#define BF_GRAPHS 1
#endif
#ifndef BF_GRAPH_MAX_PAIRS
#define BF_GRAPH_MAX_PAIRS 268435456.0  // 2^28 beam-receiver pairs (calls of ~1 ms or less)
#endif
int run_fp32_graph(DeviceCtx *c, const GbsArgs &a, const double *omegas, int64_t nf, int flags,
                   int device, cudaStream_t st) {
    auto P = [](const void *p) { return (double)(uintptr_t)p; };
    std::vector<double> key = {
        (double)device, P(st), P(a.seg_origin), P(a.seg_dir), P(a.seg_len), P(a.seg_s0),
        P(a.seg_refl), P(a.n_segs), P(a.weights), P(a.obs), P(a.acc), P(a.evals),
        (double)a.n_beams, (double)a.max_seg, (double)a.n_obs, (double)nf, (double)a.acc_stride,
        a.c, a.width_b, a.phi_amp, (double)a.use_cutoff, (double)flags, (double)c->budget,
        (double)g_kernel_timing.load()};
    for (int64_t f = 0; f < nf; ++f) key.push_back(omegas[f]);
    DeviceCtx::GraphCache &g = c->gc;
    const bool same = g.seen && g.key == key;
    if (same && g.exec && g.gen == g_pool_gen.load()) {
        // replay: the statistics land in the buffer the graph writes
        stats_begin(a.n_obs * a.n_beams);
        BF_TRY(stats_events(c->dev));
        if (g.gen != g_pool_gen.load()) return run_fp32(c, a, omegas, nf, false, flags, st);
        StatsBuf &b = g_ps.buf[g.sb];  // (a replay overwrites the previous one's statistics)
        b.timed = g_kernel_timing.load() != 0;  // as captured (part of the key)
        BF_TRY_CUDA(cudaGraphLaunch(g.exec, st));
        note_launch(g.launches);
        g_ps.cur = g.sb;
        g_ps.pending = true;
        return stats_copy(c, &b, g.d_stats, g.d_cand, g.n_tiles, st);
    }
    if (g.exec) {
        cudaGraphExecDestroy(g.exec);
        g.exec = nullptr;
    }
    if (!same) {  // first call with this key: eager
        g.key = key;
        g.seen = true;
        return run_fp32(c, a, omegas, nf, false, flags, st);
    }
    // second call: capture the whole call (the slot streams join the capture through the
    // call's fork/join events; waits on events of earlier calls are dropped -- the graph
    // launch itself is ordered after them on st)
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
        cudaGetLastError();  // a stream that cannot be captured: stay eager for this key
        g.seen = false;
        g.key.clear();
        return run_fp32(c, a, omegas, nf, false, flags, st);
    }
    for (Slot &sl : c->slot) sl.freed_valid = false;
    const uint64_t n0 = g_launches.load();
    g_capturing = true;
    const int rc = run_fp32(c, a, omegas, nf, false, flags, st);
    g_capturing = false;
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(st, &graph);
    if (rc != BF_OK) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    BF_TRY_CUDA(ce);
    const cudaError_t ie = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    BF_TRY_CUDA(ie);
    g.launches = (int)(g_launches.load() - n0);
    g.sb = g_ps.cur;
    g.d_stats = g_stats_src.d_stats;
    g.d_cand = g_stats_src.d_cand;
    g.n_tiles = g_stats_src.n_tiles;
    for (Slot &sl : c->slot) sl.freed_valid = false;  // their events were capture-internal
    BF_TRY_CUDA(cudaGraphLaunch(g.exec, st));
    BF_TRY(stats_copy(c, &g_ps.buf[g.sb], g.d_stats, g.d_cand, g.n_tiles, st));
    g.gen = g_pool_gen.load();  // (after stats_copy: its first pinned allocation bumps it)
    return BF_OK;
}

// The fp64 (oracle-mode) operator on device-resident LOCAL ranges, frequency groups of
// <= BF_MAXF (one thread per observer continues acc in ascending beam order).
// base: device padded rows of the call's beams; t: the tiling of base.obs.  Beams go in
// groups whose work-list bitmasks fit the budget: compact rows and the tight (tile, beam)
// list of the group on the work slot's stream, then the oracle-mode kernel on st over
// each tile's list (beams ascending within and across groups: the dense loop's bits).
constexpr int FP64_SLOT = NSLOT - 1;  // (the host path stages its chunks in slots 0, 1)
int run_fp64(DeviceCtx *c, const GbsArgs &base, const double *omegas, int64_t nf,
             const Tiling &t, cudaStream_t st) {
    if (base.n_obs <= 0 || base.n_beams <= 0 || nf <= 0) return BF_OK;
    double wmin = INFINITY;
    for (int64_t f = 0; f < nf; ++f) wmin = omegas[f] < wmin ? omegas[f] : wmin;
    const int64_t per_beam = t.n_tiles / 4 + 1 + base.max_seg * 68 + 16;
    int64_t G = std::max<int64_t>(32, group_budget(c) / 2 / std::max<int64_t>(per_beam, 1));
    G = std::min<int64_t>(G / 32 * 32, ((int64_t)1 << 27) / std::max<int64_t>(base.max_seg, 1));
    Slot &s = c->slot[FP64_SLOT];
    for (int64_t b0 = 0; b0 < base.n_beams; b0 += G) {
        GbsArgs gg = base;
        gg.n_beams = std::min(G, base.n_beams - b0);
        const int64_t r0 = b0 * base.max_seg;
        gg.seg_origin = base.seg_origin + 3 * r0;
        gg.seg_dir = base.seg_dir + 3 * r0;
        gg.seg_e1 = base.seg_e1 + 3 * r0;
        gg.seg_e2 = base.seg_e2 + 3 * r0;
        gg.seg_len = base.seg_len + r0;
        gg.seg_s0 = base.seg_s0 + r0;
        gg.seg_refl = base.seg_refl + r0;
        gg.n_segs = base.n_segs + b0;
        gg.weights = base.weights + b0;
        BF_TRY_CUDA(cudaEventRecord(c->pro, st));  // the slot's buffers are free again
        BF_TRY_CUDA(cudaStreamWaitEvent(s.ss, c->pro, 0));
        Rows rv;
        BF_TRY(rows_from_device(gg, s, &rv));
        const int64_t n_words = (gg.n_beams + 31) / 32;
        uint32_t *bits, *tbits;
        BF_TRY(s.get(S_WLBITS, (size_t)(t.n_tiles * n_words), &bits));
        BF_TRY(s.get(S_WLTIGHT, (size_t)(t.n_tiles * n_words), &tbits));
        BF_TRY(launch_worklist(gg, rv, t.centre, t.tbox, t.n_tiles, wmin, bits, tbits, 0, 0,
                               nullptr, nullptr, s.ss));
        BF_TRY_CUDA(cudaEventRecord(s.kdone, s.ss));
        BF_TRY_CUDA(cudaStreamWaitEvent(st, s.kdone, 0));
        for (int64_t f0 = 0; f0 < nf; f0 += BF_MAXF) {
            GbsArgs ag = gg;
            ag.nf = (int)std::min<int64_t>(BF_MAXF, nf - f0);
            for (int f = 0; f < BF_MAXF; ++f) ag.omegas[f] = f < ag.nf ? omegas[f0 + f] : 0.0;
            ag.acc = base.acc + 2 * f0;
            BF_TRY(launch_gbs_fp64(ag, t.perm, t.tile, tbits, n_words, st));
        }
    }
    return BF_OK;
}

// fp64 operator on HOST padded rows: beam chunks (budgeted) copied through two pinned
// staging slots while the previous chunk sums; per observer the beams still run in
// ascending order, so the result equals one device call bit for bit.
int run_fp64_host(DeviceCtx *c, const GbsArgs &h, const double *omegas, int64_t nf,
                  cudaStream_t st) {
    if (h.n_obs <= 0 || h.n_beams <= 0 || nf <= 0) return BF_OK;
    Tiling t;
    BF_TRY(build_tiling(c, h.obs, h.n_obs, false, st, &t));
    const int64_t S = h.max_seg;
    const int64_t per_beam = S * (4 * 24 + 3 * 8) + 4 + 8;
    const int64_t chunk = std::max<int64_t>(
        1, std::min<int64_t>(h.n_beams, group_budget(c) / 2 / per_beam));
    BF_TRY_CUDA(cudaEventRecord(c->pro, st));
    int64_t gi = 0;
    for (int64_t b0 = 0; b0 < h.n_beams; b0 += chunk, ++gi) {
        Slot &s = c->slot[gi % 2];
        const int64_t nb = std::min(chunk, h.n_beams - b0), rows = nb * S;
        BF_TRY_CUDA(cudaStreamWaitEvent(s.ss, c->pro, 0));
        if (s.freed_valid) BF_TRY_CUDA(cudaStreamWaitEvent(s.ss, s.freed, 0));
        if (s.h2d_valid) BF_TRY_CUDA(cudaEventSynchronize(s.h2d));
        const size_t bytes = (size_t)(rows * (4 * 24 + 3 * 8) + nb * 12);
        char *hp, *dp;
        BF_TRY(s.pinned(P_F64, bytes, &hp));
        BF_TRY(s.get(S_F64, bytes, &dp));
        // carve: origin, dir, e1, e2 (24 B/row), len, s0, refl (8 B/row), weights, n_segs
        const size_t off[10] = {0,
                                (size_t)rows * 24,
                                (size_t)rows * 48,
                                (size_t)rows * 72,
                                (size_t)rows * 96,
                                (size_t)rows * 104,
                                (size_t)rows * 112,
                                (size_t)rows * 120,
                                (size_t)rows * 120 + (size_t)nb * 8,
                                bytes};
        const void *src[9] = {h.seg_origin + 3 * b0 * S, h.seg_dir + 3 * b0 * S,
                              h.seg_e1 + 3 * b0 * S,     h.seg_e2 + 3 * b0 * S,
                              h.seg_len + b0 * S,        h.seg_s0 + b0 * S,
                              h.seg_refl + b0 * S,       h.weights + b0,
                              h.n_segs + b0};
        for (int i = 0; i < 9; ++i) parallel_copy(hp + off[i], src[i], off[i + 1] - off[i]);
        BF_TRY_CUDA(cudaMemcpyAsync(dp, hp, bytes, cudaMemcpyHostToDevice, s.ss));
        BF_TRY_CUDA(cudaEventRecord(s.h2d, s.ss));
        s.h2d_valid = true;
        BF_TRY_CUDA(cudaStreamWaitEvent(st, s.h2d, 0));
        GbsArgs g = h;
        g.seg_origin = (const double *)(dp + off[0]);
        g.seg_dir = (const double *)(dp + off[1]);
        g.seg_e1 = (const double *)(dp + off[2]);
        g.seg_e2 = (const double *)(dp + off[3]);
        g.seg_len = (const double *)(dp + off[4]);
        g.seg_s0 = (const double *)(dp + off[5]);
        g.seg_refl = (const double *)(dp + off[6]);
        g.weights = (const double *)(dp + off[7]);
        g.n_segs = (const int32_t *)(dp + off[8]);
        g.n_beams = nb;
        BF_TRY(run_fp64(c, g, omegas, nf, t, st));
        BF_TRY_CUDA(cudaEventRecord(s.freed, st));
        s.freed_valid = true;
    }
    return BF_OK;
}

}  // namespace
}  // namespace bf

using namespace bf;

extern "C" {

const char *bf_version(void) { return "paper_2501_13382_b200 0.2.0 (sm_100a)"; }

const char *bf_last_error(void) { return g_err; }

int bf_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

uint64_t bf_launch_count(void) { return g_launches.load(); }

int bf_set_kernel_timing(int on) {
    g_kernel_timing.store(on != 0);
    return BF_OK;
}

int bf_set_memory_budget(int device, int64_t bytes) {
    if (bytes < 0) return fail(BF_EINVAL, "negative memory budget");
    DeviceCtx *ctx;
    BF_TRY(get_ctx(device, &ctx));
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->budget = bytes;
    return BF_OK;
}

int bf_last_stats(int64_t *candidate_pairs, int64_t *total_pairs, int64_t *tie_pairs,
                  int64_t *n_tiles, int64_t *nonbehind_pairs, double *kernel_ms,
                  int64_t *candidate_pair_segs) {
    materialize_stats();
    const GbsStats &s = g_ps.last;
    if (candidate_pair_segs) *candidate_pair_segs = (int64_t)s.cand_pair_segs;
    if (nonbehind_pairs) *nonbehind_pairs = (int64_t)s.nb_pairs;
    if (kernel_ms) *kernel_ms = (double)s.kernel_ms;
    if (candidate_pairs) *candidate_pairs = (int64_t)s.candidate_pairs;
    if (total_pairs) *total_pairs = g_ps.last_total_pairs;
    if (tie_pairs) *tie_pairs = (int64_t)s.tie_pairs;
    if (n_tiles) *n_tiles = g_ps.last_tiles;
    return BF_OK;
}

int bf_last_pair_stats(int64_t *a9_pairs, int64_t *a9_pair_segs, int64_t *tight_pairs,
                       int64_t *tight_pair_segs, int64_t *live_pairs, int64_t *live_pair_segs) {
    materialize_stats();
    const GbsStats &s = g_ps.last;
    if (a9_pairs) *a9_pairs = (int64_t)s.candidate_pairs;
    if (a9_pair_segs) *a9_pair_segs = (int64_t)s.cand_pair_segs;
    if (tight_pairs) *tight_pairs = (int64_t)s.tight_pairs;
    if (tight_pair_segs) *tight_pair_segs = (int64_t)s.tight_pair_segs;
    if (live_pairs) *live_pairs = (int64_t)s.live_pairs;
    if (live_pair_segs) *live_pair_segs = (int64_t)s.live_pair_segs;
    return BF_OK;
}

int bf_last_path_stats(int64_t *culled, int64_t *single, int64_t *wedge, int64_t *multi) {
    materialize_stats();
    const GbsStats &s = g_ps.last;
    if (culled) *culled = (int64_t)s.paths[0];
    if (single) *single = (int64_t)s.paths[1];
    if (wedge) *wedge = (int64_t)s.paths[2];
    if (multi) *multi = (int64_t)s.paths[3];
    return BF_OK;
}

int bf_gbs_accumulate_dev(const double *seg_origin, const double *seg_dir,
                          const double *seg_e1, const double *seg_e2,
                          const double *seg_len, const double *seg_s0,
                          const double *seg_refl, const int32_t *n_segs, int64_t n_beams,
                          int64_t max_seg, const double *weights, const double *obs,
                          int64_t n_obs, const double *omegas, int64_t nf, double c,
                          double width_b, double phi_amp, int use_cutoff, double *acc,
                          int64_t *evals, int64_t obs_lo, int64_t obs_hi, int64_t beam_lo,
                          int64_t beam_hi, int precision, int flags, int device,
                          void *stream) {
    BF_TRY(validate(n_beams, max_seg, n_obs, nf, obs_lo, obs_hi, beam_lo, beam_hi, precision));
    if (precision == BF_PRECISION_FP64 && (!seg_e1 || !seg_e2))
        return fail(BF_EINVAL, "fp64 mode needs seg_e1/seg_e2");
    DeviceCtx *ctx;
    BF_TRY(get_ctx(device, &ctx));
    std::lock_guard<std::mutex> lk(ctx->mu);
    BF_TRY_CUDA(cudaSetDevice(device));
    CallStream cs(ctx, stream);
    const cudaStream_t st = cs.st;
    BF_TRY(cs.enter());
    StreamOrder order(ctx, st);
    GbsArgs a{};
    const int64_t r0 = beam_lo * max_seg;
    a.seg_origin = seg_origin + 3 * r0;
    a.seg_dir = seg_dir + 3 * r0;
    a.seg_e1 = seg_e1 ? seg_e1 + 3 * r0 : nullptr;
    a.seg_e2 = seg_e2 ? seg_e2 + 3 * r0 : nullptr;
    a.seg_len = seg_len + r0;
    a.seg_s0 = seg_s0 + r0;
    a.seg_refl = seg_refl + r0;
    a.n_segs = n_segs + beam_lo;
    a.weights = weights + beam_lo;
    a.obs = obs + 3 * obs_lo;
    a.max_seg = max_seg;
    a.n_beams = beam_hi - beam_lo;
    a.n_obs = obs_hi - obs_lo;
    a.nf = (int)std::min<int64_t>(nf, BF_MAXF);
    a.c = c;
    a.width_b = width_b;
    a.phi_amp = phi_amp;
    a.use_cutoff = use_cutoff ? 1 : 0;
    a.acc = acc + 2 * obs_lo * nf;
    a.acc_stride = nf;
    a.evals = evals + obs_lo;
    if (precision == BF_PRECISION_FP64) {
        stats_begin(a.n_obs * a.n_beams);
        Tiling t;
        BF_TRY(build_tiling(ctx, a.obs, a.n_obs, (flags & BF_FLAG_OBS_PRESORTED) != 0, st, &t));
        BF_TRY(run_fp64(ctx, a, omegas, nf, t, st));
    } else if (BF_GRAPHS && (double)a.n_obs * (double)a.n_beams <= BF_GRAPH_MAX_PAIRS) {
        BF_TRY(run_fp32_graph(ctx, a, omegas, nf, flags, device, st));
    } else {
        BF_TRY(run_fp32(ctx, a, omegas, nf, false, flags, st));
    }
    return cs.leave();
}

int bf_gbs_accumulate(const double *seg_origin, const double *seg_dir, const double *seg_e1,
                      const double *seg_e2, const double *seg_len, const double *seg_s0,
                      const double *seg_refl, const int32_t *n_segs, int64_t n_beams,
                      int64_t max_seg, const double *weights, const double *obs, int64_t n_obs,
                      const double *omegas, int64_t nf, double c, double width_b,
                      double phi_amp, int use_cutoff, double *acc, int64_t *evals,
                      int64_t obs_lo, int64_t obs_hi, int64_t beam_lo, int64_t beam_hi,
                      int precision, int device) {
    BF_TRY(validate(n_beams, max_seg, n_obs, nf, obs_lo, obs_hi, beam_lo, beam_hi, precision));
    if (precision == BF_PRECISION_FP64 && (!seg_e1 || !seg_e2))
        return fail(BF_EINVAL, "fp64 mode needs seg_e1/seg_e2");
    const int64_t nb = beam_hi - beam_lo, no = obs_hi - obs_lo;
    stats_begin(no * nb);
    if (nb == 0 || no == 0 || nf == 0) return BF_OK;
    DeviceCtx *ctx;
    BF_TRY(get_ctx(device, &ctx));
    std::lock_guard<std::mutex> lk(ctx->mu);
    BF_TRY_CUDA(cudaSetDevice(device));
    cudaStream_t st = ctx->stream;
    StreamOrder order(ctx, st);
    // observers go to the device first (the tiling needs them); the caller's acc/evals
    // rows are only read by the first fold, so they are staged and uploaded while the
    // first beam group sums (fp32) -- or right away (fp64)
    double *d_obs, *d_acc;
    int64_t *d_ev;
    BF_TRY(ctx->get(B_OBS, (size_t)(3 * no), &d_obs));
    BF_TRY(ctx->get(B_ACC, (size_t)(2 * no * nf), &d_acc));
    BF_TRY(ctx->get(B_EVALS, (size_t)no, &d_ev));
    // BF_DEBUG_HOST=1: host-side phase times of this call on stderr (diagnostics only)
    static const bool dbg = getenv("BF_DEBUG_HOST") != nullptr;
    const auto now = [] { return std::chrono::steady_clock::now(); };
    const auto t_a = now();
    cudaEvent_t ev_dbg[3] = {};
    if (dbg) {
        for (auto &e : ev_dbg) cudaEventCreate(&e);
        cudaEventRecord(ev_dbg[0], st);
    }
    BF_TRY(h2d(d_obs, obs + 3 * obs_lo, 24 * (size_t)no, ctx->hpin[H_OBS], st));
    const auto t_b = now();
    bool uploaded = false;
    const std::function<int()> upload_fields = [&]() -> int {
        BF_TRY(h2d(d_acc, acc + 2 * obs_lo * nf, 16 * (size_t)(no * nf), ctx->hpin[H_ACC], st));
        BF_TRY(h2d(d_ev, evals + obs_lo, 8 * (size_t)no, ctx->hpin[H_EV], st));
        uploaded = true;
        return BF_OK;
    };
    GbsArgs a{};
    const int64_t r0 = beam_lo * max_seg;
    a.seg_origin = seg_origin + 3 * r0;
    a.seg_dir = seg_dir + 3 * r0;
    a.seg_e1 = seg_e1 ? seg_e1 + 3 * r0 : nullptr;
    a.seg_e2 = seg_e2 ? seg_e2 + 3 * r0 : nullptr;
    a.seg_len = seg_len + r0;
    a.seg_s0 = seg_s0 + r0;
    a.seg_refl = seg_refl + r0;
    a.n_segs = n_segs + beam_lo;
    a.weights = weights + beam_lo;
    a.obs = d_obs;
    a.max_seg = max_seg;
    a.n_beams = nb;
    a.n_obs = no;
    a.nf = (int)std::min<int64_t>(nf, BF_MAXF);
    a.c = c;
    a.width_b = width_b;
    a.phi_amp = phi_amp;
    a.use_cutoff = use_cutoff ? 1 : 0;
    a.acc = d_acc;
    a.acc_stride = nf;
    a.evals = d_ev;
    if (precision == BF_PRECISION_FP64) {
        BF_TRY(upload_fields());
        BF_TRY(run_fp64_host(ctx, a, omegas, nf, st));
    } else {
        BF_TRY(run_fp32(ctx, a, omegas, nf, true, 0, st, &upload_fields));
    }
    if (!uploaded) BF_TRY(upload_fields());  // (no group ran: acc/evals come back unchanged)
    const auto t_c = now();
    if (dbg) cudaEventRecord(ev_dbg[1], st);
    BF_TRY(d2h_out(ctx, acc + 2 * obs_lo * nf, d_acc, 16 * (size_t)(no * nf), evals + obs_lo,
                   d_ev, 8 * (size_t)no, st));
    if (dbg) {
        const auto t_d = now();
        float gpu_ms = 0.f;
        cudaEventElapsedTime(&gpu_ms, ev_dbg[0], ev_dbg[1]);
        const auto ms = [](auto x, auto y) { return std::chrono::duration<double, std::milli>(y - x).count(); };
        fprintf(stderr, "bf host: obs upload %.2f ms, enqueue groups %.2f ms, wait+copy-out %.2f ms, "
                "total %.2f ms; GPU obs..last fold %.2f ms\n", ms(t_a, t_b), ms(t_b, t_c), ms(t_c, t_d),
                ms(t_a, t_d), gpu_ms);
        for (auto &e : ev_dbg) cudaEventDestroy(e);
    }
    return BF_OK;
}

int bf_rows_create(int device, bf_rows **out) {
    if (!out) return fail(BF_EINVAL, "null output");
    DeviceCtx *ctx;
    BF_TRY(get_ctx(device, &ctx));
    bf_rows *r = new bf_rows();
    r->device = device;
    *out = r;
    return BF_OK;
}

int bf_rows_destroy(bf_rows *rows) {
    if (!rows) return BF_OK;
    DeviceCtx *ctx;
    BF_TRY(get_ctx(rows->device, &ctx));
    std::lock_guard<std::mutex> lk(ctx->mu);
    BF_TRY_CUDA(cudaSetDevice(rows->device));
    if (ctx->done_valid) cudaEventSynchronize(ctx->done);  // no call still reads them
    cudaFree(rows->start);
    cudaFree(rows->p0);
    cudaFree(rows->p1);
    cudaFree(rows->amp);
    delete rows;
    return BF_OK;
}

int bf_rows_info(const bf_rows *rows, int64_t *n_beams, int64_t *n_rows) {
    if (!rows) return fail(BF_EINVAL, "null rows");
    if (n_beams) *n_beams = rows->n_beams;
    if (n_rows) *n_rows = rows->n_rows;
    return BF_OK;
}

int bf_rows_append_dev(bf_rows *rows, const double *seg_origin, const double *seg_dir,
                       const double *seg_len, const double *seg_s0, const double *seg_refl,
                       const int32_t *n_segs, const double *weights, int64_t n_beams,
                       int64_t max_seg, double c, double phi_amp, void *stream) {
    if (!rows) return fail(BF_EINVAL, "null rows");
    if (n_beams < 0 || max_seg < 1) return fail(BF_EINVAL, "bad sizes");
    if (max_seg > BF_FP32_MAX_SEG)
        return fail(BF_EINVAL, "compact rows serve the fp32 path: max_seg <= %d",
                    BF_FP32_MAX_SEG);
    if (rows->n_beams > 0 && (c != rows->c || phi_amp != rows->phi_amp))
        return fail(BF_EINVAL, "appended bundles must share c and amplitude_phi");
    if (n_beams == 0) return BF_OK;
    DeviceCtx *ctx;
    BF_TRY(get_ctx(rows->device, &ctx));
    std::lock_guard<std::mutex> lk(ctx->mu);
    BF_TRY_CUDA(cudaSetDevice(rows->device));
    cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
    StreamOrder order(ctx, st);
    // capacity: exact rows so far + the padded bound of this chunk (grow-only, copied)
    const int64_t need_b = rows->n_beams + n_beams + 1, need_r = rows->n_rows + n_beams * max_seg;
    if (need_b > rows->cap_beams || need_r > rows->cap_rows) {
        const int64_t cb = std::max(need_b, rows->cap_beams + rows->cap_beams / 2);
        const int64_t cr = std::max(need_r, rows->cap_rows + rows->cap_rows / 2);
        int64_t *ns;
        double4 *n0, *n1;
        float *na;
        BF_TRY_CUDA(cudaMalloc(&ns, 8 * (size_t)cb));
        BF_TRY_CUDA(cudaMalloc(&n0, 32 * (size_t)cr));
        BF_TRY_CUDA(cudaMalloc(&n1, 32 * (size_t)cr));
        BF_TRY_CUDA(cudaMalloc(&na, 4 * (size_t)cr));
        if (rows->start) {
            const auto D2D = cudaMemcpyDeviceToDevice;
            BF_TRY_CUDA(cudaMemcpyAsync(ns, rows->start, 8 * (size_t)(rows->n_beams + 1), D2D, st));
            BF_TRY_CUDA(cudaMemcpyAsync(n0, rows->p0, 32 * (size_t)rows->n_rows, D2D, st));
            BF_TRY_CUDA(cudaMemcpyAsync(n1, rows->p1, 32 * (size_t)rows->n_rows, D2D, st));
            BF_TRY_CUDA(cudaMemcpyAsync(na, rows->amp, 4 * (size_t)rows->n_rows, D2D, st));
            BF_TRY_CUDA(cudaStreamSynchronize(st));
            cudaFree(rows->start);
            cudaFree(rows->p0);
            cudaFree(rows->p1);
            cudaFree(rows->amp);
        }
        rows->start = ns;
        rows->p0 = n0;
        rows->p1 = n1;
        rows->amp = na;
        rows->cap_beams = cb;
        rows->cap_rows = cr;
    }
    GbsArgs a{};
    a.seg_origin = seg_origin;
    a.seg_dir = seg_dir;
    a.seg_len = seg_len;
    a.seg_s0 = seg_s0;
    a.seg_refl = seg_refl;
    a.n_segs = n_segs;
    a.weights = weights;
    a.n_beams = n_beams;
    a.max_seg = max_seg;
    a.c = c;
    a.phi_amp = phi_amp;
    int64_t *st0 = rows->start + rows->n_beams;  // entry 0 = rows so far
    BF_TRY(launch_rows_count(n_segs, n_beams, max_seg, rows->n_rows, st0, st));
    size_t tb = 0;
    BF_TRY_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, st0, st0, (int)(n_beams + 1), st));
    void *tmp;
    BF_TRY(ctx->buf[B_CUB].get(tb + 16, &tmp));
    BF_TRY_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, st0, st0, (int)(n_beams + 1), st));
    note_launch();
    BF_TRY(launch_rows_pack(a, st0, rows->p0, rows->p1, rows->amp, st));
    int64_t total = 0;  // the exact row count (the next append's offset): one sync
    BF_TRY_CUDA(cudaMemcpyAsync(&total, st0 + n_beams, 8, cudaMemcpyDeviceToHost, st));
    BF_TRY_CUDA(cudaStreamSynchronize(st));
    rows->n_beams += n_beams;
    rows->n_rows = total;
    rows->max_seg = std::max(rows->max_seg, max_seg);
    rows->c = c;
    rows->phi_amp = phi_amp;
    return BF_OK;
}

int bf_gbs_accumulate_rows_dev(const bf_rows *rows, const double *obs, int64_t n_obs,
                               const double *omegas, int64_t nf, double width_b, int use_cutoff,
                               double *acc, int64_t *evals, int64_t obs_lo, int64_t obs_hi,
                               int64_t beam_lo, int64_t beam_hi, int flags, void *stream) {
    if (!rows) return fail(BF_EINVAL, "null rows");
    BF_TRY(validate(rows->n_beams, std::max<int64_t>(rows->max_seg, 1), n_obs, nf, obs_lo,
                    obs_hi, beam_lo, beam_hi, BF_PRECISION_FP32));
    DeviceCtx *ctx;
    BF_TRY(get_ctx(rows->device, &ctx));
    std::lock_guard<std::mutex> lk(ctx->mu);
    BF_TRY_CUDA(cudaSetDevice(rows->device));
    CallStream cs(ctx, stream);
    const cudaStream_t st = cs.st;
    BF_TRY(cs.enter());
    StreamOrder order(ctx, st);
    GbsArgs a{};
    a.obs = obs + 3 * obs_lo;
    a.max_seg = std::max<int64_t>(rows->max_seg, 1);
    a.n_beams = beam_hi - beam_lo;
    a.n_obs = obs_hi - obs_lo;
    a.nf = (int)std::min<int64_t>(nf, BF_MAXF);
    a.c = rows->c;
    a.width_b = width_b;
    a.phi_amp = rows->phi_amp;
    a.use_cutoff = use_cutoff ? 1 : 0;
    a.acc = acc + 2 * obs_lo * nf;
    a.acc_stride = nf;
    a.evals = evals + obs_lo;
    BF_TRY(run_fp32(ctx, a, omegas, nf, false, flags, st, nullptr, rows, beam_lo));
    return cs.leave();
}

int bf_nearest_on_segments(const double *seg_origin, const double *seg_dir,
                           const double *seg_e1, const double *seg_e2, const double *seg_len,
                           const double *seg_s0, const double *seg_refl, const int32_t *n_segs,
                           int64_t n_beams, int64_t max_seg, const double *obs, int64_t n_obs,
                           const int64_t *q_obs, const int64_t *q_beam, int64_t n_query,
                           double *out, int device) {
    if (max_seg < 1 || n_query < 0) return fail(BF_EINVAL, "bad sizes");
    for (int64_t j = 0; j < n_query; ++j)
        if (q_obs[j] < 0 || q_obs[j] >= n_obs || q_beam[j] < 0 || q_beam[j] >= n_beams)
            return fail(BF_EINVAL, "query %lld out of range", (long long)j);
    if (n_query == 0) return BF_OK;
    DeviceCtx *ctx;
    BF_TRY(get_ctx(device, &ctx));
    std::lock_guard<std::mutex> lk(ctx->mu);
    BF_TRY_CUDA(cudaSetDevice(device));
    cudaStream_t st = ctx->stream;
    StreamOrder order(ctx, st);
    const int64_t rows = n_beams * max_seg;
    double *d_or, *d_dir, *d_e1, *d_e2, *d_len, *d_s0, *d_refl, *d_obs, *d_out;
    int32_t *d_ns;
    int64_t *d_qo, *d_qb;
    BF_TRY(ctx->get(B_ORIGIN, 3 * rows, &d_or));
    BF_TRY(ctx->get(B_DIR, 3 * rows, &d_dir));
    BF_TRY(ctx->get(B_E1, 3 * rows, &d_e1));
    BF_TRY(ctx->get(B_E2, 3 * rows, &d_e2));
    BF_TRY(ctx->get(B_LEN, rows, &d_len));
    BF_TRY(ctx->get(B_S0, rows, &d_s0));
    BF_TRY(ctx->get(B_REFL, rows, &d_refl));
    BF_TRY(ctx->get(B_NSEGS, n_beams, &d_ns));
    BF_TRY(ctx->get(B_OBS, 3 * n_obs, &d_obs));
    BF_TRY(ctx->get(B_QOBS, n_query, &d_qo));
    BF_TRY(ctx->get(B_QBEAM, n_query, &d_qb));
    BF_TRY(ctx->get(B_QOUT, 6 * n_query, &d_out));
    const auto H2D = cudaMemcpyHostToDevice;
    BF_TRY_CUDA(cudaMemcpyAsync(d_or, seg_origin, 24 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_dir, seg_dir, 24 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_e1, seg_e1, 24 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_e2, seg_e2, 24 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_len, seg_len, 8 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_s0, seg_s0, 8 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_refl, seg_refl, 8 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_ns, n_segs, 4 * n_beams, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_obs, obs, 24 * n_obs, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_qo, q_obs, 8 * n_query, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_qb, q_beam, 8 * n_query, H2D, st));
    GbsArgs a{};
    a.seg_origin = d_or;
    a.seg_dir = d_dir;
    a.seg_e1 = d_e1;
    a.seg_e2 = d_e2;
    a.seg_len = d_len;
    a.seg_s0 = d_s0;
    a.seg_refl = d_refl;
    a.n_segs = d_ns;
    a.obs = d_obs;
    a.max_seg = max_seg;
    a.n_beams = n_beams;
    a.n_obs = n_obs;
    BF_TRY(launch_nearest(a, d_qo, d_qb, n_query, d_out, st));
    BF_TRY_CUDA(cudaMemcpyAsync(out, d_out, 48 * n_query, cudaMemcpyDeviceToHost, st));
    BF_TRY_CUDA(cudaStreamSynchronize(st));
    return BF_OK;
}

int bf_trace_range_dev(const double *v0, const double *v1, const double *v2,
                       const double *refl_coef, int64_t n_tri, const double *bounds,
                       double diameter, const double *origin, const double *dirs,
                       const double *e1s, const double *e2s, double length_cap, int64_t r_max,
                       int64_t max_seg, double *seg_origin, double *seg_dir, double *seg_e1,
                       double *seg_e2, double *seg_len, double *seg_s0, double *seg_refl,
                       int32_t *n_segs, int32_t *n_refls, int64_t lo, int64_t hi,
                       int64_t row_base, int flags, int device, void *stream) {
    if (r_max < 0 || max_seg < r_max + 1) return fail(BF_EINVAL, "max_seg must be >= r_max+1");
    if (hi < lo || lo < row_base) return fail(BF_EINVAL, "bad ray range");
    if (n_tri < 0) return fail(BF_EINVAL, "negative triangle count");
    DeviceCtx *ctx;
    BF_TRY(get_ctx(device, &ctx));
    std::lock_guard<std::mutex> lk(ctx->mu);
    BF_TRY_CUDA(cudaSetDevice(device));
    cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
    StreamOrder order(ctx, st);
    // triangle-cluster boxes for the hit search; BF_TRACE_EXHAUSTIVE tests every
    // triangle (the self-check of the culling, same bits)
    double *cbox = nullptr;
    if (n_tri > 0 && !(flags & BF_TRACE_EXHAUSTIVE))
        BF_TRY(ctx->get(B_CBOX, (size_t)(6 * trace_cluster_count(n_tri)), &cbox));
    BF_TRY(launch_trace(v0, v1, v2, refl_coef, n_tri, cbox, bounds, diameter, origin, dirs, e1s, e2s,
                        length_cap, r_max, max_seg, seg_origin, seg_dir, seg_e1, seg_e2, seg_len,
                        seg_s0, seg_refl, n_segs, n_refls, lo, hi, row_base, st));
    if (!stream) BF_TRY_CUDA(cudaStreamSynchronize(st));
    return BF_OK;
}

int bf_field_finalize_dev(const double *acc, int64_t n, double calibration, double *pressure,
                          double *spl, int device, void *stream) {
    if (n < 0) return fail(BF_EINVAL, "negative size");
    DeviceCtx *ctx;
    BF_TRY(get_ctx(device, &ctx));
    BF_TRY_CUDA(cudaSetDevice(device));
    cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
    BF_TRY(launch_finalize(acc, n, calibration, pressure, spl, st));
    if (!stream) BF_TRY_CUDA(cudaStreamSynchronize(st));
    return BF_OK;
}

int bf_tile_size(void) { return gbs_fp32_tile(); }

int bf_worklist(const double *seg_origin, const double *seg_dir, const double *seg_len,
                const double *seg_s0, const int32_t *n_segs, int64_t n_beams, int64_t max_seg,
                const double *obs, int64_t n_obs, const double *omegas, int64_t nf, double c,
                double width_b, int use_cutoff, int32_t *perm, double *centre, double *tile_box,
                uint32_t *bits, uint32_t *tight_bits, int64_t n_tiles_cap, int64_t *n_tiles_out,
                int device) {
    if (max_seg < 1 || n_beams < 1 || n_obs < 1 || nf < 1 || nf > BF_MAXF)
        return fail(BF_EINVAL, "bad sizes");
    const int64_t T = gbs_fp32_tile(), n_tiles = (n_obs + T - 1) / T;
    *n_tiles_out = n_tiles;
    if (n_tiles > n_tiles_cap) return fail(BF_EINVAL, "need %lld tile slots", (long long)n_tiles);
    DeviceCtx *ctx;
    BF_TRY(get_ctx(device, &ctx));
    std::lock_guard<std::mutex> lk(ctx->mu);
    BF_TRY_CUDA(cudaSetDevice(device));
    cudaStream_t st = ctx->stream;
    StreamOrder order(ctx, st);
    const int64_t rows = n_beams * max_seg;
    double *d_or, *d_dir, *d_len, *d_s0, *d_obs, *d_refl, *d_w;
    int32_t *d_ns;
    BF_TRY(ctx->get(B_ORIGIN, 3 * rows, &d_or));
    BF_TRY(ctx->get(B_DIR, 3 * rows, &d_dir));
    BF_TRY(ctx->get(B_LEN, rows, &d_len));
    BF_TRY(ctx->get(B_S0, rows, &d_s0));
    BF_TRY(ctx->get(B_REFL, rows, &d_refl));
    BF_TRY(ctx->get(B_W, n_beams, &d_w));
    BF_TRY(ctx->get(B_NSEGS, n_beams, &d_ns));
    BF_TRY(ctx->get(B_OBS, 3 * n_obs, &d_obs));
    const auto H2D = cudaMemcpyHostToDevice;
    BF_TRY_CUDA(cudaMemcpyAsync(d_or, seg_origin, 24 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_dir, seg_dir, 24 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_len, seg_len, 8 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_s0, seg_s0, 8 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemsetAsync(d_refl, 0, 8 * rows, st));  // amplitudes are not used here
    BF_TRY_CUDA(cudaMemsetAsync(d_w, 0, 8 * n_beams, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_ns, n_segs, 4 * n_beams, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_obs, obs, 24 * n_obs, H2D, st));
    GbsArgs a{};
    a.seg_origin = d_or;
    a.seg_dir = d_dir;
    a.seg_len = d_len;
    a.seg_s0 = d_s0;
    a.seg_refl = d_refl;
    a.weights = d_w;
    a.n_segs = d_ns;
    a.obs = d_obs;
    a.max_seg = max_seg;
    a.n_beams = n_beams;
    a.n_obs = n_obs;
    a.nf = (int)nf;
    for (int f = 0; f < BF_MAXF; ++f) a.omegas[f] = f < nf ? omegas[f] : 0.0;
    a.c = c;
    a.width_b = width_b;
    a.phi_amp = 1.0;
    a.use_cutoff = use_cutoff ? 1 : 0;
    Tiling t;
    BF_TRY(build_tiling(ctx, d_obs, n_obs, false, st, &t));
    Slot &s = ctx->slot[0];
    BF_TRY_CUDA(cudaEventRecord(ctx->pro, st));
    BF_TRY_CUDA(cudaStreamWaitEvent(s.ss, ctx->pro, 0));
    Rows rv;
    BF_TRY(rows_from_device(a, s, &rv));
    const int64_t n_words = (n_beams + 31) / 32;
    uint32_t *d_bits, *d_tbits;
    BF_TRY(ctx->get(B_WLBITS, (size_t)(n_tiles * n_words), &d_bits));
    BF_TRY(ctx->get(B_WLTIGHT, (size_t)(n_tiles * n_words), &d_tbits));
    double wmin = INFINITY;
    for (int f = 0; f < a.nf; ++f) wmin = a.omegas[f] < wmin ? a.omegas[f] : wmin;
    BF_TRY(launch_worklist(a, rv, t.centre, t.tbox, n_tiles, wmin, d_bits, d_tbits, 0, 0, nullptr,
                           nullptr, s.ss));
    BF_TRY_CUDA(cudaEventRecord(s.kdone, s.ss));
    BF_TRY_CUDA(cudaStreamWaitEvent(st, s.kdone, 0));
    const auto D2H = cudaMemcpyDeviceToHost;
    BF_TRY_CUDA(cudaMemcpyAsync(perm, t.perm, 4 * n_obs, D2H, st));
    BF_TRY_CUDA(cudaMemcpyAsync(centre, t.centre, 32 * n_tiles, D2H, st));
    if (tile_box) BF_TRY_CUDA(cudaMemcpyAsync(tile_box, t.tbox, 32 * n_tiles, D2H, st));
    BF_TRY_CUDA(cudaMemcpyAsync(bits, d_bits, 4 * n_tiles * n_words, D2H, st));
    if (tight_bits)
        BF_TRY_CUDA(cudaMemcpyAsync(tight_bits, d_tbits, 4 * n_tiles * n_words, D2H, st));
    BF_TRY_CUDA(cudaStreamSynchronize(st));
    return BF_OK;
}

int bf_tile_order_dev(const double *obs, int64_t n, int32_t *perm, int device, void *stream) {
    if (n < 0 || n > INT32_MAX) return fail(BF_EINVAL, "bad observer count");
    if (n == 0) return BF_OK;
    DeviceCtx *ctx;
    BF_TRY(get_ctx(device, &ctx));
    std::lock_guard<std::mutex> lk(ctx->mu);
    BF_TRY_CUDA(cudaSetDevice(device));
    cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
    StreamOrder order(ctx, st);
    const int32_t *p;
    BF_TRY(hilbert_order(ctx, obs, n, st, &p));
    BF_TRY_CUDA(cudaMemcpyAsync(perm, p, 4 * n, cudaMemcpyDeviceToDevice, st));
    if (!stream) BF_TRY_CUDA(cudaStreamSynchronize(st));
    return BF_OK;
}

int bf_plan_chunks(int64_t total_rays, int64_t memory_budget, int64_t per_ray_bytes,
                   int64_t *chunk_sizes, int64_t max_chunks, int64_t *n_chunks) {
    if (total_rays < 1) return fail(BF_EINVAL, "need at least one ray to plan chunks");
    if (per_ray_bytes <= 0) return fail(BF_EINVAL, "per-ray size must be positive");
    const int64_t cap = memory_budget / per_ray_bytes;  // floor division, budget >= 0
    if (memory_budget < 0 || cap <= 0)
        return fail(BF_EBUDGET, "memory budget %lld cannot hold one ray of %lld bytes",
                    (long long)memory_budget, (long long)per_ray_bytes);
    const int64_t full = total_rays / cap, rem = total_rays % cap;
    const int64_t n = full + (rem ? 1 : 0);
    *n_chunks = n;
    if (n > max_chunks) return fail(BF_EINVAL, "need %lld chunk slots", (long long)n);
    for (int64_t i = 0; i < full; ++i) chunk_sizes[i] = cap;
    if (rem) chunk_sizes[full] = rem;
    return BF_OK;
}

}  // extern "C"
