// engine.cu -- device contexts, receiver tiling and the extern "C" ABI.
//
// The ABI (include/bf_gbs.h) is the drop-in boundary for the reference's
// kernels.gbs_accumulate (kernels.py:352-399) and its neighbours; this file
// owns everything between that boundary and the kernels: argument checks that
// mirror the reference's contracts, per-device streams and grow-only
// workspaces, host<->device staging of the caller's ranges, the Hilbert
// receiver tiling used by the fp32 kernel, and the beam segment prefix sums.
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace bf {

namespace {
thread_local char g_err[512] = "";
thread_local GbsStats g_last_stats = {};
thread_local int64_t g_last_total_pairs = 0, g_last_tiles = 0;
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

// Grow-only device buffer.
struct Buf {
    void *p = nullptr;
    size_t cap = 0;
    int get(size_t bytes, void **out) {
        if (bytes > cap) {
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

enum BufId {
    B_ORIGIN, B_DIR, B_E1, B_E2, B_LEN, B_S0, B_REFL, B_NSEGS, B_W, B_OBS, B_ACC, B_EVALS,
    B_SEGSTART, B_KEYS, B_KEYS2, B_VALS, B_VALS2, B_CUB, B_RLOC, B_CENTRE, B_BBOX, B_STATS,
    B_QOBS, B_QBEAM, B_QOUT, B_WLBITS, B_WLCNT, B_P0, B_P1, B_P2, B_PA, B_PRL, B_PCEN,
    B_DONE, B_UCTR, B_WLTIGHT, B_PARTEV, B_WLITEMS, B_WLOFF, B_WLTMP, B_PBOX, B_TBOX, B_UKEYS, B_UKEYS2, B_UVALS, B_UVALS2, B_CBOX, B_COUNT
};

struct DeviceCtx {
    int dev = -1;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // Completion of the last call that used this context's workspaces.  Calls may come
    // on different caller streams and return before their kernels finish; each call
    // orders itself after the previous one (StreamOrder) so no workspace is reused early.
    cudaEvent_t done = nullptr;
    bool done_valid = false;
    cudaStream_t aux = nullptr;              // second stream for the wide-patch kernel
    cudaEvent_t fork = nullptr, join = nullptr;
    std::mutex mu;
    Buf buf[B_COUNT];
    template <typename T>
    int get(BufId id, size_t n, T **out) {
        void *p;
        BF_TRY(buf[id].get(n * sizeof(T) + 16, &p));
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
    }
    ~StreamOrder() {
        if (cudaEventRecord(c->done, st) == cudaSuccess) c->done_valid = true;
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
        BF_TRY_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        BF_TRY_CUDA(cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming));
        BF_TRY_CUDA(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
        BF_TRY_CUDA(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
        BF_TRY_CUDA(cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming));
        g_ctx[device] = c;
    }
    *out = g_ctx[device];
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

template <int T>
__global__ void tile_kernel(const double *obs, int64_t n, const int32_t *perm, float4 *rloc,
                            double4 *centre, double4 *tbox) {
    using BR = cub::BlockReduce<double, T>;
    __shared__ typename BR::TempStorage tmp;
    __shared__ double s_c[3], s_h[3];
    __shared__ float s_r;
    const int64_t si = (int64_t)blockIdx.x * T + threadIdx.x;
    const bool valid = si < n;
    double p[3] = {0, 0, 0};
    if (valid) {
        const int64_t oi = perm[si];
        for (int d = 0; d < 3; ++d) p[d] = obs[3 * oi + d];
    }
    for (int d = 0; d < 3; ++d) {
        const double mn = BR(tmp).Reduce(valid ? p[d] : INFINITY, cub::Min());
        __syncthreads();
        const double mx = BR(tmp).Reduce(valid ? p[d] : -INFINITY, cub::Max());
        __syncthreads();
        if (threadIdx.x == 0) {
            s_c[d] = 0.5 * (mn + mx);
            s_h[d] = 0.5 * (mx - mn);
        }
    }
    __syncthreads();
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid) {
        r.x = (float)(p[0] - s_c[0]);
        r.y = (float)(p[1] - s_c[1]);
        r.z = (float)(p[2] - s_c[2]);
        rloc[si] = r;
    }
    const double rad = valid ? sqrt((double)r.x * r.x + (double)r.y * r.y + (double)r.z * r.z) : 0.0;
    const double rmax = BR(tmp).Reduce(rad, cub::Max());
    if (threadIdx.x == 0) s_r = (float)rmax;
    __syncthreads();
    if (threadIdx.x == 0) {
        centre[blockIdx.x] = make_double4(s_c[0], s_c[1], s_c[2], (double)s_r);
        tbox[blockIdx.x] = make_double4(s_h[0], s_h[1], s_h[2], (double)s_r);
    }
}

__global__ void iota_kernel(int32_t *v, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = (int32_t)i;
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
    const int32_t *perm;
    if (presorted) {
        int32_t *id;
        BF_TRY(c->get(B_VALS, n, &id));
        iota_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(id, n);
        note_launch();
        perm = id;
    } else {
        BF_TRY(hilbert_order(c, obs, n, st, &perm));
    }
    if (T == 512)
        tile_kernel<512><<<(unsigned)out->n_tiles, 512, 0, st>>>(obs, n, perm, rloc, cen, box);
    else if (T == 256)
        tile_kernel<256><<<(unsigned)out->n_tiles, 256, 0, st>>>(obs, n, perm, rloc, cen, box);
    else if (T == 1024)
        tile_kernel<1024><<<(unsigned)out->n_tiles, 1024, 0, st>>>(obs, n, perm, rloc, cen, box);
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
    if (nf < 0 || nf > BF_MAXF) return fail(BF_EINVAL, "nf=%lld outside 0..%d", (long long)nf, BF_MAXF);
    if (obs_lo < 0 || obs_hi < obs_lo || obs_hi > n_obs)
        return fail(BF_EINVAL, "observer range [%lld,%lld) outside [0,%lld)", (long long)obs_lo,
                    (long long)obs_hi, (long long)n_obs);
    if (beam_lo < 0 || beam_hi < beam_lo || beam_hi > n_beams)
        return fail(BF_EINVAL, "beam range [%lld,%lld) outside [0,%lld)", (long long)beam_lo,
                    (long long)beam_hi, (long long)n_beams);
    if (precision != BF_PRECISION_FP32 && precision != BF_PRECISION_FP64)
        return fail(BF_EINVAL, "unknown precision %d", precision);
    return BF_OK;
}

// Tile-level work list (exact fp64 candidate test, exact_fp64.cu) for tiling t.
// counts (n_tiles x n_ranges, zeroed) and wstats (4 x n_tiles, zeroed) may be null; else
// the work-list kernel also adds the tight candidates per (tile, beam range) and the
// per-tile statistics there.
int build_worklist(DeviceCtx *c, const GbsArgs &a, Tiling &t, cudaStream_t st,
                   int64_t range_beams = 0, int64_t n_ranges = 0,
                   unsigned long long *counts = nullptr, unsigned long long *wstats = nullptr) {
    const int64_t n_words = (a.n_beams + 31) / 32;
    uint32_t *bits, *tbits;
    BF_TRY(c->get(B_WLBITS, (size_t)(t.n_tiles * n_words), &bits));
    BF_TRY(c->get(B_WLTIGHT, (size_t)(t.n_tiles * n_words), &tbits));
    double wmin = INFINITY;
    for (int f = 0; f < a.nf; ++f) wmin = a.omegas[f] < wmin ? a.omegas[f] : wmin;
    BF_TRY(launch_worklist(a, t.centre, t.tbox, t.n_tiles, wmin, bits, tbits, range_beams,
                           n_ranges, counts, wstats, st));
    t.wl_bits = bits;
    t.wl_tight = tbits;
    t.wl_words = n_words;
    return BF_OK;
}

// Runs the operator on device-resident LOCAL ranges (a.obs etc. already offset).
int run_gbs(DeviceCtx *c, GbsArgs &a, int precision, int flags, cudaStream_t st) {
    g_last_stats = GbsStats{};
    g_last_total_pairs = a.n_obs * a.n_beams;
    g_last_tiles = 0;
    if (a.n_obs <= 0 || a.n_beams <= 0 || a.nf <= 0) return BF_OK;
    if (precision == BF_PRECISION_FP64) return launch_gbs_fp64(a, st);
    Tiling t;
    BF_TRY(build_tiling(c, a.obs, a.n_obs, (flags & BF_FLAG_OBS_PRESORTED) != 0, st, &t));
    Fp32Work w{};
    const int64_t rows = a.n_beams * a.max_seg;
    const int P = gbs_fp32_patch();
    w.n_patches = (a.n_obs + P - 1) / P;
    w.range_beams = gbs_fp32_range_beams(a.n_beams, a.nf);
    w.n_ranges = (a.n_beams + w.range_beams - 1) / w.range_beams;
    if (w.n_patches * w.n_ranges >= (int64_t)1 << 31)
        return fail(BF_EINVAL, "too many (patch, beam range) units; split the call");
    if (a.n_beams >= ((int64_t)1 << 27))
        return fail(BF_EINVAL, "more than 2^27 beams in one call; split the beam range");
    BF_TRY(c->get(B_P0, rows, &w.p0));
    BF_TRY(c->get(B_P1, rows, &w.p1));
    BF_TRY(c->get(B_P2, rows, &w.p2));
    BF_TRY(c->get(B_PA, 2 * rows * a.nf, &w.pa));
    BF_TRY(c->get(B_PRL, a.n_obs, &w.prl));
    BF_TRY(c->get(B_PCEN, w.n_patches, &w.pcen));
    BF_TRY(c->get(B_PBOX, w.n_patches, &w.pbox));
    w.n_pad = w.n_patches * P;
    BF_TRY(c->get(B_DONE, (size_t)(w.n_ranges * w.n_pad * a.nf), &w.part));
    BF_TRY(c->get(B_PARTEV, (size_t)(w.n_ranges * w.n_pad), &w.part_ev));
    BF_TRY(c->get(B_UCTR, 3, &w.unit_ctr));
    w.n_wide = w.unit_ctr + 2;
    BF_TRY_CUDA(cudaMemsetAsync(w.unit_ctr, 0, 3 * sizeof(unsigned), st));
    {   // wide patches (fp64 tail, see unit_keys_kernel): kappa_max RW > 16 turns or
        // omega_max RW^2 / (2 c b) > 200 (the fp32 error of r.d and q^2 grows with RW;
        // at these bounds it stays ~5x below the 0.01 dB gate at 50 dB below the maximum)
        double wmax = 0.0;
        for (int f = 0; f < a.nf; ++f) wmax = a.omegas[f] > wmax ? a.omegas[f] : wmax;
        const char *ek = getenv("BF_WIDE_TURNS"), *eq = getenv("BF_WIDE_Q");  // tuning
        const double lk = ek ? atof(ek) : 16.0, lq = eq ? atof(eq) : 200.0;
        w.wide_k = (float)(wmax / (2.0 * 3.141592653589793 * a.c) / lk);
        w.wide_q = (float)(wmax / (2.0 * a.c * a.width_b) / lq);
    }
    unsigned long long *d_cand;  // per tile: a9 beams, a9 segments, tight beams, tight segments
    BF_TRY(c->get(B_WLCNT, (size_t)(4 * t.n_tiles), &d_cand));
    BF_TRY_CUDA(cudaMemsetAsync(d_cand, 0, 4 * sizeof(unsigned long long) * t.n_tiles, st));
    const int64_t nu_wl = t.n_tiles * w.n_ranges;
    int64_t *cnt;
    {   // tight work list counts (from the work-list kernel) -> exclusive scan
        BF_TRY(c->get(B_WLTMP, (size_t)(nu_wl + 1), &cnt));
        BF_TRY(c->get(B_WLOFF, (size_t)(nu_wl + 1), &w.wl_off));
        BF_TRY_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (nu_wl + 1), st));
        BF_TRY(build_worklist(c, a, t, st, w.range_beams, w.n_ranges,
                              reinterpret_cast<unsigned long long *>(cnt), d_cand));
        size_t tmp_bytes = 0;
        BF_TRY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, w.wl_off,
                                                  (int)(nu_wl + 1), st));
        void *tmp;
        BF_TRY(c->buf[B_CUB].get(tmp_bytes + 16, &tmp));
        BF_TRY_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, w.wl_off,
                                                  (int)(nu_wl + 1), st));
        note_launch();
    }
    BF_TRY(launch_fp32_prepare(a, t, w, st));
    {   // unit queue order (wide patches last; longest-first buckets, range-major inside
        // a bucket) from the counts and the patch radii of launch_fp32_prepare
        const int64_t nu = w.n_patches * w.n_ranges;
        uint64_t *k0, *k1;
        int32_t *v0, *v1;
        BF_TRY(c->get(B_UKEYS, (size_t)nu, &k0));
        BF_TRY(c->get(B_UKEYS2, (size_t)nu, &k1));
        BF_TRY(c->get(B_UVALS, (size_t)nu, &v0));
        BF_TRY(c->get(B_UVALS2, (size_t)nu, &v1));
        BF_TRY(launch_fp32_unit_keys(t, w, cnt, k0, v0, st));
        const int end_bit = 40;  // wide << 39 | bucket (7 bits) << 32 | range
        cub::DoubleBuffer<uint64_t> dk(k0, k1);
        cub::DoubleBuffer<int32_t> dv(v0, v1);
        size_t tmp_bytes = 0;
        BF_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dk, dv, (int)nu, 0,
                                                    end_bit, st));
        void *tmp;
        BF_TRY(c->buf[B_CUB].get(tmp_bytes + 16, &tmp));
        BF_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, dk, dv, (int)nu, 0,
                                                    end_bit, st));
        note_launch();
        w.unit_order = dv.Current();
    }
    {   // one host sync: work-list length (buffer size) and wide-unit count (launches)
        int64_t total = 0;
        unsigned n_wide = 0;
        BF_TRY_CUDA(cudaMemcpyAsync(&total, w.wl_off + nu_wl, sizeof(int64_t),
                                    cudaMemcpyDeviceToHost, st));
        BF_TRY_CUDA(cudaMemcpyAsync(&n_wide, w.n_wide, sizeof(unsigned), cudaMemcpyDeviceToHost,
                                    st));
        BF_TRY_CUDA(cudaStreamSynchronize(st));
        w.n_wide_host = n_wide;
        BF_TRY(c->get(B_WLITEMS, (size_t)(total + 1), &w.wl_items));
        BF_TRY(launch_fp32_wl_compact(a, t, w, st));
    }
    GbsStats *d_stats;
    BF_TRY(c->get(B_STATS, 1, &d_stats));
    BF_TRY_CUDA(cudaMemsetAsync(d_stats, 0, sizeof(GbsStats), st));
    if (!c->ev0) {
        BF_TRY_CUDA(cudaEventCreate(&c->ev0));
        BF_TRY_CUDA(cudaEventCreate(&c->ev1));
    }
    BF_TRY_CUDA(cudaEventRecord(c->ev0, st));
    BF_TRY(launch_gbs_fp32(a, t, w, d_stats, StreamPair{st, c->aux, c->fork, c->join}));
    BF_TRY_CUDA(cudaEventRecord(c->ev1, st));
    GbsStats h;
    BF_TRY_CUDA(cudaMemcpyAsync(&h, d_stats, sizeof(GbsStats), cudaMemcpyDeviceToHost, st));
    BF_TRY_CUDA(cudaStreamSynchronize(st));
    BF_TRY_CUDA(cudaEventElapsedTime(&h.kernel_ms, c->ev0, c->ev1));
    std::vector<unsigned long long> cand((size_t)(4 * t.n_tiles));
    BF_TRY_CUDA(cudaMemcpy(cand.data(), d_cand, 4 * sizeof(unsigned long long) * t.n_tiles,
                           cudaMemcpyDeviceToHost));
    unsigned long long cp = 0, cs = 0, tp = 0, ts = 0;
    for (int64_t i = 0; i < t.n_tiles; ++i) {
        const unsigned long long in_tile =
            (unsigned long long)((i + 1 < t.n_tiles) ? t.tile : a.n_obs - i * t.tile);
        cp += cand[(size_t)i] * in_tile;
        cs += cand[(size_t)(t.n_tiles + i)] * in_tile;
        tp += cand[(size_t)(2 * t.n_tiles + i)] * in_tile;
        ts += cand[(size_t)(3 * t.n_tiles + i)] * in_tile;
    }
    h.candidate_pairs = cp;
    h.cand_pair_segs = cs;
    h.tight_pairs = tp;
    h.tight_pair_segs = ts;
    g_last_stats = h;
    if (getenv("BF_DEBUG_STATS")) {
        unsigned nw = 0;
        cudaMemcpy(&nw, w.n_wide, sizeof(unsigned), cudaMemcpyDeviceToHost);
        fprintf(stderr, "bf units: %lld, of wide patches %u\n",
                (long long)(w.n_patches * w.n_ranges), nw);
    }
    if (getenv("BF_DEBUG_STATS"))
        fprintf(stderr, "bf stats: items culled %llu single %llu wedge %llu multi %llu "
                "(surv 2:%llu 3:%llu 4:%llu 5+:%llu) ties %llu\n", h.paths[0], h.paths[1],
                h.paths[2], h.paths[3], h.multi_surv[0], h.multi_surv[1], h.multi_surv[2],
                h.multi_surv[3], h.tie_pairs);
    g_last_tiles = t.n_tiles;
    return BF_OK;
}

}  // namespace
}  // namespace bf

using namespace bf;

extern "C" {

const char *bf_version(void) { return "paper_2501_13382_b200 0.1.0 (sm_100a)"; }

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

int bf_last_stats(int64_t *candidate_pairs, int64_t *total_pairs, int64_t *tie_pairs,
                  int64_t *n_tiles, int64_t *nonbehind_pairs, double *kernel_ms,
                  int64_t *candidate_pair_segs) {
    if (candidate_pair_segs) *candidate_pair_segs = (int64_t)g_last_stats.cand_pair_segs;
    if (nonbehind_pairs) *nonbehind_pairs = (int64_t)g_last_stats.nb_pairs;
    if (kernel_ms) *kernel_ms = (double)g_last_stats.kernel_ms;
    if (candidate_pairs) *candidate_pairs = (int64_t)g_last_stats.candidate_pairs;
    if (total_pairs) *total_pairs = g_last_total_pairs;
    if (tie_pairs) *tie_pairs = (int64_t)g_last_stats.tie_pairs;
    if (n_tiles) *n_tiles = g_last_tiles;
    return BF_OK;
}

int bf_last_pair_stats(int64_t *a9_pairs, int64_t *a9_pair_segs, int64_t *tight_pairs,
                       int64_t *tight_pair_segs, int64_t *live_pairs, int64_t *live_pair_segs) {
    if (a9_pairs) *a9_pairs = (int64_t)g_last_stats.candidate_pairs;
    if (a9_pair_segs) *a9_pair_segs = (int64_t)g_last_stats.cand_pair_segs;
    if (tight_pairs) *tight_pairs = (int64_t)g_last_stats.tight_pairs;
    if (tight_pair_segs) *tight_pair_segs = (int64_t)g_last_stats.tight_pair_segs;
    if (live_pairs) *live_pairs = (int64_t)g_last_stats.live_pairs;
    if (live_pair_segs) *live_pair_segs = (int64_t)g_last_stats.live_pair_segs;
    return BF_OK;
}

int bf_last_path_stats(int64_t *culled, int64_t *single, int64_t *wedge, int64_t *multi) {
    if (culled) *culled = (int64_t)g_last_stats.paths[0];
    if (single) *single = (int64_t)g_last_stats.paths[1];
    if (wedge) *wedge = (int64_t)g_last_stats.paths[2];
    if (multi) *multi = (int64_t)g_last_stats.paths[3];
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
    DeviceCtx *ctx;
    BF_TRY(get_ctx(device, &ctx));
    std::lock_guard<std::mutex> lk(ctx->mu);
    BF_TRY_CUDA(cudaSetDevice(device));
    cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
    StreamOrder order(ctx, st);
    GbsArgs a;
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
    a.nf = (int)nf;
    for (int f = 0; f < BF_MAXF; ++f) a.omegas[f] = f < nf ? omegas[f] : 0.0;
    a.c = c;
    a.width_b = width_b;
    a.phi_amp = phi_amp;
    a.use_cutoff = use_cutoff ? 1 : 0;
    a.acc = acc + 2 * obs_lo * nf;
    a.evals = evals + obs_lo;
    if (precision == BF_PRECISION_FP64 && (!seg_e1 || !seg_e2))
        return fail(BF_EINVAL, "fp64 mode needs seg_e1/seg_e2");
    BF_TRY(run_gbs(ctx, a, precision, flags, st));
    if (!stream) BF_TRY_CUDA(cudaStreamSynchronize(st));
    return BF_OK;
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
    const int64_t nb = beam_hi - beam_lo, no = obs_hi - obs_lo;
    if (nb == 0 || no == 0 || nf == 0) return BF_OK;
    DeviceCtx *ctx;
    BF_TRY(get_ctx(device, &ctx));
    std::lock_guard<std::mutex> lk(ctx->mu);
    BF_TRY_CUDA(cudaSetDevice(device));
    cudaStream_t st = ctx->stream;
    StreamOrder order(ctx, st);
    const bool need_frame = precision == BF_PRECISION_FP64;
    const int64_t rows = nb * max_seg, r0 = beam_lo * max_seg;
    double *d_or, *d_dir, *d_e1 = nullptr, *d_e2 = nullptr, *d_len, *d_s0, *d_refl, *d_w, *d_obs,
                                *d_acc;
    int32_t *d_ns;
    int64_t *d_ev;
    BF_TRY(ctx->get(B_ORIGIN, 3 * rows, &d_or));
    BF_TRY(ctx->get(B_DIR, 3 * rows, &d_dir));
    if (need_frame) {
        BF_TRY(ctx->get(B_E1, 3 * rows, &d_e1));
        BF_TRY(ctx->get(B_E2, 3 * rows, &d_e2));
    }
    BF_TRY(ctx->get(B_LEN, rows, &d_len));
    BF_TRY(ctx->get(B_S0, rows, &d_s0));
    BF_TRY(ctx->get(B_REFL, rows, &d_refl));
    BF_TRY(ctx->get(B_NSEGS, nb, &d_ns));
    BF_TRY(ctx->get(B_W, nb, &d_w));
    BF_TRY(ctx->get(B_OBS, 3 * no, &d_obs));
    BF_TRY(ctx->get(B_ACC, 2 * no * nf, &d_acc));
    BF_TRY(ctx->get(B_EVALS, no, &d_ev));
    const auto H2D = cudaMemcpyHostToDevice;
    BF_TRY_CUDA(cudaMemcpyAsync(d_or, seg_origin + 3 * r0, 24 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_dir, seg_dir + 3 * r0, 24 * rows, H2D, st));
    if (need_frame) {
        BF_TRY_CUDA(cudaMemcpyAsync(d_e1, seg_e1 + 3 * r0, 24 * rows, H2D, st));
        BF_TRY_CUDA(cudaMemcpyAsync(d_e2, seg_e2 + 3 * r0, 24 * rows, H2D, st));
    }
    BF_TRY_CUDA(cudaMemcpyAsync(d_len, seg_len + r0, 8 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_s0, seg_s0 + r0, 8 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_refl, seg_refl + r0, 8 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_ns, n_segs + beam_lo, 4 * nb, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_w, weights + beam_lo, 8 * nb, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_obs, obs + 3 * obs_lo, 24 * no, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_acc, acc + 2 * obs_lo * nf, 16 * no * nf, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_ev, evals + obs_lo, 8 * no, H2D, st));
    GbsArgs a;
    a.seg_origin = d_or;
    a.seg_dir = d_dir;
    a.seg_e1 = d_e1;
    a.seg_e2 = d_e2;
    a.seg_len = d_len;
    a.seg_s0 = d_s0;
    a.seg_refl = d_refl;
    a.n_segs = d_ns;
    a.weights = d_w;
    a.obs = d_obs;
    a.max_seg = max_seg;
    a.n_beams = nb;
    a.n_obs = no;
    a.nf = (int)nf;
    for (int f = 0; f < BF_MAXF; ++f) a.omegas[f] = f < nf ? omegas[f] : 0.0;
    a.c = c;
    a.width_b = width_b;
    a.phi_amp = phi_amp;
    a.use_cutoff = use_cutoff ? 1 : 0;
    a.acc = d_acc;
    a.evals = d_ev;
    BF_TRY(run_gbs(ctx, a, precision, 0, st));
    const auto D2H = cudaMemcpyDeviceToHost;
    BF_TRY_CUDA(cudaMemcpyAsync(acc + 2 * obs_lo * nf, d_acc, 16 * no * nf, D2H, st));
    BF_TRY_CUDA(cudaMemcpyAsync(evals + obs_lo, d_ev, 8 * no, D2H, st));
    BF_TRY_CUDA(cudaStreamSynchronize(st));
    return BF_OK;
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
                       int64_t row_base, int device, void *stream) {
    if (r_max < 0 || max_seg < r_max + 1) return fail(BF_EINVAL, "max_seg must be >= r_max+1");
    if (hi < lo || lo < row_base) return fail(BF_EINVAL, "bad ray range");
    if (n_tri < 0) return fail(BF_EINVAL, "negative triangle count");
    DeviceCtx *ctx;
    BF_TRY(get_ctx(device, &ctx));
    std::lock_guard<std::mutex> lk(ctx->mu);
    BF_TRY_CUDA(cudaSetDevice(device));
    cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
    StreamOrder order(ctx, st);
    // triangle-cluster boxes for the hit search; BF_TRACE_EXHAUSTIVE=1 tests every
    // triangle (the self-check of the culling, same bits)
    double *cbox = nullptr;
    const char *ex = getenv("BF_TRACE_EXHAUSTIVE");
    if (n_tri > 0 && !(ex && ex[0] == '1'))
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
    std::lock_guard<std::mutex> lk(ctx->mu);
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
    double *d_or, *d_dir, *d_len, *d_s0, *d_obs;
    int32_t *d_ns;
    BF_TRY(ctx->get(B_ORIGIN, 3 * rows, &d_or));
    BF_TRY(ctx->get(B_DIR, 3 * rows, &d_dir));
    BF_TRY(ctx->get(B_LEN, rows, &d_len));
    BF_TRY(ctx->get(B_S0, rows, &d_s0));
    BF_TRY(ctx->get(B_NSEGS, n_beams, &d_ns));
    BF_TRY(ctx->get(B_OBS, 3 * n_obs, &d_obs));
    const auto H2D = cudaMemcpyHostToDevice;
    BF_TRY_CUDA(cudaMemcpyAsync(d_or, seg_origin, 24 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_dir, seg_dir, 24 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_len, seg_len, 8 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_s0, seg_s0, 8 * rows, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_ns, n_segs, 4 * n_beams, H2D, st));
    BF_TRY_CUDA(cudaMemcpyAsync(d_obs, obs, 24 * n_obs, H2D, st));
    GbsArgs a{};
    a.seg_origin = d_or;
    a.seg_dir = d_dir;
    a.seg_len = d_len;
    a.seg_s0 = d_s0;
    a.n_segs = d_ns;
    a.obs = d_obs;
    a.max_seg = max_seg;
    a.n_beams = n_beams;
    a.n_obs = n_obs;
    a.nf = (int)nf;
    for (int f = 0; f < BF_MAXF; ++f) a.omegas[f] = f < nf ? omegas[f] : 0.0;
    a.c = c;
    a.width_b = width_b;
    a.use_cutoff = use_cutoff ? 1 : 0;
    Tiling t;
    BF_TRY(build_tiling(ctx, d_obs, n_obs, false, st, &t));
    BF_TRY(build_worklist(ctx, a, t, st));
    const int64_t n_words = (n_beams + 31) / 32;
    const auto D2H = cudaMemcpyDeviceToHost;
    BF_TRY_CUDA(cudaMemcpyAsync(perm, t.perm, 4 * n_obs, D2H, st));
    BF_TRY_CUDA(cudaMemcpyAsync(centre, t.centre, 32 * n_tiles, D2H, st));
    if (tile_box) BF_TRY_CUDA(cudaMemcpyAsync(tile_box, t.tbox, 32 * n_tiles, D2H, st));
    BF_TRY_CUDA(cudaMemcpyAsync(bits, t.wl_bits, 4 * n_tiles * n_words, D2H, st));
    if (tight_bits)
        BF_TRY_CUDA(cudaMemcpyAsync(tight_bits, t.wl_tight, 4 * n_tiles * n_words, D2H, st));
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
