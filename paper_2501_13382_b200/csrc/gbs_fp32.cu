// gbs_fp32.cu -- the fast GBS summation kernel for sm_100a.
//
// Operator: kernels.gbs_accumulate (kernels.py:352-399) with its helper
// nearest_on_segments (kernels.py:304-349), re-designed for the B200 FP32/MUFU
// pipes:
//
//  * One CTA owns a tile of TILE receivers that are spatially compact (Morton
//    order, engine.cu).  Receivers are held in TILE-LOCAL fp32 coordinates
//    r = p - c_T, so fp32 rounding never sees the ~100 m absolute coordinates.
//  * Beams stream through shared memory in chunks (<= CB beams, <= ROWCAP
//    segment rows).  Staging converts each segment once per tile, in fp64, to
//    tile-local fp32 geometry (wc = c_T - o, d, len, centre projection) plus
//    fp64-exact phase anchors frac(omega/(2 pi c) * s) at the three places the
//    nearest point can sit (segment start, tile-centre projection, segment
//    end).  The per-pair axial phase is anchor + kappa * (r . d) with |r| of a
//    few metres, i.e. fp64-quality where the reference's omega*s/c reaches
//    ~1e3 rad.
//  * Per pair: fp32 nearest-segment scan (strict <, first wins), carrying the
//    best and second-best clamped distance.  If the two are closer than a
//    rigorous fp32 error bound, or the behind test (k==0, proj<0) is within
//    its error bound of 0, the pair is RE-DECIDED in fp64 with the reference
//    operation order and no FMA (__dadd_rn/__dmul_rn) -- corner ties at every
//    reflection point are exact mathematical ties that the reference breaks
//    by fp64 rounding, so only its exact arithmetic reproduces its choice.
//  * Gaussian contribution in fp32 with MUFU ex2 / sin / cos / rcp, partial
//    sums in fp32 per chunk, flushed into per-receiver fp64 accumulators that
//    start from the caller's acc (in-place continuation, kernels.py:358-359).
//    Beams are visited in ascending index order for every receiver.
#include <math.h>

#include "common.cuh"

namespace bf {
namespace {

constexpr int TILE = 256;    // receivers per CTA, one per thread
constexpr int CB = 64;       // max beams per staged chunk
constexpr int ROWCAP = 256;  // max segment rows per staged chunk

struct Fp32Consts {
    float kappa[BF_MAXF];    // omega/(2 pi c), turns per metre
    double kappa64[BF_MAXF];
    float hk[BF_MAXF];       // omega*0.5/c: g = hk*q^2/m2 (kernels.py:382)
    float omega[BF_MAXF];
    float b, b2;             // width_b, width_b^2
    double amp_scale;        // phi*sqrt(c)/(2 pi c)
};

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ double frac_turns(double x) { return x - rint(x); }

// Exact fp64 nearest-segment decision (kernels.py:320-348) for one pair,
// reference operation order, no FMA.  Returns k (or -1), and t, proj, plus the
// perpendicular q^2 of the winner.
struct Exact {
    int k;
    double t, proj, q2;
};
__device__ __noinline__ Exact nearest_exact64(const double *__restrict__ seg_origin,
                                              const double *__restrict__ seg_dir,
                                              const double *__restrict__ seg_len, int64_t base,
                                              int ns, double px, double py, double pz) {
    double best = INFINITY;
    Exact r{-1, 0.0, 0.0, 0.0};
    double bwx = 0, bwy = 0, bwz = 0, bdx = 0, bdy = 0, bdz = 0;
    for (int k = 0; k < ns; ++k) {
        const int64_t row = base + k;
        const double ox = seg_origin[3 * row], oy = seg_origin[3 * row + 1],
                     oz = seg_origin[3 * row + 2];
        const double dx = seg_dir[3 * row], dy = seg_dir[3 * row + 1], dz = seg_dir[3 * row + 2];
        const double wx = __dsub_rn(px, ox), wy = __dsub_rn(py, oy), wz = __dsub_rn(pz, oz);
        const double proj =
            __dadd_rn(__dadd_rn(__dmul_rn(wx, dx), __dmul_rn(wy, dy)), __dmul_rn(wz, dz));
        double t = proj;
        const double len = seg_len[row];
        if (t < 0.0)
            t = 0.0;
        else if (t > len)
            t = len;
        const double vx = __dsub_rn(wx, __dmul_rn(t, dx));
        const double vy = __dsub_rn(wy, __dmul_rn(t, dy));
        const double vz = __dsub_rn(wz, __dmul_rn(t, dz));
        const double d2 =
            __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz));
        if (d2 < best) {
            best = d2;
            r.k = k;
            r.t = t;
            r.proj = proj;
            bwx = wx; bwy = wy; bwz = wz;
            bdx = dx; bdy = dy; bdz = dz;
        }
    }
    const double ux = bwx - r.proj * bdx, uy = bwy - r.proj * bdy, uz = bwz - r.proj * bdz;
    r.q2 = ux * ux + uy * uy + uz * uz;
    return r;
}

template <int NF>
__global__ void __launch_bounds__(TILE, 2)
    gbs_fp32_kernel(const GbsArgs a, const Tiling tl, const int32_t *__restrict__ seg_start,
                    const Fp32Consts K, GbsStats *stats) {
    __shared__ float4 s_g0[ROWCAP];  // wc (= c_T - o), len
    __shared__ float4 s_g1[ROWCAP];  // d, centre projection Pc
    __shared__ float2 s_g2[ROWCAP];  // s0, amplitude factor A
    __shared__ float s_anc[3 * NF][ROWCAP];  // frac(kappa*s) at centre proj / start / end
    __shared__ int s_brow[CB + 1];
    __shared__ float s_bE[CB];
    __shared__ int s_nbc;

    const int tid = threadIdx.x;
    const int64_t tile = blockIdx.x;
    const int64_t si = tile * TILE + tid;
    const bool valid = si < tl.n;
    const double4 cen = tl.centre[tile];
    const float RT = (float)cen.w;

    int oi = 0;
    float rx = 0.f, ry = 0.f, rz = 0.f;
    if (valid) {
        oi = tl.perm[si];
        const float4 rl = tl.rloc[si];
        rx = rl.x;
        ry = rl.y;
        rz = rl.z;
    }
    double acc_re[NF], acc_im[NF];
    float par_re[NF], par_im[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) {
        acc_re[f] = valid ? a.acc[2 * ((int64_t)oi * NF + f)] : 0.0;
        acc_im[f] = valid ? a.acc[2 * ((int64_t)oi * NF + f) + 1] : 0.0;
        par_re[f] = 0.f;
        par_im[f] = 0.f;
    }
    int ev = 0;
    int ties = 0;
    int nbp = 0;
    const int32_t seg_base0 = seg_start[0];

    for (int64_t b0 = 0; b0 < a.n_beams;) {
        // ---- choose the chunk [b0, b0+nbc): <= CB beams and <= ROWCAP rows
        if (tid == 0) {
            int64_t hi = b0 + CB < a.n_beams ? b0 + CB : a.n_beams;
            const int32_t r0 = seg_start[b0];
            while (seg_start[hi] - r0 > ROWCAP) --hi;  // at most CB steps, S <= ROWCAP
            s_nbc = (int)(hi - b0);
        }
        __syncthreads();
        const int nbc = s_nbc;
        for (int j = tid; j <= nbc; j += TILE) s_brow[j] = seg_start[b0 + j] - seg_start[b0];
        __syncthreads();
        const int rows = s_brow[nbc];
        // ---- stage: one thread per segment row, fp64 -> tile-local fp32
        for (int r = tid; r < rows; r += TILE) {
            int lo = 0, hi = nbc;  // s_brow[lo] <= r < s_brow[hi]
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_brow[mid] <= r) lo = mid; else hi = mid;
            }
            const int jb = lo;
            const int k = r - s_brow[jb];
            const int64_t row = (b0 + jb) * a.max_seg + k;
            const double ox = a.seg_origin[3 * row], oy = a.seg_origin[3 * row + 1],
                         oz = a.seg_origin[3 * row + 2];
            const double dx = a.seg_dir[3 * row], dy = a.seg_dir[3 * row + 1],
                         dz = a.seg_dir[3 * row + 2];
            const double len = a.seg_len[row], s0 = a.seg_s0[row];
            const double wcx = cen.x - ox, wcy = cen.y - oy, wcz = cen.z - oz;
            const double pc = wcx * dx + wcy * dy + wcz * dz;
            s_g0[r] = make_float4((float)wcx, (float)wcy, (float)wcz, (float)len);
            s_g1[r] = make_float4((float)dx, (float)dy, (float)dz, (float)pc);
            const double A = K.amp_scale * a.seg_refl[row] * a.weights[b0 + jb];
            s_g2[r] = make_float2((float)s0, (float)A);
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                s_anc[3 * f + 0][r] = (float)frac_turns(K.kappa64[f] * (s0 + pc));
                s_anc[3 * f + 1][r] = (float)frac_turns(K.kappa64[f] * s0);
                s_anc[3 * f + 2][r] = (float)frac_turns(K.kappa64[f] * (s0 + len));
            }
        }
        __syncthreads();
        // Per-beam bound on the fp32 error of any |w - t d|:
        // |dv| <= 2^-18 (R_T + |wc| + len), max over the beam's segments.
        for (int j = tid; j < nbc; j += TILE) {
            float e = 0.f;
            for (int r = s_brow[j]; r < s_brow[j + 1]; ++r) {
                const float4 g = s_g0[r];
                const float m = fabsf(g.x) + fabsf(g.y) + fabsf(g.z) + g.w + RT + 1e-3f;
                e = fmaxf(e, m);
            }
            s_bE[j] = e * 3.814697265625e-06f;  // 2^-18
        }
        __syncthreads();

        // ---- summation over the chunk's beams, ascending
        if (valid) {
            for (int jb = 0; jb < nbc; ++jb) {
                const int r0 = s_brow[jb];
                const int ns = s_brow[jb + 1] - r0;
                if (ns == 0) continue;
                float best = INFINITY, second = INFINITY;
                int kb = 0;
                for (int k = 0; k < ns; ++k) {
                    const float4 g0 = s_g0[r0 + k];
                    const float4 g1 = s_g1[r0 + k];
                    const float wx = rx + g0.x, wy = ry + g0.y, wz = rz + g0.z;
                    const float proj = wx * g1.x + wy * g1.y + wz * g1.z;
                    const float t = fminf(fmaxf(proj, 0.f), g0.w);
                    const float vx = wx - t * g1.x, vy = wy - t * g1.y, vz = wz - t * g1.z;
                    const float d2 = vx * vx + vy * vy + vz * vz;
                    second = fminf(second, fmaxf(best, d2));
                    kb = (d2 < best) ? k : kb;
                    best = fminf(best, d2);
                }
                const float E = s_bE[jb];
                bool need64 = false;
                if (ns > 1) {
                    const float tol = 4.f * sqrtf(second) * E + 2.f * E * E + 1e-6f * second;
                    need64 = (second - best) <= tol;
                }
                float4 g0 = s_g0[r0 + kb];
                float4 g1 = s_g1[r0 + kb];
                float wx = rx + g0.x, wy = ry + g0.y, wz = rz + g0.z;
                float proj = wx * g1.x + wy * g1.y + wz * g1.z;
                if (kb == 0 && fabsf(proj) <= 4.f * E) need64 = true;
                float s, q2;
                int mode;  // 0: interior, 1: clamped at start, 2: clamped at end, 3: fp64 s
                double s64 = 0.0;
                int kw = kb;
                float delta = 0.f;
                if (!need64) {
                    if (kb == 0 && proj < 0.f) continue;  // behind the source
                    const float len = g0.w;
                    const float t = fminf(fmaxf(proj, 0.f), len);
                    s = s_g2[r0 + kb].x + t;
                    const float ux = wx - proj * g1.x, uy = wy - proj * g1.y,
                                uz = wz - proj * g1.z;
                    q2 = ux * ux + uy * uy + uz * uz;
                    if (proj <= 0.f) {
                        mode = 1;
                    } else if (proj >= len) {
                        mode = 2;
                    } else {
                        mode = 0;
                        delta = rx * g1.x + ry * g1.y + rz * g1.z;
                    }
                } else {
                    ++ties;
                    const int64_t gi = 3 * (int64_t)oi;
                    const Exact ex = nearest_exact64(a.seg_origin, a.seg_dir, a.seg_len,
                                                     (b0 + jb) * a.max_seg, ns, a.obs[gi],
                                                     a.obs[gi + 1], a.obs[gi + 2]);
                    if (ex.k == 0 && ex.t == 0.0 && ex.proj < 0.0) continue;  // behind
                    kw = ex.k;
                    const int64_t row = (b0 + jb) * a.max_seg + kw;
                    s64 = a.seg_s0[row] + ex.t;
                    s = (float)s64;
                    q2 = (float)ex.q2;
                    mode = 3;
                }
                ++nbp;
                const float A = s_g2[r0 + kw].y;
                const float m2 = fmaf(s, s, K.b2);
                const float inv = rcp_approx(m2);
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    const float g = K.hk[f] * q2 * inv;
                    const float ex_re = -g * K.b;
                    if (a.use_cutoff && ex_re < (float)BF_CUTOFF_EXPONENT) continue;
                    float base;
                    if (mode == 3)
                        base = (float)frac_turns(K.kappa64[f] * s64);
                    else if (mode == 0)
                        base = fmaf(K.kappa[f], delta, s_anc[3 * f + 0][r0 + kw]);
                    else
                        base = s_anc[3 * f + mode][r0 + kw];
                    float turns = fmaf(g * s, 0.15915494309189535f, base);
                    turns -= rintf(turns);
                    float sn, cs;
                    __sincosf(turns * 6.283185307179586f, &sn, &cs);
                    const float er = ex2_approx(ex_re * 1.4426950408889634f);
                    const float amp = A * K.omega[f] * er * inv;
                    par_re[f] = fmaf(-amp, fmaf(s, sn, K.b * cs), par_re[f]);
                    par_im[f] = fmaf(amp, fmaf(s, cs, -K.b * sn), par_im[f]);
                    ++ev;
                }
            }
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                acc_re[f] += (double)par_re[f];
                acc_im[f] += (double)par_im[f];
                par_re[f] = 0.f;
                par_im[f] = 0.f;
            }
        }
        __syncthreads();
        b0 += nbc;
    }
    (void)seg_base0;
    if (valid) {
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            a.acc[2 * ((int64_t)oi * NF + f)] = acc_re[f];
            a.acc[2 * ((int64_t)oi * NF + f) + 1] = acc_im[f];
        }
        a.evals[oi] += ev;
    }
    // Work-list statistics: tie re-decisions, non-behind pairs (warp-aggregated atomics).
    unsigned long long t = (unsigned long long)ties, q = (unsigned long long)nbp;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        t += __shfl_xor_sync(0xffffffffu, t, o);
        q += __shfl_xor_sync(0xffffffffu, q, o);
    }
    if ((tid & 31) == 0) {
        if (t) atomicAdd(&stats->tie_pairs, t);
        if (q) atomicAdd(&stats->nb_pairs, q);
    }
}

template <int NF>
int launch_nf(const GbsArgs &a, const Tiling &t, const int32_t *seg_start, const Fp32Consts &K,
              GbsStats *stats, cudaStream_t st) {
    gbs_fp32_kernel<NF><<<(unsigned)t.n_tiles, TILE, 0, st>>>(a, t, seg_start, K, stats);
    note_launch();
    BF_TRY_CUDA(cudaGetLastError());
    return BF_OK;
}

}  // namespace

int gbs_fp32_tile() { return TILE; }

int launch_gbs_fp32(const GbsArgs &a, const Tiling &t, const int32_t *seg_start,
                    GbsStats *d_stats, cudaStream_t st) {
    if (t.n <= 0 || a.n_beams <= 0 || a.nf <= 0) return BF_OK;
    if (a.max_seg > ROWCAP) return fail(BF_EINVAL, "max_seg %lld exceeds %d", (long long)a.max_seg, ROWCAP);
    Fp32Consts K;
    const double two_pi = 2.0 * 3.141592653589793;
    for (int f = 0; f < BF_MAXF; ++f) {
        const double w = f < a.nf ? a.omegas[f] : 0.0;
        K.kappa64[f] = w / (two_pi * a.c);
        K.kappa[f] = (float)K.kappa64[f];
        K.hk[f] = (float)(w * 0.5 / a.c);
        K.omega[f] = (float)w;
    }
    K.b = (float)a.width_b;
    K.b2 = (float)(a.width_b * a.width_b);
    K.amp_scale = a.phi_amp * sqrt(a.c) / (two_pi * a.c);
    switch (a.nf) {
        case 1: return launch_nf<1>(a, t, seg_start, K, d_stats, st);
        case 2: return launch_nf<2>(a, t, seg_start, K, d_stats, st);
        case 3: return launch_nf<3>(a, t, seg_start, K, d_stats, st);
        case 4: return launch_nf<4>(a, t, seg_start, K, d_stats, st);
        case 5: return launch_nf<5>(a, t, seg_start, K, d_stats, st);
        case 6: return launch_nf<6>(a, t, seg_start, K, d_stats, st);
        case 7: return launch_nf<7>(a, t, seg_start, K, d_stats, st);
        case 8: return launch_nf<8>(a, t, seg_start, K, d_stats, st);
        default: return fail(BF_EINVAL, "nf=%d outside 1..%d", a.nf, BF_MAXF);
    }
}

}  // namespace bf
