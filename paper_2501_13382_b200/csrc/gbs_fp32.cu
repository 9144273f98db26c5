// gbs_fp32.cu -- the fast GBS summation kernel for sm_100a.
//
// Operator: kernels.gbs_accumulate (kernels.py:352-399) with its helper
// nearest_on_segments (kernels.py:304-349), re-designed for the B200 FP32/MUFU
// pipes.  DESIGN.md holds the error analysis behind every tolerance here.
//
//  * One CTA owns a tile of TILE = THREADS x R receivers, spatially compact
//    (Morton order, engine.cu); thread t holds receivers R*t..R*t+R-1, so a
//    warp covers 128 consecutive Morton receivers (a compact patch).
//    Receivers are held in TILE-LOCAL fp32 coordinates r = p - c_T.
//  * Beams stream through shared memory in chunks (<= CB beams, <= ROWCAP
//    segment rows).  Staging converts each segment once per tile, in fp64, to
//    tile-local fp32 geometry (wc = c_T - o, d, len, centre projection Pc),
//    the cutoff radius of the segment, fp64-exact phase anchors
//    frac(omega/(2 pi c) * s) at the segment start / tile-centre projection /
//    end, and keeps the fp64 row for exact re-decisions.
//  * Per (warp, beam) a lane-parallel prepass (one lane per segment) bounds
//    the warp patch against every segment: if every segment is provably cut
//    (q_perp - R_W > R_cut) or, for segment 0, entirely behind the source,
//    the beam is skipped for the warp; segments whose distance to the patch
//    exceeds the nearest one by more than the patch diameter can never be
//    the nearest point and are pruned.  Usually ONE segment survives and the
//    pair needs no nearest-segment scan at all.
//  * Several survivors: fp32 scan (strict <, first wins) carrying best and
//    second-best clamped distance.  If the two are within the fp32 error
//    bound -- corner ties at every reflection point are exact mathematical
//    ties that the reference breaks by fp64 rounding -- the contenders are
//    re-decided in fp64 with the reference operation order and no FMA.  The
//    behind test (k==0, proj<0) is re-decided in fp64 the same way when
//    |proj| is within its error bound.
//  * Gaussian contribution in fp32 with MUFU ex2 / sin / cos / rcp, fp32
//    partial sums per chunk flushed into per-receiver fp64 accumulators (in
//    shared memory) that start from the caller's acc (in-place continuation,
//    kernels.py:358-359).  Beams are visited in ascending order per receiver.
#include <math.h>

#include "common.cuh"

namespace bf {
namespace {

#ifndef BF_CB
#define BF_CB 32
#endif
#ifndef BF_ROWCAP
#define BF_ROWCAP 128
#endif
#ifndef BF_MINB
#define BF_MINB 5
#endif
constexpr int THREADS = 128;
constexpr int R = 4;                    // receivers per thread
constexpr int TILE = THREADS * R;       // receivers per CTA
constexpr int CB = BF_CB;               // max beams per staged chunk
constexpr int ROWCAP = BF_ROWCAP;       // max segment rows per staged chunk
constexpr float TIE_REL = 3.0517578125e-05f;        // 2^-15 (x d2)
constexpr float TIE_ABS = 1.1920928955078125e-07f;  // 2^-23 (x D^2)
constexpr float PROJ_ERR = 3.814697265625e-06f;     // 2^-18 (x D): bound on |fp32 proj error|

struct Fp32Consts {
    float kappa[BF_MAXF];    // omega/(2 pi c), turns per metre
    double kappa64[BF_MAXF];
    float hk[BF_MAXF];       // omega*0.5/c: g = hk*q^2/m2 (kernels.py:382)
    float omega[BF_MAXF];
    float cutk[BF_MAXF];     // omega*b/(72 c): pair cut iff q^2*cutk > m2 (ex_re < -36)
    float hk2pi[BF_MAXF];    // hk/(2 pi): g*s in turns = (q^2/m2)*s*hk2pi
    float nhkbl2e[BF_MAXF];  // -hk*b*log2(e): exp(-g b) = ex2((q^2/m2)*nhkbl2e)
    float b, b2;             // width_b, width_b^2
    double amp_scale;        // phi*sqrt(c)/(2 pi c)
    double rcut_scale;       // 72 c / (omega_min b): R_cut^2 = rcut_scale * (s_end^2 + b^2)
    double b2_64;
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
__device__ __forceinline__ float sin_approx(float x) {
    float y;
    asm("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float cos_approx(float x) {
    float y;
    asm("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ double frac_turns(double x) { return x - rint(x); }

// Exact fp64 clamped distance of kernels.py:328-340 for padded row `row`,
// reference operation order, no FMA.
__device__ __forceinline__ double exact_d2(const GbsArgs &a, int64_t row, double px, double py,
                                           double pz, double *proj_out, double *t_out) {
    const double ox = a.seg_origin[3 * row], oy = a.seg_origin[3 * row + 1],
                 oz = a.seg_origin[3 * row + 2];
    const double dx = a.seg_dir[3 * row], dy = a.seg_dir[3 * row + 1], dz = a.seg_dir[3 * row + 2];
    const double len = a.seg_len[row];
    const double wx = __dsub_rn(px, ox), wy = __dsub_rn(py, oy), wz = __dsub_rn(pz, oz);
    const double proj =
        __dadd_rn(__dadd_rn(__dmul_rn(wx, dx), __dmul_rn(wy, dy)), __dmul_rn(wz, dz));
    double t = proj;
    if (t < 0.0)
        t = 0.0;
    else if (t > len)
        t = len;
    const double vx = __dsub_rn(wx, __dmul_rn(t, dx));
    const double vy = __dsub_rn(wy, __dmul_rn(t, dy));
    const double vz = __dsub_rn(wz, __dmul_rn(t, dz));
    *proj_out = proj;
    *t_out = t;
    return __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz));
}

constexpr int NWARPS = THREADS / 32;   // consumer warps (receiver patches)

constexpr unsigned BEHIND_CHECK = 0x80000000u;
constexpr unsigned WEDGE = 0x40000000u;

// One staged chunk of beams, as seen from this tile.
template <int NF>
struct Stage {
    float4 geo0[ROWCAP];     // wc.xyz (c_T - o), len
    float4 geo1[ROWCAP];     // d.xyz, Pc (projection of c_T)
    float4 geo2[ROWCAP];     // 2 u_c.xyz, |u_c|^2  (u_c = wc - Pc d: c_T's offset from the line)
    float4 aux[ROWCAP];      // s0, A (amplitude factor), R_cut, D (error scale)
    float anc[3 * NF][ROWCAP];  // phase anchors: centre proj / start / end (turns)
    int brow[CB + 1];
    long long b0;
    int nbc;                 // beams in the chunk; -1 terminates
};

template <int NF>
struct Smem {
    Stage<NF> st[2];         // double-buffered: chunk c+1 is staged while c is summed
    unsigned surv[NWARPS][CB];  // per warp patch and beam: surviving segments + flags
    unsigned live[NWARPS][(CB + 31) / 32];  // per warp patch: beams with any work
    float btie[NWARPS][CB];  // absolute tie tolerance of the beam
    double acc[TILE][NF][2];
};

// Gaussian-beam contribution of one pair whose cutoff test (NF == 1) already passed,
// all frequencies (kernels.py:377-399): field = phi refl sqrt(c) (s + i b)/m2
// exp(-g b) exp(i(omega s/c + g s)), contribution = i omega/(2 pi c) w_b field.
template <int NF>
__device__ __forceinline__ void eval_pair(const Fp32Consts &K, int use_cutoff, float s, float q2,
                                          float m2, float A, const float *base,
                                          float (&pre)[NF], float (&pim)[NF], int &ev) {
    const float inv = rcp_approx(m2);
    const float gq = q2 * inv;
    const float ainv = A * inv;
    const float gqs = gq * s;
#pragma unroll
    for (int f = 0; f < NF; ++f) {
        if (NF > 1 && use_cutoff && q2 * K.cutk[f] > m2) continue;  // ex_re < -36
        float turns = fmaf(gqs, K.hk2pi[f], base[f]);
        turns -= rintf(turns);
        const float ph = turns * 6.283185307179586f;
        const float sn = sin_approx(ph), cs = cos_approx(ph);
        const float amp = ainv * K.omega[f] * ex2_approx(gq * K.nhkbl2e[f]);
        pre[f] = fmaf(-amp, fmaf(s, sn, K.b * cs), pre[f]);
        pim[f] = fmaf(amp, fmaf(s, cs, -K.b * sn), pim[f]);
        ++ev;
    }
}

template <int NF>
__device__ __forceinline__ void contribute(const Fp32Consts &K, int use_cutoff, float s, float q2,
                                           float A, const float *base, float (&pre)[NF],
                                           float (&pim)[NF], int &ev) {
    const float m2 = fmaf(s, s, K.b2);
    if (NF == 1 && use_cutoff && q2 * K.cutk[0] > m2) return;  // ex_re < -36 (kernels.py:384)
    eval_pair<NF>(K, use_cutoff, s, q2, m2, A, base, pre, pim, ev);
}

// Phase anchor of the nearest point: interior -> centre anchor + kappa (r.d);
// clamped -> exact start / end anchor (turns).
template <int NF>
__device__ __forceinline__ void phase_base(const Fp32Consts &K, float proj, float dl, float len,
                                           const float *anc, float *base) {
#pragma unroll
    for (int f = 0; f < NF; ++f) {
        float bf = fmaf(K.kappa[f], dl, anc[3 * f]);
        bf = proj >= len ? anc[3 * f + 2] : bf;
        bf = proj <= 0.f ? anc[3 * f + 1] : bf;
        base[f] = bf;
    }
}

// Distance of a patch centre c to segment row `r` (fp32, tile-local), the unit
// vector from the nearest point, whether the whole patch (radius RW) is cut for
// this segment, and the centre's axial projection.
template <int NF>
__device__ __forceinline__ float patch_dist(const Stage<NF> &S, int r, float cwx, float cwy,
                                            float cwz, float RW, float *ux, float *uy, float *uz,
                                            bool *cut, float *proj_out) {
    const float4 g0 = S.geo0[r];
    const float4 g1 = S.geo1[r];
    const float wx = cwx + g0.x, wy = cwy + g0.y, wz = cwz + g0.z;
    const float proj = wx * g1.x + wy * g1.y + wz * g1.z;
    const float t = fminf(fmaxf(proj, 0.f), g0.w);
    const float vx = wx - t * g1.x, vy = wy - t * g1.y, vz = wz - t * g1.z;
    const float dc = sqrtf(vx * vx + vy * vy + vz * vz);
    const float inv = dc > 1e-6f ? 1.f / dc : 0.f;
    *ux = vx * inv;
    *uy = vy * inv;
    *uz = vz * inv;
    const float px = wx - proj * g1.x, py = wy - proj * g1.y, pz = wz - proj * g1.z;
    const float rc = (S.aux[r].z + RW) * 1.00002f + 2e-3f;
    *cut = px * px + py * py + pz * pz > rc * rc;
    *proj_out = proj;
    return dc;
}

// Bound on the angle swept by the nearest-point direction of a segment over a
// ball of radius RW around a point at distance d: I - proj is nonexpansive, so
// the residual moves by <= RW and the angle is <= asin(RW/d) <= x/sqrt(1-x^2).
__device__ __forceinline__ float sweep(float RW, float d) {
    const float x = RW / fmaxf(d, 1e-6f);
    return x < 0.7f ? x * rsqrtf(1.f - x * x) * 1.0001f : 2.f;
}

// Work generation for one (patch, beam): survivor mask + flags (0 = culled).
template <int NF>
__device__ __forceinline__ unsigned classify(const Stage<NF> &S, int r0, int ns, float cwx,
                                             float cwy, float cwz, float RW, float D) {
    if (ns <= 0) return 0u;
    // pass 1: nearest segment at the patch centre
    float best = INFINITY, p0 = 0.f;
    int kj = 0;
    for (int k = 0; k < ns; ++k) {
        float ux, uy, uz, proj;
        bool cut;
        const float dc = patch_dist(S, r0 + k, cwx, cwy, cwz, RW, &ux, &uy, &uz, &cut, &proj);
        if (k == 0) p0 = proj;
        if (dc < best) {
            best = dc;
            kj = k;
        }
    }
    // pass 2: survivors (segments that can be the nearest for some receiver of the
    // patch) and whether every survivor is dead for the whole patch -- pruned
    // segments never win, so then no pair of the patch contributes
    float ujx, ujy, ujz, pj;
    bool cj;
    const float dj = patch_dist(S, r0 + kj, cwx, cwy, cwz, RW, &ujx, &ujy, &ujz, &cj, &pj);
    const float sj = sweep(RW, dj);
    const bool behind0 = p0 + RW * 1.00002f + 2e-3f < 0.f;  // whole patch behind segment 0
    unsigned mask = 1u << kj;
    bool all_dead = cj || (kj == 0 && behind0);
    for (int k = 0; k < ns; ++k) {
        if (k == kj) continue;
        float ux, uy, uz, proj;
        bool cut;
        const float dk = patch_dist(S, r0 + k, cwx, cwy, cwz, RW, &ux, &uy, &uz, &cut, &proj);
        // d_k - d_j over the patch >= (d_k - d_j)(c) - RW * sup|grad d_k - grad d_j|
        const float ex = ux - ujx, ey = uy - ujy, ez = uz - ujz;
        const float lip = fminf(sqrtf(ex * ex + ey * ey + ez * ez) + sweep(RW, dk) + sj, 2.f);
        if (!(dk - dj > RW * lip * 1.00002f + 2e-3f + 1e-5f * dk)) {
            mask |= 1u << k;
            all_dead = all_dead && (cut || (k == 0 && behind0));
        }
    }
    if (all_dead) return 0u;
    unsigned word = mask;
    // segment 0 survives and the patch reaches its launch plane
    if ((mask & 1u) && p0 - RW * 1.00002f - 2e-3f <= PROJ_ERR * D) word |= BEHIND_CHECK;
    // corner wedge: exactly segments k, k+1 survive and every receiver projects
    // beyond the end of k and before the start of k+1, so both clamped
    // distances are distances to the shared reflection point
    const int kl = __ffs(mask) - 1;
    if (mask == (3u << kl)) {
        float ux, uy, uz, pa, pb;
        bool cut;
        patch_dist(S, r0 + kl, cwx, cwy, cwz, RW, &ux, &uy, &uz, &cut, &pa);
        patch_dist(S, r0 + kl + 1, cwx, cwy, cwz, RW, &ux, &uy, &uz, &cut, &pb);
        const float m1 = PROJ_ERR * D + RW * 1.00002f + 2e-3f;
        if (pa - S.geo0[r0 + kl].w >= m1 && pb <= -m1) word = mask | WEDGE;
    }
    return word;
}

// Live mask of the R receivers of a single-segment-0 beam whose patch reaches the
// launch plane: behind = proj < 0 (kernels.py:348,375); |proj| within the fp32
// error bound is re-decided with the reference's exact fp64 projection.
__device__ __forceinline__ unsigned behind_mask(const GbsArgs &a, const Fp32Consts &K,
                                             const float (&pj)[R], const int (&oi)[R], float D,
                                             int64_t beam, int k, int &ties) {
    const float tolp = PROJ_ERR * D;
    unsigned m = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        if (pj[j] >= tolp) {
            m |= 1u << j;
            continue;
        }
        if (pj[j] < -tolp || oi[j] < 0) continue;
        const int64_t gi = 3 * (int64_t)oi[j];
        double p64, t64;
        exact_d2(a, beam * a.max_seg + k, a.obs[gi], a.obs[gi + 1], a.obs[gi + 2], &p64, &t64);
        ++ties;
        if (!(p64 < 0.0)) m |= 1u << j;
    }
    return m;
}

template <int NF>
__device__ __forceinline__ void stage_chunk(Stage<NF> &G, const GbsArgs &a,
                                            const int32_t *__restrict__ seg_start, int64_t b0,
                                            int nbc, const double4 &cen, float RT,
                                            const Fp32Consts &K, int tid) {
    const int32_t base_row = seg_start[b0];
    for (int j = tid; j <= nbc; j += THREADS) G.brow[j] = seg_start[b0 + j] - base_row;
    if (tid == 0) {
        G.nbc = nbc;
        G.b0 = b0;
    }
    const int rows = seg_start[b0 + nbc] - base_row;
    for (int r = tid; r < rows; r += THREADS) {
        int lo = 0, hi = nbc;  // seg_start[b0+lo]-base <= r < seg_start[b0+hi]-base
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (seg_start[b0 + mid] - base_row <= r) lo = mid; else hi = mid;
        }
        const int jb = lo;
        const int k = r - (seg_start[b0 + jb] - base_row);
        const int64_t row = (b0 + jb) * a.max_seg + k;
        const double ox = a.seg_origin[3 * row], oy = a.seg_origin[3 * row + 1],
                     oz = a.seg_origin[3 * row + 2];
        const double dx = a.seg_dir[3 * row], dy = a.seg_dir[3 * row + 1],
                     dz = a.seg_dir[3 * row + 2];
        const double len = a.seg_len[row], s0 = a.seg_s0[row];
        const double wcx = cen.x - ox, wcy = cen.y - oy, wcz = cen.z - oz;
        const double pc = wcx * dx + wcy * dy + wcz * dz;
        const double ucx = wcx - pc * dx, ucy = wcy - pc * dy, ucz = wcz - pc * dz;
        G.geo0[r] = make_float4((float)wcx, (float)wcy, (float)wcz, (float)len);
        G.geo1[r] = make_float4((float)dx, (float)dy, (float)dz, (float)pc);
        G.geo2[r] = make_float4((float)(2.0 * ucx), (float)(2.0 * ucy), (float)(2.0 * ucz),
                                (float)(ucx * ucx + ucy * ucy + ucz * ucz));
        const double se = s0 + len;
        const double rcut = sqrt(K.rcut_scale * (se * se + K.b2_64)) * (1.0 + 1e-5) + 1e-3;
        const double A = K.amp_scale * a.seg_refl[row] * a.weights[b0 + jb];
        const float D = (float)(fabs(wcx) + fabs(wcy) + fabs(wcz) + len) + RT + 1.f;
        G.aux[r] = make_float4((float)s0, (float)A, (float)rcut, D);
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            G.anc[3 * f + 0][r] = (float)frac_turns(K.kappa64[f] * (s0 + pc));
            G.anc[3 * f + 1][r] = (float)frac_turns(K.kappa64[f] * s0);
            G.anc[3 * f + 2][r] = (float)frac_turns(K.kappa64[f] * se);
        }
    }
}

// Greedy chunk after beam b0: <= CB beams and <= ROWCAP segment rows.
__device__ __forceinline__ int chunk_len(const int32_t *__restrict__ seg_start, int64_t b0,
                                         int64_t n_beams) {
    if (b0 >= n_beams) return 0;
    int64_t hi = b0 + CB < n_beams ? b0 + CB : n_beams;
    const int32_t r0 = seg_start[b0];
    while (seg_start[hi] - r0 > ROWCAP) --hi;
    return (int)(hi - b0);
}

template <int NF>
__global__ void __launch_bounds__(THREADS, (NF <= 2 ? BF_MINB : 2))
    gbs_fp32_kernel(const GbsArgs a, const Tiling tl, const int32_t *__restrict__ seg_start,
                    const Fp32Consts K, GbsStats *stats) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem<NF> &S = *reinterpret_cast<Smem<NF> *>(smem_raw);

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int64_t tile = blockIdx.x;
    const double4 cen = tl.centre[tile];
    const float RT = (float)cen.w;

    // ---- receivers (tile-local coordinates); padding receivers sit at the
    //      tile centre and are computed but never written back
    float rx[R], ry[R], rz[R];
    int oi[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int64_t si = tile * TILE + R * tid + j;
        const bool valid = si < tl.n;
        oi[j] = valid ? tl.perm[si] : -1;
        float4 rl = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid) rl = tl.rloc[si];
        rx[j] = rl.x;
        ry[j] = rl.y;
        rz[j] = rl.z;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            S.acc[R * tid + j][f][0] = valid ? a.acc[2 * ((int64_t)oi[j] * NF + f)] : 0.0;
            S.acc[R * tid + j][f][1] = valid ? a.acc[2 * ((int64_t)oi[j] * NF + f) + 1] : 0.0;
        }
    }
    // ---- warp patch: bounding sphere of the warp's receivers
    float cwx, cwy, cwz, RW;
    {
        float mnx = rx[0], mny = ry[0], mnz = rz[0], mxx = rx[0], mxy = ry[0], mxz = rz[0];
#pragma unroll
        for (int j = 1; j < R; ++j) {
            mnx = fminf(mnx, rx[j]); mxx = fmaxf(mxx, rx[j]);
            mny = fminf(mny, ry[j]); mxy = fmaxf(mxy, ry[j]);
            mnz = fminf(mnz, rz[j]); mxz = fmaxf(mxz, rz[j]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mnx = fminf(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
            mny = fminf(mny, __shfl_xor_sync(0xffffffffu, mny, o));
            mnz = fminf(mnz, __shfl_xor_sync(0xffffffffu, mnz, o));
            mxx = fmaxf(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
            mxy = fmaxf(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
            mxz = fmaxf(mxz, __shfl_xor_sync(0xffffffffu, mxz, o));
        }
        cwx = 0.5f * (mnx + mxx);
        cwy = 0.5f * (mny + mxy);
        cwz = 0.5f * (mnz + mxz);
        float q = 0.f;
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const float ex = rx[j] - cwx, ey = ry[j] - cwy, ez = rz[j] - cwz;
            q = fmaxf(q, ex * ex + ey * ey + ez * ez);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) q = fmaxf(q, __shfl_xor_sync(0xffffffffu, q, o));
        RW = sqrtf(q) * 1.0001f + 1e-4f;
    }

    float pre[R][NF], pim[R][NF];
    int evr[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
        evr[j] = 0;
#pragma unroll
        for (int f = 0; f < NF; ++f) pre[j][f] = pim[j][f] = 0.f;
    }
    int ties = 0, nbp = 0;
    unsigned pc[4] = {0, 0, 0, 0};

    // ---- prologue: stage chunk 0; chunk bounds run one chunk ahead of staging
    int64_t nb0 = 0;
    int nnbc = chunk_len(seg_start, 0, a.n_beams);
    if (nnbc > 0) stage_chunk(S.st[0], a, seg_start, nb0, nnbc, cen, RT, K, tid);
    nb0 += nnbc;
    nnbc = chunk_len(seg_start, nb0, a.n_beams);
    __syncthreads();

    for (int c = 0;; ++c) {
        const Stage<NF> &G = S.st[c & 1];
        const int nbc = G.nbc;
        if (nnbc == 0 && c > 0 && nbc <= 0) break;
        if (nbc <= 0) break;
        const int64_t b0 = G.b0;
        // stage the next chunk into the other buffer (free since the last barrier)
        if (nnbc > 0) {
            stage_chunk(S.st[(c + 1) & 1], a, seg_start, nb0, nnbc, cen, RT, K, tid);
        } else if (tid == 0) {
            S.st[(c + 1) & 1].nbc = 0;
        }
        nb0 += nnbc;
        nnbc = chunk_len(seg_start, nb0, a.n_beams);
        // ---- warp work generation on this chunk: one lane per beam bounds the
        //      warp patch against the beam's segments (cut / behind / dominated)
        for (int g = 0; 32 * g < nbc; ++g) {
            const int jb = 32 * g + lane;
            unsigned word = 0;
            if (jb < nbc) {
                const int r0 = G.brow[jb], ns = G.brow[jb + 1] - r0;
                float D = 0.f;
                for (int k = 0; k < ns; ++k) D = fmaxf(D, G.aux[r0 + k].w);
                const int64_t gb = b0 + jb;  // tile-level work list (exact fp64 test)
                if ((tl.wl_bits[tile * tl.wl_words + (gb >> 5)] >> (gb & 31)) & 1u)
                    word = classify(G, r0, ns, cwx, cwy, cwz, RW, D);
                S.surv[warp][jb] = word;
                S.btie[warp][jb] = TIE_ABS * D * D;
                const unsigned m = word & ~(BEHIND_CHECK | WEDGE);
                pc[word == 0 ? 0 : (word & WEDGE) ? 2 : (m & (m - 1)) ? 3 : 1] += 1;
            }
            const unsigned live = __ballot_sync(0xffffffffu, word != 0);
            if (lane == 0) S.live[warp][g] = live;
        }
        __syncwarp();
        // ---- summation over the chunk's live beams, ascending (culled beams,
        //      where every pair of the patch is cut or behind, are never visited)
        for (int g = 0; 32 * g < nbc; ++g)
        for (unsigned lm = S.live[warp][g]; lm;) {
            const int jb = 32 * g + __ffs(lm) - 1;
            lm &= lm - 1;
            const unsigned word = S.surv[warp][jb];
            const unsigned surv = word & ~(BEHIND_CHECK | WEDGE);
            const int r0 = G.brow[jb];
            if ((surv & (surv - 1)) == 0) {
                // ---- single surviving segment: it is the nearest for every receiver
                const int k = __ffs(surv) - 1;
                const int row = r0 + k;
                const float4 g0 = G.geo0[row];
                const float4 g1 = G.geo1[row];
                const float4 g2 = G.geo2[row];
                const float4 ax = G.aux[row];
                float anc[3 * NF];
#pragma unroll
                for (int q = 0; q < 3 * NF; ++q) anc[q] = G.anc[q][row];
                // geometry of all R receivers, branch-free (independent chains)
                float sj[R], q2j[R], pj[R], m2j[R], base[R][NF];
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const float dl = fmaf(rx[j], g1.x, fmaf(ry[j], g1.y, rz[j] * g1.z));
                    const float proj = dl + g1.w;
                    const float rr = fmaf(rx[j], rx[j], fmaf(ry[j], ry[j], rz[j] * rz[j]));
                    pj[j] = proj;
                    sj[j] = ax.x + fminf(fmaxf(proj, 0.f), g0.w);
                    q2j[j] = fmaxf(
                        fmaf(-dl, dl, fmaf(g2.x, rx[j], fmaf(g2.y, ry[j], fmaf(g2.z, rz[j], g2.w + rr)))),
                        0.f);
                    m2j[j] = fmaf(sj[j], sj[j], K.b2);
                    phase_base<NF>(K, proj, dl, g0.w, anc, base[j]);
                }
                unsigned lvm = (1u << R) - 1;
                if (word & BEHIND_CHECK) lvm = behind_mask(a, K, pj, oi, ax.w, b0 + jb, k, ties);
                nbp += __popc(lvm);
                if (NF == 1 && a.use_cutoff) {
#pragma unroll
                    for (int j = 0; j < R; ++j)
                        if (q2j[j] * K.cutk[0] > m2j[j]) lvm &= ~(1u << j);  // ex_re < -36
                }
#pragma unroll
                for (int j = 0; j < R; ++j)
                    if (lvm & (1u << j))
                        eval_pair<NF>(K, a.use_cutoff, sj[j], q2j[j], m2j[j], ax.y, base[j],
                                      pre[j], pim[j], evr[j]);
            } else if (word & WEDGE) {
                // ---- corner wedge of segments k, k+1: both clamp to the reflection point;
                //      the reference picks by fp64 rounding, reproduced exactly here
                const int k = __ffs(surv) - 1;
                const int ra = r0 + k, rb = ra + 1;
                const int64_t grow = (b0 + jb) * a.max_seg + k;
                const double lena = a.seg_len[grow];
                const double oax = a.seg_origin[3 * grow], oay = a.seg_origin[3 * grow + 1],
                             oaz = a.seg_origin[3 * grow + 2];
                const double obx = a.seg_origin[3 * grow + 3], oby = a.seg_origin[3 * grow + 4],
                             obz = a.seg_origin[3 * grow + 5];
                const double ldx = __dmul_rn(lena, a.seg_dir[3 * grow]);
                const double ldy = __dmul_rn(lena, a.seg_dir[3 * grow + 1]);
                const double ldz = __dmul_rn(lena, a.seg_dir[3 * grow + 2]);
                const float sa = (float)(a.seg_s0[grow] + lena);  // s0_k + t, t = len
                const float sb = (float)a.seg_s0[grow + 1];       // s0_{k+1} + 0
                const float4 g1a = G.geo1[ra], g2a = G.geo2[ra];
                const float4 g1b = G.geo1[rb], g2b = G.geo2[rb];
                const float Aa = G.aux[ra].y, Ab = G.aux[rb].y;
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    if (oi[j] < 0) continue;
                    const int64_t gi = 3 * (int64_t)oi[j];
                    const double px = a.obs[gi], py = a.obs[gi + 1], pz = a.obs[gi + 2];
                    const double vx = __dsub_rn(__dsub_rn(px, oax), ldx);
                    const double vy = __dsub_rn(__dsub_rn(py, oay), ldy);
                    const double vz = __dsub_rn(__dsub_rn(pz, oaz), ldz);
                    const double da = __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)),
                                                __dmul_rn(vz, vz));
                    const double wx = __dsub_rn(px, obx), wy = __dsub_rn(py, oby),
                                 wz = __dsub_rn(pz, obz);
                    const double db = __dadd_rn(__dadd_rn(__dmul_rn(wx, wx), __dmul_rn(wy, wy)),
                                                __dmul_rn(wz, wz));
                    const bool wb = db < da;  // strict: equal distances keep segment k
                    const float4 g1 = wb ? g1b : g1a;
                    const float4 g2 = wb ? g2b : g2a;
                    const float rr = fmaf(rx[j], rx[j], fmaf(ry[j], ry[j], rz[j] * rz[j]));
                    const float dl = fmaf(rx[j], g1.x, fmaf(ry[j], g1.y, rz[j] * g1.z));
                    const float q2 = fmaxf(
                        fmaf(-dl, dl, fmaf(g2.x, rx[j], fmaf(g2.y, ry[j], fmaf(g2.z, rz[j], g2.w + rr)))),
                        0.f);
                    float base[NF];
#pragma unroll
                    for (int f = 0; f < NF; ++f) base[f] = wb ? G.anc[3 * f + 1][rb] : G.anc[3 * f + 2][ra];
                    ++ties;
                    ++nbp;
                    contribute<NF>(K, a.use_cutoff, wb ? sb : sa, q2, wb ? Ab : Aa, base, pre[j],
                                   pim[j], evr[j]);
                }
            } else {
                // ---- several candidate segments: fp32 scan, fp64 re-decision of ties
                const float tie_abs = S.btie[warp][jb];
                float best[R], second[R];
                int kb[R];
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    best[j] = INFINITY;
                    second[j] = INFINITY;
                    kb[j] = 0;
                }
                for (unsigned m = surv; m; m &= m - 1) {
                    const int k = __ffs(m) - 1;
                    const float4 g0 = G.geo0[r0 + k];
                    const float4 g1 = G.geo1[r0 + k];
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const float wx = rx[j] + g0.x, wy = ry[j] + g0.y, wz = rz[j] + g0.z;
                        const float proj = wx * g1.x + wy * g1.y + wz * g1.z;
                        const float t = fminf(fmaxf(proj, 0.f), g0.w);
                        const float vx = wx - t * g1.x, vy = wy - t * g1.y, vz = wz - t * g1.z;
                        const float d2 = vx * vx + vy * vy + vz * vz;
                        second[j] = fminf(second[j], fmaxf(best[j], d2));
                        kb[j] = d2 < best[j] ? k : kb[j];
                        best[j] = fminf(best[j], d2);
                    }
                }
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const int k = kb[j];
                    bool exact = second[j] - best[j] <= fmaf(TIE_REL, second[j], tie_abs);
                    const float4 g0 = G.geo0[r0 + k];
                    const float4 g1 = G.geo1[r0 + k];
                    const float4 ax = G.aux[r0 + k];
                    const float dl = fmaf(rx[j], g1.x, fmaf(ry[j], g1.y, rz[j] * g1.z));
                    const float proj = dl + g1.w;
                    const float rr = fmaf(rx[j], rx[j], fmaf(ry[j], ry[j], rz[j] * rz[j]));
                    if (k == 0 && fabsf(proj) <= PROJ_ERR * ax.w) exact = true;
                    float s, q2, A, base[NF];
                    if (!exact) {
                        if (k == 0 && proj < 0.f) continue;  // behind the source
                        const float4 g2 = G.geo2[r0 + k];
                        s = ax.x + fminf(fmaxf(proj, 0.f), g0.w);
                        A = ax.y;
                        q2 = fmaxf(fmaf(-dl, dl, fmaf(g2.x, rx[j], fmaf(g2.y, ry[j], fmaf(g2.z, rz[j], g2.w + rr)))),
                                   0.f);
                        float anc[3 * NF];
#pragma unroll
                        for (int q = 0; q < 3 * NF; ++q) anc[q] = G.anc[q][r0 + k];
                        phase_base<NF>(K, proj, dl, g0.w, anc, base);
                    } else {
                        // exact re-decision among the contenders, ascending k, strict <
                        if (oi[j] < 0) continue;
                        ++ties;
                        const int64_t gi = 3 * (int64_t)oi[j];
                        const double px = a.obs[gi], py = a.obs[gi + 1], pz = a.obs[gi + 2];
                        double bd = INFINITY, bt = 0.0, bp = 0.0;
                        int bk = -1;
                        for (unsigned m = surv; m; m &= m - 1) {
                            const int kk = __ffs(m) - 1;
                            // a segment can beat the fp32 winner only within the error bound
                            const float4 h0 = G.geo0[r0 + kk];
                            const float4 h1 = G.geo1[r0 + kk];
                            const float vx0 = rx[j] + h0.x, vy0 = ry[j] + h0.y, vz0 = rz[j] + h0.z;
                            const float pjj = vx0 * h1.x + vy0 * h1.y + vz0 * h1.z;
                            const float tt = fminf(fmaxf(pjj, 0.f), h0.w);
                            const float ex = vx0 - tt * h1.x, ey = vy0 - tt * h1.y,
                                        ez = vz0 - tt * h1.z;
                            const float d2k = ex * ex + ey * ey + ez * ez;
                            if (kk != k && fmaf(-TIE_REL, d2k, d2k - best[j]) > tie_abs) continue;
                            double p64, t64;
                            const double d2 = exact_d2(a, (b0 + jb) * a.max_seg + kk, px, py, pz,
                                                       &p64, &t64);
                            if (d2 < bd) {
                                bd = d2;
                                bk = kk;
                                bt = t64;
                                bp = p64;
                            }
                        }
                        if (bk == 0 && bt == 0.0 && bp < 0.0) continue;  // behind
                        const int64_t grow = (b0 + jb) * a.max_seg + bk;
                        const double s_ref = a.seg_s0[grow] + bt;  // reference s (kernels.py:344)
                        s = (float)s_ref;
                        const float4 h1 = G.geo1[r0 + bk];
                        const float4 h2 = G.geo2[r0 + bk];
                        A = G.aux[r0 + bk].y;
                        const float dk = fmaf(rx[j], h1.x, fmaf(ry[j], h1.y, rz[j] * h1.z));
                        q2 = fmaxf(fmaf(-dk, dk, fmaf(h2.x, rx[j], fmaf(h2.y, ry[j], fmaf(h2.z, rz[j], h2.w + rr)))),
                                   0.f);
#pragma unroll
                        for (int f = 0; f < NF; ++f) base[f] = (float)frac_turns(K.kappa64[f] * s_ref);
                    }
                    ++nbp;
                    contribute<NF>(K, a.use_cutoff, s, q2, A, base, pre[j], pim[j], evr[j]);
                }
            }
        }
        // flush fp32 partial sums into the fp64 accumulators
#pragma unroll
        for (int j = 0; j < R; ++j)
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                S.acc[R * tid + j][f][0] += (double)pre[j][f];
                S.acc[R * tid + j][f][1] += (double)pim[j][f];
                pre[j][f] = pim[j][f] = 0.f;
            }
        __syncthreads();  // next chunk staged; this chunk's buffer may be reused
    }
    // ---- write back (in-place continuation) and evaluation counts (kernels.py:399)
#pragma unroll
    for (int j = 0; j < R; ++j) {
        if (oi[j] < 0) continue;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            a.acc[2 * ((int64_t)oi[j] * NF + f)] = S.acc[R * tid + j][f][0];
            a.acc[2 * ((int64_t)oi[j] * NF + f) + 1] = S.acc[R * tid + j][f][1];
        }
        a.evals[oi[j]] += evr[j];
    }
    unsigned long long t[6] = {(unsigned long long)ties, (unsigned long long)nbp, pc[0], pc[1],
                               pc[2], pc[3]};
#pragma unroll
    for (int i = 0; i < 6; ++i) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t[i] += __shfl_xor_sync(0xffffffffu, t[i], o);
    }
    if (lane == 0) {
        if (t[0]) atomicAdd(&stats->tie_pairs, t[0]);
        if (t[1]) atomicAdd(&stats->nb_pairs, t[1]);
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (t[2 + i]) atomicAdd(&stats->paths[i], t[2 + i]);
    }
}

template <int NF>
int launch_nf(const GbsArgs &a, const Tiling &t, const int32_t *seg_start, const Fp32Consts &K,
              GbsStats *stats, cudaStream_t st) {
    const size_t smem = sizeof(Smem<NF>);
    BF_TRY_CUDA(cudaFuncSetAttribute(gbs_fp32_kernel<NF>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    gbs_fp32_kernel<NF><<<(unsigned)t.n_tiles, THREADS, smem, st>>>(a, t, seg_start, K, stats);
    note_launch();
    BF_TRY_CUDA(cudaGetLastError());
    return BF_OK;
}

}  // namespace

int gbs_fp32_tile() { return TILE; }

int launch_gbs_fp32(const GbsArgs &a, const Tiling &t, const int32_t *seg_start,
                    GbsStats *d_stats, cudaStream_t st) {
    if (t.n <= 0 || a.n_beams <= 0 || a.nf <= 0) return BF_OK;
    if (a.max_seg > 32)
        return fail(BF_EINVAL, "max_seg %lld exceeds 32 (r_max <= 31)", (long long)a.max_seg);
    Fp32Consts K;
    const double two_pi = 2.0 * 3.141592653589793;
    double wmin = INFINITY;
    for (int f = 0; f < BF_MAXF; ++f) {
        const double w = f < a.nf ? a.omegas[f] : 0.0;
        if (f < a.nf && w < wmin) wmin = w;
        K.kappa64[f] = w / (two_pi * a.c);
        K.kappa[f] = (float)K.kappa64[f];
        K.hk[f] = (float)(w * 0.5 / a.c);
        K.omega[f] = (float)w;
        K.cutk[f] = (float)(w * a.width_b / (72.0 * a.c));
        K.hk2pi[f] = (float)(w * 0.5 / a.c / two_pi);
        K.nhkbl2e[f] = (float)(-(w * 0.5 / a.c) * a.width_b * 1.4426950408889634);
    }
    K.b = (float)a.width_b;
    K.b2 = (float)(a.width_b * a.width_b);
    K.b2_64 = a.width_b * a.width_b;
    K.amp_scale = a.phi_amp * sqrt(a.c) / (two_pi * a.c);
    // Cut radius for the warp-patch prepass; without the cutoff nothing is ever cut.
    K.rcut_scale = (a.use_cutoff && wmin > 0) ? 72.0 * a.c / (wmin * a.width_b) : INFINITY;
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
