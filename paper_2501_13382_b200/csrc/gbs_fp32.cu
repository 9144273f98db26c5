// gbs_fp32.cu -- the fast GBS summation kernel for sm_100a.
//
// Operator: kernels.gbs_accumulate (kernels.py:352-399) with its helper
// nearest_on_segments (kernels.py:304-349), re-designed for the B200 FP32/MUFU
// pipes.  DESIGN.md holds the error analysis behind every tolerance here.
//
//  * Receivers are Hilbert-sorted (engine.cu); 128 consecutive receivers form a
//    warp PATCH (lane l holds receivers 4l..4l+3), four patches a work-list
//    TILE.  patch_kernel stores every receiver in PATCH-LOCAL fp32
//    coordinates r = p - c_P (fp64 subtraction) with |r|^2, so fp32 never
//    represents ~100 m absolute coordinates.
//  * pack_kernel converts the reference's padded fp64 bundle once per call into
//    a row SoA: origin/len and direction/s0 in fp64, the amplitude factor and
//    cutoff radius in fp32, and fp64-exact phase anchors (radians, reduced in fp64) at
//    both ends.
//  * The kernel is PERSISTENT: every warp is an independent worker that pulls
//    (patch, beam range) units from an atomic queue, longest units first in
//    half-octave buckets and range-major inside a bucket (concurrent warps share
//    an L2-resident slice of the bundle).  No CTA barriers at all.  Units of WIDE
//    patches (sparse receiver sets) go to a second instantiation with an fp64 tail,
//    launched concurrently (gbs_fp32_kernel<NF, true>).
//  * Per unit the warp reads its tile's slice of the compacted tight work list
//    (entries (n_segs - 1) << 27 | beam: counted by the work-list kernel of
//    exact_fp64.cu, scanned, written by wl_compact from its exact fp64 bitmask),
//    <= 32 beams / ROWCAP rows per chunk:
//    stages the rows into warp-private shared memory in patch-local fp32 (fp64
//    conversion), classifies each (patch, beam) with one lane per beam (cut / behind /
//    dominated segments from the patch's bounding box, first- and second-order
//    bounds), then sums the live beams in ascending order through the
//    single-survivor path, the junction block (corner wedges and junction ties) and the
//    several-candidate scan with fp64 re-decision of near ties (exact_pending).
//  * fp32 partial sums are flushed into fp64 accumulators per chunk (every
//    BF_FLUSHN chunks with several frequencies); a unit
//    stores its fp64 partial per (beam range, receiver) and fold_kernel adds the
//    ranges in ascending order to the caller's acc (in-place continuation,
//    kernels.py:358-359) -- the result is deterministic and independent of
//    scheduling and of the number of ranks.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

// Compile-time switches (tuning and diagnostics; the defaults are the product):
//   BF_ROWCAP rows per staged chunk, BF_MINB CTAs/SM for NF = 1, BF_RANGES beam ranges per
//   call, BF_EVG receivers per evaluation branch, BF_WARPS warps per CTA, BF_FLUSHN (chunks per fp64 flush with
//   several frequencies), BF_NOPF (no junction-row prefetch); BF_ABL skips work for
//   ablation timings (results invalid), BF_HIST prints debug counters.
namespace bf {
namespace {

#ifndef BF_ROWCAP
#define BF_ROWCAP 96
#endif
#ifndef BF_MINB
#define BF_MINB 4
#endif
#ifndef BF_ABL
#define BF_ABL 0
#endif
#ifndef BF_MULTI_BF
#define BF_MULTI_BF 1  // several candidates: branch-free per-receiver block
#endif
#ifndef BF_STAGE2
#define BF_STAGE2 1
#endif
#ifndef BF_JP_ALL
#define BF_JP_ALL 1
#endif
#ifndef BF_HIST
#define BF_HIST 0
#endif
#ifndef BF_EVG
#define BF_EVG 4
#endif
#ifndef BF_RANGES
#define BF_RANGES 64
#endif
static_assert(BF_RANGES <= 64, "unit sort keys hold the beam range in 6 bits");
#ifndef BF_FLUSHN
#define BF_FLUSHN 16  // several frequencies: chunks per fp64 flush of the partials (power of 2)
#endif
constexpr int R = 4;                    // receivers per lane
constexpr int PATCH = 32 * R;           // receivers per warp patch
#ifndef BF_TILEP
#define BF_TILEP 8
#endif
constexpr int TILE = BF_TILEP * PATCH;  // receivers per work-list tile
#ifndef BF_WARPS
#define BF_WARPS 4
#endif
constexpr int WARPS = BF_WARPS;         // independent warps per CTA
#ifndef BF_FUNROLL
#define BF_FUNROLL 2  // measured: 1 -> 42.68 ms, 2 -> 42.36, 5 -> 42.64 (F = 5)
#endif
constexpr int FUNROLL = BF_FUNROLL;     // unroll of the several-frequency loop
// several frequencies (and the wide-patch kernel): warps per CTA, CTAs per SM, and whether
// the fp64 receiver positions stay in shared memory (else the sorted global copy)
#ifndef BF_WARPS_MF
#define BF_WARPS_MF 4
#endif
#ifndef BF_MF_P64_SMEM
#define BF_MF_P64_SMEM 0
#endif
template <bool MF>
constexpr int WARPS_OF = MF ? BF_WARPS_MF : WARPS;
template <bool MF>
constexpr bool P64G = MF && !BF_MF_P64_SMEM;  // fp64 receiver positions from global memory
constexpr int CB = 32;                  // max beams per staged chunk
constexpr int ROWCAP = BF_ROWCAP;       // max segment rows per staged chunk (one frequency)
#ifndef BF_ROWCAP_MF
#define BF_ROWCAP_MF 64
#endif
constexpr int ROWCAP_MF = BF_ROWCAP_MF;  // ... several frequencies (a multiple of 32)
template <bool MF>
constexpr int ROWS = MF ? ROWCAP_MF : ROWCAP;
constexpr int EVG = BF_EVG;             // receivers evaluated per branch of the tail
constexpr float TIE_REL = 3.0517578125e-05f;        // 2^-15 (x d2)
constexpr float TIE_ABS = 1.1920928955078125e-07f;  // 2^-23 (x D^2)
constexpr float PROJ_ERR = 3.814697265625e-06f;     // 2^-18 (x D): bound on |fp32 proj error|
constexpr float TIE_DD = 3.814697265625e-06f;       // 2^-18 (x d D)   tight tie bound terms
constexpr float TIE_D2 = 4.76837158203125e-07f;     // 2^-21 (x d^2)
constexpr float TIE_DSQ = 1.8189894035458565e-12f;  // 2^-39 (x D^2)

#if BF_HIST
__device__ unsigned long long g_hist[16];  // debug counters (BF_HIST builds only)
#endif
#ifndef BF_UNIT_TIMES
#define BF_UNIT_TIMES 0  // debug: clock64 cycles of every unit to $BF_UNIT_TIMES_OUT
#endif
#if BF_UNIT_TIMES
__device__ long long *g_unit_cycles;
#endif

template <typename T>
__device__ __forceinline__ T pick4(const T (&v)[4], int j) {
    return j == 0 ? v[0] : j == 1 ? v[1] : j == 2 ? v[2] : v[3];
}

struct Fp32Consts {
    double kappa64[BF_MAXF]; // omega/(2 pi c), turns per metre (fp64 anchors)
    float omega[BF_MAXF];
    float omrel[BF_MAXF];    // omega_f / omega_0 (the staged amplitude carries omega_0)
    float lomrel[BF_MAXF];   // log2(omrel)
    float gcut[BF_MAXF];     // 72 c/(omega b): q^2/m2 > gcut iff ex_re < -36 (kernels.py:384)
    float kh[BF_MAXF];       // omega/(2 c): phase = an' + kh (c2 + (q^2/m2) s) radians
    float nhkbl2e[BF_MAXF];  // -kh*b*log2(e): exp(-g b) = ex2((q^2/m2)*nhkbl2e)
    double nhkbl2e64[BF_MAXF];
    // the summation tail works with the arc length in units of b, s' = s/b, and
    // g' = q^2/(s'^2 + 1) = b^2 q^2/m2 (section 5 of DESIGN.md): the same terms with b folded
    float gcutq[BF_MAXF];    // gcut b^2: g' > gcutq iff ex_re < -36
    float khq[BF_MAXF];      // kh/b: phase = an' + kh c2 + khq g' s'
    float nhkq[BF_MAXF];     // nhkbl2e/b^2: exp(-g b) = ex2(g' nhkq)
    double nhkq64[BF_MAXF];
    float hinvb;             // 0.5/b: s' = (s0 + Pc')/b + c2 hinvb
    float invb;              // 1/b
    double invb64;           // 1/b
    float b, b2;             // width_b, width_b^2
    int ascending;           // omegas nondecreasing (gcut nonincreasing)
    double amp_scale;        // phi*sqrt(c)/(2 pi c)
    double rcut_scale;       // 72 c / (omega_min b): R_cut^2 = rcut_scale * (s_end^2 + b^2)
    float rscale;            // (float) rcut_scale
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
// 1/x on the FMA pipe (x > 0 normal): bit-trick seed (|rel err| <= 5.1e-2) and three
// Newton steps (6.6e-6, then rounding level ~6e-8).  The evaluation is bound by the
// MUFU (XU) pipe -- rcp, ex2, sin, cos per pair at 16/clk/SM -- so the reciprocal moves
// to the FMA pipe, which has the issue slots to spare.
#ifndef BF_RCP_NR
#define BF_RCP_NR 0  // measured: slower (the kernel is issue-bound, not XU-bound)
#endif
__device__ __forceinline__ float rcp_nr(float x) {
#if BF_RCP_NR
    float y = __int_as_float(0x7ef311c3 - __float_as_int(x));
#pragma unroll
    for (int i = 0; i < 3; ++i) y = fmaf(y, fmaf(-x, y, 1.f), y);
    return y;
#else
    return rcp_approx(x);
#endif
}
__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// x turns reduced to [-1/2, 1/2] and expressed in radians (fp64), rounded once
__device__ __forceinline__ float frac_rad(double x) {
    return (float)(6.283185307179586 * (x - rint(x)));
}

// Packed fp32 pairs (receivers 2h, 2h+1 of a lane): FFMA2 / FMUL2 / FADD2 do the two
// receivers' operations in one issue slot (sm_100), each with the rounding of the scalar
// instruction; a scalar operand is broadcast (.F32 operand, no extra moves).
#ifndef BF_PACKED_EVAL
#define BF_PACKED_EVAL 0  // packed pairs in the evaluation tail (measured: no gain)
#endif
#ifndef BF_PACKED_GEOM
#define BF_PACKED_GEOM 0  // packed pairs in the nearest-point geometry (no gain)
#endif
__device__ __forceinline__ float2 bc2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }
template <bool P>
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    if constexpr (P) return __ffma2_rn(a, b, c);
    return make_float2(fmaf(a.x, b.x, c.x), fmaf(a.y, b.y, c.y));
}
template <bool P>
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    if constexpr (P) return __fmul2_rn(a, b);
    return make_float2(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y));
}
template <bool P>
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    if constexpr (P) return __fadd2_rn(a, b);
    return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y));
}
constexpr bool PE = BF_PACKED_EVAL, PG = BF_PACKED_GEOM;
__device__ __forceinline__ float2 pair(const float (&v)[4], int h) { return make_float2(v[h], v[h + 1]); }


constexpr unsigned BEHIND_CHECK = 0x80000000u;
constexpr unsigned WEDGE = 0x40000000u;

// Warp-private shared memory: one staged chunk of beams as seen from the patch,
// plus the patch's fp64 accumulators.
// MF: the several-frequency representation of the summation (phase references, fp32
// chunk sums in shared memory, fp64 partials in the global buffer); also used with one
// frequency by the wide-patch kernel.
template <int NF, bool MF = (NF > 1)>
struct WarpSmem {
    // first, at the same offset in both layouts (a wide unit aliases the warp's memory):
    unsigned long long cnt[8];  // statistics: ties, non-behind, culled/single/wedge/multi
                                // items, live pairs, live pair-segments
    float4 geo0[ROWS<MF>];     // wc.xyz (c_P - o), len
    float4 geo1[ROWS<MF>];     // d.xyz, Pc (projection of c_P)
    float4 geo2[ROWS<MF>];     // 2 u_c.xyz, |u_c|^2  (u_c = wc - Pc d: c_P's offset from the line)
    float2 aux[ROWS<MF>];      // (s0 + Pc')/b, A/b (A: amplitude factor x omega_0); Pc' = clamp(Pc, 0, len)
    float4 anc[ROWS<MF>];      // an' (exact phase at s0 + Pc', radians), lo2, hi2, d2 (clamp2)
    float ancf[MF ? NF : 1][MF ? ROWS<MF> : 1];  // several frequencies: an' per frequency
    unsigned rowinfo[ROWS<MF>];  // chunk row -> compact row (Rows) of the group
    short brow[CB + 1];      // chunk beam -> first chunk row
    unsigned grow0[CB];      // chunk beam -> compact row of its segment 0
    int4 desc[CB];           // chunk beam -> (segment-0 row, survivor word, first row, D bits)
    // fp64 accumulators of the unit (NF == 1); with several frequencies they live in
    // the unit's slice of the global partial buffer instead (shared memory is the
    // occupancy limit there)
    double acc[MF ? 1 : PATCH][NF][2];
    // several frequencies: the chunk's fp32 partial sums, [f][receiver j][lane]
    // (receivers 2h, 2h+1 of lane l in facc[f][h][l] as (re, im, re, im))
    float4 facc[MF ? NF : 1][MF ? R / 2 : 1][32];
    int evc[PATCH];          // evaluation counts of the unit
    // fp64 receiver positions (exact re-decisions); the several-frequency kernels read
    // them from the sorted global copy w.pos64 instead (shared memory is their occupancy
    // limit)
    double p64[P64G<MF> ? 1 : PATCH][3];
};

// fp64 position of receiver j of the lane: the lane's slice of S.p64 (one frequency) or
// the sorted global copy at sb + j (several frequencies)
struct D3 {
    double x, y, z;
};
template <bool G>
struct Recv64 {
    const double (*p64)[3];  // S.p64 + R * lane (G = false)
    const double4 *pos;      // w.pos64 + sb (G = true)
    __device__ __forceinline__ D3 operator()(int j) const {
        if constexpr (G) {
            const double4 v = pos[j];
            return D3{v.x, v.y, v.z};
        } else {
            return D3{p64[j][0], p64[j][1], p64[j][2]};
        }
    }
};

// Gaussian-beam contribution of one pair (kernels.py:377-399): field = phi refl
// sqrt(c) (s + i b)/m2 exp(-g b) exp(i(omega s/c + g s)), contribution
// i omega/(2 pi c) w_b field.
//
// Axial phase.  Staging clamps the patch centre's projection to the segment, Pc' =
// clamp(Pc, 0, len), and stores the exact phase there (an' = omega (s0 + Pc')/c reduced
// modulo 2 pi in fp64), lo2 = -2 Pc', hi2 = 2 (len - Pc') and d2 = 2 (Pc - Pc').  A
// receiver's clamped arc length is then s = s0 + Pc' + c2/2 with c2 = clamp(2 r.d + d2,
// lo2, hi2) = 2 (clamp(proj, 0, len) - Pc'), and its phase is an' + kh (c2 + g s) with
// kh = omega/(2c) (g s = q^2 s/m2 is the off-axis term).  |c2| stays within a few patch
// radii (a receiver clamped at an end has its patch centre projecting near that end, or
// beyond it where Pc' is the end itself and c2 = 0), so the fp32 phase carries the same
// ~eps kh RW error as an interior point.
//
// Without the cutoff (kernels.py:384-385 skipped) exp(-g b) falls below the fp32 range
// for pairs far off a beam's axis: a receiver with only such pairs has a reference value
// ~1e-40..1e-300 of the field maximum.  The kernels for calls without the cutoff
// (TINY = true) therefore sum every pair beyond the cutoff exponent (ex_re < -36) in
// fp64 instead: tiny_contribution redoes the evaluation from the same fp32 s, g = q^2/m2,
// 1/m2, amplitude factor and phase with the exponential and products in fp64, added
// straight into the fp64 accumulator.  Pairs within the exponent range stay fp32 (their
// amplitude is >= e^-36 times the amplitude factor).  Calls with the cutoff never reach
// this code (TINY = false kernels do not contain it).
__device__ __forceinline__ void tiny_contribution(const Fp32Consts &K, int f, float s, float gq,
                                                  float inv, float A, float ph, double *acc64) {
    // scaled inputs (s' = s/b, g', 1/(s'^2 + 1), A/b): amp b (s' sin + cos), amp b (s' cos - sin)
    const float sn = sin_approx(ph), cs = cos_approx(ph);
    const double e = exp2((double)gq * K.nhkq64[f]);
    const double amp = (double)(A * inv) * e * (double)(f > 0 ? K.omrel[f] : 1.f);
    acc64[0] += -amp * ((double)s * (double)sn + (double)cs);
    acc64[1] += amp * ((double)s * (double)cs - (double)sn);
}

// One frequency of a pair's contribution (the several-frequency tail): ph the phase,
// gq = g', s = s', ainv = (A/b)/(s'^2 + 1) shared across frequencies; omrel[f] folded
// into the exponent (lomrel[f] = log2(omega_f/omega_0)).
__device__ __forceinline__ void eval_freq(const Fp32Consts &K, int f, float ph, float gq,
                                          float s, float ainv, float &are, float &aim,
                                          bool live) {
    const float sn = sin_approx(ph), cs = cos_approx(ph);
    const float amp = ainv * ex2_approx(fmaf(gq, K.nhkq[f], K.lomrel[f]));
    if (live) {  // i amp (s + i b)(cos + i sin) = amp b (-(s' sin + cos) + i (s' cos - sin))
        are = fmaf(-amp, fmaf(s, sn, cs), are);
        aim = fmaf(amp, fmaf(s, cs, -sn), aim);
    }
}

// One frequency, receivers 2h, 2h+1 as packed pairs: s = s' = s/b, gq = g' = q^2/(s'^2 + 1),
// inv = 1/(s'^2 + 1), A = A/b, base = an' + kh c2 (the axial phase); with m2 = b^2 (s'^2 + 1)
// the contribution i (A/m2) e (s + i b)(cos + i sin) is amp (-(s' sin + cos) + i (s' cos -
// sin)), amp = (A/b) inv e: two products fewer than with s and b apart.  A receiver that is
// not live adds zero (its amplitude factor is selected to 0, so its inputs must be finite:
// every path leaves finite s, q^2, A, b).
__device__ __forceinline__ void eval_pair2(const Fp32Consts &K, float2 s, float2 gq, float2 inv,
                                           float2 A, float2 base, float2 &pre, float2 &pim,
                                           bool l0, bool l1) {
    float2 ainv = mul2<PE>(A, inv);
    ainv.x = l0 ? ainv.x : 0.f;
    ainv.y = l1 ? ainv.y : 0.f;
    const float2 gk = mul2<PE>(gq, bc2(K.khq[0]));
    const float2 ph = fma2<PE>(gk, s, base);
    const float2 sn = make_float2(sin_approx(ph.x), sin_approx(ph.y));
    const float2 cs = make_float2(cos_approx(ph.x), cos_approx(ph.y));
    const float2 ex = mul2<PE>(gq, bc2(K.nhkq[0]));
    const float2 amp = mul2<PE>(ainv, make_float2(ex2_approx(ex.x), ex2_approx(ex.y)));
    pre = fma2<PE>(neg2(amp), fma2<PE>(s, sn, cs), pre);
    pim = fma2<PE>(amp, fma2<PE>(s, cs, neg2(sn)), pim);
}

// Evaluation counts (kernels.py:399) of a lane's R = 4 receivers as byte fields: bit j of a
// receiver mask -> byte j (one multiply, no carries: the shifted copies never overlap).
// A chunk adds at most CB * NF evaluations per receiver (checked where it is used).
__device__ __forceinline__ unsigned spread4(unsigned m) { return (m * 0x00204081u) & 0x01010101u; }

// c2 = 2 (clamp(proj, 0, len) - Pc') from r.d and the row's (lo2, hi2, d2) (see above).
__device__ __forceinline__ float clamp2(float dl, const float4 &an) {
    return fminf(fmaxf(fmaf(2.f, dl, an.w), an.y), an.z);
}

// Distance of the patch centre (the origin of patch-local coordinates) to
// segment row `r` (fp32), the unit vector from the nearest point, whether the
// whole patch (radius RW) is cut for this segment, and the centre's projection.
// Largest |r.g| over the patch: min of the box bound sum_i h_i |g_i| and the ball bound
// RW |g| (both hold for every receiver; the box is much tighter along a flat patch's normal).
__device__ __forceinline__ float reach(const float4 &B, float gx, float gy, float gz, float gn) {
    return fminf(fmaf(B.x, fabsf(gx), fmaf(B.y, fabsf(gy), B.z * fabsf(gz))), B.w * gn);
}

template <int NF, bool MF>
__device__ __forceinline__ float patch_dist(const WarpSmem<NF, MF> &S, const Fp32Consts &K, int r,
                                            const float4 &B, float *ux, float *uy, float *uz,
                                            bool *cut, float *proj_out) {
    const float4 g0 = S.geo0[r];
    const float4 g1 = S.geo1[r];
    const float4 g2 = S.geo2[r];
    const float wx = g0.x, wy = g0.y, wz = g0.z;
    const float proj = g1.w;
    const float t = fminf(fmaxf(proj, 0.f), g0.w);
    const float vx = wx - t * g1.x, vy = wy - t * g1.y, vz = wz - t * g1.z;
    const float dc = sqrt_approx(vx * vx + vy * vy + vz * vz);
    const float inv = dc > 1e-6f ? rcp_approx(dc) : 0.f;
    *ux = vx * inv;
    *uy = vy * inv;
    *uz = vz * inv;
    // cut for every receiver if this segment wins (kernels.py:382-385): q is convex with
    // subgradient n = u_c/|u_c| at the centre, so q >= |u_c| - reach(n) (|u_c|: the
    // centre's distance to the infinite line), and s <= s_hi = s0 + clamp(Pc + reach(d));
    // the patch is cut when |u_c| > R_cut(s_hi) + reach(n),
    // R_cut(s)^2 = 72 c (s^2 + b^2)/(omega_min b)
    const float uc = sqrt_approx(g2.w);
    const float hn = uc > 1e-6f ? 0.5f * rcp_approx(uc) : 0.f;
    const float rn = uc > 1e-6f ? reach(B, g2.x * hn, g2.y * hn, g2.z * hn, 1.f) : B.w;
    const float rd = reach(B, g1.x, g1.y, g1.z, 1.f);
    const float s0 = fmaf(0.5f, S.anc[r].y, S.aux[r].x * K.b);  // s0 = (s0 + Pc') - Pc'
    const float s_hi = s0 + fminf(fmaxf(proj + rd * 1.00002f + 2e-3f, 0.f), g0.w);
    const float rk = sqrt_approx(K.rscale * fmaf(s_hi, s_hi, K.b2)) * 1.00002f + 1e-3f;
    *cut = uc * 0.99999f > (rk + rn) * 1.00002f + 2e-3f;
    *proj_out = proj;
    return dc;
}

// Bound on the angle swept by the nearest-point direction of a segment over a
// ball of radius RW around a point at distance d: I - proj is nonexpansive, so
// the residual moves by <= RW and the angle is <= asin(RW/d) <= x/sqrt(1-x^2).
__device__ __forceinline__ float sweep(float RW, float d) {
    const float x = RW * rcp_approx(fmaxf(d, 1e-6f));
    return x < 0.7f ? x * rsqrtf(1.f - x * x) * 1.0001f : 2.f;
}

// Second-order drop of the distance to a segment over the ball of radius RW around a
// point at distance d > RW: RW^2 / (2 (d - RW)) (gradient 1/(d - RW)-Lipschitz there).
__device__ __forceinline__ float curv(float RW, float d) {
    return d > RW * 1.0001f + 1e-4f ? 0.5f * RW * RW * rcp_approx(d - RW) * 1.0001f : INFINITY;
}

// Work generation for one (patch, beam): survivor mask + flags (0 = culled).
template <int NF, bool MF>
__device__ __forceinline__ unsigned classify(const WarpSmem<NF, MF> &S, const Fp32Consts &K, int r0,
                                             int ns, const float4 &B, float &D) {
    const float RW = B.w;
    D = 0.f;
    if (ns <= 0) return 0u;
    // pass 1: nearest segment at the patch centre; error scale D of the beam
    float best = INFINITY;
    int kj = 0;
#pragma unroll 1
    for (int k = 0; k < ns; ++k) {
        const float4 g0 = S.geo0[r0 + k];
        D = fmaxf(D, fabsf(g0.x) + fabsf(g0.y) + fabsf(g0.z) + g0.w);
        const float4 g1 = S.geo1[r0 + k];
        const float t = fminf(fmaxf(g1.w, 0.f), g0.w);
        const float vx = g0.x - t * g1.x, vy = g0.y - t * g1.y, vz = g0.z - t * g1.z;
        const float d2 = vx * vx + vy * vy + vz * vz;
        if (d2 < best) {
            best = d2;
            kj = k;
        }
    }
    D = D * 1.000001f + RW + 1.f;  // error scale |c_P - o|_1 + len + R_W + 1 (DESIGN 5)
    const float p0 = S.geo1[r0].w;
    // pass 2: survivors (segments that can be the nearest for some receiver of the
    // patch) and whether every survivor is dead for the whole patch -- pruned
    // segments never win, so then no pair of the patch contributes
    float ujx, ujy, ujz, pj;
    bool cj;
    const float dj = patch_dist(S, K, r0 + kj, B, &ujx, &ujy, &ujz, &cj, &pj);
    const float sj = sweep(RW, dj);
    const float hj = curv(RW, dj);
    const float4 d0 = S.geo1[r0];
    const float r0d = reach(B, d0.x, d0.y, d0.z, 1.f);  // max |r.d_0| over the patch
    const bool behind0 = p0 + r0d * 1.00002f + 2e-3f < 0.f;  // whole patch behind segment 0
    unsigned mask = 1u << kj;
    bool all_dead = cj || (kj == 0 && behind0);
#if BF_HIST
    bool all_cut = all_dead;  // debug: every segment cut (no pruning needed)
#endif
#pragma unroll 1
    for (int k = 0; k < ns; ++k) {
        if (k == kj) continue;
        float ux, uy, uz, proj;
        bool cut;
        const float dk = patch_dist(S, K, r0 + k, B, &ux, &uy, &uz, &cut, &proj);
        // d_k - d_j over the patch >= (d_k - d_j)(c) + g.r - |r| sup|grad(d_k - d_j) - g|
        // with g = grad(d_k - d_j)(c) = u_k - u_j; each gradient turns by at most the
        // sweep angle over the ball, so the drop is <= reach(g) + RW (sweep_k + sweep_j)
        const float ex = ux - ujx, ey = uy - ujy, ez = uz - ujz;
        const float gn = sqrt_approx(ex * ex + ey * ey + ez * ez);
        // second order: grad d is 1/delta-Lipschitz at distance >= delta from a convex
        // set, delta >= d - RW in the ball, so the drop is also <= reach(g) +
        // RW^2 (1/(d_k - RW) + 1/(d_j - RW)) / 2
        const float rg = reach(B, ex, ey, ez, gn);
        const float drop = fminf(fminf(rg + RW * (sweep(RW, dk) + sj), rg + curv(RW, dk) + hj),
                                 2.f * RW);
        if (!(dk - dj > drop * 1.00002f + 2e-3f + 1e-5f * dk)) {
            mask |= 1u << k;
            all_dead = all_dead && (cut || (k == 0 && behind0));
        }
#if BF_HIST
        all_cut = all_cut && (cut || (k == 0 && behind0));
#endif
    }
#if BF_HIST
    if (all_cut) atomicAdd(&g_hist[4], 1ull);
    if (all_dead) atomicAdd(&g_hist[5], 1ull);
#endif
    if (all_dead) return 0u;
    unsigned word = mask;
    // segment 0 survives and the patch reaches its launch plane
    if ((mask & 1u) && p0 - r0d * 1.00002f - 2e-3f <= PROJ_ERR * D) word |= BEHIND_CHECK;
    // corner wedge: exactly segments k, k+1 survive and every receiver projects
    // beyond the end of k and before the start of k+1, so both clamped
    // distances are distances to the shared reflection point
    const int kl = __ffs(mask) - 1;
    if (mask == (3u << kl)) {
        const float4 da = S.geo1[r0 + kl], db = S.geo1[r0 + kl + 1];
        const float ma = PROJ_ERR * D + reach(B, da.x, da.y, da.z, 1.f) * 1.00002f + 2e-3f;
        const float mb = PROJ_ERR * D + reach(B, db.x, db.y, db.z, 1.f) * 1.00002f + 2e-3f;
        if (da.w - S.geo0[r0 + kl].w >= ma && db.w <= -mb) word = mask | WEDGE;
    }
    return word;
}

// Live mask of the R receivers of a single-segment-0 beam whose patch reaches the
// launch plane: behind = proj < 0 (kernels.py:348,375); |proj| within the fp32
// error bound is re-decided with the reference's exact fp64 projection.
template <bool G>
__device__ __forceinline__ unsigned behind_mask(const Fp32Work &w, const float (&pj)[R],
                                             const Recv64<G> &P64, int nvalid, float D,
                                             int64_t row, unsigned &ties) {
    const float tolp = PROJ_ERR * D;
    unsigned m = 0, amb = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        if (pj[j] >= tolp)
            m |= 1u << j;
        else if (pj[j] >= -tolp && j < nvalid)
            amb |= 1u << j;
    }
    if (amb) {  // rare: one copy of the fp64 code
        const double4 o4 = w.p0[row], d4 = w.p1[row];  // compact fp64 rows (exact copies)
        const double ox = o4.x, oy = o4.y, oz = o4.z;
        const double dx = d4.x, dy = d4.y, dz = d4.z;
        ties += __popc(amb);
#pragma unroll 1
        for (; amb; amb &= amb - 1) {
            const int j = __ffs(amb) - 1;
            // proj of kernels.py:328-331, reference operation order, no FMA
            const D3 P = P64(j);
            const double wx = __dsub_rn(P.x, ox), wy = __dsub_rn(P.y, oy), wz = __dsub_rn(P.z, oz);
            const double proj =
                __dadd_rn(__dadd_rn(__dmul_rn(wx, dx), __dmul_rn(wy, dy)), __dmul_rn(wz, dz));
            if (!(proj < 0.0)) m |= 1u << j;
        }
    }
    return m;
}

// Segments k, k+1 meeting at a reflection point, in fp64 (packed rows): when a
// receiver projects beyond the end of k and before the start of k+1, both clamped
// distances (kernels.py:332-340) are distances to the reflection point and the
// reference's choice is decided by fp64 rounding, reproduced here op for op.
struct Junction {
    double ox, oy, oz;  // o_k
    double lx, ly, lz;  // len_k * d_k (t = len, kernels.py:337-339)
    double bx, by, bz;  // o_{k+1}
    float sa, sb;       // s' = s/b of either winner: s0_k + len_k, s0_{k+1}
};

__device__ __forceinline__ Junction load_junction(const double4 *__restrict__ p0,
                                                  const double4 *__restrict__ p1, int64_t grow,
                                                  double invb = 1.0) {
    const double4 a0 = p0[grow], a1 = p1[grow], b0 = p0[grow + 1], b1 = p1[grow + 1];
    Junction J;
    J.ox = a0.x, J.oy = a0.y, J.oz = a0.z;
    J.lx = __dmul_rn(a0.w, a1.x), J.ly = __dmul_rn(a0.w, a1.y), J.lz = __dmul_rn(a0.w, a1.z);
    J.bx = b0.x, J.by = b0.y, J.bz = b0.z;
    J.sa = (float)((a1.w + a0.w) * invb);  // s' = s/b
    J.sb = (float)(b1.w * invb);
    return J;
}

// true -> segment k+1 is the reference's nearest segment (strict <: ties keep k)
__device__ __forceinline__ bool junction_pick(const Junction &J, const D3 &p) {
    const double vx = __dsub_rn(__dsub_rn(p.x, J.ox), J.lx);
    const double vy = __dsub_rn(__dsub_rn(p.y, J.oy), J.ly);
    const double vz = __dsub_rn(__dsub_rn(p.z, J.oz), J.lz);
    const double da = __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz));
    const double wx = __dsub_rn(p.x, J.bx), wy = __dsub_rn(p.y, J.by), wz = __dsub_rn(p.z, J.bz);
    const double db = __dadd_rn(__dadd_rn(__dmul_rn(wx, wx), __dmul_rn(wy, wy)), __dmul_rn(wz, wz));
    return db < da;
}

struct ExactPick {
    double bt, bp, len;  // clamped t, projection and length of the winning segment
    int bk;              // winning segment (ascending k, strict <)
};

// Exact re-decision of a near tie among the surviving segments `surv` of one
// beam (kernels.py:320-348 with the reference's fp64 operations): only segments
// whose fp32 distance is within the tie bound of the fp32 best can win.  Out of
// line: one copy of the code serves every call site of the multi path.
__device__ __forceinline__ ExactPick exact_pick(const double4 *__restrict__ p0,
                                             const double4 *__restrict__ p1, int64_t row0,
                                             const float4 *geo0, const float4 *geo1,
                                             unsigned surv, int kf, float rx, float ry, float rz,
                                             float best, float Db, const D3 &p) {
    const double px = p.x, py = p.y, pz = p.z;
    ExactPick e{0.0, 0.0, 0.0, -1};
    // pass 1 (fp32): contenders, the segments within the fp32 error of two distances of
    // the fp32 best (tight bound, DESIGN 5.8)
    unsigned cm = 0;
#pragma unroll 1
    for (unsigned m = surv; m; m &= m - 1) {
        const int kk = __ffs(m) - 1;
        const float4 h0 = geo0[kk];
        const float4 h1 = geo1[kk];
        const float vx0 = rx + h0.x, vy0 = ry + h0.y, vz0 = rz + h0.z;
        const float pjj = vx0 * h1.x + vy0 * h1.y + vz0 * h1.z;
        const float tt = fminf(fmaxf(pjj, 0.f), h0.w);
        const float ex = vx0 - tt * h1.x, ey = vy0 - tt * h1.y, ez = vz0 - tt * h1.z;
        const float d2k = ex * ex + ey * ey + ez * ez;
        if (kk == kf || d2k - best <= fmaf(TIE_DD * Db, sqrt_approx(d2k) * 1.0001f,
                                           fmaf(TIE_D2, d2k, TIE_DSQ * Db * Db)))
            cm |= 1u << kk;
    }
    // two adjacent contenders k, k+1 and the receiver beyond the end of k and before the
    // start of k+1: the junction decision (both clamped, kernels.py:332-336)
    const int ka = __ffs(cm) - 1;
    if (cm == (3u << ka)) {
        const float4 a0 = geo0[ka], a1 = geo1[ka], b1 = geo1[ka + 1];
        const float pa = fmaf(rx, a1.x, fmaf(ry, a1.y, rz * a1.z)) + a1.w;
        const float pb = fmaf(rx, b1.x, fmaf(ry, b1.y, rz * b1.z)) + b1.w;
        const float tol = PROJ_ERR * Db;
        if (pa - a0.w >= tol && pb <= -tol) {
            const Junction J = load_junction(p0, p1, row0 + ka);
            const bool wb = junction_pick(J, p);
            e.bk = ka + (wb ? 1 : 0);
            e.len = wb ? p0[row0 + ka + 1].w : p0[row0 + ka].w;
            e.bt = wb ? 0.0 : e.len;
            e.bp = wb ? -1.0 : e.len;  // clamped at the start of k+1 / the end of k
            return e;
        }
    }
    // pass 2 (fp64, reference operation order): argmin over the contenders, strict <
    double bd = INFINITY;
#pragma unroll 1
    for (unsigned m = cm; m; m &= m - 1) {
        const int kk = __ffs(m) - 1;
        const double4 o = p0[row0 + kk], d = p1[row0 + kk];  // packed fp64 rows (exact copies)
        const double ox = o.x, oy = o.y, oz = o.z, len = o.w;
        const double dx = d.x, dy = d.y, dz = d.z;
        const double wx = __dsub_rn(px, ox), wy = __dsub_rn(py, oy), wz = __dsub_rn(pz, oz);
        const double proj =
            __dadd_rn(__dadd_rn(__dmul_rn(wx, dx), __dmul_rn(wy, dy)), __dmul_rn(wz, dz));
        const double t = proj < 0.0 ? 0.0 : (proj > len ? len : proj);
        const double vx = __dsub_rn(wx, __dmul_rn(t, dx));
        const double vy = __dsub_rn(wy, __dmul_rn(t, dy));
        const double vz = __dsub_rn(wz, __dmul_rn(t, dz));
        const double d2 =
            __dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz));
        if (d2 < bd) {
            bd = d2;
            e.bk = kk;
            e.bt = t;
            e.bp = proj;
            e.len = len;
        }
    }
    return e;
}


// Exact re-decision (fp64, reference operation order) of the receivers in `pend`
// among the surviving segments `surv` (ascending k, strict <), one pending
// receiver per lane per round; fills the nearest point of each decided receiver.
template <int NF, bool MF>
__device__ __forceinline__ void exact_pending(const GbsArgs &a, const Fp32Consts &K,
                                              const WarpSmem<NF, MF> &S,
                                              int64_t row0, int r0, unsigned surv, unsigned pend,
                                              const float (&rx)[R], const float (&ry)[R],
                                              const float (&rz)[R], const float (&rr)[R],
                                              const float (&best)[R], const int (&kb)[R],
                                              float Db, int lane, float (&sj)[R],
                                              float (&q2j)[R], float (&Aj)[R],
                                              float (&bj)[R][1], int (&pref)[R], unsigned &lvm,
                                              unsigned &ties, const Fp32Work &w,
                                              const Recv64<P64G<MF>> &P64) {
    ties += __popc(pend);
    // two adjacent candidates k, k+1 (most multi items): a receiver that projects
    // beyond the end of k and before the start of k+1 is decided like the corner wedge
#pragma unroll 1
    while (__any_sync(0xffffffffu, pend != 0)) {
#if BF_HIST
        if ((threadIdx.x & 31) == 0) atomicAdd(&g_hist[2], 1ull);
#endif
        if (!pend) continue;
        const int j = __ffs(pend) - 1;
        pend &= pend - 1;
        const float x = pick4(rx, j), y = pick4(ry, j), z = pick4(rz, j);
        const ExactPick e = exact_pick(w.p0, w.p1, row0,
                                       S.geo0 + r0, S.geo1 + r0, surv, pick4(kb, j), x, y, z,
                                       pick4(best, j), Db, P64(j));
        if (e.bk == 0 && e.bt == 0.0 && e.bp < 0.0) continue;  // behind
        const int k = e.bk;
        const float4 g1 = S.geo1[r0 + k];
        const float4 g2 = S.geo2[r0 + k];
        const float dl = fmaf(x, g1.x, fmaf(y, g1.y, z * g1.z));
        const float q2 =
            fmaxf(fmaf(-dl, dl, fmaf(g2.x, x, fmaf(g2.y, y, fmaf(g2.z, z, g2.w + pick4(rr, j))))),
                  0.f);
        const float s = (float)((w.p1[row0 + k].w + e.bt) * K.invb64);  // kernels.py:344, s' = s/b
        // phase reference follows the exact clamp
        const float4 an = S.anc[r0 + k];
        const float c2 = e.bt == 0.0 ? an.y : e.bt == e.len ? an.z : clamp2(dl, an);
        const float A = S.aux[r0 + k].y;
        const float b = MF ? c2 : fmaf(K.kh[0], c2, an.x);
        const int ref = r0 + k;
#pragma unroll
        for (int jj = 0; jj < R; ++jj)
            if (jj == j) {
                q2j[jj] = q2;
                sj[jj] = s;
                Aj[jj] = A;
                bj[jj][0] = b;
                if constexpr (MF) pref[jj] = ref;
            }
        lvm |= 1u << j;
    }
}

// Stage chunk rows [0, nrows) into warp-private shared memory, patch-local.
template <int NF, bool MF>
__device__ __forceinline__ void stage_rows(WarpSmem<NF, MF> &S, const Fp32Work &w, int nrows,
                                           double cx, double cy, double cz, float RW,
                                           const Fp32Consts &K, int lane) {
#if BF_STAGE2
    // two rows per lane at a time (rows r and r + 32): both rows' loads in flight together
    // and their fp64 chains interleave
    auto row_out = [&](int r, const double4 &p0, const double4 &p1, float p2, bool st) {
        const double wcx = cx - p0.x, wcy = cy - p0.y, wcz = cz - p0.z;
        const double pc = wcx * p1.x + wcy * p1.y + wcz * p1.z;
        const double ucx = wcx - pc * p1.x, ucy = wcy - pc * p1.y, ucz = wcz - pc * p1.z;
        if (st) S.geo0[r] = make_float4((float)wcx, (float)wcy, (float)wcz, (float)p0.w);
        if (st) S.geo1[r] = make_float4((float)p1.x, (float)p1.y, (float)p1.z, (float)pc);
        if (st) S.geo2[r] = make_float4((float)(2.0 * ucx), (float)(2.0 * ucy), (float)(2.0 * ucz),
                                (float)(ucx * ucx + ucy * ucy + ucz * ucz));
        // the centre's projection clamped to the segment; phase references (clamp2)
        const double pcc = pc < 0.0 ? 0.0 : (pc > p0.w ? p0.w : pc);
        const double sp = p1.w + pcc;
        if (st) S.aux[r] = make_float2((float)(sp * K.invb64), (float)((double)(p2 * K.omega[0]) * K.invb64));
        if (st) S.anc[r] = make_float4(frac_rad(K.kappa64[0] * sp), (float)(-2.0 * pcc),
                               (float)(2.0 * (p0.w - pcc)), (float)(2.0 * (pc - pcc)));
        if constexpr (MF) {
#pragma unroll
            for (int f = 0; f < NF; ++f) if (st) S.ancf[f][r] = frac_rad(K.kappa64[f] * sp);
        }
    };
#pragma unroll 1
    for (int r = lane; r < nrows; r += 64) {
        const bool two = r + 32 < nrows;
        const int64_t ga = (int64_t)S.rowinfo[r];
        const int64_t gb = two ? (int64_t)S.rowinfo[r + 32] : ga;
        const double4 a0 = w.p0[ga], a1 = w.p1[ga];
        const float a2 = w.amp[ga];
        const double4 b0 = w.p0[gb], b1 = w.p1[gb];
        const float b2 = w.amp[gb];
        row_out(r, a0, a1, a2, true);
        row_out(two ? r + 32 : r, b0, b1, b2, two);  // (computed either way: the chains interleave)
    }
}
#else
    // software-pipelined: the next row's loads are in flight while this row converts
    auto grow = [&](int r) { return (int64_t)S.rowinfo[r]; };
    int r = lane;
    double4 p0 = make_double4(0, 0, 0, 0), p1 = p0;
    float p2 = 0.f;
    if (r < nrows) {
        const int64_t g = grow(r);
        p0 = w.p0[g];  // o.xyz, len
        p1 = w.p1[g];  // d.xyz, s0
        p2 = w.amp[g];  // A
    }
#pragma unroll 1
    for (; r < nrows; r += 32) {
        const int rn = r + 32;
        double4 p0n = p0, p1n = p1;
        float p2n = p2;
        if (rn < nrows) {
            const int64_t gn = grow(rn);
            p0n = w.p0[gn];
            p1n = w.p1[gn];
            p2n = w.amp[gn];
        }
        const double wcx = cx - p0.x, wcy = cy - p0.y, wcz = cz - p0.z;
        const double pc = wcx * p1.x + wcy * p1.y + wcz * p1.z;
        const double ucx = wcx - pc * p1.x, ucy = wcy - pc * p1.y, ucz = wcz - pc * p1.z;
        S.geo0[r] = make_float4((float)wcx, (float)wcy, (float)wcz, (float)p0.w);
        S.geo1[r] = make_float4((float)p1.x, (float)p1.y, (float)p1.z, (float)pc);
        S.geo2[r] = make_float4((float)(2.0 * ucx), (float)(2.0 * ucy), (float)(2.0 * ucz),
                                (float)(ucx * ucx + ucy * ucy + ucz * ucz));
        // the centre's projection clamped to the segment; phase references (clamp2)
        const double pcc = pc < 0.0 ? 0.0 : (pc > p0.w ? p0.w : pc);
        const double sp = p1.w + pcc;
        S.aux[r] = make_float2((float)(sp * K.invb64), (float)((double)(p2 * K.omega[0]) * K.invb64));
        S.anc[r] = make_float4(frac_rad(K.kappa64[0] * sp), (float)(-2.0 * pcc),
                               (float)(2.0 * (p0.w - pcc)), (float)(2.0 * (pc - pcc)));
        if constexpr (MF) {
#pragma unroll
            for (int f = 0; f < NF; ++f) S.ancf[f][r] = frac_rad(K.kappa64[f] * sp);
        }
        p0 = p0n;
        p1 = p1n;
        p2 = p2n;
    }
}
#endif


// One (patch, beam range) unit.
template <int NF, bool WIDE, bool TINY, bool MF = (NF > 1 || WIDE)>
__device__ __forceinline__ void run_unit(const GbsArgs &a, const Tiling &tl, const Fp32Work &w,
                                         const Fp32Consts &K, WarpSmem<NF, MF> &S, int64_t p,
                                         int64_t q, int lane, GbsStats *stats) {
    const float RW = (float)w.pcen[p].w;
    // ---- receivers (patch-local); padding receivers sit at the centre and are
    //      computed but never written back
    float rx[R], ry[R], rz[R], rr[R];
    const int64_t sb = p * PATCH + R * lane;  // sorted position of receiver j = sb + j
    const int32_t *perm = tl.perm + sb;       // observer index of receiver j = perm[j]
    const int nvalid =  // receivers j < nvalid are real
        tl.n - sb < R ? (tl.n - sb > 0 ? (int)(tl.n - sb) : 0) : R;
    const Recv64<P64G<MF>> P64{S.p64 + (P64G<MF> ? 0 : R * lane), w.pos64 + sb};
#pragma unroll
    for (int j = 0; j < R; ++j) {
        float4 rl = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j < nvalid) rl = w.prl[sb + j];
        rx[j] = rl.x;
        ry[j] = rl.y;
        rz[j] = rl.z;
        rr[j] = rl.w;
        if (!MF) {
            S.acc[R * lane + j][0][0] = S.acc[R * lane + j][0][1] = 0.0;
        } else if (j < nvalid) {
#pragma unroll
            for (int f = 0; f < NF; ++f)
                w.part[((q * w.n_pad + sb + j) * NF) + f] = make_double2(0.0, 0.0);
        }
        S.evc[R * lane + j] = 0;
        if (j < nvalid) {
            const int64_t oi = perm[j];
            if constexpr (!P64G<MF>) {
                S.p64[R * lane + j][0] = a.obs[3 * oi];
                S.p64[R * lane + j][1] = a.obs[3 * oi + 1];
                S.p64[R * lane + j][2] = a.obs[3 * oi + 2];
            }
        }
    }
    // fp32 partial sums of the chunk: registers with one frequency, shared memory
    // (S.facc) with several
    float2 pre2[R / 2], pim2[R / 2];  // (one frequency) receivers 2h, 2h+1
    // byte counters: a receiver gets <= CBN * NF <= 255 evaluations per chunk
    constexpr int CBN = NF * CB <= 255 ? CB : 255 / NF;
    static_assert(R == 4 && CBN * NF <= 255, "byte evaluation counters");
    unsigned evb = 0;  // evaluation counts of the lane's receivers in the chunk (byte fields)
    unsigned ties = 0, nbp = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        if (!(j & 1)) pre2[j >> 1] = pim2[j >> 1] = make_float2(0.f, 0.f);
        if constexpr (MF) {
            if (!(j & 1)) {
#pragma unroll
                for (int f = 0; f < NF; ++f) S.facc[f][j >> 1][lane] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    }

    // ---- candidate beams: the unit's slice of the compacted tight work list
    const int64_t ui = (p / (TILE / PATCH)) * w.n_ranges + q;
    const uint32_t *items = w.wl_items + w.wl_off[ui];
    const int n_items = (int)(w.wl_off[ui + 1] - w.wl_off[ui]);
    int cur = 0, nch = 0;
    uint32_t e = lane < n_items ? items[lane] : 0u;  // entries of the next chunk
    while (cur < n_items) {
        const int nbn = min(CBN, n_items - cur);
        const int ns = lane < nbn ? (int)(e >> 27) + 1 : 0;
        const unsigned row_l = e & 0x7ffffffu;  // compact row of the beam's segment 0
        // ---- row capacity: keep the prefix of beams whose rows fit ROWS<MF>
        int incl = ns;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const unsigned fit = __ballot_sync(0xffffffffu, lane < nbn && incl <= ROWS<MF>);
        const int nbc = __popc(fit);
        const int nrows = __shfl_sync(0xffffffffu, incl, nbc - 1);
        if (lane < nbc) {
            S.grow0[lane] = row_l;
            S.brow[lane] = incl - ns;
#pragma unroll 1
            for (int k = 0; k < ns; ++k) S.rowinfo[incl - ns + k] = row_l + k;
        }
        cur += nbc;
        // the next chunk's entries: in flight during this chunk
        e = cur + lane < n_items ? items[cur + lane] : 0u;
        if (lane == 0) S.brow[nbc] = nrows;
        __syncwarp();
        {
            const double4 c = w.pcen[p];  // re-read (L1) rather than held in registers
#if !(BF_ABL & 64)
            stage_rows<NF, MF>(S, w, nrows, c.x, c.y, c.z, RW, K, lane);
#endif
        }
        __syncwarp();
        // ---- work generation: one lane per beam bounds the patch against the
        //      beam's segments (cut / behind / dominated)
        unsigned word = 0;
        if (lane < nbc) {
            const int r0 = S.brow[lane], nsb = S.brow[lane + 1] - r0;
            float D = 0.f;
#if BF_ABL & 32
            word = 0;  // ablation: no classification
#else
            word = classify<NF, MF>(S, K, r0, nsb, w.pbox[p], D);
#endif
#if !BF_NOPF
            {   // corner wedges and two-adjacent-survivor items read the fp64 rows of the
                // junction (load_junction): start those loads now, into L1
                const unsigned m = word & ~(BEHIND_CHECK | WEDGE);
                const int ka = __ffs(m) - 1;
                if ((word & WEDGE) || (m != 0 && m == (3u << ka))) {
                    const int64_t g = (int64_t)S.grow0[lane] + ka;
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(w.p0 + g));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(w.p1 + g));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(w.p0 + g + 1));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(w.p1 + g + 1));
                }
            }
#endif
            S.desc[lane] = make_int4((int)S.grow0[lane], (int)word, r0, __float_as_int(D));
        }
        const unsigned live = __ballot_sync(0xffffffffu, word != 0);
        {
            const unsigned m = word & ~(BEHIND_CHECK | WEDGE);
            const unsigned nw = __popc(__ballot_sync(0xffffffffu, (word & WEDGE) != 0));
            const unsigned nm = __popc(__ballot_sync(0xffffffffu, word != 0 && !(word & WEDGE) &&
                                                                      (m & (m - 1)) != 0));
#if BF_HIST
            {
                const bool mul = word != 0 && !(word & WEDGE) && (m & (m - 1)) != 0;
                const int ns_ = __popc(m);
                const unsigned h2 = __popc(__ballot_sync(0xffffffffu, mul && ns_ == 2));
                const unsigned h3 = __popc(__ballot_sync(0xffffffffu, mul && ns_ == 3));
                const unsigned h4 = __popc(__ballot_sync(0xffffffffu, mul && ns_ == 4));
                const unsigned h5 = __popc(__ballot_sync(0xffffffffu, mul && ns_ >= 5));
                if (lane == 0) {
                    atomicAdd(&stats->multi_surv[0], (unsigned long long)h2);
                    atomicAdd(&stats->multi_surv[1], (unsigned long long)h3);
                    atomicAdd(&stats->multi_surv[2], (unsigned long long)h4);
                    atomicAdd(&stats->multi_surv[3], (unsigned long long)h5);
                }
            }
#endif
            // pairs of the evaluated items and their segment counts (FLOP model)
            const unsigned lsegs = __reduce_add_sync(
                0xffffffffu, word != 0 ? (unsigned)(S.brow[lane + 1] - S.brow[lane]) : 0u);
            const unsigned long long pv = (unsigned long long)min((int64_t)PATCH, tl.n - p * PATCH);
            if (lane == 0) {
                S.cnt[6] += pv * __popc(live);
                S.cnt[7] += pv * lsegs;
                S.cnt[2] += nbc - __popc(live);
                S.cnt[3] += __popc(live) - nw - nm;
                S.cnt[4] += nw;
                S.cnt[5] += nm;
            }
        }
        __syncwarp();
        // ---- summation over the chunk's live beams, ascending.  Each path yields
        //      the nearest point of every receiver (s, q^2, row, proj, r.d) and the
        //      mask of non-behind receivers; one shared tail applies the cutoff and
        //      evaluates the contributions.
        // the next item's descriptor is loaded one item ahead (its shared-memory latency
        // overlaps the current item)
        int4 dnext = S.desc[live ? __ffs(live) - 1 : 0];
#pragma unroll 1
#if BF_ABL & 16
        for (unsigned lm = 0; lm;) {  // ablation: no summation at all
#else
        for (unsigned lm = live; lm;) {
#endif
            const int4 dsc = dnext;
            lm &= lm - 1;
            dnext = S.desc[lm ? __ffs(lm) - 1 : 0];
            const int64_t row0 = (unsigned)dsc.x;  // compact row of segment 0
            const unsigned bword = (unsigned)dsc.y;
            const unsigned surv = bword & ~(BEHIND_CHECK | WEDGE);
            const int r0 = dsc.z;
#if BF_ABL
            // ablation (timing experiments only; results are wrong): skip item kinds
            {
                const bool is_single = (surv & (surv - 1)) == 0, is_wedge = (bword & WEDGE) != 0;
                if ((BF_ABL & 1) && is_single) continue;
                if ((BF_ABL & 2) && !is_single && is_wedge) continue;
                if ((BF_ABL & 4) && !is_single && !is_wedge) continue;
            }
#endif
            // nearest point of every receiver: s, q^2, amplitude factor, axial phase base
            // (one frequency) or its (row, clamp) reference and r.d (several, pref/bj)
            float sj[R], q2j[R], Aj[R], bj[R][1];
            int pref[R] = {};
            unsigned lvm;
            if ((surv & (surv - 1)) == 0) {
                // ---- single surviving segment: it is the nearest for every receiver
                const int k = __ffs(surv) - 1;
                const int row = r0 + k;
                const float4 g1 = S.geo1[row];
                const float4 g2 = S.geo2[row];
                const float2 ax = S.aux[row];
                const float4 an = S.anc[row];
                float dlj[R];
#pragma unroll
                for (int h = 0; h < R; h += 2) {  // receivers h, h+1 as packed pairs
                    const float2 X = pair(rx, h), Y = pair(ry, h), Z = pair(rz, h);
                    const float2 dl = fma2<PG>(X, bc2(g1.x), fma2<PG>(Y, bc2(g1.y), mul2<PG>(Z, bc2(g1.z))));
                    const float2 qq = fma2<PG>(neg2(dl), dl,
                                           fma2<PG>(bc2(g2.x), X, fma2<PG>(bc2(g2.y), Y,
                                                fma2<PG>(bc2(g2.z), Z, add2<PG>(bc2(g2.w), pair(rr, h))))));
                    const float2 c2 = make_float2(clamp2(dl.x, an), clamp2(dl.y, an));
                    const float2 sv = fma2<PG>(bc2(K.hinvb), c2, bc2(ax.x));  // s' = s/b
                    float2 bf;
                    if constexpr (!MF) bf = fma2<PG>(bc2(K.kh[0]), c2, bc2(an.x));
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int j = h + u;
                        dlj[j] = u ? dl.y : dl.x;
                        Aj[j] = ax.y;
                        if constexpr (!MF) {
                            bj[j][0] = u ? bf.y : bf.x;
                        } else {
                            bj[j][0] = u ? c2.y : c2.x;
                            pref[j] = row;
                        }
                        sj[j] = u ? sv.y : sv.x;
                        q2j[j] = u ? qq.y : qq.x;  // may round below 0: harmless (g ~ -eps)
                    }
                }
                lvm = (1u << R) - 1;
                if (bword & BEHIND_CHECK) {
                    float pj[R];
#pragma unroll
                    for (int j = 0; j < R; ++j) pj[j] = dlj[j] + g1.w;
                    lvm = behind_mask(w, pj, P64, nvalid, __int_as_float(dsc.w),
                                      row0 + k, ties);
                }
            } else {
                // receivers decided at the junction of segments ka, ka+1 (corner wedge):
                // both clamped distances are distances to the reflection point, an exact
                // tie the reference breaks by fp64 rounding, reproduced op for op
                unsigned jp;
                int ka = __ffs(surv) - 1;
                unsigned pend = 0;  // receivers re-decided by the general fp64 search
                // receivers no path decides (behind, padding) still go through the
                // evaluation with a zero amplitude: finite inputs
#pragma unroll
                for (int j = 0; j < R; ++j) sj[j] = q2j[j] = Aj[j] = bj[j][0] = 0.f;
                float best[R];
                int kb[R];
                float Db = 0.f;
                if (bword & WEDGE) {
                    // ---- corner wedge: every receiver of the patch is at the junction
                    jp = (1u << nvalid) - 1u;
                    lvm = 0;
                } else {
                // ---- several candidate segments: fp32 distances, fp64 re-decision of ties
                Db = __int_as_float(dsc.w);
#if BF_HIST
                {   // debug: lane-level pruning potential of this several-candidate item
                    float rl = 0.f;
#pragma unroll
                    for (int j = 1; j < R; ++j) {
                        const float ex_ = rx[j] - rx[0], ey_ = ry[j] - ry[0], ez_ = rz[j] - rz[0];
                        if (j < nvalid) rl = fmaxf(rl, sqrtf(ex_ * ex_ + ey_ * ey_ + ez_ * ez_));
                    }
                    auto dist0 = [&](int k) {
                        const float4 g0 = S.geo0[r0 + k], g1 = S.geo1[r0 + k];
                        const float wx = rx[0] + g0.x, wy = ry[0] + g0.y, wz = rz[0] + g0.z;
                        const float pr = wx * g1.x + wy * g1.y + wz * g1.z;
                        const float t = fminf(fmaxf(pr, 0.f), g0.w);
                        const float vx = wx - t * g1.x, vy = wy - t * g1.y, vz = wz - t * g1.z;
                        return sqrtf(vx * vx + vy * vy + vz * vz);
                    };
                    float bd = INFINITY;
                    for (unsigned m = surv; m; m &= m - 1) bd = fminf(bd, dist0(__ffs(m) - 1));
                    unsigned keep = 0;
                    for (unsigned m = surv; m; m &= m - 1) {
                        const int k = __ffs(m) - 1;
                        const float d = dist0(k);
                        if (d - bd <= 2.f * rl * 1.0001f + 2e-3f + 1e-5f * d) keep |= 1u << k;
                    }
                    if (nvalid == 0) keep = 0;
                    const unsigned wk = __reduce_or_sync(0xffffffffu, keep);
                    const unsigned mx = __reduce_max_sync(0xffffffffu, (unsigned)__popc(keep));
                    const unsigned l1 = __popc(__ballot_sync(0xffffffffu, __popc(keep) == 1));
                    if (lane == 0) {
                        const int n = __popc(surv);
                        atomicAdd(&g_hist[6], (unsigned long long)n);
                        atomicAdd(&g_hist[7], (unsigned long long)__popc(wk));
                        atomicAdd(&g_hist[8], (unsigned long long)(__popc(wk) == 1));
                        atomicAdd(&g_hist[9], 1ull);
                        atomicAdd(&g_hist[10], (unsigned long long)l1);
                        atomicAdd(&g_hist[11], (unsigned long long)mx);
                        atomicAdd(&g_hist[n == 2 ? 12 : n == 3 ? 13 : n == 4 ? 14 : 15], 1ull);
                    }
                }
#endif
                const float tie_abs = TIE_ABS * Db * Db;
                jp = 0;
                lvm = 0;
                float second[R];
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    best[j] = INFINITY;
                    second[j] = INFINITY;
                    kb[j] = 0;
                }
#pragma unroll 1
                for (unsigned m = surv; m; m &= m - 1) {
                    const int k = __ffs(m) - 1;
                    const float4 g0 = S.geo0[r0 + k];
                    const float4 g1 = S.geo1[r0 + k];
#pragma unroll
                    for (int h = 0; h < R; h += 2) {  // receivers h, h+1 as packed pairs
                        const float2 wx = add2<PG>(pair(rx, h), bc2(g0.x));
                        const float2 wy = add2<PG>(pair(ry, h), bc2(g0.y));
                        const float2 wz = add2<PG>(pair(rz, h), bc2(g0.z));
                        const float2 proj =
                            fma2<PG>(wz, bc2(g1.z), fma2<PG>(wy, bc2(g1.y), mul2<PG>(wx, bc2(g1.x))));
                        const float2 nt = make_float2(-fminf(fmaxf(proj.x, 0.f), g0.w),
                                                      -fminf(fmaxf(proj.y, 0.f), g0.w));
                        const float2 vx = fma2<PG>(nt, bc2(g1.x), wx), vy = fma2<PG>(nt, bc2(g1.y), wy),
                                     vz = fma2<PG>(nt, bc2(g1.z), wz);
                        const float2 d2p = fma2<PG>(vz, vz, fma2<PG>(vy, vy, mul2<PG>(vx, vx)));
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const int j = h + u;
                            const float d2 = u ? d2p.y : d2p.x;
                            second[j] = fminf(second[j], fmaxf(best[j], d2));
                            kb[j] = d2 < best[j] ? k : kb[j];
                            best[j] = fminf(best[j], d2);
                        }
                    }
                }
                // two adjacent candidates: ties at the junction go to the wedge decision
                const bool pair = surv == (3u << ka);
                const float jtol = pair ? PROJ_ERR * Db : 0.f;  // Db >= either row's D
#if BF_MULTI_BF
                // every receiver's nearest point from its fp32 winner, unconditionally (the
                // four blocks interleave); near ties and behind receivers only flagged here
                unsigned exm = 0;
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const int k = kb[j];
                    const float gap = second[j] - best[j];
                    // fp32 error of the two distances: loose test first,
                    // then 2^-18 d D + 2^-21 d^2 + 2^-39 D^2 with d^2 <= second
                    bool exact = gap <= fmaf(TIE_REL, second[j], tie_abs) &&
                                 gap <= fmaf(TIE_DD * Db, sqrt_approx(second[j]) * 1.0001f,
                                             fmaf(TIE_D2, second[j], TIE_DSQ * Db * Db));
                    const float4 g1 = S.geo1[r0 + k];
                    const float4 g2 = S.geo2[r0 + k];
                    const float2 ax = S.aux[r0 + k];
                    const float4 an = S.anc[r0 + k];
                    const float dl = fmaf(rx[j], g1.x, fmaf(ry[j], g1.y, rz[j] * g1.z));
                    const float proj = dl + g1.w;
                    exact = exact || (k == 0 && fabsf(proj) <= PROJ_ERR * Db);
                    const bool behind = k == 0 && proj < 0.f;  // behind the source
                    q2j[j] = fmaf(-dl, dl, fmaf(g2.x, rx[j], fmaf(g2.y, ry[j], fmaf(g2.z, rz[j], g2.w + rr[j]))));
                    const float c2 = clamp2(dl, an);
                    sj[j] = fmaf(K.hinvb, c2, ax.x);
                    Aj[j] = ax.y;
                    if constexpr (!MF) {
                        bj[j][0] = fmaf(K.kh[0], c2, an.x);
                    } else {
                        bj[j][0] = c2;
                        pref[j] = r0 + k;
                    }
                    exm |= (exact ? 1u : 0u) << j;
                    lvm |= (!exact && !behind ? 1u : 0u) << j;
                }
                exm &= (1u << nvalid) - 1u;
                for (unsigned m = exm; m; m &= m - 1) {  // near ties: junction or fp64 search
                    const int j = __ffs(m) - 1;
                    if (pair) {
                        // beyond the end of ka and before the start of ka+1?
                        const float4 a0 = S.geo0[r0 + ka], a1 = S.geo1[r0 + ka];
                        const float4 b1 = S.geo1[r0 + ka + 1];
                        const float x = pick4(rx, j), y = pick4(ry, j), z = pick4(rz, j);
                        const float pa = fmaf(x, a1.x, fmaf(y, a1.y, z * a1.z)) + a1.w;
                        const float pb = fmaf(x, b1.x, fmaf(y, b1.y, z * b1.z)) + b1.w;
                        if (pa - a0.w >= jtol && pb <= -jtol) {
                            jp |= 1u << j;
                            continue;
                        }
                    }
                    pend |= 1u << j;
                }
                }
#else
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const int k = kb[j];
                    const float gap = second[j] - best[j];
                    // fp32 error of the two distances: loose test first,
                    // then 2^-18 d D + 2^-21 d^2 + 2^-39 D^2 with d^2 <= second
                    bool exact = gap <= fmaf(TIE_REL, second[j], tie_abs);
                    if (exact)
                        exact = gap <= fmaf(TIE_DD * Db, sqrt_approx(second[j]) * 1.0001f,
                                            fmaf(TIE_D2, second[j], TIE_DSQ * Db * Db));
                    const float4 g1 = S.geo1[r0 + k];
                    const float dl = fmaf(rx[j], g1.x, fmaf(ry[j], g1.y, rz[j] * g1.z));
                    const float proj = dl + g1.w;
                    if (k == 0 && fabsf(proj) <= PROJ_ERR * Db) exact = true;
                    if (exact) {
                        if (j >= nvalid) continue;
                        if (pair) {
                            // beyond the end of ka and before the start of ka+1?
                            const float4 a0 = S.geo0[r0 + ka], a1 = S.geo1[r0 + ka];
                            const float4 b1 = S.geo1[r0 + ka + 1];
                            const float pa = fmaf(rx[j], a1.x, fmaf(ry[j], a1.y, rz[j] * a1.z)) + a1.w;
                            const float pb = fmaf(rx[j], b1.x, fmaf(ry[j], b1.y, rz[j] * b1.z)) + b1.w;
                            if (pa - a0.w >= jtol && pb <= -jtol) {
                                jp |= 1u << j;
                                continue;
                            }
                        }
                        pend |= 1u << j;
                        continue;
                    }
                    if (k == 0 && proj < 0.f) continue;  // behind the source
                    const float4 g2 = S.geo2[r0 + k];
                    q2j[j] = fmaf(-dl, dl, fmaf(g2.x, rx[j], fmaf(g2.y, ry[j], fmaf(g2.z, rz[j], g2.w + rr[j]))));
                    const float2 ax = S.aux[r0 + k];
                    const float4 an = S.anc[r0 + k];
                    const float c2 = clamp2(dl, an);
                    sj[j] = fmaf(K.hinvb, c2, ax.x);
                    Aj[j] = ax.y;
                    if constexpr (!MF) {
                        bj[j][0] = fmaf(K.kh[0], c2, an.x);
                    } else {
                        bj[j][0] = c2;
                        pref[j] = r0 + k;
                    }
                    lvm |= 1u << j;
                }
                }
#endif
                if (__any_sync(0xffffffffu, jp != 0)) {
                    const int ra = r0 + ka, rb = ra + 1;
                    const Junction J = load_junction(w.p0, w.p1, row0 + ka, K.invb64);
                    const float Aa = S.aux[ra].y, Ab = S.aux[rb].y;
                    // phase references at the end of ka (c2 = hi2) and the start of ka+1
                    // (c2 = lo2)
                    const float4 ana = S.anc[ra], anb = S.anc[rb];
                    const float ea = MF ? ana.z : fmaf(K.kh[0], ana.z, ana.x);
                    const float sb_ = MF ? anb.y : fmaf(K.kh[0], anb.y, anb.x);
                    ties += __popc(jp);
#if BF_JP_ALL
                    // the four decisions first and unconditionally: independent fp64 chains
                    // the scheduler can interleave (a receiver not in jp is computed from
                    // whatever its position slot holds and ignored)
                    bool wbj[R];
#pragma unroll
                    for (int j = 0; j < R; ++j) wbj[j] = junction_pick(J, P64(j));
#endif
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        if (!((jp >> j) & 1u)) continue;
#if BF_JP_ALL
                        const bool wb = wbj[j];
#else
                        const bool wb = junction_pick(J, P64(j));
#endif
                        const int rw = wb ? rb : ra;  // the winner's row (loads, not selects)
                        const float4 g1 = S.geo1[rw];
                        const float4 g2 = S.geo2[rw];
                        const float dl = fmaf(rx[j], g1.x, fmaf(ry[j], g1.y, rz[j] * g1.z));
                        q2j[j] = fmaf(-dl, dl, fmaf(g2.x, rx[j], fmaf(g2.y, ry[j], fmaf(g2.z, rz[j], g2.w + rr[j]))));
                        sj[j] = wb ? J.sb : J.sa;
                        Aj[j] = wb ? Ab : Aa;
                        bj[j][0] = wb ? sb_ : ea;
                        if constexpr (MF) pref[j] = wb ? rb : ra;
                        lvm |= 1u << j;
                    }
                }
#if BF_HIST
                if (pend) atomicAdd(&g_hist[__popc(surv) <= 2 ? 0 : 1], (unsigned long long)__popc(pend));
                if (jp) atomicAdd(&g_hist[3], (unsigned long long)__popc(jp));
#endif
                if (__any_sync(0xffffffffu, pend != 0))
                    exact_pending<NF, MF>(a, K, S, row0, r0, surv, pend, rx, ry, rz, rr, best, kb,
                                      Db, lane, sj, q2j, Aj, bj, pref, lvm, ties, w, P64);
            }
            // ---- shared tail: cutoff (kernels.py:384) and contributions (:386-399)
            nbp += __popc(lvm);
#if BF_ABL & 8
            if (lvm != 0x7u) continue;  // ablation: no evaluation
#endif
            double s64[WIDE ? R : 1];
            if constexpr (WIDE) {
                // wide patch: the winner's arc length, q^2 and axial phase from the fp64
                // rows and receiver positions (patch-local fp32 loses ~eps RW in r.d and
                // eps RW^2 in q^2); clamp as kernels.py:331-336, q^2 to the infinite line
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    s64[j] = 0.0;
                    if ((lvm >> j) & 1u) {
                        const int64_t g = S.rowinfo[pref[j]];
                        const double4 o = w.p0[g], d = w.p1[g];
                        const D3 P = P64(j);
                        const double wx = __dsub_rn(P.x, o.x), wy = __dsub_rn(P.y, o.y),
                                     wz = __dsub_rn(P.z, o.z);
                        const double proj = __dadd_rn(
                            __dadd_rn(__dmul_rn(wx, d.x), __dmul_rn(wy, d.y)), __dmul_rn(wz, d.z));
                        const double t = proj < 0.0 ? 0.0 : (proj > o.w ? o.w : proj);
                        const double ux = wx - proj * d.x, uy = wy - proj * d.y,
                                     uz = wz - proj * d.z;
                        s64[j] = __dadd_rn(d.w, t);  // kernels.py:344
                        sj[j] = (float)(s64[j] * K.invb64);
                        q2j[j] = (float)(ux * ux + uy * uy + uz * uz);
                    }
                }
            }
            // 1/(s'^2 + 1) and g' = q^2/(s'^2 + 1) of every receiver (s' = s/b; m2 = s^2 + b^2 =
            // b^2 (s'^2 + 1))
            float invj[R], gqj[R];
            unsigned tiny = 0;  // (TINY) receivers beyond the cutoff exponent: fp64
#pragma unroll
            for (int h = 0; h < R; h += 2) {
                const float2 m2p = fma2<PG>(pair(sj, h), pair(sj, h), bc2(1.f));  // m2/b^2
                invj[h] = rcp_nr(m2p.x);
                invj[h + 1] = rcp_nr(m2p.y);
                const float2 gp = mul2<PG>(pair(q2j, h), pair(invj, h));
                gqj[h] = gp.x;
                gqj[h + 1] = gp.y;
            }
            if constexpr (!MF) {
            {   // ex_re < -36 (kernels.py:384) as one mask (no cutoff: fp64 below)
                unsigned cutm = 0;
#pragma unroll
                for (int j = 0; j < R; ++j) cutm |= (gqj[j] > K.gcutq[0] ? 1u : 0u) << j;
                if (TINY) tiny = cutm & lvm;
                lvm &= ~cutm;
            }
            // receivers evaluated in groups of EVG (one branch, EVG independent chains),
            // as packed pairs
#pragma unroll
            for (int g = 0; g < R; g += EVG)
                if (lvm & (((1u << EVG) - 1u) << g)) {
#pragma unroll
                    for (int h = g; h < g + EVG; h += 2)
                        eval_pair2(K, pair(sj, h), pair(gqj, h), pair(invj, h), pair(Aj, h),
                                   make_float2(bj[h][0], bj[h + 1][0]), pre2[h >> 1],
                                   pim2[h >> 1], (lvm >> h) & 1u, (lvm >> (h + 1)) & 1u);
                }
            if constexpr (TINY) {
                if (tiny) {
#pragma unroll 1
                    for (int j = 0; j < R; ++j)
                        if ((tiny >> j) & 1u) {
                            const float sv = pick4(sj, j), gv = pick4(gqj, j);
                            const float bv = j == 0 ? bj[0][0] : j == 1 ? bj[1][0]
                                           : j == 2 ? bj[2][0] : bj[3][0];
                            tiny_contribution(K, 0, sv, gv, pick4(invj, j), pick4(Aj, j),
                                              fmaf(gv * K.khq[0], sv, bv), S.acc[R * lane + j][0]);
                        }
                }
            }
            evb += spread4(lvm | tiny);
            } else {
            // several frequencies: phase an'_f + kh_f X with X = c2 + g s (frequency
            // independent; WIDE: c2 = 0 and an'_f from the fp64 arc length), amplitude
            // A/m2 (s + i b) shared; the cutoff grows with omega, so each frequency is
            // evaluated only if some receiver of the warp is live for it
            float X[R], ainv[R];
#pragma unroll
            for (int j = 0; j < R; ++j) {
                // X = c2 + g s = c2 + g' s'/b
                X[j] = fmaf(gqj[j] * K.invb, sj[j], WIDE ? 0.f : bj[j][0]);
                ainv[j] = Aj[j] * invj[j];
            }
            // per frequency: partial sums in shared memory (no per-frequency registers)
#pragma unroll FUNROLL
            for (int f = 0; f < NF; ++f) {
                // fp32 / (TINY) fp64 receivers of frequency f: ex_re < -36 (kernels.py:384)
                const float gc = K.gcutq[f];
                unsigned cutm = 0;
#pragma unroll
                for (int j = 0; j < R; ++j) cutm |= (gqj[j] > gc ? 1u : 0u) << j;
                const unsigned lf = lvm & ~cutm, tf = TINY ? (lvm & cutm) : 0u;
                if (!__any_sync(0xffffffffu, (lf | tf) != 0)) {
                    // ascending frequencies: the cut radius shrinks with omega, so every
                    // later frequency is cut for the whole warp as well
                    if (K.ascending) break;
                    continue;
                }
                {
                    float ph[R];
                    // phase references an'_f of the receivers' rows: one load when the
                    // item is a single-segment one (the same row for every receiver)
                    float an[R];
                    if constexpr (WIDE) {
#pragma unroll
                        for (int j = 0; j < R; ++j) an[j] = frac_rad(K.kappa64[f] * s64[j]);
                    } else {
                        an[0] = S.ancf[f][pref[0]];
                        if ((surv & (surv - 1)) == 0) {
                            an[1] = an[2] = an[3] = an[0];
                        } else {
#pragma unroll
                            for (int j = 1; j < R; ++j) an[j] = S.ancf[f][pref[j]];
                        }
                    }
#pragma unroll
                    for (int h = 0; h < R; h += 2) {
                        float4 v = S.facc[f][h >> 1][lane];
                        ph[h] = fmaf(K.kh[f], X[h], an[h]);
                        ph[h + 1] = fmaf(K.kh[f], X[h + 1], an[h + 1]);
                        eval_freq(K, f, ph[h], gqj[h], sj[h], ainv[h], v.x, v.y, (lf >> h) & 1u);
                        eval_freq(K, f, ph[h + 1], gqj[h + 1], sj[h + 1], ainv[h + 1], v.z, v.w,
                                  (lf >> (h + 1)) & 1u);
                        S.facc[f][h >> 1][lane] = v;
                    }
                    evb += spread4(lf | tf);
                    if (TINY && tf) {
#pragma unroll 1
                        for (int j = 0; j < R; ++j)
                            if ((tf >> j) & 1u) {
                                tiny_contribution(
                                    K, f, pick4(sj, j), pick4(gqj, j), pick4(invj, j), pick4(Aj, j),
                                    pick4(ph, j),
                                    reinterpret_cast<double *>(
                                        w.part + (q * w.n_pad + sb + j) * NF + f));
                            }
                    }
                }
            }
            }
        }
        // flush fp32 partial sums into the fp64 accumulators (several frequencies: the
        // global fp64 partials every BF_FLUSHN-th chunk and after the last one)
        const bool flush64 = !MF || (++nch & (BF_FLUSHN - 1)) == 0 || cur >= n_items;
#pragma unroll
        for (int j = 0; j < R; ++j) {
            if (!MF) {
                S.acc[R * lane + j][0][0] += (double)((j & 1) ? pre2[j >> 1].y : pre2[j >> 1].x);
                S.acc[R * lane + j][0][1] += (double)((j & 1) ? pim2[j >> 1].y : pim2[j >> 1].x);
            } else if (flush64) {
                if (j < nvalid) {
                    double2 *pp = w.part + (q * w.n_pad + sb + j) * NF;
#pragma unroll
                    for (int f = 0; f < NF; ++f) {
                        const double2 v = pp[f];
                        const float4 c4 = S.facc[f][j >> 1][lane];
                        const float2 c = (j & 1) ? make_float2(c4.z, c4.w) : make_float2(c4.x, c4.y);
                        pp[f] = make_double2(v.x + (double)c.x, v.y + (double)c.y);
                    }
                }
                if (j & 1) {
#pragma unroll
                    for (int f = 0; f < NF; ++f) S.facc[f][j >> 1][lane] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
            if (j & 1) pre2[j >> 1] = pim2[j >> 1] = make_float2(0.f, 0.f);  // pair flushed
        }
#pragma unroll
        for (int j = 0; j < R; ++j) S.evc[R * lane + j] += (evb >> (8 * j)) & 0xffu;
        evb = 0;
        __syncwarp();  // every lane is done with this chunk's shared rows
    }
    // ---- the unit's partial sums (fp64) for fold_kernel, which adds the beam
    //      ranges in ascending order: deterministic, kernels.py:358-359 continuation
#pragma unroll
    for (int j = 0; j < R; ++j) {
        if (j >= nvalid) continue;
        const int64_t slot = q * w.n_pad + sb + j;
        if (!MF) w.part[slot] = make_double2(S.acc[R * lane + j][0][0], S.acc[R * lane + j][0][1]);
        w.part_ev[slot] = S.evc[R * lane + j];
    }
    ties = __reduce_add_sync(0xffffffffu, ties);
    nbp = __reduce_add_sync(0xffffffffu, nbp);
    if (lane == 0) {
        S.cnt[0] += ties;
        S.cnt[1] += nbp;
    }
}

__device__ __forceinline__ bool wide_patch(const Fp32Work &w, int64_t p) {
    const float RW = (float)w.pcen[p].w;
    return !(RW * w.wide_k <= 1.f && RW * RW * w.wide_q <= 1.f);
}

// One launch per patch class, on two streams: WIDE = false takes queue positions
// [0, n_units - n_wide), WIDE = true the rest (unit_keys_kernel sorts wide patches last).
template <int NF, bool WIDE, bool TINY>
#ifndef BF_MINB_MF
#define BF_MINB_MF 4
#endif
__global__ void __launch_bounds__(32 * WARPS_OF<(NF > 1 || WIDE)>,
                                  (NF == 1 && !WIDE ? BF_MINB : NF <= 5 ? BF_MINB_MF : 2))
    gbs_fp32_kernel(const GbsArgs a, const Tiling tl, const Fp32Work w, const Fp32Consts K,
                    GbsStats *stats) {
    constexpr bool MF = NF > 1 || WIDE;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpSmem<NF, MF> &S = reinterpret_cast<WarpSmem<NF, MF> *>(smem_raw)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const unsigned n_units = (unsigned)(w.n_patches * w.n_ranges);
    const unsigned n_wide = *w.n_wide;
    if (WIDE && n_wide == 0) return;  // (uniform over the grid) no atomics, no statistics
    const unsigned n_split = n_units - n_wide;
    const unsigned u0 = WIDE ? n_split : 0u, u1 = WIDE ? n_units : n_split;
    const unsigned n_patches = (unsigned)w.n_patches;
    if (lane < 8) S.cnt[lane] = 0;
    __syncwarp();
    for (;;) {
        unsigned u = 0;
        if (lane == 0) u = u0 + atomicAdd(w.unit_ctr + (WIDE ? 1 : 0), 1u);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= u1) break;
        const unsigned id = (unsigned)w.unit_order[u];  // longest-first, see unit_keys_kernel
        const unsigned q = id / n_patches;
        const unsigned p = id - q * n_patches;
#if BF_UNIT_TIMES
        const long long c0 = clock64();
#endif
        run_unit<NF, WIDE, TINY>(a, tl, w, K, S, p, q, lane, stats);
#if BF_UNIT_TIMES
        if (lane == 0 && g_unit_cycles) g_unit_cycles[id] = clock64() - c0;
#endif
    }
    // the CTA's warp counters summed in shared memory, then one set of atomics per CTA
    // (per-warp atomics on the same eight addresses serialised into a tail of ~10 us)
    __syncthreads();
    if (threadIdx.x < 8) {
        unsigned long long v = 0;
#pragma unroll
        for (int wi = 0; wi < WARPS_OF<MF>; ++wi)
            v += reinterpret_cast<WarpSmem<NF, MF> *>(smem_raw)[wi].cnt[threadIdx.x];
        unsigned long long *dst = threadIdx.x == 0 ? &stats->tie_pairs
                                : threadIdx.x == 1 ? &stats->nb_pairs
                                : threadIdx.x < 6  ? &stats->paths[threadIdx.x - 2]
                                : threadIdx.x == 6 ? &stats->live_pairs
                                                   : &stats->live_pair_segs;
        if (v) atomicAdd(dst, v);
    }
}

// ------------------------------------------------------------ preparation ----

// Padded reference bundle (beamtrace.py:274-288) -> compact rows: thread per padded row,
// rows k < n_segs[b] go to start[b] + k.  p0 = (o, len), p1 = (d, s0) are exact fp64
// copies; amp = (float)(phi sqrt(c)/(2 pi c) * refl * w_b) (kernels.py:388,397).
__global__ void rows_pack_kernel(const GbsArgs a, double amp_scale, const int64_t *start,
                                 double4 *p0, double4 *p1, float *amp) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= a.n_beams * a.max_seg) return;
    const int64_t b = row / a.max_seg;
    const int64_t k = row - b * a.max_seg;
    const int64_t dst = start[b] + k;
    if (dst >= start[b + 1]) return;
    p0[dst] = make_double4(a.seg_origin[3 * row], a.seg_origin[3 * row + 1],
                           a.seg_origin[3 * row + 2], a.seg_len[row]);
    p1[dst] = make_double4(a.seg_dir[3 * row], a.seg_dir[3 * row + 1], a.seg_dir[3 * row + 2],
                           a.seg_s0[row]);
    amp[dst] = (float)(amp_scale * a.seg_refl[row] * a.weights[b]);
}

// start[b + 1] = n_segs[b] clamped to [0, max_seg] (the scan input; start[0] = base).
__global__ void rows_count_kernel(const int32_t *n_segs, int64_t n_beams, int64_t max_seg,
                                  int64_t base, int64_t *cnt) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b > n_beams) return;
    if (b == n_beams) {
        cnt[0] = base;
        return;
    }
    int64_t n = n_segs[b];
    n = n < 0 ? 0 : (n > max_seg ? max_seg : n);
    cnt[b + 1] = n;
}

// Beams [b0, b0 + nb) of resident compact rows -> a group's own rows starting at 0:
// start rebased, rows copied (thread i: start entry i <= nb and row i < nb * max_seg).
__global__ void rows_slice_kernel(const Rows src, int64_t b0, int64_t nb, int64_t *start,
                                  double4 *p0, double4 *p1, float *amp) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t base = src.start[b0];
    if (i <= nb) start[i] = src.start[b0 + i] - base;
    if (i < nb * src.max_seg) {
        const int64_t row = base + i;
        if (row < src.start[b0 + nb]) {
            p0[i] = src.p0[row];
            p1[i] = src.p1[row];
            amp[i] = src.amp[row];
        }
    }
}

// One warp per patch: fp64 bounding-box centre c_P, patch-local r = p - c_P in
// fp32 (w = |r|^2) and the patch radius (max |r|, padded).
__global__ void patch_kernel(const double *obs, int64_t n, const int32_t *perm,
                             int64_t n_patches, float4 *prl, double4 *pos64, double4 *pcen,
                             float4 *pbox) {
    const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (p >= n_patches) return;
    double px[R], py[R], pz[R];
    bool valid[R];
    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int64_t si = p * PATCH + R * lane + j;
        valid[j] = si < n;
        px[j] = py[j] = pz[j] = 0.0;
        if (valid[j]) {
            const int64_t oi = perm[si];
            px[j] = obs[3 * oi];
            py[j] = obs[3 * oi + 1];
            pz[j] = obs[3 * oi + 2];
            pos64[si] = make_double4(px[j], py[j], pz[j], 0.0);
            mn[0] = fmin(mn[0], px[j]); mx[0] = fmax(mx[0], px[j]);
            mn[1] = fmin(mn[1], py[j]); mx[1] = fmax(mx[1], py[j]);
            mn[2] = fmin(mn[2], pz[j]); mx[2] = fmax(mx[2], pz[j]);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            mn[d] = fmin(mn[d], __shfl_xor_sync(0xffffffffu, mn[d], o));
            mx[d] = fmax(mx[d], __shfl_xor_sync(0xffffffffu, mx[d], o));
        }
    const double cx = 0.5 * (mn[0] + mx[0]), cy = 0.5 * (mn[1] + mx[1]),
                 cz = 0.5 * (mn[2] + mx[2]);
    float q = 0.f, hx = 0.f, hy = 0.f, hz = 0.f;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        if (!valid[j]) continue;
        const float rx = (float)(px[j] - cx), ry = (float)(py[j] - cy), rz = (float)(pz[j] - cz);
        const float r2 = rx * rx + ry * ry + rz * rz;
        prl[p * PATCH + R * lane + j] = make_float4(rx, ry, rz, r2);
        q = fmaxf(q, r2);
        hx = fmaxf(hx, fabsf(rx));
        hy = fmaxf(hy, fabsf(ry));
        hz = fmaxf(hz, fabsf(rz));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        q = fmaxf(q, __shfl_xor_sync(0xffffffffu, q, o));
        hx = fmaxf(hx, __shfl_xor_sync(0xffffffffu, hx, o));
        hy = fmaxf(hy, __shfl_xor_sync(0xffffffffu, hy, o));
        hz = fmaxf(hz, __shfl_xor_sync(0xffffffffu, hz, o));
    }
    const float RW = sqrtf(q) * 1.0001f + 1e-4f;
    if (lane == 0) {
        pcen[p] = make_double4(cx, cy, cz, (double)RW);
        pbox[p] = make_float4(hx * 1.0001f + 1e-4f, hy * 1.0001f + 1e-4f, hz * 1.0001f + 1e-4f, RW);
    }
}

// acc[oi] += sum over beam ranges q (ascending) of the units' partials; evals alike.  The
// adds stay one sequential chain per receiver, acc + v_0 + v_1 + ... (so beam groups and
// chunk plans that split the same ranges give the same bits), but a block of 32 receivers
// stages the partials through shared memory with FOLD_G threads per receiver: FOLD_G times
// the loads in flight of a thread per receiver (small calls are latency bound here).
constexpr int FOLD_G = 8, FOLD_Q = 64;
__global__ void __launch_bounds__(32 * FOLD_G)
    fold_kernel(const Tiling tl, const Fp32Work w, int nf, int64_t stride, double *acc,
                int64_t *evals) {
    __shared__ double2 vals[FOLD_Q][32];
    __shared__ int rev[FOLD_G][32];
    const int x = threadIdx.x, g = threadIdx.y;
    const int64_t si = (int64_t)blockIdx.x * 32 + x;
    const bool ok = si < tl.n;
    const int64_t oi = ok ? tl.perm[si] : 0;
    for (int f = 0; f < nf; ++f) {
        double re = 0.0, im = 0.0;
        if (g == 0 && ok) {
            re = acc[2 * (oi * stride + f)];
            im = acc[2 * (oi * stride + f) + 1];
        }
        for (int64_t qb = 0; qb < w.n_ranges; qb += FOLD_Q) {
            const int nq = (int)(w.n_ranges - qb < FOLD_Q ? w.n_ranges - qb : FOLD_Q);
            if (ok)
                for (int j = g; j < nq; j += FOLD_G)
                    vals[j][x] = w.part[((qb + j) * w.n_pad + si) * nf + f];
            __syncthreads();
            if (g == 0 && ok)
                for (int j = 0; j < nq; ++j) {
                    re += vals[j][x].x;
                    im += vals[j][x].y;
                }
            __syncthreads();
        }
        if (g == 0 && ok) {
            acc[2 * (oi * stride + f)] = re;
            acc[2 * (oi * stride + f) + 1] = im;
        }
    }
    int ev = 0;  // integer: any order
    if (ok)
        for (int64_t q = g; q < w.n_ranges; q += FOLD_G) ev += w.part_ev[q * w.n_pad + si];
    rev[g][x] = ev;
    __syncthreads();
    if (g == 0 && ok) {
        int64_t e = 0;
#pragma unroll
        for (int j = 0; j < FOLD_G; ++j) e += rev[j][x];
        evals[oi] += e;
    }
}

// Sort keys of the unit queue: longest-first in half-octave buckets of the unit's
// candidate count, range-major inside a bucket (concurrent units share a beam range, so
// its rows stay L2-resident).  A unit near the source can run for ~10 ms; started late
// it would be the launch's tail, which matters once ranks hold few receivers each.
// Units of WIDE patches sort last and are summed by the wide-patch kernel: with
// patch-local fp32 geometry the nearest point's r.d carries an error ~eps RW and q^2
// ~eps RW^2, which with strong cancellation between beams (a receiver 50 dB below the
// field maximum) reaches the 0.01 dB gate once kappa RW is tens of turns (sparse
// receiver sets); the wide kernel recomputes s, q^2 and the phase in fp64.
__device__ __forceinline__ unsigned unit_key(const Fp32Work &w, const int64_t *counts,
                                             int64_t q, int64_t p, bool *wide) {
    const int64_t tile = p / (TILE / PATCH);
    const uint64_t c = (uint64_t)counts[tile * w.n_ranges + q] + 1;
    const int msb = 63 - __clzll((long long)c);
    const int bucket = 2 * msb + (msb > 0 ? (int)((c >> (msb - 1)) & 1) : 0);  // < 128
    *wide = wide_patch(w, p);
    // 14 significant bits (wide, 7-bit bucket, range q < 64): the radix sort needs 2
    // passes (8-bit digits) instead of 5 over 40 bits
    return ((unsigned)*wide << 13) | ((unsigned)(127 - bucket) << 6) | (unsigned)q;
}

__global__ void unit_keys_kernel(const Tiling tl, const Fp32Work w, const int64_t *counts,
                                 uint64_t *keys, int32_t *vals) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= w.n_patches * w.n_ranges) return;
    bool wide;
    const int64_t q = u / w.n_patches;
    keys[u] = unit_key(w, counts, q, u - q * w.n_patches, &wide);
    if (wide) atomicAdd(w.n_wide, 1u);
    vals[u] = (int32_t)u;
}

// Small calls (<= SMALL_QUEUE_N units): the keys, a counting sort and the wide-unit count
// in one CTA and one launch (instead of the keys kernel and a radix sort).  The sort key is
// the unit key without its range bits (wide, bucket: 256 values); units enter it in
// ascending u = q n_patches + p, so inside a bucket the order stays range-major up to the
// interleaving of concurrent warps.  That order only decides which warp takes a unit
// first, never a result (every unit writes its own partial slot, fold_kernel adds them in
// range order).
constexpr int SQ_T = 1024, SQ_BINS = 256;
__global__ void __launch_bounds__(SQ_T)
    small_queue_kernel(const Fp32Work w, const int64_t *counts, int32_t *order) {
    extern __shared__ unsigned char sq_key[];  // per unit: wide << 7 | (127 - bucket)
    __shared__ int hist[SQ_BINS];
    __shared__ unsigned nwide;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nu = (int)(w.n_patches * w.n_ranges);
    if (tid < SQ_BINS) hist[tid] = 0;
    if (tid == 0) nwide = 0;
    __syncthreads();
    unsigned nw = 0;
    // keys first (independent global loads, unrolled so several are in flight; 32-bit
    // index math: nu <= SMALL_QUEUE_N), then the histogram with one shared-memory atomic
    // per distinct key of a warp (the 32 units of a warp are mostly one bucket)
    const int np = (int)w.n_patches;
#pragma unroll 4
    for (int u = tid; u < nu; u += SQ_T) {
        bool wide;
        const int q = u / np;
        sq_key[u] = (unsigned char)(unit_key(w, counts, q, u - q * np, &wide) >> 6);
        nw += wide;
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    for (int u0 = wid * 32; u0 < nu; u0 += SQ_T) {
        const int u = u0 + lane;
        const unsigned live = __ballot_sync(0xffffffffu, u < nu);
        const unsigned k = u < nu ? sq_key[u] : 0xffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, k) & live;
        if (u < nu && (peers & lt) == 0) atomicAdd(&hist[k], __popc(peers));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) nw += __shfl_xor_sync(0xffffffffu, nw, o);
    if (lane == 0 && nw) atomicAdd(&nwide, nw);
    __syncthreads();
    if (wid == 0) {  // exclusive scan of the 256 counters, rows of 32
        int carry = 0;
#pragma unroll
        for (int r = 0; r < SQ_BINS / 32; ++r) {
            const int v = hist[32 * r + lane];
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            hist[32 * r + lane] = carry + incl - v;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    __syncthreads();
    for (int u0 = wid * 32; u0 < nu; u0 += SQ_T) {
        const int u = u0 + lane;
        const unsigned live = __ballot_sync(0xffffffffu, u < nu);
        const unsigned k = u < nu ? sq_key[u] : 0xffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, k) & live;
        const int leader = __ffs(peers) - 1;
        int base = 0;
        if (u < nu && lane == leader) base = atomicAdd(&hist[k], __popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader < 0 ? 0 : leader);
        if (u < nu) order[base + __popc(peers & lt)] = u;
    }
    if (tid == 0) {  // the two queue heads and the wide count (w.n_wide = w.unit_ctr + 2)
        w.unit_ctr[0] = 0u;
        w.unit_ctr[1] = 0u;
        *w.n_wide = nwide;
    }
}

// One warp per (tile, beam range): ascending candidate beams with their segment
// counts, (n_segs - 1) << 27 | compact row of segment 0, at the scanned offset.
__global__ void wl_compact_kernel(const Tiling tl, const Fp32Work w) {
    const int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (u >= tl.n_tiles * w.n_ranges) return;
    const int64_t tile = u / w.n_ranges, q = u - tile * w.n_ranges;
    const int64_t w0 = q * w.range_beams / 32;
    const int64_t w1 = min(tl.wl_words, (q + 1) * w.range_beams / 32);
    const uint32_t *bits = tl.wl_tight + tile * tl.wl_words;
    uint32_t *out = w.wl_items + w.wl_off[u];
    int64_t base = 0;
    for (int64_t i0 = w0; i0 < w1; i0 += 32) {
        const int64_t i = i0 + lane;
        unsigned m = i < w1 ? bits[i] : 0u;
        const int c = __popc(m);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        int64_t pos = base + incl - c;
        for (; m; m &= m - 1) {
            const int64_t beam = 32 * i + __ffs(m) - 1;
            const int64_t r0 = w.start[beam];
            const uint32_t ns = (uint32_t)(w.start[beam + 1] - r0);
            out[pos++] = ((ns - 1u) << 27) | (uint32_t)r0;
        }
        base += __shfl_sync(0xffffffffu, incl, 31);
    }
}

template <int NF, bool WIDE, bool TINY>
int launch_class(const GbsArgs &a, const Tiling &t, const Fp32Work &w, const Fp32Consts &K,
                 GbsStats *stats, cudaStream_t st) {
    constexpr bool MF = NF > 1 || WIDE;
    constexpr int NW = WARPS_OF<MF>;
    const size_t smem = NW * sizeof(WarpSmem<NF, MF>);
    // per-device launch geometry, computed once (attribute + occupancy queries cost host time
    // on every call otherwise); a benign race writes the same values
    constexpr int MAXDEV = 64;
    static int grid_cache[MAXDEV] = {};
    int dev = 0;
    BF_TRY_CUDA(cudaGetDevice(&dev));
    if (dev >= MAXDEV) return fail(BF_ENODEV, "device index %d >= %d", dev, MAXDEV);
    if (grid_cache[dev] == 0) {
        BF_TRY_CUDA(cudaFuncSetAttribute(gbs_fp32_kernel<NF, WIDE, TINY>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int sms = 0, per_sm = 0;
        BF_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        BF_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, gbs_fp32_kernel<NF, WIDE, TINY>, 32 * NW, smem));
        if (per_sm < 1)
            return fail(BF_ECUDA, "fp32 kernel does not fit on an SM (smem %zu)", smem);
        if (getenv("BF_DEBUG_STATS"))
            fprintf(stderr, "bf fp32 kernel%s: %zu B shared per CTA (%zu per warp), %d CTAs/SM\n",
                    WIDE ? " (wide patches)" : "", smem, sizeof(WarpSmem<NF, MF>), per_sm);
        grid_cache[dev] = sms * per_sm;
    }
    const int64_t units = w.n_patches * w.n_ranges;
    int64_t grid = grid_cache[dev];
    const int64_t need = (units + NW - 1) / NW;
    if (grid > need) grid = need;
    gbs_fp32_kernel<NF, WIDE, TINY><<<(unsigned)grid, 32 * NW, smem, st>>>(a, t, w, K, stats);
    note_launch();
    BF_TRY_CUDA(cudaGetLastError());
    return BF_OK;
}

// The wide-patch kernel goes first on the auxiliary stream; the common kernel's CTAs
// take the SM slots as the wide ones retire (no tail of a second sequential launch).
// Both are always launched: the wide-unit count is on the device (unit_keys_kernel), and
// with none every warp of the wide kernel exits after one atomic (no host round trip).
template <int NF>
int launch_nf(const GbsArgs &a, const Tiling &t, const Fp32Work &w, const Fp32Consts &K,
              GbsStats *stats, const StreamPair &sp) {
#if BF_HIST
    {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbolAsync(g_hist, z, sizeof(z), 0, cudaMemcpyHostToDevice, sp.st);
    }
#endif
    BF_TRY_CUDA(cudaEventRecord(sp.fork, sp.st));
    BF_TRY_CUDA(cudaStreamWaitEvent(sp.aux, sp.fork, 0));
    if (a.use_cutoff) {
        BF_TRY((launch_class<NF, true, false>(a, t, w, K, stats, sp.aux)));
        BF_TRY((launch_class<NF, false, false>(a, t, w, K, stats, sp.st)));
    } else {  // kernels with the fp64 path for pairs beyond the cutoff exponent
        BF_TRY((launch_class<NF, true, true>(a, t, w, K, stats, sp.aux)));
        BF_TRY((launch_class<NF, false, true>(a, t, w, K, stats, sp.st)));
    }
    BF_TRY_CUDA(cudaEventRecord(sp.join, sp.aux));
    BF_TRY_CUDA(cudaStreamWaitEvent(sp.st, sp.join, 0));
#if BF_UNIT_TIMES
    {
        const int64_t nu = w.n_patches * w.n_ranges;
        long long *buf = nullptr;
        cudaStreamSynchronize(sp.st);
        cudaMalloc(&buf, 8 * nu);
        cudaMemcpyToSymbol(g_unit_cycles, &buf, sizeof(buf));
        cudaMemsetAsync(w.unit_ctr, 0, sizeof(unsigned), sp.st);
        launch_class<NF, false, false>(a, t, w, K, stats, sp.st);  // re-run, timed per unit
        cudaStreamSynchronize(sp.st);
        std::vector<long long> h(nu);
        cudaMemcpy(h.data(), buf, 8 * nu, cudaMemcpyDeviceToHost);
        long long sum = 0;
        for (long long v : h) sum += v;
        fprintf(stderr, "bf unit times: %lld units, %lld cycles, err %s\n", (long long)nu, sum,
                cudaGetErrorString(cudaGetLastError()));
        long long *nul = nullptr;
        cudaMemcpyToSymbol(g_unit_cycles, &nul, sizeof(nul));
        cudaFree(buf);
        if (const char *out = getenv("BF_UNIT_TIMES_OUT")) {
            FILE *f = fopen(out, "wb");
            const int64_t hdr[3] = {w.n_patches, w.n_ranges, TILE / PATCH};
            fwrite(hdr, 8, 3, f);
            fwrite(h.data(), 8, nu, f);
            fclose(f);
        }
    }
#endif
#if BF_HIST
    {
        unsigned long long h[16];
        cudaMemcpyFromSymbolAsync(h, g_hist, sizeof(h), 0, cudaMemcpyDeviceToHost, sp.st);
        cudaStreamSynchronize(sp.st);
        fprintf(stderr, "bf hist: items all-cut %llu culled %llu\n", h[4], h[5]);
        fprintf(stderr, "bf hist: pend(<=2 surv) %llu pend(>=3 surv) %llu exact rounds %llu junction %llu\n", h[0], h[1], h[2], h[3]);
        fprintf(stderr, "bf hist: multi items %llu sum n %llu sum n_lane_union %llu union==1 %llu lanes single %llu sum max lane n %llu; n=2 %llu n=3 %llu n=4 %llu n>=5 %llu\n", h[9], h[6], h[7], h[8], h[10], h[11], h[12], h[13], h[14], h[15]);
    }
#endif
    return BF_OK;
}

Fp32Consts make_consts(const GbsArgs &a) {
    Fp32Consts K;
    const double two_pi = 2.0 * 3.141592653589793;
    double wmin = INFINITY;
    for (int f = 0; f < BF_MAXF; ++f) {
        const double w = f < a.nf ? a.omegas[f] : 0.0;
        if (f < a.nf && w < wmin) wmin = w;
        K.kappa64[f] = w / (two_pi * a.c);
        K.omega[f] = (float)w;
        K.omrel[f] = f < a.nf ? (float)(w / a.omegas[0]) : 0.f;
        K.lomrel[f] = f < a.nf && w > 0 ? (float)log2(w / a.omegas[0]) : 0.f;
        K.gcut[f] = w > 0 ? (float)(72.0 * a.c / (w * a.width_b)) : INFINITY;
        K.kh[f] = (float)(w * 0.5 / a.c);
        K.nhkbl2e64[f] = -(w * 0.5 / a.c) * a.width_b * 1.4426950408889634;
        K.nhkbl2e[f] = (float)K.nhkbl2e64[f];
    }
    K.ascending = 1;
    for (int f = 1; f < a.nf; ++f)
        if (!(K.gcut[f] <= K.gcut[f - 1])) K.ascending = 0;
    K.b = (float)a.width_b;
    K.invb64 = 1.0 / a.width_b;
    K.hinvb = (float)(0.5 / a.width_b);
    K.invb = (float)(1.0 / a.width_b);
    for (int f = 0; f < BF_MAXF; ++f) {
        const double b2 = a.width_b * a.width_b;
        K.gcutq[f] = K.gcut[f] == INFINITY ? INFINITY : (float)((double)K.gcut[f] * b2);
        K.khq[f] = (float)((double)K.kh[f] / a.width_b);
        K.nhkq64[f] = K.nhkbl2e64[f] / b2;
        K.nhkq[f] = (float)K.nhkq64[f];
    }
    K.b2 = (float)(a.width_b * a.width_b);
    K.b2_64 = a.width_b * a.width_b;
    K.amp_scale = a.phi_amp * sqrt(a.c) / (two_pi * a.c);
    // Cut radius for the patch prepass; without the cutoff nothing is ever cut.
    K.rcut_scale = (a.use_cutoff && wmin > 0) ? 72.0 * a.c / (wmin * a.width_b) : INFINITY;
    K.rscale = (float)K.rcut_scale;
    return K;
}

}  // namespace

int gbs_fp32_tile() { return TILE; }
int gbs_fp32_patch() { return PATCH; }

// Beams per range unit: depends on the beam and frequency counts only, so the
// per-receiver summation order (and result bits) does not depend on how receivers are
// sharded over ranks.
int64_t gbs_fp32_range_beams(int64_t n_beams, int nf) {
    // BF_RANGES ranges for one frequency, fewer with several (the partial buffer holds
    // ranges x receivers x frequencies complex values)
    // (small calls get 32-beam ranges: more (patch, range) units to spread over the SMs)
    const int64_t ranges = BF_RANGES / nf > 8 ? BF_RANGES / nf : 8;
    int64_t rb = (n_beams + ranges - 1) / ranges;
    rb = (rb + 31) / 32 * 32;
    return rb < 32 ? 32 : rb;
}

int launch_rows_count(const int32_t *n_segs, int64_t n_beams, int64_t max_seg, int64_t base,
                      int64_t *cnt, cudaStream_t st) {
    rows_count_kernel<<<(unsigned)((n_beams + 1 + 255) / 256), 256, 0, st>>>(n_segs, n_beams,
                                                                             max_seg, base, cnt);
    note_launch();
    BF_TRY_CUDA(cudaGetLastError());
    return BF_OK;
}

int launch_rows_slice(const Rows &src, int64_t b0, int64_t nb, int64_t *start, double4 *p0,
                      double4 *p1, float *amp, cudaStream_t st) {
    const int64_t n = std::max<int64_t>(nb + 1, nb * src.max_seg);
    rows_slice_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src, b0, nb, start, p0, p1,
                                                                   amp);
    note_launch();
    BF_TRY_CUDA(cudaGetLastError());
    return BF_OK;
}

int launch_rows_pack(const GbsArgs &a, const int64_t *start, double4 *p0, double4 *p1,
                     float *amp, cudaStream_t st) {
    const int64_t rows = a.n_beams * a.max_seg;
    if (rows <= 0) return BF_OK;
    const double amp_scale = a.phi_amp * sqrt(a.c) / (2.0 * 3.141592653589793 * a.c);
    rows_pack_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(a, amp_scale, start, p0, p1,
                                                                     amp);
    note_launch();
    BF_TRY_CUDA(cudaGetLastError());
    return BF_OK;
}

int launch_fp32_patches(const GbsArgs &a, const Tiling &t, Fp32Work &w, cudaStream_t st) {
    if (w.n_patches > 0) {
        patch_kernel<<<(unsigned)((w.n_patches * 32 + 127) / 128), 128, 0, st>>>(
            a.obs, t.n, t.perm, w.n_patches, w.prl, w.pos64, w.pcen, w.pbox);
        note_launch();
    }
    BF_TRY_CUDA(cudaGetLastError());
    return BF_OK;
}

int launch_fp32_unit_keys(const Tiling &t, const Fp32Work &w,
                          const int64_t *counts, uint64_t *keys, int32_t *vals, cudaStream_t st) {
    const int64_t nu = w.n_patches * w.n_ranges;
    if (nu > 0) {
        unit_keys_kernel<<<(unsigned)((nu + 255) / 256), 256, 0, st>>>(t, w, counts, keys, vals);
        note_launch();
    }
    BF_TRY_CUDA(cudaGetLastError());
    return BF_OK;
}

int launch_fp32_small_queue(const Fp32Work &w, const int64_t *counts, int32_t *order,
                            cudaStream_t st) {
    const int64_t nu = w.n_patches * w.n_ranges;
    if (nu <= 0) return BF_OK;
    if (nu > SMALL_QUEUE_N) return fail(BF_EINVAL, "small queue of %lld units", (long long)nu);
    const size_t smem = SMALL_QUEUE_N;  // one key byte per unit
    constexpr int MAXDEV = 64;
    static bool attr_set[MAXDEV] = {};
    int dev = 0;
    BF_TRY_CUDA(cudaGetDevice(&dev));
    if (dev >= MAXDEV) return fail(BF_ENODEV, "device index %d >= %d", dev, MAXDEV);
    if (!attr_set[dev]) {
        BF_TRY_CUDA(cudaFuncSetAttribute(small_queue_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_set[dev] = true;
    }
    small_queue_kernel<<<1, SQ_T, smem, st>>>(w, counts, order);
    note_launch();
    BF_TRY_CUDA(cudaGetLastError());
    return BF_OK;
}

int launch_fp32_wl_compact(const Tiling &t, const Fp32Work &w, cudaStream_t st) {
    const int64_t nu = t.n_tiles * w.n_ranges;
    if (nu > 0) {
        wl_compact_kernel<<<(unsigned)((nu * 32 + 127) / 128), 128, 0, st>>>(t, w);
        note_launch();
    }
    BF_TRY_CUDA(cudaGetLastError());
    return BF_OK;
}

int launch_gbs_fp32(const GbsArgs &a, const Tiling &t, const Fp32Work &w, GbsStats *d_stats,
                    const StreamPair &st) {
    if (t.n <= 0 || a.nf <= 0 || w.n_ranges <= 0) return BF_OK;
    const Fp32Consts K = make_consts(a);
    switch (a.nf) {
        case 1: return launch_nf<1>(a, t, w, K, d_stats, st);
        case 2: return launch_nf<2>(a, t, w, K, d_stats, st);
        case 3: return launch_nf<3>(a, t, w, K, d_stats, st);
        case 4: return launch_nf<4>(a, t, w, K, d_stats, st);
        case 5: return launch_nf<5>(a, t, w, K, d_stats, st);
        case 6: return launch_nf<6>(a, t, w, K, d_stats, st);
        case 7: return launch_nf<7>(a, t, w, K, d_stats, st);
        case 8: return launch_nf<8>(a, t, w, K, d_stats, st);
        default: return fail(BF_EINVAL, "nf=%d outside 1..%d", a.nf, BF_MAXF);
    }
}

int launch_fp32_fold(const GbsArgs &a, const Tiling &t, const Fp32Work &w, cudaStream_t st) {
    if (t.n <= 0 || w.n_ranges <= 0) return BF_OK;
    fold_kernel<<<(unsigned)((t.n + 31) / 32), dim3(32, FOLD_G), 0, st>>>(
        t, w, a.nf, a.acc_stride, a.acc, a.evals);
    note_launch();
    BF_TRY_CUDA(cudaGetLastError());
    return BF_OK;
}

}  // namespace bf
