// exact_fp64.cu -- fp64 kernels that follow the reference operation order.
//
// THIS FILE IS COMPILED WITH -fmad=false: every + and * rounds separately,
// exactly as the numba reference (kernels.py:20, fastmath=False; its x86 asm
// has no vfmadd).  Division and sqrt are IEEE (nvcc defaults -prec-div=true,
// -prec-sqrt=true), so everything except exp/cos/sin (CUDA libdevice, <=2 ulp
// vs glibc) is bit-identical to the reference.
//
//   gbs_fp64_kernel   kernels.gbs_accumulate      kernels.py:352-399  (oracle mode)
//   nearest_kernel    kernels.nearest_on_segments kernels.py:304-349
//   trace_kernel      kernels.trace_one/range     kernels.py:143-301 (nearest hit of
//                     bvh_nearest, kernels.py:54-116, by exhaustive search; same
//                     (t, triangle index) lexicographic minimum)
//   finalize_kernel   parallel.py:343-344 + gbs.spl (gbs.py:39-46)
#include <math.h>

#include "common.cuh"

namespace bf {
namespace {

struct Nearest {
    int k;
    double s, q1, q2, refl;
    bool behind;
};

// kernels.py:304-349, operation for operation.  Rows are read through the
// read-only path; all lanes of a warp read the same row (broadcast).
__device__ __forceinline__ Nearest nearest_exact(const GbsArgs &a, int64_t base, int ns,
                                                 double px, double py, double pz) {
    double best_d2 = INFINITY;
    Nearest r;
    r.k = -1;
    r.s = 0.0;
    r.q1 = 0.0;
    r.q2 = 0.0;
    r.refl = 1.0;
    r.behind = false;
    for (int k = 0; k < ns; ++k) {
        const int64_t row = base + k;
        const double ox = __ldg(a.seg_origin + 3 * row + 0);
        const double oy = __ldg(a.seg_origin + 3 * row + 1);
        const double oz = __ldg(a.seg_origin + 3 * row + 2);
        const double dx = __ldg(a.seg_dir + 3 * row + 0);
        const double dy = __ldg(a.seg_dir + 3 * row + 1);
        const double dz = __ldg(a.seg_dir + 3 * row + 2);
        const double wx = px - ox, wy = py - oy, wz = pz - oz;
        const double proj = wx * dx + wy * dy + wz * dz;
        double t = proj;
        const double len = __ldg(a.seg_len + row);
        if (t < 0.0)
            t = 0.0;
        else if (t > len)
            t = len;
        const double vx = wx - t * dx, vy = wy - t * dy, vz = wz - t * dz;
        const double d2 = vx * vx + vy * vy + vz * vz;
        if (d2 < best_d2) {
            best_d2 = d2;
            r.k = k;
            r.s = __ldg(a.seg_s0 + row) + t;
            r.q1 = vx * __ldg(a.seg_e1 + 3 * row + 0) + vy * __ldg(a.seg_e1 + 3 * row + 1) +
                   vz * __ldg(a.seg_e1 + 3 * row + 2);
            r.q2 = vx * __ldg(a.seg_e2 + 3 * row + 0) + vy * __ldg(a.seg_e2 + 3 * row + 1) +
                   vz * __ldg(a.seg_e2 + 3 * row + 2);
            r.refl = __ldg(a.seg_refl + row);
            r.behind = (k == 0) && (t == 0.0) && (proj < 0.0);
        }
    }
    return r;
}

// One thread per observer, in tile order (sorted position si -> observer perm[si]);
// the beams of the receiver's tile's TIGHT work list in ascending order
// (kernels.py:364-399).  Every pair off the list is cut for every segment or behind
// segment 0 (the list is sound: exact fp64 bounds with margins, oracle-pinned), so the
// reference adds nothing for it: skipping it leaves acc and evals bit-identical to the
// dense loop over all beams.  A warp's 32 receivers share a tile, so the beam loop is
// warp-uniform.
template <int NF>
__global__ void __launch_bounds__(128)
    gbs_fp64_kernel(const GbsArgs a, const int32_t *perm, int tile, const uint32_t *tbits,
                    int64_t n_words) {
    const int64_t si = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (si >= a.n_obs) return;
    const int64_t oi = perm[si];
    const uint32_t *words = tbits + (si / tile) * n_words;
    const double pi = 3.141592653589793;  // np.pi
    const double c = a.c, width_b = a.width_b;
    const double sqrt_c = sqrt(c);
    const double px = a.obs[3 * oi + 0], py = a.obs[3 * oi + 1], pz = a.obs[3 * oi + 2];
    const int nf = NF > 0 ? NF : a.nf;
    double acc_re[NF > 0 ? NF : BF_MAXF], acc_im[NF > 0 ? NF : BF_MAXF];
#pragma unroll
    for (int f = 0; f < (NF > 0 ? NF : BF_MAXF); ++f) {
        if (f < nf) {
            acc_re[f] = a.acc[2 * (oi * a.acc_stride + f) + 0];
            acc_im[f] = a.acc[2 * (oi * a.acc_stride + f) + 1];
        }
    }
    int64_t ev = 0;
    for (int64_t wi = 0; wi < n_words; ++wi)
    for (uint32_t m = __ldg(words + wi); m; m &= m - 1) {
        const int64_t b = 32 * wi + __ffs(m) - 1;
        const int ns = __ldg(a.n_segs + b);
        if (ns == 0) continue;
        const Nearest r = nearest_exact(a, b * a.max_seg, ns, px, py, pz);
        if (r.behind) continue;
        const double s = r.s;
        const double q_sq = r.q1 * r.q1 + r.q2 * r.q2;
        const double m2 = s * s + width_b * width_b;
        const double inv_m2 = 1.0 / m2;
        const double wb = __ldg(a.weights + b);
#pragma unroll
        for (int f = 0; f < (NF > 0 ? NF : BF_MAXF); ++f) {
            if (f >= nf) break;
            const double w = a.omegas[f];
            const double g = w * q_sq * 0.5 / c * inv_m2;
            const double ex_re = -g * width_b;
            if (a.use_cutoff && ex_re < BF_CUTOFF_EXPONENT) continue;
            const double ex_im = w * s / c + g * s;
            const double amp = a.phi_amp * r.refl * sqrt_c;
            const double q_re = s * inv_m2;
            const double q_im = width_b * inv_m2;
            const double er = exp(ex_re);
            double sn, cs;
            sincos(ex_im, &sn, &cs);
            const double cr = er * cs;
            const double ci = er * sn;
            const double f_re = amp * (q_re * cr - q_im * ci);
            const double f_im = amp * (q_re * ci + q_im * cr);
            const double pref = w / (2.0 * pi * c) * wb;
            acc_re[f] += -pref * f_im;
            acc_im[f] += pref * f_re;
            ev += 1;
        }
    }
#pragma unroll
    for (int f = 0; f < (NF > 0 ? NF : BF_MAXF); ++f) {
        if (f < nf) {
            a.acc[2 * (oi * a.acc_stride + f) + 0] = acc_re[f];
            a.acc[2 * (oi * a.acc_stride + f) + 1] = acc_im[f];
        }
    }
    a.evals[oi] += ev;
}

__global__ void nearest_kernel(const GbsArgs a, const int64_t *q_obs, const int64_t *q_beam,
                               int64_t n_query, double *out) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_query) return;
    const int64_t oi = q_obs[j], b = q_beam[j];
    double *o = out + 6 * j;
    const int ns = a.n_segs[b];
    if (ns == 0) {
        o[0] = -1.0;
        o[1] = 0.0;
        o[2] = 0.0;
        o[3] = 0.0;
        o[4] = 1.0;
        o[5] = 0.0;
        return;
    }
    const Nearest r = nearest_exact(a, b * a.max_seg, ns, a.obs[3 * oi], a.obs[3 * oi + 1],
                                    a.obs[3 * oi + 2]);
    o[0] = (double)r.k;
    o[1] = r.s;
    o[2] = r.q1;
    o[3] = r.q2;
    o[4] = r.refl;
    o[5] = r.behind ? 1.0 : 0.0;
}

// ---------------------------------------------------------------- tracer ----

// Python's min/max on two floats: min(a, b) returns a unless b < a.
__device__ __forceinline__ double pymin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double pymax(double a, double b) { return (b > a) ? b : a; }

// kernels.py:23-51 (Moller-Trumbore, inclusive edges).
__device__ __forceinline__ double tri_intersect(double ox, double oy, double oz, double dx,
                                                double dy, double dz, const double *A,
                                                const double *B, const double *C) {
    const double ax = A[0], ay = A[1], az = A[2];
    const double e1x = B[0] - ax, e1y = B[1] - ay, e1z = B[2] - az;
    const double e2x = C[0] - ax, e2y = C[1] - ay, e2z = C[2] - az;
    const double px = dy * e2z - dz * e2y;
    const double py = dz * e2x - dx * e2z;
    const double pz = dx * e2y - dy * e2x;
    const double det = e1x * px + e1y * py + e1z * pz;
    if (-1e-12 < det && det < 1e-12) return INFINITY;
    const double inv = 1.0 / det;
    const double tx = ox - ax, ty = oy - ay, tz = oz - az;
    const double u = (tx * px + ty * py + tz * pz) * inv;
    if (u < 0.0 || u > 1.0) return INFINITY;
    const double qx = ty * e1z - tz * e1y;
    const double qy = tz * e1x - tx * e1z;
    const double qz = tx * e1y - ty * e1x;
    const double v = (dx * qx + dy * qy + dz * qz) * inv;
    if (v < 0.0 || u + v > 1.0) return INFINITY;
    return (e2x * qx + e2y * qy + e2z * qz) * inv;
}

// kernels.py:119-140
__device__ __forceinline__ double ray_box_exit(const double *bounds, double ox, double oy,
                                               double oz, double dx, double dy, double dz) {
    const double big = 1e300;
    const double idx = (dx > 1e-300 || dx < -1e-300) ? 1.0 / dx : (dx >= 0 ? big : -big);
    const double idy = (dy > 1e-300 || dy < -1e-300) ? 1.0 / dy : (dy >= 0 ? big : -big);
    const double idz = (dz > 1e-300 || dz < -1e-300) ? 1.0 / dz : (dz >= 0 ? big : -big);
    double t1 = (bounds[0] - ox) * idx;
    double t2 = (bounds[3] - ox) * idx;
    double tmin = pymin(t1, t2);
    double tmax = pymax(t1, t2);
    t1 = (bounds[1] - oy) * idy;
    t2 = (bounds[4] - oy) * idy;
    tmin = pymax(tmin, pymin(t1, t2));
    tmax = pymin(tmax, pymax(t1, t2));
    t1 = (bounds[2] - oz) * idz;
    t2 = (bounds[5] - oz) * idz;
    tmin = pymax(tmin, pymin(t1, t2));
    tmax = pymin(tmax, pymax(t1, t2));
    if (tmax < tmin || tmax < 0.0) return 0.0;
    return tmax;
}

struct TraceArgs {
    const double *v0, *v1, *v2, *refl;
    int64_t n_tri;
    const double *cbox;  // per cluster of TRI_CLUSTER consecutive triangles: expanded AABB
    int64_t n_clu;       // 0: exhaustive search
    const double *bounds;
    double diameter;
    const double *origin, *dirs, *e1s, *e2s;
    double length_cap;
    int64_t r_max, max_seg;
    double *seg_origin, *seg_dir, *seg_e1, *seg_e2, *seg_len, *seg_s0, *seg_refl;
    int32_t *n_segs, *n_refls;
    int64_t lo, hi, row_base;
};

__device__ __forceinline__ void write_row(const TraceArgs &a, int64_t row, double px, double py,
                                          double pz, double dx, double dy, double dz,
                                          double e1x, double e1y, double e1z, double e2x,
                                          double e2y, double e2z, double len, double s0,
                                          double refl) {
    a.seg_origin[3 * row + 0] = px;
    a.seg_origin[3 * row + 1] = py;
    a.seg_origin[3 * row + 2] = pz;
    a.seg_dir[3 * row + 0] = dx;
    a.seg_dir[3 * row + 1] = dy;
    a.seg_dir[3 * row + 2] = dz;
    a.seg_e1[3 * row + 0] = e1x;
    a.seg_e1[3 * row + 1] = e1y;
    a.seg_e1[3 * row + 2] = e1z;
    a.seg_e2[3 * row + 0] = e2x;
    a.seg_e2[3 * row + 1] = e2y;
    a.seg_e2[3 * row + 2] = e2z;
    a.seg_len[row] = len;
    a.seg_s0[row] = s0;
    a.seg_refl[row] = refl;
}

// Triangle clusters for the hit search: TRI_CLUSTER consecutive triangles (the scene
// generators emit a building's faces contiguously) share an axis-aligned box, expanded
// by 1e-7 + 1e-9 |x| so that it contains every point the exact intersection test can
// accept.  A cluster is skipped when the ray misses its box or enters it beyond the best
// hit so far; the selection -- lexicographic minimum of (t, triangle index) over the
// accepted hits -- does not depend on the order triangles are visited, so the result is
// bit-identical to the exhaustive search (tests/test_gbs_gpu.py checks both).
constexpr int TRI_CLUSTER = 16;

__global__ void cluster_box_kernel(const double *v0, const double *v1, const double *v2,
                                   int64_t n_tri, int64_t n_clu, double *cbox) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_clu) return;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    const int64_t t1 = min(n_tri, (c + 1) * TRI_CLUSTER);
    for (int64_t t = c * TRI_CLUSTER; t < t1; ++t)
        for (int d = 0; d < 3; ++d) {
            const double a = v0[3 * t + d], b = v1[3 * t + d], e = v2[3 * t + d];
            lo[d] = fmin(lo[d], fmin(a, fmin(b, e)));
            hi[d] = fmax(hi[d], fmax(a, fmax(b, e)));
        }
    for (int d = 0; d < 3; ++d) {
        cbox[6 * c + d] = lo[d] - (1e-7 + 1e-9 * fabs(lo[d]));
        cbox[6 * c + 3 + d] = hi[d] + (1e-7 + 1e-9 * fabs(hi[d]));
    }
}

// Can the ray (o, d) meet box B at a parameter t <= tmax_allowed?  Conservative: slab
// intervals widened by a relative 1e-9 (the box itself is already expanded).
__device__ __forceinline__ bool ray_may_hit_box(const double *B, double ox, double oy,
                                                double oz, double dx, double dy, double dz,
                                                double tmax_allowed) {
    double tmin = -INFINITY, tmax = INFINITY;
    const double o[3] = {ox, oy, oz}, dd[3] = {dx, dy, dz};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (fabs(dd[k]) < 1e-300) {
            if (o[k] < B[k] || o[k] > B[3 + k]) return false;
            continue;
        }
        const double inv = 1.0 / dd[k];
        double t1 = (B[k] - o[k]) * inv, t2 = (B[3 + k] - o[k]) * inv;
        if (t1 > t2) {
            const double t = t1;
            t1 = t2;
            t2 = t;
        }
        tmin = fmax(tmin, t1);
        tmax = fmin(tmax, t2);
    }
    const double slack = 1e-9 * (1.0 + fabs(tmin) + fabs(tmax));
    return tmax >= -slack && tmin <= tmax + slack && tmin <= tmax_allowed + slack;
}

// One thread per ray (kernels.py:282-301 / 143-279).
__global__ void __launch_bounds__(128) trace_kernel(const TraceArgs a) {
    const int64_t i = a.lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.hi) return;
    const bool have_scene = a.n_tri > 0;
    double px = a.origin[0], py = a.origin[1], pz = a.origin[2];
    double dx = a.dirs[3 * i + 0], dy = a.dirs[3 * i + 1], dz = a.dirs[3 * i + 2];
    double e1x = a.e1s[3 * i + 0], e1y = a.e1s[3 * i + 1], e1z = a.e1s[3 * i + 2];
    double e2x = a.e2s[3 * i + 0], e2y = a.e2s[3 * i + 1], e2z = a.e2s[3 * i + 2];
    double s_acc = 0.0;
    int n_refl = 0;
    double cum_refl = 1.0;
    const int64_t row0 = (i - a.row_base) * a.max_seg;
    int64_t row = row0;
    while (true) {
        const double remaining = a.length_cap - s_acc;
        if (remaining <= 0.0) break;
        // Nearest hit with t in (EPS_HIT, remaining]; ties -> lower triangle index.
        double best_t = remaining;
        int64_t best_i = -1;
        auto visit = [&](int64_t t0, int64_t t1) {
            for (int64_t tri = t0; tri < t1; ++tri) {
                const double t = tri_intersect(px, py, pz, dx, dy, dz, a.v0 + 3 * tri,
                                               a.v1 + 3 * tri, a.v2 + 3 * tri);
                if (t > BF_EPS_HIT && t <= best_t) {
                    if (t < best_t || best_i < 0 || tri < best_i) {
                        best_t = t;
                        best_i = tri;
                    }
                }
            }
        };
        if (a.n_clu > 0) {
            for (int64_t c = 0; c < a.n_clu; ++c)
                if (ray_may_hit_box(a.cbox + 6 * c, px, py, pz, dx, dy, dz, best_t))
                    visit(c * TRI_CLUSTER, min(a.n_tri, (c + 1) * TRI_CLUSTER));
        } else {
            visit(0, a.n_tri);
        }
        if (best_i < 0) {
            double seg = remaining;
            if (have_scene) {
                const double allow = ray_box_exit(a.bounds, px, py, pz, dx, dy, dz) + a.diameter;
                if (allow < seg) seg = allow;
            }
            write_row(a, row, px, py, pz, dx, dy, dz, e1x, e1y, e1z, e2x, e2y, e2z, seg, s_acc,
                      cum_refl);
            ++row;
            break;
        }
        const double t = best_t;
        const int64_t tri = best_i;
        write_row(a, row, px, py, pz, dx, dy, dz, e1x, e1y, e1z, e2x, e2y, e2z, t, s_acc,
                  cum_refl);
        ++row;
        if (n_refl == a.r_max) break;

        s_acc += t;
        px += t * dx;
        py += t * dy;
        pz += t * dz;

        const double ax = a.v0[3 * tri + 0], ay = a.v0[3 * tri + 1], az = a.v0[3 * tri + 2];
        const double ux = a.v1[3 * tri + 0] - ax, uy = a.v1[3 * tri + 1] - ay,
                     uz = a.v1[3 * tri + 2] - az;
        const double wx = a.v2[3 * tri + 0] - ax, wy = a.v2[3 * tri + 1] - ay,
                     wz = a.v2[3 * tri + 2] - az;
        double nx = uy * wz - uz * wy;
        double ny = uz * wx - ux * wz;
        double nz = ux * wy - uy * wx;
        const double nn = sqrt(nx * nx + ny * ny + nz * nz);
        nx /= nn;
        ny /= nn;
        nz /= nn;
        if (nx * dx + ny * dy + nz * dz > 0.0) {
            nx = -nx;
            ny = -ny;
            nz = -nz;
        }
        // Householder mirror of direction and frame, then re-orthonormalize.
        const double dn = dx * nx + dy * ny + dz * nz;
        dx -= 2.0 * dn * nx;
        dy -= 2.0 * dn * ny;
        dz -= 2.0 * dn * nz;
        const double dnorm = sqrt(dx * dx + dy * dy + dz * dz);
        dx /= dnorm;
        dy /= dnorm;
        dz /= dnorm;

        double h = e1x * nx + e1y * ny + e1z * nz;
        e1x -= 2.0 * h * nx;
        e1y -= 2.0 * h * ny;
        e1z -= 2.0 * h * nz;
        h = e2x * nx + e2y * ny + e2z * nz;
        e2x -= 2.0 * h * nx;
        e2y -= 2.0 * h * ny;
        e2z -= 2.0 * h * nz;

        h = e1x * dx + e1y * dy + e1z * dz;
        e1x -= h * dx;
        e1y -= h * dy;
        e1z -= h * dz;
        double en = sqrt(e1x * e1x + e1y * e1y + e1z * e1z);
        e1x /= en;
        e1y /= en;
        e1z /= en;
        h = e2x * dx + e2y * dy + e2z * dz;
        e2x -= h * dx;
        e2y -= h * dy;
        e2z -= h * dz;
        h = e2x * e1x + e2y * e1y + e2z * e1z;
        e2x -= h * e1x;
        e2y -= h * e1y;
        e2z -= h * e1z;
        en = sqrt(e2x * e2x + e2y * e2y + e2z * e2z);
        e2x /= en;
        e2y /= en;
        e2z /= en;

        n_refl += 1;
        cum_refl *= a.refl[tri];
    }
    a.n_segs[i - a.row_base] = (int32_t)(row - row0);
    a.n_refls[i - a.row_base] = n_refl;
}

// ------------------------------------------------------------ work list ----
// Candidate (receiver tile, beam) pairs, SURVEY.md 8(a) row a9.  A beam is NOT a
// candidate for a tile (centre c, radius R_T) when for every segment k either
//   * the whole tile lies outside the cutoff cylinder of k's infinite line:
//     |w - (w.d) d| - R_T > R_k (1 + 1e-6) + 1e-6 with w = c - o_k and
//     R_k^2 = 72 c (s_end^2 + b^2) / (omega_min b), s_end = s0 + len
//     (q^2 of the winner is measured to its infinite line, kernels.py:345-346,377, and
//     s <= s_end, so ex_re < -36 for every receiver if k wins, kernels.py:382-385), or
//   * k == 0 and the tile lies behind the launch plane: w.d + R_T < -1e-6 (if k = 0
//     wins it is `behind`, kernels.py:348,375).
// Fixed fp64 operation order, no FMA (this file is -fmad=false), IEEE sqrt/div:
// oracle/worklist_oracle.c reproduces the bitmask bit for bit.
// Returns bit 0 = dead under the a9 bound above (R_k from s_end), bit 1 = dead under
// the TIGHT bound that uses the largest arc length the tile can reach on segment k,
// s_hi = s0 + clamp(w.d + R_T, 0, len) <= s_end (every receiver's nearest point on k
// projects within R_T of the centre's), R_k(s_hi)^2 = 72 c (s_hi^2 + b^2)/(omega_min b).
// Tight-dead implies nothing about a9; a9-dead implies tight-dead.
// qp - rt > sqrt(r2) (1 + 1e-6) + 1e-6 with qp = sqrt(q2), decided in fp64 exactly as
// the C restatement does, but the two square roots are only taken when an fp32
// estimate (relative error ~1e-7) is within 1e-4 of the threshold.
__device__ __forceinline__ bool cut_beyond(double q2, double r2, double rt) {
    const float x = sqrtf((float)r2) * 1.000001f + 1e-6f + (float)rt;  // threshold for qp
    const float x2 = x * x, qf = (float)q2;
    if (qf > x2 * 1.0001f + 1e-12f) return true;
    if (qf < x2 * 0.9999f - 1e-12f) return false;
    return sqrt(q2) - rt > sqrt(r2) * (1.0 + 1e-6) + 1e-6;
}

// The rows of one 32-beam word, staged in shared memory as [segment][beam] arrays.
struct WordRows {
    const double *ox, *oy, *oz, *dx, *dy, *dz, *s0, *len;
};

// Tight cut: qn - min(hu/qn, rt) > sqrt(r2) (1 + 1e-6) + 1e-6 with qn = sqrt(q2), in
// fp64 exactly as the C restatement, after an fp32 screen (relative margin 1e-4).
__device__ __forceinline__ bool tight_cut(double q2, double hu, double rt, double r2) {
    const float qf = sqrtf((float)q2);
    const float rnf = qf > 0.f ? fminf((float)hu / qf, (float)rt) : (float)rt;
    const float lhs = qf - rnf, rhs = sqrtf((float)r2) * 1.000001f + 1e-6f;
    const float tol = 1e-4f * (qf + rnf + rhs) + 1e-6f;
    if (lhs > rhs + tol) return true;
    if (lhs < rhs - tol) return false;
    const double qn = sqrt(q2);
    double rn = rt;
    if (qn > 0.0) {
        rn = hu / qn;
        rn = rn < rt ? rn : rt;
    }
    return qn - rn > sqrt(r2) * (1.0 + 1e-6) + 1e-6;
}

__device__ __forceinline__ unsigned beam_dead_for_tile(const WordRows &w, int jb, int ns,
                                                       double width_b, double cx, double cy,
                                                       double cz, double rt, double hx, double hy,
                                                       double hz, double rscale) {
    bool loose = true, tight = true;
    for (int k = 0; k < ns && tight; ++k) {
        const int i = 32 * k + jb;
        const double wx = cx - w.ox[i], wy = cy - w.oy[i], wz = cz - w.oz[i];
        const double dx = w.dx[i], dy = w.dy[i], dz = w.dz[i];
        const double proj = wx * dx + wy * dy + wz * dz;
        const double ux = wx - proj * dx, uy = wy - proj * dy, uz = wz - proj * dz;
        const double q2 = ux * ux + uy * uy + uz * uz;
        const double s0 = w.s0[i], len = w.len[i];
        const double se = s0 + len;
        // tight: the tile's bounding box bounds r.d and (q convex, subgradient u/|u| at
        // the centre) the drop of q; each bound is also capped by the radius R_T
        double rd = hx * fabs(dx) + hy * fabs(dy) + hz * fabs(dz);
        rd = rd < rt ? rd : rt;
        double reach = proj + rd;
        reach = reach < 0.0 ? 0.0 : (reach > len ? len : reach);
        const double sh = s0 + reach;
        if (!(k == 0 && proj + rt < -1e-6))
            loose = loose && cut_beyond(q2, rscale * (se * se + width_b * width_b), rt);
        if (!(k == 0 && proj + rd < -1e-6) && tight)
            tight = tight_cut(q2, hx * fabs(ux) + hy * fabs(uy) + hz * fabs(uz), rt,
                              rscale * (sh * sh + width_b * width_b));
    }
    return (loose ? 1u : 0u) | (tight ? 2u : 0u);
}

// One block per 32-beam word: the word's rows are read once into shared memory and
// every warp sweeps a share of the tiles; bit j of (tile, word) = beam 32*word + j is a
// candidate (bits: a9 bound, tbits: tight bound, tbits subset of bits).
// With counts != null it also adds popc(tight word) to counts[tile * n_ranges + range]
// (compaction offsets of the fp32 kernel's work list) and the per-tile statistics
// wstats[{0,1,2,3} * n_tiles + tile] = a9 beams, a9 beam segments, tight beams, tight
// beam segments (the FLOP model of bench.py).
__global__ void worklist_kernel(const GbsArgs a, const Rows r, const double4 *centre,
                                const double4 *tbox, int64_t n_tiles, int64_t n_words,
                                double rscale, uint32_t *bits, uint32_t *tbits,
                                int64_t range_beams, int64_t n_ranges,
                                unsigned long long *counts, unsigned long long *wstats) {
    extern __shared__ double wsm[];
    __shared__ int ns_s[32];
    __shared__ int64_t st_s[33];
    const int S = (int)r.max_seg;
    const int64_t word = blockIdx.x;
    WordRows w{wsm, wsm + 32 * S, wsm + 64 * S, wsm + 96 * S, wsm + 128 * S, wsm + 160 * S,
               wsm + 192 * S, wsm + 224 * S};
    if (threadIdx.x < 33) {
        const int64_t b = min(32 * word + threadIdx.x, r.n_beams);
        st_s[threadIdx.x] = r.start[b];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * S; i += blockDim.x) {
        const int jb = i / S, k = i - jb * S;  // beam-major
        const int64_t row = st_s[jb] + k;
        if (row >= st_s[jb + 1]) continue;
        const int o = 32 * k + jb;
        const double4 q0 = r.p0[row], q1 = r.p1[row];  // exact copies of the bundle's fp64
        const_cast<double *>(w.ox)[o] = q0.x;
        const_cast<double *>(w.oy)[o] = q0.y;
        const_cast<double *>(w.oz)[o] = q0.z;
        const_cast<double *>(w.dx)[o] = q1.x;
        const_cast<double *>(w.dy)[o] = q1.y;
        const_cast<double *>(w.dz)[o] = q1.z;
        const_cast<double *>(w.s0)[o] = q1.w;
        const_cast<double *>(w.len)[o] = q0.w;
    }
    const int lane = threadIdx.x & 31;
    const int64_t b = 32 * word + lane;
    if (threadIdx.x < 32) ns_s[lane] = (int)(st_s[lane + 1] - st_s[lane]);
    __syncthreads();
    const int ns = ns_s[lane];
    for (int64_t t = threadIdx.x >> 5; t < n_tiles; t += blockDim.x >> 5) {
        const double4 c = centre[t], h = tbox[t];
        unsigned dead = 3u;
        if (b < r.n_beams)
            dead = beam_dead_for_tile(w, lane, ns, a.width_b, c.x, c.y, c.z, c.w, h.x, h.y, h.z,
                                      rscale);
        const unsigned m = __ballot_sync(0xffffffffu, !(dead & 1u));
        const unsigned mt = __ballot_sync(0xffffffffu, !(dead & 2u));
        if (lane == 0) {
            bits[t * n_words + word] = m;
            tbits[t * n_words + word] = mt;
        }
        if (counts && m) {
            const unsigned sg = __reduce_add_sync(0xffffffffu, (dead & 1u) ? 0u : (unsigned)ns);
            const unsigned sgt = __reduce_add_sync(0xffffffffu, (dead & 2u) ? 0u : (unsigned)ns);
            if (lane == 0) {
                atomicAdd(&wstats[t], (unsigned long long)__popc(m));
                atomicAdd(&wstats[n_tiles + t], (unsigned long long)sg);
                if (mt) {
                    const int64_t q = 32 * word / range_beams;
                    atomicAdd(&counts[t * n_ranges + q], (unsigned long long)__popc(mt));
                    atomicAdd(&wstats[2 * n_tiles + t], (unsigned long long)__popc(mt));
                    atomicAdd(&wstats[3 * n_tiles + t], (unsigned long long)sgt);
                }
            }
        }
    }
}

__global__ void finalize_kernel(const double *acc, int64_t n, double calibration,
                                double *pressure, double *spl) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double re = calibration * acc[2 * i], im = calibration * acc[2 * i + 1];
    if (pressure) {
        pressure[2 * i] = re;
        pressure[2 * i + 1] = im;
    }
    if (spl) {
        const double mag = hypot(re, im);
        spl[i] = (mag == 0.0) ? -INFINITY : 20.0 * log10(mag / 2e-5);
    }
}

}  // namespace

int launch_gbs_fp64(const GbsArgs &a, const int32_t *perm, int tile, const uint32_t *tbits,
                    int64_t n_words, cudaStream_t st) {
    if (a.n_obs <= 0) return BF_OK;
    const int threads = 128;
    const unsigned blocks = (unsigned)((a.n_obs + threads - 1) / threads);
    switch (a.nf) {
        case 1: gbs_fp64_kernel<1><<<blocks, threads, 0, st>>>(a, perm, tile, tbits, n_words); break;
        case 2: gbs_fp64_kernel<2><<<blocks, threads, 0, st>>>(a, perm, tile, tbits, n_words); break;
        case 3: gbs_fp64_kernel<3><<<blocks, threads, 0, st>>>(a, perm, tile, tbits, n_words); break;
        case 4: gbs_fp64_kernel<4><<<blocks, threads, 0, st>>>(a, perm, tile, tbits, n_words); break;
        case 5: gbs_fp64_kernel<5><<<blocks, threads, 0, st>>>(a, perm, tile, tbits, n_words); break;
        default: gbs_fp64_kernel<0><<<blocks, threads, 0, st>>>(a, perm, tile, tbits, n_words); break;
    }
    note_launch();
    BF_TRY_CUDA(cudaGetLastError());
    return BF_OK;
}

int launch_nearest(const GbsArgs &a, const int64_t *q_obs, const int64_t *q_beam,
                   int64_t n_query, double *out, cudaStream_t st) {
    if (n_query <= 0) return BF_OK;
    const unsigned blocks = (unsigned)((n_query + 127) / 128);
    nearest_kernel<<<blocks, 128, 0, st>>>(a, q_obs, q_beam, n_query, out);
    note_launch();
    BF_TRY_CUDA(cudaGetLastError());
    return BF_OK;
}

int trace_cluster_count(int64_t n_tri) { return (int)((n_tri + TRI_CLUSTER - 1) / TRI_CLUSTER); }

int launch_trace(const double *v0, const double *v1, const double *v2, const double *refl,
                 int64_t n_tri, double *cbox, const double *bounds, double diameter,
                 const double *origin,
                 const double *dirs, const double *e1s, const double *e2s, double length_cap,
                 int64_t r_max, int64_t max_seg, double *seg_origin, double *seg_dir,
                 double *seg_e1, double *seg_e2, double *seg_len, double *seg_s0,
                 double *seg_refl, int32_t *n_segs, int32_t *n_refls, int64_t lo, int64_t hi,
                 int64_t row_base, cudaStream_t st) {
    if (hi <= lo) return BF_OK;
    const int64_t n_clu = cbox ? (n_tri + TRI_CLUSTER - 1) / TRI_CLUSTER : 0;
    if (n_clu > 0) {
        cluster_box_kernel<<<(unsigned)((n_clu + 127) / 128), 128, 0, st>>>(v0, v1, v2, n_tri,
                                                                           n_clu, cbox);
        note_launch();
    }
    TraceArgs a{v0, v1, v2, refl, n_tri, cbox, n_clu, bounds, diameter, origin, dirs, e1s, e2s,
                length_cap, r_max, max_seg, seg_origin, seg_dir, seg_e1, seg_e2, seg_len,
                seg_s0, seg_refl, n_segs, n_refls, lo, hi, row_base};
    const unsigned blocks = (unsigned)((hi - lo + 127) / 128);
    trace_kernel<<<blocks, 128, 0, st>>>(a);
    note_launch();
    BF_TRY_CUDA(cudaGetLastError());
    return BF_OK;
}

int launch_worklist(const GbsArgs &a, const Rows &r, const double4 *centre, const double4 *tbox,
                    int64_t n_tiles, double omega_min, uint32_t *bits, uint32_t *tbits,
                    int64_t range_beams, int64_t n_ranges, unsigned long long *counts,
                    unsigned long long *wstats, cudaStream_t st) {
    if (n_tiles <= 0 || r.n_beams <= 0) return BF_OK;
    const int64_t n_words = (r.n_beams + 31) / 32;
    // no cutoff -> nothing is ever cut (only the behind test of segment 0 remains)
    const double rscale = a.use_cutoff ? 72.0 * a.c / (omega_min * a.width_b) : INFINITY;
    const size_t smem = 8 * 32 * sizeof(double) * (size_t)r.max_seg;
    BF_TRY_CUDA(cudaFuncSetAttribute(worklist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    worklist_kernel<<<(unsigned)n_words, 256, smem, st>>>(a, r, centre, tbox, n_tiles, n_words,
                                                          rscale, bits, tbits, range_beams,
                                                          n_ranges, counts, wstats);
    note_launch();
    BF_TRY_CUDA(cudaGetLastError());
    return BF_OK;
}

int launch_finalize(const double *acc, int64_t n, double calibration, double *pressure,
                    double *spl, cudaStream_t st) {
    if (n <= 0) return BF_OK;
    finalize_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(acc, n, calibration, pressure,
                                                                   spl);
    note_launch();
    BF_TRY_CUDA(cudaGetLastError());
    return BF_OK;
}

}  // namespace bf
