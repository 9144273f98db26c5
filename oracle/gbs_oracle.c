/*
 * CPU ORACLE -- test infrastructure only, never the product path.
 *
 * A plain-C, operation-for-operation restatement of the reference GBS hot path
 *   - nearest_on_segments   /root/reference/pkg/src/beamfield/kernels.py:304-349
 *   - gbs_accumulate        /root/reference/pkg/src/beamfield/kernels.py:352-399
 * and of the reference's flat CPU scheduler
 *   - WorkerPool.flat / block_partition   parallel.py:108-140 (static blocks of the
 *     observer range, one per thread)
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg (and the
 * `--impl reference` arm) may load this library, and only as the checker/baseline.
 *
 * Numerics: the reference is numba-compiled with fastmath=False and no FMA
 * contraction (kernels.py:20); this file must be compiled with
 * -ffp-contract=off -fno-fast-math so every + and * rounds separately, in the
 * same left-to-right order as the Python source.  exp/cos/sin come from the
 * platform libm, as numba's llvm.exp/cos/sin.f64 do.
 *
 * Pinned against the reference's own outputs: the tests/golden npz files were produced by
 * executing the reference (tests/golden/make_golden.py); tests/test_oracle.py checks
 * this restatement against every fixture.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define CUTOFF_EXPONENT (-36.0) /* kernels.py:18 */

typedef struct {
    int64_t k;
    double s, q1, q2, refl;
    int behind;
} nearest_t;

/* kernels.py:304-349.  Rows are (N,3) C-contiguous fp64 arrays. */
static nearest_t nearest_on_segments(const double *seg_origin, const double *seg_dir,
                                     const double *seg_e1, const double *seg_e2,
                                     const double *seg_len, const double *seg_s0,
                                     const double *seg_refl, int64_t base, int64_t n_seg,
                                     double px, double py, double pz) {
    double best_d2 = INFINITY;
    nearest_t r = {-1, 0.0, 0.0, 0.0, 1.0, 0};
    for (int64_t k = 0; k < n_seg; ++k) {
        int64_t row = base + k;
        double ox = seg_origin[3 * row + 0], oy = seg_origin[3 * row + 1], oz = seg_origin[3 * row + 2];
        double dx = seg_dir[3 * row + 0], dy = seg_dir[3 * row + 1], dz = seg_dir[3 * row + 2];
        double wx = px - ox, wy = py - oy, wz = pz - oz;
        double proj = wx * dx + wy * dy + wz * dz;
        double t = proj;
        if (t < 0.0)
            t = 0.0;
        else if (t > seg_len[row])
            t = seg_len[row];
        double vx = wx - t * dx, vy = wy - t * dy, vz = wz - t * dz;
        double d2 = vx * vx + vy * vy + vz * vz;
        if (d2 < best_d2) { /* strict: the smallest k wins exact ties */
            best_d2 = d2;
            r.k = k;
            r.s = seg_s0[row] + t;
            r.q1 = vx * seg_e1[3 * row + 0] + vy * seg_e1[3 * row + 1] + vz * seg_e1[3 * row + 2];
            r.q2 = vx * seg_e2[3 * row + 0] + vy * seg_e2[3 * row + 1] + vz * seg_e2[3 * row + 2];
            r.refl = seg_refl[row];
            r.behind = (k == 0) && (t == 0.0) && (proj < 0.0);
        }
    }
    return r;
}

/* Exported for the nearest-segment golden test. out = (k, s, q1, q2, refl, behind). */
void oracle_nearest_on_segments(const double *seg_origin, const double *seg_dir,
                                const double *seg_e1, const double *seg_e2,
                                const double *seg_len, const double *seg_s0,
                                const double *seg_refl, int64_t base, int64_t n_seg,
                                double px, double py, double pz, double *out) {
    nearest_t r = nearest_on_segments(seg_origin, seg_dir, seg_e1, seg_e2, seg_len, seg_s0,
                                      seg_refl, base, n_seg, px, py, pz);
    out[0] = (double)r.k;
    out[1] = r.s;
    out[2] = r.q1;
    out[3] = r.q2;
    out[4] = r.refl;
    out[5] = (double)r.behind;
}

typedef struct {
    const double *seg_origin, *seg_dir, *seg_e1, *seg_e2, *seg_len, *seg_s0, *seg_refl;
    const int32_t *n_segs;
    int64_t max_seg;
    const double *weights, *obs, *omegas;
    int64_t nf;
    double c, width_b, phi_amp;
    int use_cutoff;
    double *acc; /* complex128 interleaved (n_obs, nf) */
    int64_t *evals;
    int64_t obs_lo, obs_hi, beam_lo, beam_hi;
} gbs_args_t;

/* kernels.py:352-399 */
static void gbs_range(const gbs_args_t *a) {
    const double pi = 3.141592653589793; /* np.pi */
    int64_t nf = a->nf;
    double c = a->c, width_b = a->width_b;
    double sqrt_c = sqrt(c);
    for (int64_t oi = a->obs_lo; oi < a->obs_hi; ++oi) {
        double px = a->obs[3 * oi + 0], py = a->obs[3 * oi + 1], pz = a->obs[3 * oi + 2];
        for (int64_t b = a->beam_lo; b < a->beam_hi; ++b) {
            int64_t ns = a->n_segs[b];
            if (ns == 0)
                continue;
            nearest_t r = nearest_on_segments(a->seg_origin, a->seg_dir, a->seg_e1, a->seg_e2,
                                              a->seg_len, a->seg_s0, a->seg_refl,
                                              b * a->max_seg, ns, px, py, pz);
            if (r.behind)
                continue;
            double s = r.s;
            double q_sq = r.q1 * r.q1 + r.q2 * r.q2;
            double m2 = s * s + width_b * width_b;
            double inv_m2 = 1.0 / m2;
            for (int64_t f = 0; f < nf; ++f) {
                double w = a->omegas[f];
                double g = w * q_sq * 0.5 / c * inv_m2;
                double ex_re = -g * width_b;
                if (a->use_cutoff && ex_re < CUTOFF_EXPONENT)
                    continue;
                double ex_im = w * s / c + g * s;
                double amp = a->phi_amp * r.refl * sqrt_c;
                double q_re = s * inv_m2;
                double q_im = width_b * inv_m2;
                double er = exp(ex_re);
                double cr = er * cos(ex_im);
                double ci = er * sin(ex_im);
                double f_re = amp * (q_re * cr - q_im * ci);
                double f_im = amp * (q_re * ci + q_im * cr);
                double pref = w / (2.0 * pi * c) * a->weights[b];
                double *acc = a->acc + 2 * (oi * nf + f);
                acc[0] += -pref * f_im;
                acc[1] += pref * f_re;
                a->evals[oi] += 1;
            }
        }
    }
}

static void *gbs_thread(void *p) {
    gbs_range((const gbs_args_t *)p);
    return NULL;
}

/*
 * Same argument list and in-place semantics as the reference gbs_accumulate
 * (kernels.py:352-355) plus a thread count.  Observer range [obs_lo, obs_hi) is cut
 * into `threads` contiguous near-even blocks (parallel.py:108-118), which
 * cannot change any result bit: each observer's sum is private and runs over the
 * beams in ascending order.
 */
int oracle_gbs_accumulate(const double *seg_origin, const double *seg_dir,
                          const double *seg_e1, const double *seg_e2, const double *seg_len,
                          const double *seg_s0, const double *seg_refl, const int32_t *n_segs,
                          int64_t max_seg, const double *weights, const double *obs,
                          const double *omegas, int64_t nf, double c, double width_b,
                          double phi_amp, int use_cutoff, double *acc, int64_t *evals,
                          int64_t obs_lo, int64_t obs_hi, int64_t beam_lo, int64_t beam_hi,
                          int threads) {
    gbs_args_t base = {seg_origin, seg_dir, seg_e1, seg_e2, seg_len, seg_s0, seg_refl,
                       n_segs, max_seg, weights, obs, omegas, nf, c, width_b, phi_amp,
                       use_cutoff, acc, evals, obs_lo, obs_hi, beam_lo, beam_hi};
    int64_t n = obs_hi - obs_lo;
    if (n <= 0)
        return 0;
    if (threads < 1)
        threads = 1;
    if (threads > n)
        threads = (int)n;
    if (threads == 1) {
        gbs_range(&base);
        return 0;
    }
    pthread_t *tid = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    gbs_args_t *args = (gbs_args_t *)calloc((size_t)threads, sizeof(gbs_args_t));
    if (!tid || !args) {
        free(tid);
        free(args);
        return -1;
    }
    int64_t q = n / threads, rem = n % threads, lo = obs_lo;
    for (int t = 0; t < threads; ++t) {
        int64_t size = q + (t < rem ? 1 : 0);
        args[t] = base;
        args[t].obs_lo = lo;
        args[t].obs_hi = lo + size;
        lo += size;
        pthread_create(&tid[t], NULL, gbs_thread, &args[t]);
    }
    for (int t = 0; t < threads; ++t)
        pthread_join(tid[t], NULL);
    free(tid);
    free(args);
    return 0;
}
