/*
 * CPU ORACLE -- test infrastructure only.  Plain-C restatement of the reference
 * tracer used to build identical GBS inputs on the CPU side (the `--impl
 * reference` arm and large-config parity tests):
 *   tri_intersect  kernels.py:23-51      ray_box_exit  kernels.py:119-140
 *   trace_one      kernels.py:143-279    trace_range   kernels.py:282-301
 * Nearest hit = the (t, triangle index) lexicographic minimum over t in
 * (EPS_HIT, remaining] -- the result bvh_nearest (kernels.py:54-116) returns --
 * found by exhaustive search.  Compiled with -ffp-contract=off (no FMA).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

#define EPS_HIT 1e-6

static double pymin(double a, double b) { return (b < a) ? b : a; }
static double pymax(double a, double b) { return (b > a) ? b : a; }

static double tri_intersect(double ox, double oy, double oz, double dx, double dy, double dz,
                            const double *A, const double *B, const double *C) {
    double ax = A[0], ay = A[1], az = A[2];
    double e1x = B[0] - ax, e1y = B[1] - ay, e1z = B[2] - az;
    double e2x = C[0] - ax, e2y = C[1] - ay, e2z = C[2] - az;
    double px = dy * e2z - dz * e2y, py = dz * e2x - dx * e2z, pz = dx * e2y - dy * e2x;
    double det = e1x * px + e1y * py + e1z * pz;
    if (-1e-12 < det && det < 1e-12) return INFINITY;
    double inv = 1.0 / det;
    double tx = ox - ax, ty = oy - ay, tz = oz - az;
    double u = (tx * px + ty * py + tz * pz) * inv;
    if (u < 0.0 || u > 1.0) return INFINITY;
    double qx = ty * e1z - tz * e1y, qy = tz * e1x - tx * e1z, qz = tx * e1y - ty * e1x;
    double v = (dx * qx + dy * qy + dz * qz) * inv;
    if (v < 0.0 || u + v > 1.0) return INFINITY;
    return (e2x * qx + e2y * qy + e2z * qz) * inv;
}

static double ray_box_exit(const double *bd, double ox, double oy, double oz, double dx,
                           double dy, double dz) {
    const double big = 1e300;
    double idx = (dx > 1e-300 || dx < -1e-300) ? 1.0 / dx : (dx >= 0 ? big : -big);
    double idy = (dy > 1e-300 || dy < -1e-300) ? 1.0 / dy : (dy >= 0 ? big : -big);
    double idz = (dz > 1e-300 || dz < -1e-300) ? 1.0 / dz : (dz >= 0 ? big : -big);
    double t1 = (bd[0] - ox) * idx, t2 = (bd[3] - ox) * idx;
    double tmin = pymin(t1, t2), tmax = pymax(t1, t2);
    t1 = (bd[1] - oy) * idy;
    t2 = (bd[4] - oy) * idy;
    tmin = pymax(tmin, pymin(t1, t2));
    tmax = pymin(tmax, pymax(t1, t2));
    t1 = (bd[2] - oz) * idz;
    t2 = (bd[5] - oz) * idz;
    tmin = pymax(tmin, pymin(t1, t2));
    tmax = pymin(tmax, pymax(t1, t2));
    if (tmax < tmin || tmax < 0.0) return 0.0;
    return tmax;
}

typedef struct {
    const double *v0, *v1, *v2, *refl;
    int64_t n_tri;
    const double *bounds;
    double diameter;
    const double *origin, *dirs, *e1s, *e2s;
    double length_cap;
    int64_t r_max, max_seg;
    double *so, *sd, *se1, *se2, *sl, *ss0, *sr;
    int32_t *n_segs, *n_refls;
    int64_t lo, hi;
} targs_t;

static void put_row(const targs_t *a, int64_t r, const double *p, const double *d,
                    const double *e1, const double *e2, double len, double s0, double refl) {
    for (int k = 0; k < 3; ++k) {
        a->so[3 * r + k] = p[k];
        a->sd[3 * r + k] = d[k];
        a->se1[3 * r + k] = e1[k];
        a->se2[3 * r + k] = e2[k];
    }
    a->sl[r] = len;
    a->ss0[r] = s0;
    a->sr[r] = refl;
}

static void trace_range(const targs_t *a) {
    for (int64_t i = a->lo; i < a->hi; ++i) {
        double p[3] = {a->origin[0], a->origin[1], a->origin[2]};
        double d[3] = {a->dirs[3 * i], a->dirs[3 * i + 1], a->dirs[3 * i + 2]};
        double e1[3] = {a->e1s[3 * i], a->e1s[3 * i + 1], a->e1s[3 * i + 2]};
        double e2[3] = {a->e2s[3 * i], a->e2s[3 * i + 1], a->e2s[3 * i + 2]};
        double s_acc = 0.0, cum = 1.0;
        int n_refl = 0;
        int64_t row0 = i * a->max_seg, row = row0;
        for (;;) {
            double remaining = a->length_cap - s_acc;
            if (remaining <= 0.0) break;
            double best_t = remaining;
            int64_t best_i = -1;
            for (int64_t tri = 0; tri < a->n_tri; ++tri) {
                double t = tri_intersect(p[0], p[1], p[2], d[0], d[1], d[2], a->v0 + 3 * tri,
                                         a->v1 + 3 * tri, a->v2 + 3 * tri);
                if (t > EPS_HIT && t <= best_t && (t < best_t || best_i < 0 || tri < best_i)) {
                    best_t = t;
                    best_i = tri;
                }
            }
            if (best_i < 0) {
                double seg = remaining;
                if (a->n_tri > 0) {
                    double allow = ray_box_exit(a->bounds, p[0], p[1], p[2], d[0], d[1], d[2]) +
                                   a->diameter;
                    if (allow < seg) seg = allow;
                }
                put_row(a, row++, p, d, e1, e2, seg, s_acc, cum);
                break;
            }
            double t = best_t;
            int64_t tri = best_i;
            put_row(a, row++, p, d, e1, e2, t, s_acc, cum);
            if (n_refl == a->r_max) break;
            s_acc += t;
            p[0] += t * d[0];
            p[1] += t * d[1];
            p[2] += t * d[2];
            const double *A = a->v0 + 3 * tri, *B = a->v1 + 3 * tri, *C = a->v2 + 3 * tri;
            double ux = B[0] - A[0], uy = B[1] - A[1], uz = B[2] - A[2];
            double wx = C[0] - A[0], wy = C[1] - A[1], wz = C[2] - A[2];
            double nx = uy * wz - uz * wy, ny = uz * wx - ux * wz, nz = ux * wy - uy * wx;
            double nn = sqrt(nx * nx + ny * ny + nz * nz);
            nx /= nn;
            ny /= nn;
            nz /= nn;
            if (nx * d[0] + ny * d[1] + nz * d[2] > 0.0) {
                nx = -nx;
                ny = -ny;
                nz = -nz;
            }
            double dn = d[0] * nx + d[1] * ny + d[2] * nz;
            d[0] -= 2.0 * dn * nx;
            d[1] -= 2.0 * dn * ny;
            d[2] -= 2.0 * dn * nz;
            double dnorm = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
            d[0] /= dnorm;
            d[1] /= dnorm;
            d[2] /= dnorm;
            double h = e1[0] * nx + e1[1] * ny + e1[2] * nz;
            e1[0] -= 2.0 * h * nx;
            e1[1] -= 2.0 * h * ny;
            e1[2] -= 2.0 * h * nz;
            h = e2[0] * nx + e2[1] * ny + e2[2] * nz;
            e2[0] -= 2.0 * h * nx;
            e2[1] -= 2.0 * h * ny;
            e2[2] -= 2.0 * h * nz;
            h = e1[0] * d[0] + e1[1] * d[1] + e1[2] * d[2];
            e1[0] -= h * d[0];
            e1[1] -= h * d[1];
            e1[2] -= h * d[2];
            double en = sqrt(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2]);
            e1[0] /= en;
            e1[1] /= en;
            e1[2] /= en;
            h = e2[0] * d[0] + e2[1] * d[1] + e2[2] * d[2];
            e2[0] -= h * d[0];
            e2[1] -= h * d[1];
            e2[2] -= h * d[2];
            h = e2[0] * e1[0] + e2[1] * e1[1] + e2[2] * e1[2];
            e2[0] -= h * e1[0];
            e2[1] -= h * e1[1];
            e2[2] -= h * e1[2];
            en = sqrt(e2[0] * e2[0] + e2[1] * e2[1] + e2[2] * e2[2]);
            e2[0] /= en;
            e2[1] /= en;
            e2[2] /= en;
            n_refl += 1;
            cum *= a->refl[tri];
        }
        a->n_segs[i] = (int32_t)(row - row0);
        a->n_refls[i] = n_refl;
    }
}

static void *trace_thread(void *p) {
    trace_range((const targs_t *)p);
    return NULL;
}

/* Trace rays [0, n_rays) into padded rows i*max_seg (bundle arrays zeroed/ones by caller). */
int oracle_trace(const double *v0, const double *v1, const double *v2, const double *refl,
                 int64_t n_tri, const double *bounds, double diameter, const double *origin,
                 const double *dirs, const double *e1s, const double *e2s, int64_t n_rays,
                 double length_cap, int64_t r_max, int64_t max_seg, double *so, double *sd,
                 double *se1, double *se2, double *sl, double *ss0, double *sr, int32_t *n_segs,
                 int32_t *n_refls, int threads) {
    targs_t base = {v0, v1, v2, refl, n_tri, bounds, diameter, origin, dirs, e1s, e2s,
                    length_cap, r_max, max_seg, so, sd, se1, se2, sl, ss0, sr, n_segs, n_refls,
                    0, n_rays};
    if (threads < 1) threads = 1;
    if (threads > n_rays) threads = n_rays > 0 ? (int)n_rays : 1;
    pthread_t *tid = calloc((size_t)threads, sizeof(pthread_t));
    targs_t *args = calloc((size_t)threads, sizeof(targs_t));
    if (!tid || !args) {
        free(tid);
        free(args);
        return -1;
    }
    /* interleaved blocks of 64 rays balance the per-ray cost */
    int64_t q = n_rays / threads, rem = n_rays % threads, lo = 0;
    for (int t = 0; t < threads; ++t) {
        int64_t size = q + (t < rem ? 1 : 0);
        args[t] = base;
        args[t].lo = lo;
        args[t].hi = lo + size;
        lo += size;
        pthread_create(&tid[t], NULL, trace_thread, &args[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    free(tid);
    free(args);
    return 0;
}
