/*
 * CPU ORACLE -- test infrastructure only.  Bit-exact restatement of the tile-level
 * work list of the fp32 GBS path (repo:paper_2501_13382_b200/csrc/exact_fp64.cu,
 * beam_dead_for_tile / worklist_kernel), i.e. of SURVEY.md 8(a) row a9:
 * a beam is not a candidate for a receiver tile (centre c, radius R_T) when every
 * segment k is either cut for the whole tile (its infinite line is farther than
 * R_k + R_T, R_k^2 = 72 c (s_end^2 + b^2)/(omega_min b), kernels.py:377-385) or,
 * for k == 0, the tile lies behind the launch plane (kernels.py:348,375).
 * Same fp64 operation order, no FMA (-ffp-contract=off), IEEE sqrt.
 *
 * tight = 1 restates the TIGHT list the fp32 kernel walks (a subset): with the tile's
 * bounding-box half extents h (box = n_tiles x 4: hx, hy, hz, R_T), the arc length the
 * tile reaches on k is s_hi = s0 + clamp(w.d + min(h.|d|, R_T), 0, len), the line
 * distance drops by at most min(h.|u|/|u|, R_T) (q convex, subgradient u/|u|), and the
 * behind test uses w.d + min(h.|d|, R_T) < -1e-6.
 */
#include <math.h>
#include <stdint.h>

static int beam_dead(const double *so, const double *sd, const double *sl, const double *ss0,
                     const int32_t *n_segs, int64_t max_seg, double width_b, int64_t b,
                     double cx, double cy, double cz, double rt, const double *h, double rscale,
                     int tight) {
    int ns = n_segs[b];
    for (int k = 0; k < ns; ++k) {
        int64_t row = b * max_seg + k;
        double wx = cx - so[3 * row], wy = cy - so[3 * row + 1], wz = cz - so[3 * row + 2];
        double dx = sd[3 * row], dy = sd[3 * row + 1], dz = sd[3 * row + 2];
        double proj = wx * dx + wy * dy + wz * dz;
        double ux = wx - proj * dx, uy = wy - proj * dy, uz = wz - proj * dz;
        double q2 = ux * ux + uy * uy + uz * uz;
        int dead;
        if (!tight) {
            double se = ss0[row] + sl[row];
            double rk = sqrt(rscale * (se * se + width_b * width_b));
            dead = sqrt(q2) - rt > rk * (1.0 + 1e-6) + 1e-6;
            if (k == 0) dead = dead || (proj + rt < -1e-6);
        } else {
            double rd = h[0] * fabs(dx) + h[1] * fabs(dy) + h[2] * fabs(dz);
            rd = rd < rt ? rd : rt;
            double reach = proj + rd;
            reach = reach < 0.0 ? 0.0 : (reach > sl[row] ? sl[row] : reach);
            double sh = ss0[row] + reach;
            double qn = sqrt(q2), rn = rt;
            if (qn > 0.0) {
                rn = (h[0] * fabs(ux) + h[1] * fabs(uy) + h[2] * fabs(uz)) / qn;
                rn = rn < rt ? rn : rt;
            }
            double rh = sqrt(rscale * (sh * sh + width_b * width_b));
            dead = qn - rn > rh * (1.0 + 1e-6) + 1e-6;
            if (k == 0) dead = dead || (proj + rd < -1e-6);
        }
        if (!dead) return 0;
    }
    return 1;
}

/* centre: (n_tiles, 4) = x, y, z, R_T; box: (n_tiles, 4) = hx, hy, hz, R_T (tight only,
 * may be NULL for the a9 list).  bits: (n_tiles, ceil(n_beams/32)). */
void oracle_worklist(const double *so, const double *sd, const double *sl, const double *ss0,
                     const int32_t *n_segs, int64_t n_beams, int64_t max_seg,
                     const double *centre, const double *box, int64_t n_tiles, double c,
                     double width_b, double omega_min, int use_cutoff, int tight,
                     uint32_t *bits) {
    const double rscale = use_cutoff ? 72.0 * c / (omega_min * width_b) : INFINITY;
    const int64_t n_words = (n_beams + 31) / 32;
    for (int64_t t = 0; t < n_tiles; ++t) {
        const double *ct = centre + 4 * t;
        const double *h = box ? box + 4 * t : ct;  /* unused by the a9 test */
        for (int64_t w = 0; w < n_words; ++w) {
            uint32_t m = 0;
            for (int j = 0; j < 32; ++j) {
                int64_t b = 32 * w + j;
                if (b < n_beams &&
                    !beam_dead(so, sd, sl, ss0, n_segs, max_seg, width_b, b, ct[0], ct[1], ct[2],
                               ct[3], h, rscale, tight))
                    m |= 1u << j;
            }
            bits[t * n_words + w] = m;
        }
    }
}
