// common.cuh -- shared definitions of the B200 GBS engine (internal).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bf_gbs.h"

#define BF_MAXF 8            // frequencies per kernel launch (calls loop over groups of <= 8)
#define BF_FP32_MAX_SEG 30   // fp32 path: survivor masks share a word with two flag bits
#define BF_CUTOFF_EXPONENT (-36.0)  // kernels.py:18
#define BF_EPS_HIT 1e-6              // kernels.py:14

namespace bf {

// Records a failure message for bf_last_error() and returns the status.
int fail(int status, const char *fmt, ...);
// Counts one kernel launch of this library (bf_launch_count()).
void note_launch(int n = 1);
// Converts a CUDA error (if any) into BF_ECUDA with a message.
int check_cuda(cudaError_t e, const char *what);

#define BF_TRY_CUDA(expr)                                   \
    do {                                                    \
        cudaError_t _e = (expr);                            \
        if (_e != cudaSuccess) return ::bf::check_cuda(_e, #expr); \
    } while (0)

#define BF_TRY(expr)                 \
    do {                             \
        int _s = (expr);             \
        if (_s != BF_OK) return _s;  \
    } while (0)

// Arguments of one summation over LOCAL ranges: beam 0 here is the caller's
// beam_lo, observer 0 is obs_lo.  Row r of beam b is b*max_seg + r (padded
// reference layout, beamtrace.py:274-288).
struct GbsArgs {
    const double *seg_origin, *seg_dir, *seg_e1, *seg_e2, *seg_len, *seg_s0, *seg_refl;
    const int32_t *n_segs;
    const double *weights;
    const double *obs;
    int64_t max_seg;
    int64_t n_beams;  // local beam count
    int64_t n_obs;    // local observer count
    int nf;
    double omegas[BF_MAXF];
    double c, width_b, phi_amp;
    int use_cutoff;
    double *acc;      // (n_obs, acc_stride) complex, interleaved; columns [0, nf) are ours
    int64_t acc_stride;  // complex values per observer row of acc (>= nf)
    int64_t *evals;   // (n_obs,)
};

// Compact segment rows on the device (the fp32 path's input layout): beam b owns rows
// [start[b], start[b] + n_segs[b]) of p0/p1/amp, no padding (the reference's padded
// PathBundle rows beyond n_segs, beamtrace.py:274-288, are dropped when packing).
// start has n_beams + 1 entries; start[n_beams] = end of the last beam's rows.
// p0/p1 are exact copies of the reference's fp64 values (the exact re-decisions and the
// work-list bound use them bit for bit); amp is the fp32 amplitude factor
// A = phi sqrt(c)/(2 pi c) * refl * w_b (kernels.py:388,397 without omega).
struct Rows {
    const int64_t *start;
    const double4 *p0;  // per row: origin xyz, len
    const double4 *p1;  // per row: direction xyz, s0
    const float *amp;   // per row: A
    int64_t n_beams;
    int64_t max_seg;    // bound on segments per beam (the padded row count)
};

// Work-list statistics of the fp32 path (device counters, copied back).
struct GbsStats {
    unsigned long long candidate_pairs;  // (beam, receiver) pairs inside candidate tiles
    unsigned long long tie_pairs;        // pairs re-decided in fp64
    unsigned long long nb_pairs;         // non-behind pairs (P_nb of SURVEY 8(d))
    unsigned long long cand_pair_segs;   // sum over candidate pairs of the beam's n_segs
    unsigned long long paths[4];         // (warp patch, beam) items: culled, single, wedge, multi
    unsigned long long multi_surv[4];    // multi items with 2, 3, 4, >= 5 surviving segments
    unsigned long long tight_pairs;      // (beam, receiver) pairs on the tight work list
    unsigned long long tight_pair_segs;  // sum over those pairs of the beam's n_segs
    unsigned long long live_pairs;       // pairs of the (patch, beam) items the kernel evaluates
    unsigned long long live_pair_segs;   // sum over those pairs of the beam's n_segs
    float kernel_ms;                     // CUDA-event duration of the summation kernel
};

// Receiver tiling built per call for the fp32 path (engine.cu).
struct Tiling {
    int64_t n;          // receivers
    int64_t n_tiles;
    int tile;           // receivers per tile
    const int32_t *perm;      // sorted position -> local observer index
    const float4 *rloc;       // sorted position -> (p - centre) fp32, w = unused
    const double4 *centre;    // per tile: centre xyz, radius
    const double4 *tbox;      // per tile: bounding-box half extents xyz, radius
    const uint32_t *wl_bits;  // work list: (tile, beam) candidate bits, wl_words per tile
    const uint32_t *wl_tight; // tight work list (subset of wl_bits) the fp32 kernel walks
    int64_t wl_words;
};

// Workspace of the fp32 path (engine.cu allocates, gbs_fp32.cu fills and uses).
// Row arrays use the padded row index b*max_seg + k of the reference bundle.
struct Fp32Work {
    const int64_t *start;     // compact rows (Rows): beam -> first row
    const double4 *p0;        // per row: origin xyz, len
    const double4 *p1;        // per row: direction xyz, s0
    const float *amp;         // per row: amplitude factor A
    float4 *prl;              // sorted receiver -> patch-local fp32 coordinates, |r|^2
    double4 *pos64;           // sorted receiver -> fp64 position (exact re-decisions)
    double4 *pcen;            // per patch: centre xyz, radius
    float4 *pbox;             // per patch: bounding-box half extents xyz, radius (patch-local)
    double2 *part;            // per (beam range, sorted receiver, frequency): unit partial sum
    int *part_ev;             // per (beam range, sorted receiver): unit evaluation count
    unsigned *unit_ctr;       // persistent-kernel work queue head
    unsigned *n_wide;         // units of wide patches (device; the wide kernel takes them)
    float wide_k, wide_q;     // patch radius RW is wide iff RW wide_k > 1 or RW^2 wide_q > 1
    uint32_t *wl_items;       // compacted tight work list: per (tile, beam range), ascending
                              // beams, entry = (n_segs - 1) << 27 | beam
    int64_t *wl_off;          // n_tiles * n_ranges + 1 offsets into wl_items
    const int32_t *unit_order;  // queue position -> unit q * n_patches + p (longest-first
                                // buckets, range-major inside; see unit_keys_kernel)
    int64_t n_patches, n_ranges, range_beams, n_pad;  // n_pad = n_patches * patch
};

// A launch's stream plus an auxiliary stream and two events for a fork/join inside it.
struct StreamPair {
    cudaStream_t st, aux;
    cudaEvent_t fork, join;
};

// Launchers (return BF_OK or an error status).
// oracle-mode summation of the observers in tile order over each tile's tight work list
// (a.obs / a.acc / a.evals indexed by perm[sorted position])
int launch_gbs_fp64(const GbsArgs &a, const int32_t *perm, int tile, const uint32_t *tbits,
                    int64_t n_words, cudaStream_t st);
int gbs_fp32_tile();
int gbs_fp32_patch();
int64_t gbs_fp32_range_beams(int64_t n_beams, int nf);
// Padded reference bundle (GbsArgs, local beams) -> compact rows.  start must already
// hold the exclusive scan of n_segs (n_beams + 1 entries); amp_scale = phi sqrt(c)/(2 pi c).
int launch_rows_pack(const GbsArgs &a, const int64_t *start, double4 *p0, double4 *p1,
                     float *amp, cudaStream_t st);
// cnt[0] = base, cnt[b + 1] = n_segs[b] clamped to [0, max_seg]; an inclusive scan of cnt
// (engine.cu, cub) then gives the compact row starts (rows from `base` on).
int launch_rows_count(const int32_t *n_segs, int64_t n_beams, int64_t max_seg, int64_t base,
                      int64_t *cnt, cudaStream_t st);
// Beams [b0, b0 + nb) of resident rows src -> rows of their own (start rebased to 0).
int launch_rows_slice(const Rows &src, int64_t b0, int64_t nb, int64_t *start, double4 *p0,
                      double4 *p1, float *amp, cudaStream_t st);
// Patch-local receivers of the tiling (w.prl, w.pcen, w.pbox).
int launch_fp32_patches(const GbsArgs &a, const Tiling &t, Fp32Work &w, cudaStream_t st);
// Work-list compaction (north star: prefix-sum compaction into (beam, tile) lists):
// counts per (tile, range) into w.wl_off (pass 1), then, after an exclusive scan of
// the counts, the entries (pass 2).
// wstats (4 x n_tiles, zeroed): per tile a9 candidate beams, their segments, tight
// candidate beams, their segments.
// Queue order: keys (wide << 13 | longest-first bucket << 6 | range) and unit values,
// radix-sorted.
int launch_fp32_unit_keys(const Tiling &t, const Fp32Work &w,
                          const int64_t *counts, uint64_t *keys, int32_t *vals, cudaStream_t st);
// one CTA: unit keys + counting sort + wide count, for n_patches * n_ranges <= SMALL_QUEUE_N
constexpr int64_t SMALL_QUEUE_N = 32768;
int launch_fp32_small_queue(const Fp32Work &w, const int64_t *counts, int32_t *order,
                            cudaStream_t st);
int launch_fp32_wl_compact(const Tiling &t, const Fp32Work &w, cudaStream_t st);
// The summation of one group of beam ranges (wide-patch kernel on st.aux first, the
// common kernel on st.st), without the fold.
int launch_gbs_fp32(const GbsArgs &a, const Tiling &t, const Fp32Work &w, GbsStats *d_stats,
                    const StreamPair &st);
// acc[:, :nf] += the group's unit partials over its ranges (ascending), evals alike.
int launch_fp32_fold(const GbsArgs &a, const Tiling &t, const Fp32Work &w, cudaStream_t st);
int launch_nearest(const GbsArgs &a, const int64_t *q_obs, const int64_t *q_beam,
                   int64_t n_query, double *out, cudaStream_t st);
// cbox: scratch for ceil(n_tri/16) cluster boxes (6 doubles each), or null for the
// exhaustive hit search.
int trace_cluster_count(int64_t n_tri);
int launch_trace(const double *v0, const double *v1, const double *v2, const double *refl,
                 int64_t n_tri, double *cbox, const double *bounds, double diameter, const double *origin,
                 const double *dirs, const double *e1s, const double *e2s, double length_cap,
                 int64_t r_max, int64_t max_seg, double *seg_origin, double *seg_dir,
                 double *seg_e1, double *seg_e2, double *seg_len, double *seg_s0,
                 double *seg_refl, int32_t *n_segs, int32_t *n_refls, int64_t lo, int64_t hi,
                 int64_t row_base, cudaStream_t st);
// Work lists of tiling (centre, tbox) against the compact rows r (beams [0, r.n_beams)).
int launch_worklist(const GbsArgs &a, const Rows &r, const double4 *centre, const double4 *tbox,
                    int64_t n_tiles, double omega_min, uint32_t *bits, uint32_t *tbits,
                    int64_t range_beams, int64_t n_ranges, unsigned long long *counts,
                    unsigned long long *wstats, cudaStream_t st);
int launch_finalize(const double *acc, int64_t n, double calibration, double *pressure,
                    double *spl, cudaStream_t st);

}  // namespace bf
