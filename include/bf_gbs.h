/*
 * bf_gbs.h -- C ABI of the B200-native Gaussian Beam Summation (GBS) engine.
 *
 * Plain pointers and sizes only (no torch / C++ types).  Every entry point
 * returns a bf_status; on failure bf_last_error() returns a thread-local
 * message.  All functions are thread-safe.  A *_dev call given a caller stream
 * returns once its work is enqueued -- it never waits on the device (work-list
 * buffers are sized from a bound, statistics are copied back asynchronously) --
 * and the next call that uses the device's workspaces (on any stream) is ordered
 * after it by an event, so concurrent callers on different streams never see
 * each other's scratch buffers.  Results never depend on environment variables.
 *
 * Reference interface each entry point replaces (paths relative to
 * /root/reference/pkg/src/beamfield/):
 *
 *   bf_gbs_accumulate        kernels.gbs_accumulate           kernels.py:352-399
 *                            (called by parallel.run_pipeline.gbs_range,
 *                             parallel.py:320-327, and gbs.sum_at_observer,
 *                             gbs.py:196-201)
 *   bf_gbs_accumulate_dev    same operator, device-resident buffers (the
 *                            engine path used by run_pipeline on the GPU)
 *   bf_nearest_on_segments   kernels.nearest_on_segments      kernels.py:304-349
 *   bf_trace_range_dev       kernels.trace_range/trace_one    kernels.py:143-301
 *                            (+ bvh_nearest semantics kernels.py:54-116)
 *   bf_field_finalize_dev    parallel.py:343-344 (pressure = calibration*acc)
 *                            + gbs.spl                        gbs.py:39-46
 *   bf_plan_chunks           parallel.plan_chunks             parallel.py:91-105
 *   bf_tile_order_dev        parallel.block_partition/WorkerPool.flat observer split
 *                            (parallel.py:108-140), re-cut as spatial receiver tiles
 *
 * Array layouts are exactly the reference PathBundle's (beamtrace.py:218-288):
 * seg_origin/seg_dir/seg_e1/seg_e2 are (n_beams*max_seg, 3) C-contiguous fp64,
 * seg_len/seg_s0/seg_refl are (n_beams*max_seg,) fp64, beam b owns rows
 * [b*max_seg, b*max_seg + n_segs[b]); obs is (n_obs, 3) fp64; acc is
 * (n_obs, nf) complex128 stored as interleaved (re, im) doubles; evals is
 * (n_obs,) int64.  acc/evals rows [obs_lo, obs_hi) are CONTINUED in place
 * (kernels.py:358-359); nothing outside that range is touched.
 */
#ifndef BF_GBS_H
#define BF_GBS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    BF_OK = 0,
    BF_EINVAL = 1,  /* bad argument (maps to ValueError in the Python shim) */
    BF_ENOMEM = 2,  /* device or pinned-host allocation failed (MemoryError) */
    BF_ECUDA = 3,   /* CUDA runtime / launch failure (RuntimeError) */
    BF_ENODEV = 4,  /* no usable sm_100 device (RuntimeError) */
    BF_EBUDGET = 5, /* memory budget cannot hold one ray (BudgetError, parallel.py:98-100) */
    BF_EIO = 6      /* file output failed (OSError) */
} bf_status;

/* Arithmetic of the summation kernel. */
enum {
    BF_PRECISION_FP32 = 0, /* fast path: fp32 FMA/MUFU, fp64 tie re-decision,
                              fp64-anchored axial phase, fp64 accumulators */
    BF_PRECISION_FP64 = 1  /* oracle mode: reference operation order, no FMA */
};

/* Flags of bf_trace_range_dev. */
enum {
    BF_TRACE_EXHAUSTIVE = 1 /* test every triangle (self-check of the cluster culling) */
};

/* Library identification and diagnostics. */
const char *bf_version(void);
const char *bf_last_error(void);
int bf_device_count(void);
/* Number of CUDA kernels this library has launched in this process. */
uint64_t bf_launch_count(void);

/* Device-memory budget (bytes) of the summation's beam-group workspaces and
 * staging on `device`; 0 = automatic (1/8 of device memory, at most 24 GiB).
 * Changes the grouping only, never the results. */
int bf_set_memory_budget(int device, int64_t bytes);

/* Process-wide: record the fp32 summation's GPU time for bf_last_stats' kernel_ms
 * (two events around the kernels of every later call; ~10 us of graph-node latency on a
 * small call).  0 (default) = not recorded, kernel_ms reads 0.  Never changes results. */
int bf_set_kernel_timing(int on);

/*
 * Drop-in for kernels.gbs_accumulate (kernels.py:352-355) on HOST buffers
 * (pageable or pinned).  Argument order follows the reference; array sizes
 * (n_beams = rows/max_seg, n_obs, nf) are passed right after the array they size.
 * The call streams the beam range through the device in groups: host threads
 * pack each group's valid rows (no padding) into pinned staging, 68 B per segment
 * in fp32 mode (origin, direction, len, s0 in fp64 -- the exact re-decisions
 * need them bit for bit -- and the fp32 amplitude refl*w_b*phi sqrt(c)/(2 pi c)),
 * and the copy of group g+1 overlaps the summation of group g; device memory
 * stays within the budget however large the bundle.  fp64 mode streams padded
 * beam chunks the same way.  acc/evals[obs_lo:obs_hi] are copied back at the end.
 * Result bits equal bf_gbs_accumulate_dev's on the same inputs.
 */
int bf_gbs_accumulate(const double *seg_origin, const double *seg_dir,
                      const double *seg_e1, const double *seg_e2,
                      const double *seg_len, const double *seg_s0,
                      const double *seg_refl, const int32_t *n_segs, int64_t n_beams,
                      int64_t max_seg, const double *weights, const double *obs,
                      int64_t n_obs, const double *omegas, int64_t nf, double c,
                      double width_b, double phi_amp, int use_cutoff, double *acc,
                      int64_t *evals, int64_t obs_lo, int64_t obs_hi, int64_t beam_lo,
                      int64_t beam_hi, int precision, int device);

/* Flags of bf_gbs_accumulate_dev. */
enum {
    /* Observers [obs_lo, obs_hi) are already in spatial tile order (e.g. from
     * bf_tile_order_dev): consecutive blocks of bf_tile_size() receivers form
     * the kernel's tiles.  Used by the multi-GPU receiver-tile partition so a
     * receiver's result does not depend on the number of ranks. */
    BF_FLAG_OBS_PRESORTED = 1
};

/*
 * Same operator on DEVICE buffers (all pointers are device pointers on
 * `device`).  Asynchronous on `stream` (cudaStream_t, NULL = the engine's own
 * stream, which the call synchronises before returning; cudaStreamLegacy or
 * cudaStreamPerThread = the work runs on the engine's stream fenced in and out
 * of that stream by events, asynchronous and graph-capturable -- torch's
 * default stream is passed this way).  `omegas` is a HOST
 * array.  Any nf: frequencies are summed in groups of 8 (acc columns are
 * independent).  fp32 mode needs max_seg <= 30 (BF_EINVAL otherwise, before any
 * work) and fewer than 2^27 beams per call.
 *
 * The beams are summed in groups of whole beam ranges (the range size depends
 * only on the beam and frequency counts) whose workspaces fit the memory budget
 * (bf_set_memory_budget); the fp32 result bits do not depend on the budget, on
 * device vs host inputs, or on how receivers are sharded (BF_FLAG_OBS_PRESORTED).
 * They do depend on the call's beam and observer sets (patch-local fp32
 * geometry): splitting a call changes fp32 results within the fp32 tolerance,
 * while fp64 mode is bit-identical under any split of beams or observers.
 *
 * Small fp32 calls (<= 2^28 beam-receiver pairs) repeated with identical
 * arguments (pointers, sizes, scalars, frequencies, flags, stream) replay a CUDA
 * graph of the whole call captured on the second one; the graph reads the
 * buffers at replay time, the bits equal an eager call's, and it is dropped when
 * a workspace is reallocated.
 */
int bf_gbs_accumulate_dev(const double *seg_origin, const double *seg_dir,
                          const double *seg_e1, const double *seg_e2,
                          const double *seg_len, const double *seg_s0,
                          const double *seg_refl, const int32_t *n_segs, int64_t n_beams,
                          int64_t max_seg, const double *weights, const double *obs,
                          int64_t n_obs, const double *omegas, int64_t nf, double c,
                          double width_b, double phi_amp, int use_cutoff, double *acc,
                          int64_t *evals, int64_t obs_lo, int64_t obs_hi, int64_t beam_lo,
                          int64_t beam_hi, int precision, int flags, int device,
                          void *stream);

/*
 * Compact segment rows resident on one device -- the traced-ray output repacked into
 * the fp32 path's SoA (beam b owns rows [start[b], start[b+1]); per row origin/len and
 * direction/s0 in fp64, the fp32 amplitude A = phi sqrt(c)/(2 pi c) refl w_b: 68 B per
 * segment, no padding).  run_pipeline appends each traced chunk
 * (parallel.py:297-338) and sums ALL rays in one call, so the field does not depend on
 * the chunk plan.  Handles are not thread-safe; calls on them serialise on the device.
 */
typedef struct bf_rows bf_rows;
int bf_rows_create(int device, bf_rows **out);
int bf_rows_destroy(bf_rows *rows);
/* Beams and (exact) rows appended so far. */
int bf_rows_info(const bf_rows *rows, int64_t *n_beams, int64_t *n_rows);
/* Appends the valid rows of padded DEVICE bundle beams [0, n_beams) (reference PathBundle
 * layout, beamtrace.py:218-288; max_seg <= 30).  Ordered on `stream` (NULL = engine
 * stream); returns after the append (one sync for the exact row count). */
int bf_rows_append_dev(bf_rows *rows, const double *seg_origin, const double *seg_dir,
                       const double *seg_len, const double *seg_s0, const double *seg_refl,
                       const int32_t *n_segs, const double *weights, int64_t n_beams,
                       int64_t max_seg, double c, double phi_amp, void *stream);
/* bf_gbs_accumulate_dev (fp32 mode) over beams [beam_lo, beam_hi) of the resident rows:
 * same result bits as bf_gbs_accumulate_dev on the concatenated padded bundle. */
int bf_gbs_accumulate_rows_dev(const bf_rows *rows, const double *obs, int64_t n_obs,
                               const double *omegas, int64_t nf, double width_b, int use_cutoff,
                               double *acc, int64_t *evals, int64_t obs_lo, int64_t obs_hi,
                               int64_t beam_lo, int64_t beam_hi, int flags, void *stream);

/*
 * Work list of the fp32 path, exposed for verification: the
 * Hilbert receiver order perm (n_obs), tile centres/radii centre (n_tiles x 4:
 * x, y, z, R_T) and the candidate bitmask bits (n_tiles x ceil(n_beams/32)
 * uint32, bit b%32 of word b/32 = beam b may contribute to some receiver of the
 * tile).  tight_bits (same shape, may be NULL) is the subset the fp32 kernel
 * walks: with the tile's bounding box (half extents h, tile_box = n_tiles x 4:
 * hx, hy, hz, R_T, may be NULL), R_k from the largest arc length
 * s_hi = s0 + clamp(w.d + min(h.|d|, R_T), 0, len) the tile reaches and the line
 * distance lowered by min(h.|u|/|u|, R_T) (u: the centre's offset from the line).
 * Host buffers; exact fp64 tests, reproduced bit for bit by oracle/worklist_oracle.c.
 */
int bf_worklist(const double *seg_origin, const double *seg_dir, const double *seg_len,
                const double *seg_s0, const int32_t *n_segs, int64_t n_beams, int64_t max_seg,
                const double *obs, int64_t n_obs, const double *omegas, int64_t nf, double c,
                double width_b, int use_cutoff, int32_t *perm, double *centre, double *tile_box,
                uint32_t *bits, uint32_t *tight_bits, int64_t n_tiles_cap, int64_t *n_tiles_out,
                int device);

/*
 * Pair counts of the last fp32 summation on this thread (FLOP model of the roofline,
 * SURVEY 8(d)): (beam, receiver) pairs and pair-segments (sum of the beam's n_segs)
 * on the a9 work list, on the tight work list the kernel walks, and in the
 * (patch, beam) items the kernel evaluated (after its own patch-level culling).
 */
int bf_last_pair_stats(int64_t *a9_pairs, int64_t *a9_pair_segs, int64_t *tight_pairs,
                       int64_t *tight_pair_segs, int64_t *live_pairs, int64_t *live_pair_segs);

/*
 * Field CSV writer, replaces beamfield.harness.write_field_csv (harness.py:197-208):
 * header "x,y,z,freq_hz,re_p,im_p,spl_db", one row per (observer, frequency),
 * observer-major, numbers as Python format(x, ".17g") (harness.py:39-40).  points is
 * (n_obs, 3), pressure (n_obs, nf) complex128 interleaved, spl (n_obs, nf); host
 * buffers.  Rows are formatted on `threads` host threads (<= 0: all) and written in
 * order, byte-identical to the reference's row loop.
 */
int bf_write_field_csv(const char *path, const double *points, int64_t n_obs,
                       const double *freqs, int64_t nf, const double *pressure,
                       const double *spl, int threads);

/* Receivers per tile of the fp32 summation kernel. */
int bf_tile_size(void);

/*
 * Spatial order of n device observers (Hilbert curve, 21 bits per axis, isotropic
 * over the bounding box; the 2-D curve for planar sets): perm[i] = index of the i-th
 * receiver in tile order.  Deterministic,
 * so every rank of a multi-GPU run derives the same receiver-tile partition.
 */
int bf_tile_order_dev(const double *obs, int64_t n, int32_t *perm, int device, void *stream);

/*
 * kernels.nearest_on_segments (kernels.py:304-349) for n_query (observer,
 * beam) pairs on the device (fp64, reference operation order).  Host
 * buffers.  out is (n_query, 6): k, s, q1, q2, refl, behind.
 */
int bf_nearest_on_segments(const double *seg_origin, const double *seg_dir,
                           const double *seg_e1, const double *seg_e2,
                           const double *seg_len, const double *seg_s0,
                           const double *seg_refl, const int32_t *n_segs, int64_t n_beams,
                           int64_t max_seg, const double *obs, int64_t n_obs,
                           const int64_t *q_obs, const int64_t *q_beam, int64_t n_query,
                           double *out, int device);

/*
 * Ray marching (kernels.trace_range, kernels.py:282-301) of launch rays
 * [lo, hi) into bundle rows [(lo-row_base)*max_seg, ...), on DEVICE buffers.
 * Nearest-hit semantics of bvh_nearest (kernels.py:54-116): smallest t in
 * (EPS_HIT, remaining], ties to the lower triangle index.  fp64, reference
 * operation order, no FMA.  v0/v1/v2 are (n_tri, 3); refl_coef (n_tri,);
 * bounds = (bmin xyz, bmax xyz); dirs/e1s/e2s are (n_rays, 3).
 */
int bf_trace_range_dev(const double *v0, const double *v1, const double *v2,
                       const double *refl_coef, int64_t n_tri, const double *bounds,
                       double diameter, const double *origin, const double *dirs,
                       const double *e1s, const double *e2s, double length_cap,
                       int64_t r_max, int64_t max_seg, double *seg_origin, double *seg_dir,
                       double *seg_e1, double *seg_e2, double *seg_len, double *seg_s0,
                       double *seg_refl, int32_t *n_segs, int32_t *n_refls, int64_t lo,
                       int64_t hi, int64_t row_base, int flags, int device, void *stream);

/*
 * pressure = calibration * acc (parallel.py:343) and spl = 20 log10(|p|/2e-5),
 * -inf for |p| == 0 (gbs.py:39-46), over n complex values on the device.
 */
int bf_field_finalize_dev(const double *acc, int64_t n, double calibration,
                          double *pressure, double *spl, int device, void *stream);

/* parallel.plan_chunks (parallel.py:91-105): greedy maximal chunks.
 * Writes up to max_chunks sizes, returns the count in *n_chunks. */
int bf_plan_chunks(int64_t total_rays, int64_t memory_budget, int64_t per_ray_bytes,
                   int64_t *chunk_sizes, int64_t max_chunks, int64_t *n_chunks);

/* Statistics of the last fp32 bf_gbs_accumulate* call on this thread:
 * candidate (beam, receiver) pairs of the tile work list, total pairs, fp64
 * tie re-decisions, receiver tiles, non-behind pairs (P_nb), the CUDA-event
 * duration of the summation (first summation kernel start to last kernel end; 0
 * unless bf_set_kernel_timing(1) was in effect for the call),
 * and the sum of n_segs over candidate pairs (the scan term of the FLOP model).
 * Any pointer may be NULL.  The counters are copied back asynchronously by the
 * call; this function waits for that copy (the only place the engine waits on
 * the device for statistics). */
int bf_last_stats(int64_t *candidate_pairs, int64_t *total_pairs, int64_t *tie_pairs,
                  int64_t *n_tiles, int64_t *nonbehind_pairs, double *kernel_ms,
                  int64_t *candidate_pair_segs);

/* Work-generation outcome of the last fp32 call on this thread, counted per
 * (warp patch of 128 receivers, beam) item: culled (every pair cut/behind),
 * single surviving segment, corner wedge (two segments, exact fp64 pick),
 * general multi-segment scan. */
int bf_last_path_stats(int64_t *culled, int64_t *single, int64_t *wedge, int64_t *multi);

/* Microbenchmarks of the pipes the summation is bound by, on `device`:
 * dependent-free FFMA stream (TFLOP/s, 2 flop per FFMA) and MUFU ex2 stream
 * (Tops/s).  Used for the roofline denominators in bench.py. */
int bf_probe_peaks(int device, double *fp32_tflops, double *mufu_tops);

#ifdef __cplusplus
}
#endif
#endif /* BF_GBS_H */
