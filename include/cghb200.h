/*
 * cghb200 — C ABI of the B200-native hologram-generation hot path.
 *
 * Plain C types only (no torch, no CUDA types in signatures). Every entry
 * point is reentrant: state lives in the caller's arguments or in an opaque
 * plan owned by one thread at a time; each call/plan has its own CUDA stream.
 * All host arrays are caller-owned, C-contiguous, row-major; complex arrays
 * are interleaved (re, im) float64 — numpy complex128 layout.
 *
 * Each function names the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/cghkit/).
 */
#ifndef CGHB200_H
#define CGHB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: one per reference exception class (errors.py:79-108) --- */
#define CGH_OK 0
#define CGH_ERR_DIMENSION 1      /* DimensionMismatchError */
#define CGH_ERR_ZERO_TARGET 2    /* ZeroTargetError */
#define CGH_ERR_EMPTY_MASK 3     /* EmptyMaskError */
#define CGH_ERR_INVALID_SPEC 4   /* InvalidSpecError */
#define CGH_ERR_NONFINITE 5      /* NonFiniteError */
#define CGH_ERR_ZERO_FIELD 6     /* ZeroFieldError */
#define CGH_ERR_VALUE 7          /* ValueError (bad init mode / direction / argument) */
#define CGH_ERR_UNSUPPORTED 8    /* shape outside the implemented set (raised loudly) */
#define CGH_ERR_CUDA 9           /* CUDA runtime failure */
#define CGH_ERR_NO_DEVICE 10     /* no CUDA device / library built without GPU */
#define CGH_ERR_MEMORY 11        /* device or host allocation failed */

#define CGH_FP32 0
#define CGH_FP64 1

#define CGH_SCHEME_PHASE 0       /* slm.py:18-31 PhaseOnly (binary_phase = 2 levels) */
#define CGH_SCHEME_AMPLITUDE 1   /* slm.py:34-42 AmplitudeOnly */
#define CGH_SCHEME_MULTI 2       /* slm.py:45-55 MultiAmp */

#define CGH_FOURIER 0
#define CGH_FRESNEL 1

#define CGH_COMPLETED 0          /* algorithms.py:48-50 */
#define CGH_CONVERGED 1
#define CGH_CANCELLED 2

#define CGH_INIT_RANDOM_PHASE 0  /* algorithms.py:42-43 */
#define CGH_INIT_BACKPROPAGATE 1

/* numpy PCG64 state (bit_generator.state): 128-bit state and increment, the
 * buffered 32-bit half (has_uint32/uinteger). */
typedef struct cgh_pcg64 {
    uint64_t state_hi, state_lo;
    uint64_t inc_hi, inc_lo;
    int32_t has_uint32;
    uint32_t uinteger;
} cgh_pcg64;

/* One generation problem: SLM (slm.py:58-64), scheme states (slm.py:71-79,
 * computed by the caller exactly as the reference does), propagation
 * (propagation.py:38-55) and metric flag (propagation.py:58-63). */
typedef struct cgh_problem {
    int32_t height, width;
    int32_t precision;          /* CGH_FP32 | CGH_FP64 (GS/OSPR/transforms) */
    int32_t device;
    int32_t scheme_kind;
    int32_t n_states;
    double phase_offset;        /* PhaseOnly.phase_offset */
    const double *states;       /* n_states complex128 */
    int32_t prop_kind;          /* CGH_FOURIER | CGH_FRESNEL */
    double wavelength, distance, pitch_x, pitch_y;
    int32_t rescale;            /* MetricSpec.rescale */
} cgh_problem;

typedef int (*cgh_cancel_fn)(void *user);
typedef void (*cgh_progress_fn)(void *user, int64_t k, double err);
/* audit(k, incremental_unscaled_error, index_plane int32[H*W]) — SA/DBS test hook */
typedef void (*cgh_audit_fn)(void *user, int64_t k, double inc_err, const int32_t *indices);

typedef struct cgh_callbacks {
    cgh_cancel_fn cancel;       /* polled before each iteration/frame/checkpoint chunk */
    cgh_progress_fn progress;   /* called in order on the calling thread */
    cgh_audit_fn audit;
    void *user;
} cgh_callbacks;

/* RunReport (algorithms.py:84-94) minus the Python-side fields. The trace is
 * written to caller arrays trace_k/trace_v of capacity trace_cap. */
typedef struct cgh_report {
    double final_error;
    double efficiency;
    int64_t iterations_executed;
    int32_t termination;        /* CGH_COMPLETED | CGH_CONVERGED | CGH_CANCELLED */
    int64_t trace_len;
    int64_t kernel_launches;    /* kernels this call launched (evidence/bench) */
    double device_ms;           /* CUDA-event time of the device work */
} cgh_report;

typedef struct cgh_gs_params {   /* algorithms.py:57-81 (gs fields) */
    int32_t iterations;
    double feedback_gain;
    int32_t quantize_each_iteration;
    int32_t init_mode;           /* CGH_INIT_* */
    cgh_pcg64 rng;               /* PCG64(seed) — algorithms.py:160 */
} cgh_gs_params;

typedef struct cgh_ospr_params { /* algorithms.py:473-487 */
    int32_t subframes;
    const cgh_pcg64 *frame_rng;  /* subframes entries: PCG64(SeedSequence(seed).spawn(S)[i]) */
} cgh_ospr_params;

typedef struct cgh_sa_params {   /* algorithms.py:343-404 */
    int64_t proposals;
    double initial_temperature;  /* < 0 : auto (100 warm-up proposals) */
    double cooling_factor;
    int32_t init_mode;
    cgh_pcg64 rng;               /* PCG64(seed) at draw 0 */
    int64_t log_cap;             /* record the first log_cap proposals (0 = off) */
    int64_t *log_pixel;          /* [log_cap] proposal pixel m*W+n (warm-up excluded) */
    int32_t *log_level;          /* [log_cap] proposed level */
    uint8_t *log_accept;         /* [log_cap] 1 = committed */
} cgh_sa_params;

typedef struct cgh_dbs_params {  /* algorithms.py:410-467 */
    int32_t max_passes;
    int32_t scan_random;         /* scan_order == "random" */
    int32_t init_mode;
    cgh_pcg64 rng;               /* PCG64(SeedSequence(seed)) at draw 0 */
    /* random order: per-pass permutation streams PCG64(root.spawn(1)[0]),
       one per pass (max_passes entries) — algorithms.py:437-439 */
    const cgh_pcg64 *pass_rng;
    int64_t log_cap;             /* record the first log_cap pixel visits */
    int64_t *log_pixel;
    int32_t *log_level;          /* committed level or -1 */
    double *log_change;
} cgh_dbs_params;

/* ---- library ---------------------------------------------------------- */
int cgh_version(void);
const char *cgh_last_error(void);               /* thread-local message of the last failure */
int cgh_device_count(int32_t *count);

/* ---- transforms: propagation.py:81-94 (fft2), 110-123 (propagate[_inverse])
 * op 0 = fft2 forward (centred), 1 = fft2 inverse, 2 = propagate,
 * 3 = propagate_inverse. in/out: H*W complex128. Power-of-two sides up to 4096
 * run the row/column passes; any other shape runs Bluestein line transforms
 * (sides up to 4096 in fp64, 8192 in fp32). */
int cgh_transform(const cgh_problem *pb, const double *in, double *out, int32_t op);

/* ---- masked metric sums on the device, fp64, fixed order (mse_error /
 * efficiency, propagation.py:164-202). r = |replay|, t = |target|:
 * out[6] = {count_in, sum_in t^2, sum_in r^2, sum_in r t, sum_in (scale r - t)^2, sum_all r^2}. */
int cgh_masked_sums(int32_t device, const double *replay, const double *target, const uint8_t *mask,
                    int64_t count, double scale, double *out);

/* ---- slm.py:86-108 quantize_indices on the device (fp64). */
int cgh_quantize(const cgh_problem *pb, const double *values, int64_t count, int32_t *out_idx);

/* ---- runners. target: H*W complex128 (centred, as given to the reference);
 * mask: H*W bytes (centred MetricSpec.mask); illumination: H*W complex128 or
 * NULL. out_idx: index plane(s), uint8 when n_states <= 256 else int32.
 * out_field (GS only, nullable): complex128 hologram after the last
 * iteration's projection, before the final snap (parity checks). */
int cgh_gs_run(const cgh_problem *pb, const cgh_gs_params *gp, const double *target, const uint8_t *mask,
               const double *illumination, void *out_idx, double *out_field, int64_t *trace_k,
               double *trace_v, int64_t trace_cap, cgh_report *rep, const cgh_callbacks *cb);   /* algorithms.py:147 run_gs */
int cgh_ospr_run(const cgh_problem *pb, const cgh_ospr_params *op, const double *target, const uint8_t *mask,
                 const double *illumination, void *out_idx, int64_t *trace_k, double *trace_v,
                 int64_t trace_cap, cgh_report *rep, const cgh_callbacks *cb);                 /* algorithms.py:473 run_ospr */
int cgh_sa_run(const cgh_problem *pb, const cgh_sa_params *sp, const double *target, const uint8_t *mask,
               const double *illumination, void *out_idx, int64_t *trace_k, double *trace_v,
               int64_t trace_cap, cgh_report *rep, const cgh_callbacks *cb);                   /* algorithms.py:343 run_sa */
int cgh_dbs_run(const cgh_problem *pb, const cgh_dbs_params *dp, const double *target, const uint8_t *mask,
                const double *illumination, void *out_idx, int64_t *trace_k, double *trace_v,
                int64_t trace_cap, cgh_report *rep, const cgh_callbacks *cb);                  /* algorithms.py:410 run_dbs */

/* ---- device-resident plans (benchmarks / batched callers) --------------
 * A plan owns the device buffers and stream for one (H, W, precision, device).
 * set_target uploads and prepares the target once; run_* then execute with
 * inputs resident in HBM and leave the index planes on the device
 * (cgh_plan_download_idx copies them out). */
typedef struct cgh_plan cgh_plan;
int cgh_plan_create(const cgh_problem *pb, cgh_plan **out);
int cgh_plan_destroy(cgh_plan *plan);
int cgh_plan_set_target(cgh_plan *plan, const double *target, const uint8_t *mask, const double *illumination);
/* As cgh_plan_set_target; flags bit 0 (CGH_TARGET_AMPLITUDE_ONLY): the runs of
 * this target never start from the backpropagated target (random-phase GS /
 * SA / DBS, OSPR), so fp32 plans build the shifted amplitude plane on host
 * threads and upload 4 B/px instead of the complex128 target and the mask. A
 * backpropagation start then fails with CGH_ERR_VALUE until the target is set
 * again with flags = 0. */
#define CGH_TARGET_AMPLITUDE_ONLY 1
int cgh_plan_set_target_ex(cgh_plan *plan, const double *target, const uint8_t *mask, const double *illumination,
                           int32_t flags);
int cgh_plan_gs(cgh_plan *plan, const cgh_gs_params *gp, int64_t *trace_k, double *trace_v, int64_t trace_cap,
                cgh_report *rep, const cgh_callbacks *cb);
int cgh_plan_ospr(cgh_plan *plan, const cgh_ospr_params *op, int64_t *trace_k, double *trace_v,
                  int64_t trace_cap, cgh_report *rep, const cgh_callbacks *cb);
int cgh_plan_sa(cgh_plan *plan, const cgh_sa_params *sp, int64_t *trace_k, double *trace_v, int64_t trace_cap,
                cgh_report *rep, const cgh_callbacks *cb);      /* plan must be CGH_FP64 */
int cgh_plan_dbs(cgh_plan *plan, const cgh_dbs_params *dp, int64_t *trace_k, double *trace_v, int64_t trace_cap,
                 cgh_report *rep, const cgh_callbacks *cb);     /* plan must be CGH_FP64 */
int cgh_plan_download_idx(cgh_plan *plan, void *out_idx, int64_t frames);
/* OSPR sharded over subframes: this plan's contiguous
 * part [frame0, frame0 + op->subframes) (1..64 frames, op->frame_rng = their
 * streams) of an nframes_total-subframe run. Phase 1 generates the part
 * (index planes final) and leaves its own |R|^2 total in the plan's intensity
 * plane; the caller sets the plane to the lower parts' totals
 * (cgh_plan_set_intensity) and phase 2 re-accumulates with the global frame
 * numbers: trace = the reference's cumulative errors of these frames, and the
 * efficiency when the part ends the run. */
int cgh_plan_ospr_part(cgh_plan *plan, const cgh_ospr_params *op, int32_t frame0, int32_t nframes_total,
                       int32_t phase, int64_t *trace_k, double *trace_v, int64_t trace_cap, cgh_report *rep);
/* intensity plane := sum of `count` device planes (H*W of the plan's real
 * type; peer pointers allowed), fixed order 0, 1, ...; count 0 zeroes it. */
int cgh_plan_set_intensity(cgh_plan *plan, const void *const *planes, int32_t count);
/* copy the intensity plane (H*W reals) to device address dst */
int cgh_plan_copy_intensity(cgh_plan *plan, void *dst);
/* device address / bytes of the plan's intensity plane */
int cgh_plan_intensity(cgh_plan *plan, void **out_ptr, int64_t *out_bytes);
void *cgh_plan_stream(cgh_plan *plan);          /* cudaStream_t of the plan */
/* Per-pass CUDA-event timing: returns the accumulated ms / launch counts per
 * pass id since the last call (ids: row modes 0-7, column modes 8-15, search
 * kernels 16-23; n entries), clears them, and switches timing on/off. */
int cgh_plan_profile(cgh_plan *plan, int32_t enable, double *ms, int64_t *counts, int32_t n);
/* Timing experiments: with profiling on and CGHB200_WL_STAMPS set, the
 * warp-line 2048^2 passes record per-warp stage timestamps (globaltimer,
 * clock64 pairs: [pass 0 row / 1 column][1024 CTAs][16 warps][8 marks][2]). */
int cgh_debug_wl_stamps(cgh_plan *plan, int64_t *out, int64_t cap);
int cgh_plan_sync(cgh_plan *plan);

/* ---- reference-kernel seam: kernels/__init__.py:42-44 (delta_error,
 * commit_update, best_delta, _core.pyx:20-83) on the device, fp64.
 * replay_m: count complex128 (in/out for commit); target_m: count float64;
 * row_tw/col_tw: the pixel's DFT-table rows (complex128, lengths H and W). */
int cgh_delta_error(int32_t device, const double *replay_m, const double *target_m, const double *row_tw,
                    const double *col_tw, const int32_t *mu, const int32_t *mv, int64_t count, int32_t h,
                    int32_t w, double delta_re, double delta_im, double *out);
int cgh_commit_update(int32_t device, double *replay_m, const double *row_tw, const double *col_tw,
                      const int32_t *mu, const int32_t *mv, int64_t count, int32_t h, int32_t w,
                      double delta_re, double delta_im);
int cgh_best_delta(int32_t device, const double *replay_m, const double *target_m, const double *row_tw,
                   const double *col_tw, const int32_t *mu, const int32_t *mv, int64_t count, int32_t h,
                   int32_t w, const double *deltas, int64_t levels, int64_t *best_index, double *best_change);

/* ---- row-distributed GS slabs (config C6: one N x N run over G ranks) -----
 * Replaces the pass loop of run_gs (algorithms.py:147-202) for one rank of a
 * row-slab decomposition; the caller (paper_2006_10509_b200/slab.py) owns the
 * device buffers and runs the all-to-all (NCCL) between passes on `stream`.
 * A slab holds R = N/G lines as G segments of S = N/G points, segment-major:
 * element (line i, position n) at ((n/S)*R + i)*S + n%S; block g (S*S
 * elements) is the chunk exchanged with rank g. pb->height = pb->width = N
 * (global). Pass modes: 0 random-phase init [-> snap] -> forward; 1 hologram
 * pass (inverse -> beam*x/|x| [-> snap] -> forward); 2 replay pass (forward ->
 * error sums + amplitude projection -> inverse); 3 final replay (sums only);
 * 4 inverse (backpropagation start); 6 forward, unscaled (transform only). Sums: 4 doubles {S_dd, S_rr, S_rd,
 * S_all} of this rank written to the device pointer `sums` (modes 2, 3). */
typedef struct cgh_slab cgh_slab;
int cgh_slab_create(const cgh_problem *pb, int32_t world, int32_t rank, void *stream, cgh_slab **out);
int cgh_slab_destroy(cgh_slab *slab);
/* tgt_local: R x N float64, the ifftshifted |target| of this rank's columns
 * (transposed), sign bit set outside the mask; beam_local: R x N |illumination|
 * of this rank's hologram rows, or NULL. */
int cgh_slab_set_local(cgh_slab *slab, const double *tgt_local, const double *beam_local);
int cgh_slab_pass(cgh_slab *slab, int32_t mode, void *data, const cgh_gs_params *gp, int32_t quantize,
                  void *idx_out, double *sums);
/* dst[g] = transpose(src[g]) for every S x S block (the corner turn). */
int cgh_slab_transpose(cgh_slab *slab, const void *src, void *dst);
/* Corner turn fused with the exchange: transpose(src[g]) is stored directly
 * to dst_blocks[g] (G device pointers, e.g. rank g's receive buffer at chunk
 * [this rank] through NVLink peer mappings). The caller orders the peers'
 * next reads after it with a device barrier (one per turn). */
int cgh_slab_turn(cgh_slab *slab, const void *src, void *const *dst_blocks);

/* ---- multi-GPU plumbing (one process per GPU; SURVEY.md §8(b) cgh_multi_*,
 * §8(e)): NCCL communicators (NCCL resolved at run time from the process's
 * libnccl.so.2), CUDA IPC peer mappings and a device barrier on peer flags.
 * Used by the distributed modes for the C6 corner turn (fused peer-store turn
 * cgh_slab_turn + cgh_multi_device_barrier, or cgh_multi_all_to_all), the
 * all-reduce of error sums and the all-gather of OSPR |R|^2 totals.
 * Replaces the torch.distributed data plane of the round-1 drivers; torch
 * only bootstraps (broadcast of the 128-byte id, exchange of IPC handles). */
typedef struct cgh_multi cgh_multi;
int cgh_multi_available(void);                 /* 1 when NCCL could be resolved */
int cgh_multi_unique_id(uint8_t *out128);      /* rank 0: ncclGetUniqueId */
int cgh_multi_create(int32_t device, int32_t world, int32_t rank, const uint8_t *id128, void *stream,
                     cgh_multi **out);         /* ncclCommInitRank; stream NULL = own stream */
int cgh_multi_destroy(cgh_multi *m);
/* block g (bytes_per_peer) of send -> rank g, block g of recv <- rank g */
int cgh_multi_all_to_all(cgh_multi *m, const void *send, void *recv, int64_t bytes_per_peer, void *stream);
int cgh_multi_all_reduce_sum_f64(cgh_multi *m, double *buf, int64_t count, void *stream);
int cgh_multi_all_gather(cgh_multi *m, const void *send, void *recv, int64_t bytes, void *stream);
int cgh_multi_ipc_handle(cgh_multi *m, void *ptr, uint8_t *out64);
int cgh_multi_ipc_open(cgh_multi *m, const uint8_t *handle64, void **out);
int cgh_multi_flags(cgh_multi *m, void **out);
int cgh_multi_set_peer_flags(cgh_multi *m, void *const *flags);
int cgh_multi_device_barrier(cgh_multi *m, void *stream);
/* cudaMalloc / cudaFree on a device (IPC-exportable allocation bases) */
int cgh_device_alloc(int32_t device, int64_t bytes, void **out);
int cgh_device_free(int32_t device, void *ptr);

/* ---- .hgi payload (cghkit/serialio.py:167-185 save_field): the complex128
 * payload states[idx] of an index plane, expanded on the device and copied to
 * out_payload (count x 16 bytes, may be NULL), and zlib's CRC-32 of those
 * payload bytes computed on the device from the index plane. */
int cgh_hgi_payload(int32_t device, const void *idx, int32_t idx_bytes, int64_t count, const double *states,
                    int32_t n_states, double *out_payload, uint32_t *out_crc);
/* zlib crc32_combine (host, no GPU): CRC-32 of A||B from crc(A), crc(B), len(B). */
int cgh_crc32_combine(uint32_t crc1, uint32_t crc2, int64_t len2, uint32_t *out);

/* ---- propagation.py:205-218 delta_replay_update on the device: in-place
 * rank-1 update of an uncentred replay (h x w complex128, host memory) for a
 * change `delta` of hologram pixel (m, n). */
int cgh_delta_replay_update(int32_t device, double *replay, int32_t h, int32_t w, int32_t m, int32_t n,
                            double delta_re, double delta_im);

/* ---- host: materialise states[indices] as complex128 (the returned
 * hologram of every runner) with `threads` host threads (no GPU needed). */
int cgh_expand_states(const void *idx, int32_t idx_bytes, int64_t count, const double *states, int32_t n_states,
                      double *out, int32_t threads);
/* ---- host: touch one byte per 4 KB page of [p, p + bytes) (writes zeros)
 * with `threads` host threads, so a fresh output array is faulted in while the
 * device runs instead of during cgh_expand_states. No reference counterpart. */
int cgh_prefault(void *p, int64_t bytes, int32_t threads);

/* ---- host-side numpy-stream emulation (no GPU needed) -----------------
 * Generator.permutation(n) of a PCG64 stream (algorithms.py:437-439). */
int cgh_permutation(const cgh_pcg64 *rng, int64_t n, int64_t *out);
/* n doubles of Generator.random after skipping `skip` draws, on the device
 * when device >= 0 (parity tests of the device emulation), else on the host. */
int cgh_random_doubles(int32_t device, const cgh_pcg64 *rng, int64_t skip, int64_t n, double *out);

#ifdef __cplusplus
}
#endif
#endif /* CGHB200_H */
