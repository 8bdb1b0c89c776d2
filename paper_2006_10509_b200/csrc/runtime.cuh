// Host runtime shared by the C-ABI translation units: plans, buffers, errors.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <shared_mutex>
#include <string>
#include <vector>

#include "../../include/cghb200.h"
#include "dispatch.cuh"

namespace cgh {

// ----------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);

// Kernels whose CTAs wait on each other (grid barriers: the SA/DBS search
// kernels, the warp-line loops) need every CTA resident. Launched onto one
// device while another host thread's work is on it (run_batch workers
// sharing a GPU), such a grid can be left partly resident behind CTAs that
// themselves wait — another grid-barrier kernel, or kernels launched early
// with programmatic dependent launch waiting for their predecessor — and
// both sides wait forever (seen in the 3-thread run_batch test). Runs take
// this per-device gate for their whole duration (every run synchronizes
// before it returns): shared by runs that only launch ordinary kernels,
// exclusive for runs that may launch a grid-barrier kernel.
std::shared_mutex& device_gate(int dev);
struct GateLock {
    std::shared_mutex& m;
    bool ex;
    GateLock(int dev, bool exclusive) : m(device_gate(dev)), ex(exclusive) {
        if (ex) m.lock();
        else m.lock_shared();
    }
    ~GateLock() {
        if (ex) m.unlock();
        else m.unlock_shared();
    }
    GateLock(const GateLock&) = delete;
    GateLock& operator=(const GateLock&) = delete;
};

#define CGH_CUDA(call)                                                                      \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return ::cgh::fail(e_ == cudaErrorMemoryAllocation ? CGH_ERR_MEMORY : CGH_ERR_CUDA, \
                               "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

#define CGH_TRY(call)            \
    do {                         \
        int s_ = (call);         \
        if (s_ != CGH_OK) return s_; \
    } while (0)

inline Pcg64 to_pcg(const cgh_pcg64& g) {
    Pcg64 r;
    r.state = (u128(g.state_hi) << 64) | u128(g.state_lo);
    r.inc = (u128(g.inc_hi) << 64) | u128(g.inc_lo);
    r.has_uint32 = g.has_uint32;
    r.uinteger = g.uinteger;
    return r;
}

inline bool is_pow2(int n) { return n >= 2 && (n & (n - 1)) == 0; }

// ------------------------------------------------------------------ plan
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
};

}  // namespace cgh

struct cgh_plan {
    int dev = 0, H = 0, W = 0, prec = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::vector<cudaEvent_t> evpool;
    // scheme / propagation / metric
    int scheme_kind = 0, nstates = 0;
    double offset = 0, step = 0;
    int prop_kind = 0;
    double wl = 0, dist = 0, px = 0, py = 0;
    int rescale = 0;
    // device buffers
    cgh::DevBuf states64, states32, tw_row, tw_col, q_row, q_col;
    cgh::DevBuf data, tgt, beam, idx, field, partials, counter, stats, stage, mask, frame_rng, intensity;
    cgh::DevBuf sa_buf;   // search state (SA/DBS)
    void* fast = nullptr; // FastState of the pipelined complex64 GS passes (fast.cu)
    void* wlst = nullptr; // WlState of the warp-line 2048^2 GS passes (wl.cu)
    int idx_bytes = 1;
    bool has_beam = false, target_ready = false;
    // mapped host results
    double* res_h = nullptr;
    // pinned staging for large host->device uploads (upload_staged)
    std::vector<void*> pin;
    std::vector<cudaStream_t> pin_st;
    std::vector<cudaEvent_t> pin_ev;
    // host-side amplitude preparation (cgh_plan_set_target_ex, fp32): pinned
    // plane, one stream per host thread
    void* pin_amp = nullptr;
    size_t pin_amp_cap = 0;
    std::vector<cudaStream_t> amp_st;
    std::vector<cudaEvent_t> amp_ev;
    bool stage_valid = false;   // the complex target is on the device (P->stage)
    double* res_d = nullptr;
    size_t res_cap = 0;
    // prep statistics
    double count_in = 0, denom = 0, nf_in = 0, nf_all = 0, nf_beam = 0;
    long launches = 0;
    // per-pass CUDA-event timing (cgh_plan_profile): (pass id, start, end)
    bool profiling = false;
    std::vector<int> prof_id;
    std::vector<cudaEvent_t> prof_ev;
    int idx_frames = 0;   // index planes currently held
};

namespace cgh {

// fp64 tables (long-double evaluation): exp(-2 pi i k / n); separable Fresnel chirp
void twiddle_table(int n, std::vector<double>& out);
// centred transform of any H x W (anysize.cu; Bluestein line DFTs)
int transform_any(const cgh_problem* pb, const double* in, double* out, int op);
// packed Bluestein tables of non-power-of-two plan axes (anysize.cu)
void blue_pack_table(int N, std::vector<double>& out);
int blue_finish_table(int prec, int N, void* dev_table, cudaStream_t st);
void chirp_table(int n, double pitch, double wl, double dist, std::vector<double>& out);

int plan_init(cgh_plan* P, const cgh_problem* pb);
void plan_free(cgh_plan* P);
int ensure(cgh_plan* P, DevBuf& b, size_t bytes);
int ensure_res(cgh_plan* P, size_t n);
int ensure_events(cgh_plan* P, size_t n);
int plan_upload_target(cgh_plan* P, const double* target, const uint8_t* mask, const double* illum);
// Host -> device copy of a large pageable buffer through pinned staging:
// host threads copy slices into double-buffered pinned chunks and issue the
// DMAs on their own streams; P->st waits for them. Small copies go direct.
int upload_staged(cgh_plan* P, void* dst, const void* src, size_t bytes);

template <class T>
PassArgs<T> base_args(cgh_plan* P);

// Pipelined complex64 GS passes (fast.cu): eligibility, per-plan setup, launches.
bool fast_eligible(cgh_plan* P);
int fast_prepare(cgh_plan* P);
int fast_row(cgh_plan* P, const PassArgs<float>& a);
int fast_col(cgh_plan* P, const PassArgs<float>& a);
void fast_free(cgh_plan* P);
void fast_invalidate_target(cgh_plan* P);
// Warp-line complex64 GS passes for 2048 x 2048 planes (wl.cu): the plane is
// kept column-tiled ("T4") in a buffer of their own between the relayouts.
bool wl_eligible(cgh_plan* P);
int wl_prepare(cgh_plan* P);
int wl_relayout(cgh_plan* P, int to_t4);
int wl_col(cgh_plan* P, const PassArgs<float>& a);
int wl_row(cgh_plan* P, const PassArgs<float>& a);
int wl_gs_loop(cgh_plan* P, const PassArgs<float>& a, int iters);
bool wl_ospr_eligible(cgh_plan* P);
int wl_ospr_run(cgh_plan* P, const PassArgs<float>& a, int S_frames);
void wl_free(cgh_plan* P);
void wl_invalidate_target(cgh_plan* P);
bool fast_ospr_eligible(cgh_plan* P);
int fast_ospr_holo(cgh_plan* P, const PassArgs<float>& a, int frames, int cap, uint8_t* idx_out);
int fast_ospr_gen(cgh_plan* P, const PassArgs<float>& a);
int fast_ospr_acc(cgh_plan* P, const PassArgs<float>& a);

// Record a timing event before (start) / after a pass launch. Pass ids:
// row modes 0..7, column modes 8 + mode, search kernels 16+.
int prof_mark(cgh_plan* P, int id, bool start);

template <class T>
inline int run_row(cgh_plan* P, int mode, const PassArgs<T>& a, int frames) {
    if (P->profiling) CGH_TRY(prof_mark(P, mode, true));
    cudaError_t e = launch_row<T>(mode, P->W, a, frames, P->st);
    if (P->profiling) CGH_TRY(prof_mark(P, mode, false));
    P->launches += 1;
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "row pass (mode %d, W=%d): %s", mode, P->W, cudaGetErrorString(e));
    return CGH_OK;
}
template <class T>
inline int run_col(cgh_plan* P, int mode, const PassArgs<T>& a, int frames) {
    if (P->profiling) CGH_TRY(prof_mark(P, 8 + mode, true));
    cudaError_t e = launch_col<T>(mode, P->H, a, frames, P->st);
    if (P->profiling) CGH_TRY(prof_mark(P, 8 + mode, false));
    P->launches += 1;
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "column pass (mode %d, H=%d): %s", mode, P->H, cudaGetErrorString(e));
    return CGH_OK;
}

inline bool cancelled(const cgh_callbacks* cb) { return cb && cb->cancel && cb->cancel(cb->user); }

inline int grid_for(long total) {
    long g = (total + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
    return int(g);
}

// In-order progress delivery with a bounded number of iterations in flight:
// after each enqueue, completed entries are reported; if more than `depth`
// are pending the oldest is waited for (the GPU keeps the rest queued).
struct ProgressQueue {
    cgh_plan* P = nullptr;
    const cgh_callbacks* cb = nullptr;
    size_t depth = 64;
    const double* values = nullptr;   // mapped host results
    long stride = 1;                  // values[k * stride] is entry k
    long kbias = 0;                   // progress(k + kbias, ...)
    std::vector<long> ks;
    std::vector<cudaEvent_t> evs;
    size_t head = 0, used = 0;
    int init(cgh_plan* P_, const cgh_callbacks* cb_, size_t depth_, const double* values_, long stride_);
    int push(long k);
    int poll(bool all);
};

}  // namespace cgh
