// Per-device launch setup shared by the persistent-kernel launchers.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

namespace cgh {

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device property of a
// kernel: set it once per (kernel, device) and report its status. Safe when
// several host threads drive different devices (multi.run_batch). SMEM must be
// the kernel's fixed dynamic shared-memory size.
template <auto Kernel>
cudaError_t ensure_smem_attr(size_t smem) {
    static std::atomic<uint64_t> done{0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = uint64_t(1) << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

// Resident CTAs of a kernel on the current device (cached per device).
template <auto Kernel>
int resident_ctas(int threads, size_t smem) {
    static std::atomic<int> cached[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 1;
    int v = cached[dev & 63].load(std::memory_order_relaxed);
    if (v > 0) return v;
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, Kernel, threads, smem);
    v = (sms > 0 ? sms : 1) * (per > 0 ? per : 1);
    cached[dev & 63].store(v, std::memory_order_relaxed);
    return v;
}

}  // namespace cgh
