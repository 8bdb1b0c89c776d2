// Micro-benchmark: how fast can persistent CTAs stream a 2048 x 2048 complex64
// field (32 MB, L2-resident) through shared memory in 64 KB tiles?
//   colC : column tiles of C columns via 2-D TMA boxes (row segment = 8C bytes)
//   bulk : contiguous 64 KB 1-D bulk copies (row tiles)
//   blk4 : 4x4-blocked layout, 2-D TMA boxes of 128-B rows
//   ldgsts: column tiles of 4 columns gathered by cp.async (16 B per thread)
// Two slots per CTA, one CTA per SM, static tile order, no compute.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_tiles tma_tiles.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#include "../../paper_2006_10509_b200/csrc/tma.cuh"

using namespace cgh;
constexpr int N = 2048;
constexpr int TILE = 64 * 1024;

template <int MODE, int C>
__global__ void __launch_bounds__(512, 1) stream(const __grid_constant__ CUtensorMap tm, const float2* base,
                                                 int ntiles, float* sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t full[2];
    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    constexpr int ROWS = TILE / (8 * C);   // rows per column tile
    auto issue = [&](int s, int tile) {
        unsigned char* dst = sm + s * TILE;
        if constexpr (MODE == 0) {   // column tile: C cols x ROWS rows, boxes of 256 rows
            const int tiles_x = N / C;
            const int tx = tile % tiles_x, ty = tile / tiles_x;
            mbar_expect_tx(&full[s], TILE);
            for (int y = 0; y < ROWS; y += 256)
                tma_g2s_2d(dst + y * C * 8, &tm, 2 * C * tx, ty * ROWS + y, &full[s]);
        } else if constexpr (MODE == 1) {
            mbar_expect_tx(&full[s], TILE);
            bulk_g2s(dst, reinterpret_cast<const char*>(base) + size_t(tile) * TILE, TILE, &full[s]);
        } else if constexpr (MODE == 2) {   // blocked: 512 blocks of 128 B per tile, boxes of 256 blocks
            mbar_expect_tx(&full[s], TILE);
            tma_g2s_2d(dst, &tm, 0, tile * 512, &full[s]);
            tma_g2s_2d(dst + 32768, &tm, 0, tile * 512 + 256, &full[s]);
        }
    };
    float acc = 0.f;
    if constexpr (MODE == 3) {
        // cp.async gathers: tile = 4 columns x 2048 rows; thread copies 16 B
        // (2 columns of one row) per op: 4096 ops / 512 threads = 8 per tile
        auto gather = [&](int s, int tile) {
            unsigned char* dst = sm + s * TILE;
            for (int i = tid; i < 2 * N; i += 512) {
                const int row = i >> 1, half = i & 1;
                const float2* src = base + size_t(row) * N + tile * 4 + half * 2;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + (row * 4 + half * 2) * 8)),
                             "l"(src)
                             : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        if (blockIdx.x < ntiles) gather(0, blockIdx.x);
        int it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int s = it & 1;
            if (tile + gridDim.x < ntiles) {
                gather(s ^ 1, tile + gridDim.x);
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            } else {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            __syncthreads();
            acc += reinterpret_cast<float*>(sm + s * TILE)[tid];
            __syncthreads();
        }
        if (acc == 12345.f) sink[0] = acc;
        return;
    }
    if (tid == 0) {
        if (blockIdx.x < ntiles) issue(0, blockIdx.x);
        if (blockIdx.x + gridDim.x < ntiles) issue(1, blockIdx.x + gridDim.x);
    }
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int s = it & 1;
        mbar_wait(&full[s], (it >> 1) & 1);
        acc += reinterpret_cast<float*>(sm + s * TILE)[tid];
        __syncthreads();
        if (tid == 0 && tile + 2 * gridDim.x < ntiles) issue(s, tile + 2 * gridDim.x);
    }
    if (acc == 12345.f) sink[0] = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

template <int MODE, int C>
static void run(const char* name, CUtensorMap tm, const float2* base, int ntiles, float* sink) {
    auto k = stream<MODE, C>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * TILE);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) k<<<sms, 512, 2 * TILE>>>(tm, base, ntiles, sink);
    const int reps = 20;
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) k<<<sms, 512, 2 * TILE>>>(tm, base, ntiles, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1e3 / reps;
    printf("%-10s %8.2f us per 32 MB pass  %7.1f GB/s  (%s)\n", name, us, 32.0 * 1048576 / (us * 1e3),
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    float2* d;
    float* sink;
    cudaMalloc(&d, size_t(N) * N * 8);
    cudaMalloc(&sink, 64);
    cudaMemset(d, 0, size_t(N) * N * 8);
    auto e = enc();
    const int ntiles = N * N * 8 / TILE;   // 512
    auto colmap = [&](int C) {
        CUtensorMap m;
        cuuint64_t dims[2] = {cuuint64_t(2 * N), cuuint64_t(N)};
        cuuint64_t strides[1] = {cuuint64_t(N) * 8};
        cuuint32_t box[2] = {cuuint32_t(2 * C), 256u};
        cuuint32_t es[2] = {1, 1};
        CUresult r = e(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r) printf("encode C=%d failed %d\n", C, int(r));
        return m;
    };
    CUtensorMap m4 = colmap(4), m8 = colmap(8), m16 = colmap(16);
    CUtensorMap mb;
    {
        cuuint64_t dims[2] = {32, cuuint64_t(N) * N / 16};
        cuuint64_t strides[1] = {128};
        cuuint32_t box[2] = {32u, 256u};
        cuuint32_t es[2] = {1, 1};
        CUresult r = e(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r) printf("encode blk failed %d\n", int(r));
    }
    for (int rep = 0; rep < 2; ++rep) {
        run<0, 4>("col4", m4, d, ntiles, sink);
        run<0, 8>("col8", m8, d, ntiles, sink);
        run<0, 16>("col16", m16, d, ntiles, sink);
        run<1, 4>("bulk", m4, d, ntiles, sink);
        run<2, 4>("blk4x4", mb, d, ntiles, sink);
        run<3, 4>("ldgsts4", m4, d, ntiles, sink);
    }
    return 0;
}
