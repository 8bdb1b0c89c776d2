// FP32 issue-rate microbenchmark (FADD / FFMA reg-reg / FFMA-imm / FMUL), 8 chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(float* out, float a, float b, int iters) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    float y0 = a, y1 = a + 1, y2 = a + 2, y3 = a + 3, y4 = b, y5 = b + 1, y6 = b + 2, y7 = b + 3;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (OP == 0) { x0 = x0 + y0; x1 = x1 + y1; x2 = x2 + y2; x3 = x3 + y3; x4 = x4 + y4; x5 = x5 + y5; x6 = x6 + y6; x7 = x7 + y7; }
            if (OP == 1) { x0 = fmaf(x0, y0, y4); x1 = fmaf(x1, y1, y5); x2 = fmaf(x2, y2, y6); x3 = fmaf(x3, y3, y7); x4 = fmaf(x4, y4, y0); x5 = fmaf(x5, y5, y1); x6 = fmaf(x6, y6, y2); x7 = fmaf(x7, y7, y3); }
            if (OP == 2) { x0 = fmaf(x0, 1.0001f, y0); x1 = fmaf(x1, 1.0001f, y1); x2 = fmaf(x2, 1.0001f, y2); x3 = fmaf(x3, 1.0001f, y3); x4 = fmaf(x4, 1.0001f, y4); x5 = fmaf(x5, 1.0001f, y5); x6 = fmaf(x6, 1.0001f, y6); x7 = fmaf(x7, 1.0001f, y7); }
            if (OP == 3) { x0 = x0 * y0; x1 = x1 * y1; x2 = x2 * y2; x3 = x3 * y3; x4 = x4 * y4; x5 = x5 * y5; x6 = x6 * y6; x7 = x7 * y7; }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
template <int OP>
void run(const char* name, float* d) {
    int iters = 4096, blocks = 148 * 4, threads = 512;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<OP><<<blocks, threads>>>(d, 1.0f, 2.0f, 16);
    cudaEventRecord(e0);
    k<OP><<<blocks, threads>>>(d, 1.0f, 2.0f, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = double(blocks) * threads * iters * 64;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%s: %.2f Tops/s = %.1f thread-ops/clk/SM at %d MHz (%.3f ms)\n", name, ops / ms / 1e9, ops / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000, ms);
}
int main() {
    float* d; cudaMalloc(&d, 148 * 4 * 512 * 4);
    run<0>("FADD", d); run<1>("FFMA rrr", d); run<2>("FFMA imm", d); run<3>("FMUL", d);
    return 0;
}
