// FFT code-efficiency microbenchmark: K forward+inverse 2048-point line FFT
// pairs per block in registers (+ shared exchanges unless NOEX), no global I/O.
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2006_10509_b200/csrc/fast_passes.cuh"
using namespace cgh;
constexpr int N = 2048, TH = 256;
template <bool NOEX>
__global__ void __launch_bounds__(TH, 2) kfft(const cx<float>* tw_tab, float2* out, int K) {
    using S = FastShape<N, TH>;
    extern __shared__ __align__(128) float2 fsm[];
    const int tid = threadIdx.x, g = tid / S::TF, t = tid - g * S::TF;
    float2* line = fsm + g * ((S::LW + 15) / 16 * 16);
    FastTw<N, TH> tw;
    fast_tw_init<N, TH>(tw, t, tw_tab);
    cx<float> v[16];
    for (int r = 0; r < 16; ++r) v[r] = mk(float(t + r), float(r - t));
    const int bid = NOEX ? -1 : 1 + g;
    for (int k = 0; k < K; ++k) {
        fast_fft<N, TH, +1>(v, line, t, padc(t), tw, bid, S::TF);
        for (int r = 0; r < 16; ++r) { float m2 = v[r].x * v[r].x + v[r].y * v[r].y; float s = rsqrtf(m2 + 1e-30f); v[r] = mk(v[r].x * s, v[r].y * s); }
        fast_fft<N, TH, -1>(v, line, t, padc(t), tw, bid, S::TF);
    }
    float acc = 0; for (int r = 0; r < 16; ++r) acc += v[r].x + v[r].y;
    out[blockIdx.x * TH + tid] = make_float2(acc, 0);
}
int main() {
    cx<float>* tab; cudaMalloc(&tab, N * 8);
    float2 h[N]; for (int k = 0; k < N; ++k) { double a = -2 * 3.14159265358979 * k / N; h[k] = make_float2(cos(a), sin(a)); }
    cudaMemcpy(tab, h, N * 8, cudaMemcpyHostToDevice);
    float2* out; cudaMalloc(&out, 148 * 2 * TH * 8 * 4);
    using S = FastShape<N, TH>;
    size_t smem = size_t(S::LINES) * ((S::LW + 15) / 16 * 16) * 8;
    cudaFuncSetAttribute(kfft<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(kfft<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int blocks = 148 * 2;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int K : {64, 7})
    for (int noex = 0; noex < 2; ++noex) {
        auto k = noex ? kfft<true> : kfft<false>;
        k<<<blocks, TH, smem>>>(tab, out, 2);
        cudaEventRecord(e0); k<<<blocks, TH, smem>>>(tab, out, K); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double elems = double(blocks) * S::LINES * N * K;   // element-passes (fwd+inv pair)
        printf("K=%d %s: %.3f ms, %.2f ps per element-pair, equivalent 2048^2 pass %.1f us\n", K, noex ? "no-exchange" : "exchange", ms,
               ms * 1e9 / elems, ms * 1e3 / elems * 4194304.0);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
