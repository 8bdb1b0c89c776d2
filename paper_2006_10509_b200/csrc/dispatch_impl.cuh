// Line-length switch for one precision (pass_fp32.cu / pass_fp64.cu); the
// kernels themselves are instantiated in inst_*.cu so they compile in parallel.
#pragma once
#include "dispatch.cuh"

namespace cgh {

#define CGH_ALL_SIZES(X) X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096)
#define CGH_ROW_CASE(N) case N: return row_dispatch<CGH_T, N>(mode, a, frames, st);
#define CGH_COL_CASE(N) case N: return col_dispatch<CGH_T, N>(mode, a, frames, st);
#define CGH_RB_CASE(N) case N: return row_blocks<CGH_T, N>(H);
#define CGH_CB_CASE(N) case N: return col_blocks<CGH_T, N>(W);

template <>
cudaError_t launch_row<CGH_T>(int mode, int N, const PassArgs<CGH_T>& a, int frames, cudaStream_t st) {
    switch (N) {
        CGH_ALL_SIZES(CGH_ROW_CASE)
        default: return launch_row_any<CGH_T>(mode, N, a, frames, st);
    }
}

template <>
cudaError_t launch_col<CGH_T>(int mode, int N, const PassArgs<CGH_T>& a, int frames, cudaStream_t st) {
    switch (N) {
        CGH_ALL_SIZES(CGH_COL_CASE)
        default: return launch_col_any<CGH_T>(mode, N, a, frames, st);
    }
}

template <>
int row_grid_blocks<CGH_T>(int N, int H) {
    switch (N) {
        CGH_ALL_SIZES(CGH_RB_CASE)
        default: return H;   // Bluestein rows: one CTA per line
    }
}
template <>
int col_grid_blocks<CGH_T>(int N, int W) {
    switch (N) {
        CGH_ALL_SIZES(CGH_CB_CASE)
        default: return W;   // Bluestein columns: one CTA per line
    }
}

}  // namespace cgh
