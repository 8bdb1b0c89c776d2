// Mode dispatch for one line length N (instantiated per size group in inst_*.cu).
#pragma once
#include "dispatch.cuh"

namespace cgh {

template <class T, int N>
cudaError_t row_dispatch(int mode, const PassArgs<T>& a, int frames, cudaStream_t st) {
    switch (mode) {
        case ROW_FWD: return launch_row_n<T, N, ROW_FWD>(a, frames, st);
        case ROW_INV: return launch_row_n<T, N, ROW_INV>(a, frames, st);
        case ROW_HOLO: return launch_row_n<T, N, ROW_HOLO>(a, frames, st);
        case ROW_INIT: return launch_row_n<T, N, ROW_INIT>(a, frames, st);
        case ROW_OSPR_GEN: return launch_row_n<T, N, ROW_OSPR_GEN>(a, frames, st);
        case ROW_OSPR_ACC: return launch_row_n<T, N, ROW_OSPR_ACC>(a, frames, st);
        default: return cudaErrorInvalidValue;
    }
}

template <class T, int N>
cudaError_t col_dispatch(int mode, const PassArgs<T>& a, int frames, cudaStream_t st) {
    switch (mode) {
        case COL_FWD: return launch_col_n<T, N, COL_FWD>(a, frames, st);
        case COL_INV: return launch_col_n<T, N, COL_INV>(a, frames, st);
        case COL_GS: return launch_col_n<T, N, COL_GS>(a, frames, st);
        case COL_FINAL: return launch_col_n<T, N, COL_FINAL>(a, frames, st);
        case COL_HOLO: return launch_col_n<T, N, COL_HOLO>(a, frames, st);
        default: return cudaErrorInvalidValue;
    }
}

#define CGH_INSTANTIATE(T, N)                                                                        \
    template cudaError_t row_dispatch<T, N>(int, const PassArgs<T>&, int, cudaStream_t);            \
    template cudaError_t col_dispatch<T, N>(int, const PassArgs<T>&, int, cudaStream_t);

}  // namespace cgh
