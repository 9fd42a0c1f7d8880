// Host-side description of the instantiated sweep kernels, one entry per
// (precision, log2 length). Filled by pm_inst_f32.cu / pm_inst_f64.cu.
#pragma once

namespace pm {

struct KernelSet {
    const void* row_iter;   // row_iter_kernel<T, lg, lgR>
    const void* col_iter;   // col_iter_kernel<T, lg, lgR>
    const void* row_fft;    // row_fft_kernel<T, lg, lgR>
    const void* col_fft;    // col_fft_kernel<T, lg, lgR>
    int lgR;                // log2 points per thread
    int TG;                 // threads per transform
    int NP;                 // Stockham passes
    int SM;                 // shared-memory elements per transform (0 if NP <= 1)
    int TW;                 // twiddle-table entries
};

constexpr int kMaxLg = 12;  // n_x, n_y up to 4096

const KernelSet& kernels_f32(int lg);
const KernelSet& kernels_f64(int lg);

}  // namespace pm
