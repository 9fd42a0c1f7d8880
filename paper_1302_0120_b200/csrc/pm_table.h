// Host-side description of the instantiated sweep kernels, one entry per
// (precision, log2 length). Filled by pm_inst_f32.cu / pm_inst_f64.cu.
#pragma once

namespace pm {

struct AxisShape {
    int lgR;                // log2 points per thread
    int TG;                 // threads per transform
    int NP;                 // Stockham passes
    int SM;                 // shared-memory elements per transform (0 if NP <= 1)
    int TW;                 // twiddle-table entries
};

// Row kernels (contiguous axis, length n_x) and column kernels (strided
// axis, length n_y) may use different points-per-thread.
struct KernelSet {
    const void* row_iter;   // row_iter_kernel<T, lg, lgR_row>
    const void* row_final;  // row_final_kernel<T, lg, lgR_row>
    const void* row_fft;    // row_fft_kernel<T, lg, lgR_row>
    const void* col_iter;   // col_iter_kernel<T, lg, lgR_col>
    const void* col_fft;    // col_fft_kernel<T, lg, lgR_col>
    const void* solve;      // solve_kernel<T, lg, lgR_row, lgR_col, GS> (square grids, lg >= 7) or null
    const void* solve_raar; // the same for RAAR
    int solve_smem;         // its dynamic shared memory (bytes)
    int solve_smem_raar;    // the RAAR kernel's (x staged as well)
    // variants whose column phase streams tiles through TMA (used when a CTA
    // has several column tasks per phase: batches), or null
    const void* solve_tma;
    const void* solve_raar_tma;
    int solve_smem_tma;
    int solve_smem_raar_tma;
    int solve_tma_m;        // the TMA variant streams m too (else it stages m by cp.async)
    int solve_threads;      // its CTA size
    AxisShape row, col;
};

constexpr int kMaxLg = 12;  // n_x, n_y up to 4096


const KernelSet& kernels_f32(int lg);
const KernelSet& kernels_f64(int lg);

}  // namespace pm
