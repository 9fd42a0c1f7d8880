// Instantiates the sweep kernels for ONE (precision, log2 length). Compiled
// once per pair with -DPM_F64=0|1 -DPM_LG=<0..12> (see build.py) so the
// 26 instantiations build in parallel.
#include "pm_kernels.cuh"
#include "pm_table.h"

#if PM_F64
#define PM_T double
#define PM_TAG f64
#ifndef PM_LGR_ROW
#define PM_LGR_ROW 4
#endif
#ifndef PM_LGR_COL
#define PM_LGR_COL 3
#endif
#else
#define PM_T float
#define PM_TAG f32
#ifndef PM_LGR_ROW
#define PM_LGR_ROW 4
#endif
#ifndef PM_LGR_COL
#define PM_LGR_COL 4
#endif
#endif
#define PM_CAT3_(a, b, c) a##b##_##c
#define PM_CAT3(a, b, c) PM_CAT3_(a, b, c)

namespace pm {
KernelSet PM_CAT3(make_set_, PM_TAG, PM_LG)() {
    using FR = FftShape<PM_LG, PM_LGR_ROW>;
    using FC = FftShape<PM_LG, PM_LGR_COL>;
    KernelSet s;
    s.row_iter = (const void*)&row_iter_kernel<PM_T, PM_LG, PM_LGR_ROW>;
    s.row_final = (const void*)&row_final_kernel<PM_T, PM_LG, PM_LGR_ROW>;
    s.row_fft = (const void*)&row_fft_kernel<PM_T, PM_LG, PM_LGR_ROW>;
    s.col_iter = (const void*)&col_iter_kernel<PM_T, PM_LG, PM_LGR_COL>;
    s.col_fft = (const void*)&col_fft_kernel<PM_T, PM_LG, PM_LGR_COL>;
    s.solve = nullptr;
    s.solve_raar = nullptr;
    s.solve_tma = nullptr;
    s.solve_raar_tma = nullptr;
    s.solve_smem_tma = 0;
    s.solve_smem_raar_tma = 0;
    s.solve_tma_m = 0;
    s.solve_smem = 0;
    s.solve_smem_raar = 0;
    s.solve_threads = 0;
    // persistent kernel: square grids n >= 128 whose transforms fit one CTA
    if constexpr (PM_LG >= 7 && FR::TG <= kSolveThreads && FC::TG <= kSolveThreads) {
        s.solve = (const void*)&solve_kernel<PM_T, PM_LG, PM_LGR_ROW, PM_LGR_COL, 0>;
        s.solve_raar = (const void*)&solve_kernel<PM_T, PM_LG, PM_LGR_ROW, PM_LGR_COL, 1>;
        using LT = SolveSmem<PM_T, PM_LG, PM_LGR_ROW, PM_LGR_COL, true>;
        if constexpr (LT::TMA) {
            s.solve_tma = (const void*)&solve_kernel<PM_T, PM_LG, PM_LGR_ROW, PM_LGR_COL, 0, true>;
            s.solve_raar_tma = (const void*)&solve_kernel<PM_T, PM_LG, PM_LGR_ROW, PM_LGR_COL, 1, true>;
            s.solve_smem_tma = LT::BYTES_ALL + 128;
            s.solve_smem_raar_tma = LT::BYTES_ALL_RAAR + 128;
            s.solve_tma_m = LT::TMA_M ? 1 : 0;
        }
        s.solve_smem = SolveSmem<PM_T, PM_LG, PM_LGR_ROW, PM_LGR_COL>::BYTES_ALL + 128;
        s.solve_smem_raar = SolveSmem<PM_T, PM_LG, PM_LGR_ROW, PM_LGR_COL>::BYTES_ALL_RAAR + 128;
        s.solve_threads = kSolveThreads;
    }
    s.row = AxisShape{FR::lgR, FR::TG, FR::NP, FR::SM, FR::TW};
    s.col = AxisShape{FC::lgR, FC::TG, FC::NP, FC::SM, FC::TW};
    return s;
}
}  // namespace pm
