// Instantiates the sweep kernels for ONE (precision, log2 length). Compiled
// once per pair with -DPM_F64=0|1 -DPM_LG=<0..12> (see build.py) so the
// 26 instantiations build in parallel.
#include "pm_kernels.cuh"
#include "pm_table.h"

#if PM_F64
#define PM_T double
#define PM_LGR 4
#define PM_TAG f64
#else
#define PM_T float
#define PM_LGR 5
#define PM_TAG f32
#endif
#define PM_CAT3_(a, b, c) a##b##_##c
#define PM_CAT3(a, b, c) PM_CAT3_(a, b, c)

namespace pm {
KernelSet PM_CAT3(make_set_, PM_TAG, PM_LG)() {
    using F = FftShape<PM_LG, PM_LGR>;
    KernelSet s;
    s.row_iter = (const void*)&row_iter_kernel<PM_T, PM_LG, PM_LGR>;
    s.col_iter = (const void*)&col_iter_kernel<PM_T, PM_LG, PM_LGR>;
    s.row_fft = (const void*)&row_fft_kernel<PM_T, PM_LG, PM_LGR>;
    s.col_fft = (const void*)&col_fft_kernel<PM_T, PM_LG, PM_LGR>;
    s.lgR = F::lgR;
    s.TG = F::TG;
    s.NP = F::NP;
    s.SM = F::SM;
    s.TW = F::TW;
    return s;
}
}  // namespace pm
