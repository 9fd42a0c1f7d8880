// Kernel tables: one KernelSet per (precision, log2 length), gathered from
// the per-size instantiation objects (pm_inst.cu).
#include "pm_table.h"

namespace pm {

#define PM_DECL(tag, lg) KernelSet make_set_##tag##lg();
#define PM_DECL_ALL(tag)                                                                       \
    PM_DECL(tag, _0) PM_DECL(tag, _1) PM_DECL(tag, _2) PM_DECL(tag, _3) PM_DECL(tag, _4)       \
    PM_DECL(tag, _5) PM_DECL(tag, _6) PM_DECL(tag, _7) PM_DECL(tag, _8) PM_DECL(tag, _9)       \
    PM_DECL(tag, _10) PM_DECL(tag, _11) PM_DECL(tag, _12)
PM_DECL_ALL(f32)
PM_DECL_ALL(f64)

#define PM_LIST(tag)                                                                           \
    {make_set_##tag##_0(), make_set_##tag##_1(), make_set_##tag##_2(), make_set_##tag##_3(),   \
     make_set_##tag##_4(), make_set_##tag##_5(), make_set_##tag##_6(), make_set_##tag##_7(),   \
     make_set_##tag##_8(), make_set_##tag##_9(), make_set_##tag##_10(), make_set_##tag##_11(), \
     make_set_##tag##_12()}

const KernelSet& kernels_f32(int lg) {
    static const KernelSet t[kMaxLg + 1] = PM_LIST(f32);
    return t[lg];
}
const KernelSet& kernels_f64(int lg) {
    static const KernelSet t[kMaxLg + 1] = PM_LIST(f64);
    return t[lg];
}

}  // namespace pm
