// rs_i8.cu — reduce-scatter transport kernels for I8 U8, all four ops (see kernels.cu).
#include "transport.cuh"

namespace pat {
using KernelFn = void (*)(const KPlan);
#define PAT_RS_ROW(DT, NAME) \
  extern const KernelFn NAME[4] = {pat_kernel<DT, kSum, kRS>, pat_kernel<DT, kProd, kRS>, pat_kernel<DT, kMax, kRS>, \
                                  pat_kernel<DT, kMin, kRS>};
PAT_RS_ROW(kI8, kRsRowI8)
PAT_RS_ROW(kU8, kRsRowU8)
using GroupFn = void (*)(const KPlan2);
extern const GroupFn kGroupI8 = pat_group_kernel<kI8>;
extern const GroupFn kGroupU8 = pat_group_kernel<kU8>;
}  // namespace pat
