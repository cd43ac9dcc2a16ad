// rs_i32.cu — reduce-scatter transport kernels for I32 U32, all four ops (see kernels.cu).
#include "transport.cuh"

namespace pat {
using KernelFn = void (*)(const KPlan);
#define PAT_RS_ROW(DT, NAME) \
  extern const KernelFn NAME[4] = {pat_kernel<DT, kSum, kRS>, pat_kernel<DT, kProd, kRS>, pat_kernel<DT, kMax, kRS>, \
                                  pat_kernel<DT, kMin, kRS>};
PAT_RS_ROW(kI32, kRsRowI32)
PAT_RS_ROW(kU32, kRsRowU32)
using GroupFn = void (*)(const KPlan2);
extern const GroupFn kGroupI32 = pat_group_kernel<kI32>;
extern const GroupFn kGroupU32 = pat_group_kernel<kU32>;
}  // namespace pat
