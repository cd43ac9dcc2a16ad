// rs_f32.cu — reduce-scatter transport kernels for F32, all four ops (see kernels.cu).
#include "transport.cuh"

namespace pat {
using KernelFn = void (*)(const KPlan);
#define PAT_RS_ROW(DT, NAME) \
  extern const KernelFn NAME[4] = {pat_kernel<DT, kSum, kRS>, pat_kernel<DT, kProd, kRS>, pat_kernel<DT, kMax, kRS>, \
                                  pat_kernel<DT, kMin, kRS>};
PAT_RS_ROW(kF32, kRsRowF32)
using GroupFn = void (*)(const KPlan2);
extern const GroupFn kGroupF32 = pat_group_kernel<kF32>;
}  // namespace pat
