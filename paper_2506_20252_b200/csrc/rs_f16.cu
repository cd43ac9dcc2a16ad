// rs_f16.cu — reduce-scatter transport kernels for F16 BF16, all four ops (see kernels.cu).
#include "transport.cuh"

namespace pat {
using KernelFn = void (*)(const KPlan);
#define PAT_RS_ROW(DT, NAME) \
  extern const KernelFn NAME[4] = {pat_kernel<DT, kSum, kRS>, pat_kernel<DT, kProd, kRS>, pat_kernel<DT, kMax, kRS>, \
                                  pat_kernel<DT, kMin, kRS>};
PAT_RS_ROW(kF16, kRsRowF16)
PAT_RS_ROW(kBF16, kRsRowBF16)
using GroupFn = void (*)(const KPlan2);
extern const GroupFn kGroupF16 = pat_group_kernel<kF16>;
extern const GroupFn kGroupBF16 = pat_group_kernel<kBF16>;
}  // namespace pat
