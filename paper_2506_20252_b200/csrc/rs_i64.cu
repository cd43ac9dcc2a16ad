// rs_i64.cu — reduce-scatter transport kernels for I64 U64, all four ops (see kernels.cu).
#include "transport.cuh"

namespace pat {
using KernelFn = void (*)(const KPlan);
#define PAT_RS_ROW(DT, NAME) \
  extern const KernelFn NAME[4] = {pat_kernel<DT, kSum, kRS>, pat_kernel<DT, kProd, kRS>, pat_kernel<DT, kMax, kRS>, \
                                  pat_kernel<DT, kMin, kRS>};
PAT_RS_ROW(kI64, kRsRowI64)
PAT_RS_ROW(kU64, kRsRowU64)
using GroupFn = void (*)(const KPlan2);
extern const GroupFn kGroupI64 = pat_group_kernel<kI64>;
extern const GroupFn kGroupU64 = pat_group_kernel<kU64>;
}  // namespace pat
