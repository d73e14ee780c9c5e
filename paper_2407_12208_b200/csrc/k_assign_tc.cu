// k_assign_tc.cu — K4 tcgen05 distance + argmin (placeholder until the kernel lands).
#include <string>

#include "common.cuh"
#include "internal.h"

namespace mpk {
struct TcPlan { int dummy; };
bool tc_supported(int, int, int) { return false; }
int tc_dpad(int, int d) { return d; }
TcPlan* tc_plan_create(int, int64_t, int, int, int, const void*, const void*, std::string* err) {
    if (err) *err = "tcgen05 kernel not built";
    return nullptr;
}
void tc_plan_destroy(TcPlan* p) { delete p; }
cudaError_t launch_assign_tc(TcPlan*, const Problem&, const float*, const float*, const float*,
                             const float*, int32_t*, double*, double*, cudaStream_t) {
    return cudaErrorNotSupported;
}
}  // namespace mpk
