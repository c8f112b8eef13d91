// GEMM template (KB5): placeholder until the tcgen05 kernel lands.
#include "../../include/korch.h"
#include "codegen.h"

namespace korch {

KernelPlan generate_gemm(const Graph& g, const Candidate& c) {
  (void)g;
  (void)c;
  KernelPlan kp;
  kp.klass = KORCH_CLASS_REJECTED;
  kp.reject = "GEMM template not available";
  return kp;
}

}  // namespace korch
