// tcgen05 wide pass (placeholder until the tensor-core kernel lands).
#include <stdexcept>

#include "kernels.hpp"

namespace ltfb_dev {

bool wide_tc_supported(const StepArgs&) { return false; }
void launch_wide_tc(const StepArgs&, cudaStream_t) { throw std::runtime_error("tcgen05 wide kernel unavailable"); }

}  // namespace ltfb_dev
