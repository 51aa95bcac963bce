// explicit instantiation: conv kernel variants for (DT_F16, EPI_NONE)
#include "conv_tc_kernel.cuh"

namespace abed_host {
template cudaError_t launch_epi<abed_dev::DT_F16, abed_dev::EPI_NONE, 0>(const ConvTcParams&, int, bool, cudaStream_t);
}  // namespace abed_host
