// explicit instantiation: conv kernel variants for (DT_BF16, EPI_COMPARE)
#include "conv_tc_kernel.cuh"

namespace abed_host {
template cudaError_t launch_epi<abed_dev::DT_BF16, abed_dev::EPI_COMPARE, 0>(const ConvTcParams&, int, bool, cudaStream_t);
}  // namespace abed_host
