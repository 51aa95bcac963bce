// explicit instantiation: conv kernel variants with the FIC staged input-checksum source for (DT_I8, EPI_NONE)
#include "conv_tc_kernel.cuh"

namespace abed_host {
template cudaError_t launch_epi<abed_dev::DT_I8, abed_dev::EPI_NONE, 4>(const ConvTcParams&, int, bool, cudaStream_t);
}  // namespace abed_host
