// abed/abed.hpp -- umbrella header of the B200 drop-in for the reference's ABED
// convolution path (reference: proj/include/abed/abed.hpp), plus the ABFT-GEMM
// comparison (abft_gemm.hpp).  The reference's analytic cost model is out of the
// hot-path scope and not included.
#pragma once

#include "abft_gemm.hpp"
#include "checksum.hpp"
#include "convolution.hpp"
#include "faults.hpp"
#include "protected_conv.hpp"
#include "rng.hpp"
#include "tensor.hpp"
