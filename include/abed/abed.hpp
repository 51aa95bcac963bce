// abed/abed.hpp -- umbrella header of the B200 drop-in for the reference's ABED
// convolution path (reference: proj/include/abed/abed.hpp), plus the ABFT-GEMM
// comparison (abft_gemm.hpp) and the analytic op / byte model (cost_model.hpp).
#pragma once

#include "abft_gemm.hpp"
#include "checksum.hpp"
#include "cost_model.hpp"
#include "convolution.hpp"
#include "faults.hpp"
#include "protected_conv.hpp"
#include "rng.hpp"
#include "tensor.hpp"
