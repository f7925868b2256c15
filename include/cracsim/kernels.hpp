// cracsim B200 build — the standard kernel set as CUDA bodies.
// Same names, arities and byte semantics as the reference host bodies
// (ref: include/cracsim/kernels.hpp:9-23, src/kernels.cpp:10-117); each body
// enqueues one sm_100a kernel on the launch stream.  The f32 kernels keep the
// reference's fixed four-lane accumulation order and are compiled without FMA
// contraction, so results are bit-identical to the host reference.
//   fill8   (1 buffer; value, len)       add8 (1 buffer; addend, len)
//   affine8 (1 buffer; mul, add, len)    dot_f32 (x, y, out; n)
//   gemv_f32(A, x, y; m, k)              gemm_f32(A, B, C; m, k, n)
#pragma once

#include "cracsim/ckpt_engine.hpp"

namespace cracsim {

std::vector<KernelDescriptor> standard_kernels();
const KernelCatalog& standard_catalog();

}  // namespace cracsim
