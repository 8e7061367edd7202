// tcgen05 3xTF32 contraction kernels (placeholder: declines every shape until landed).
#include "common.cuh"

extern "C" {
int pb_matmul_tc(const pb_tensor*, const pb_tensor*, const pb_tensor*) { return PB_ERR_UNSUPPORTED; }
int pb_conv2d_tc(const pb_tensor*, const pb_tensor*, const pb_tensor*, const pb_conv*, const pb_tensor*) {
  return PB_ERR_UNSUPPORTED;
}
int pb_conv2d_grad_input_tc(const pb_tensor*, const pb_tensor*, const pb_conv*, const pb_tensor*) {
  return PB_ERR_UNSUPPORTED;
}
int pb_conv2d_grad_weight_tc(const pb_tensor*, const pb_tensor*, const pb_conv*, const pb_tensor*) {
  return PB_ERR_UNSUPPORTED;
}
}
