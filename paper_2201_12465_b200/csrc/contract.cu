// Contraction dispatch: f32 x f32 matmul / conv go to the tcgen05 3xTF32 kernels
// (gemm_tc.cu) when that path is enabled and the shape is supported; everything else
// (f64, integer, mixed dtypes, unsupported shapes) runs the SIMT kernels (gemm_simt.cu).
#include "common.cuh"

extern "C" {
int pb_matmul_simt(const pb_tensor* a, const pb_tensor* b, const pb_tensor* out);
int pb_conv2d_simt(const pb_tensor* x, const pb_tensor* w, const pb_tensor* bias, const pb_conv* p, const pb_tensor* out);
int pb_conv2d_grad_input_simt(const pb_tensor* g, const pb_tensor* w, const pb_conv* p, const pb_tensor* out);
int pb_conv2d_grad_weight_simt(const pb_tensor* x, const pb_tensor* g, const pb_conv* p, const pb_tensor* out);
// tensor-core path: returns PB_ERR_UNSUPPORTED (without side effects) when it declines
int pb_matmul_tc(const pb_tensor* a, const pb_tensor* b, const pb_tensor* out);
int pb_conv2d_tc(const pb_tensor* x, const pb_tensor* w, const pb_tensor* bias, const pb_conv* p, const pb_tensor* out);
int pb_conv2d_grad_input_tc(const pb_tensor* g, const pb_tensor* w, const pb_conv* p, const pb_tensor* out);
int pb_conv2d_grad_weight_tc(const pb_tensor* x, const pb_tensor* g, const pb_conv* p, const pb_tensor* out);
}

static int g_tc = 1;

extern "C" {

int pb_gemm_path(void) { return g_tc; }
int pb_set_gemm_path(int tc) {
  g_tc = tc ? 1 : 0;
  return PB_OK;
}

int pb_matmul(const pb_tensor* a, const pb_tensor* b, const pb_tensor* out) {
  if (g_tc) {
    int rc = pb_matmul_tc(a, b, out);
    if (rc != PB_ERR_UNSUPPORTED) return rc;
  }
  return pb_matmul_simt(a, b, out);
}

int pb_conv2d(const pb_tensor* x, const pb_tensor* w, const pb_tensor* bias, const pb_conv* p, const pb_tensor* out) {
  if (g_tc) {
    int rc = pb_conv2d_tc(x, w, bias, p, out);
    if (rc != PB_ERR_UNSUPPORTED) return rc;
  }
  return pb_conv2d_simt(x, w, bias, p, out);
}

int pb_conv2d_grad_input(const pb_tensor* g, const pb_tensor* w, const pb_conv* p, const pb_tensor* out) {
  if (g_tc) {
    int rc = pb_conv2d_grad_input_tc(g, w, p, out);
    if (rc != PB_ERR_UNSUPPORTED) return rc;
  }
  return pb_conv2d_grad_input_simt(g, w, p, out);
}

int pb_conv2d_grad_weight(const pb_tensor* x, const pb_tensor* g, const pb_conv* p, const pb_tensor* out) {
  if (g_tc) {
    int rc = pb_conv2d_grad_weight_tc(x, g, p, out);
    if (rc != PB_ERR_UNSUPPORTED) return rc;
  }
  return pb_conv2d_grad_weight_simt(x, g, p, out);
}

}  // extern "C"
