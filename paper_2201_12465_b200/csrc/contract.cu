// Contraction dispatch.  Path 2 (default): f32 convs whose channel counts are multiples of 32
// go to the TMA-fed tcgen05 3xTF32 kernels (gemm_tma.cu); path >= 1: other f32 matmul / conv
// shapes go to the SIMT-fed tcgen05 kernels (gemm_tc.cu); everything else (f64, integer,
// mixed dtypes, unsupported shapes) and path 0 run the SIMT kernels (gemm_simt.cu).
#include "common.cuh"

extern "C" {
int pb_matmul_simt(const pb_tensor* a, const pb_tensor* b, const pb_tensor* out);
int pb_conv2d_simt(const pb_tensor* x, const pb_tensor* w, const pb_tensor* bias, const pb_conv* p, const pb_tensor* out);
int pb_conv2d_grad_input_simt(const pb_tensor* g, const pb_tensor* w, const pb_conv* p, const pb_tensor* out);
int pb_conv2d_grad_weight_simt(const pb_tensor* x, const pb_tensor* g, const pb_conv* p, const pb_tensor* out);
// tensor-core path: returns PB_ERR_UNSUPPORTED (without side effects) when it declines
int pb_matmul_tc(const pb_tensor* a, const pb_tensor* b, const pb_tensor* out);
int pb_matmul_tma(const pb_tensor* a, const pb_tensor* b, const pb_tensor* out);
int pb_conv2d_grad_weight_mm(const pb_tensor* x, const pb_tensor* g, const pb_conv* p, const pb_tensor* out);
int pb_conv2d_tc(const pb_tensor* x, const pb_tensor* w, const pb_tensor* bias, const pb_conv* p, const pb_tensor* out);
int pb_conv2d_grad_input_tc(const pb_tensor* g, const pb_tensor* w, const pb_conv* p, const pb_tensor* out);
int pb_conv2d_grad_weight_tc(const pb_tensor* x, const pb_tensor* g, const pb_conv* p, const pb_tensor* out);
int pb_conv2d_tma(const pb_tensor* x, const pb_tensor* w, const pb_tensor* bias, const pb_conv* p, const pb_tensor* out);
int pb_conv2d_grad_input_tma(const pb_tensor* g, const pb_tensor* w, const pb_conv* p, const pb_tensor* out);
int pb_conv2d_grad_weight_tma(const pb_tensor* x, const pb_tensor* g, const pb_conv* p, const pb_tensor* out);
}

static int g_tc = 2;

extern "C" {

int pb_gemm_path(void) { return g_tc; }
int pb_set_gemm_path(int path) {
  if (path < 0 || path > 2) return PB_ERR_ARG;
  g_tc = path;
  return PB_OK;
}

int pb_matmul(const pb_tensor* a, const pb_tensor* b, const pb_tensor* out) {
  if (g_tc == 2) {
    int rc = pb_matmul_tma(a, b, out);
    if (rc != PB_ERR_UNSUPPORTED) return rc;
  }
  if (g_tc) {
    int rc = pb_matmul_tc(a, b, out);
    if (rc != PB_ERR_UNSUPPORTED) return rc;
  }
  return pb_matmul_simt(a, b, out);
}

int pb_conv2d(const pb_tensor* x, const pb_tensor* w, const pb_tensor* bias, const pb_conv* p, const pb_tensor* out) {
  if (g_tc == 2) {
    int rc = pb_conv2d_tma(x, w, bias, p, out);
    if (rc != PB_ERR_UNSUPPORTED) return rc;
  }
  if (g_tc) {
    int rc = pb_conv2d_tc(x, w, bias, p, out);
    if (rc != PB_ERR_UNSUPPORTED) return rc;
  }
  return pb_conv2d_simt(x, w, bias, p, out);
}

int pb_conv2d_grad_input(const pb_tensor* g, const pb_tensor* w, const pb_conv* p, const pb_tensor* out) {
  if (g_tc == 2) {
    int rc = pb_conv2d_grad_input_tma(g, w, p, out);
    if (rc != PB_ERR_UNSUPPORTED) return rc;
  }
  if (g_tc) {
    int rc = pb_conv2d_grad_input_tc(g, w, p, out);
    if (rc != PB_ERR_UNSUPPORTED) return rc;
  }
  return pb_conv2d_grad_input_simt(g, w, p, out);
}

int pb_conv2d_grad_weight(const pb_tensor* x, const pb_tensor* g, const pb_conv* p, const pb_tensor* out) {
  if (g_tc == 2) {
    int rc = pb_conv2d_grad_weight_mm(x, g, p, out);
    if (rc != PB_ERR_UNSUPPORTED) return rc;
  }
  if (g_tc == 2) {
    int rc = pb_conv2d_grad_weight_tma(x, g, p, out);
    if (rc != PB_ERR_UNSUPPORTED) return rc;
  }
  if (g_tc) {
    int rc = pb_conv2d_grad_weight_tc(x, g, p, out);
    if (rc != PB_ERR_UNSUPPORTED) return rc;
  }
  return pb_conv2d_grad_weight_simt(x, g, p, out);
}

}  // extern "C"
