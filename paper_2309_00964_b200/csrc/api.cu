// api.cu -- the C ABI of libedkm.so (include/edkm.h): argument validation,
// buffer layout of `saved` / `ws`, and the launch sequence of each entry point.
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <vector>

#include "../../include/edkm.h"
#include "common.cuh"
#include "launch.h"

using namespace edkm;

namespace {

thread_local char g_err[512] = "";
thread_local int g_launches = 0;
thread_local int g_max_ctas = 0;  // edkm_set_max_ctas: cap on the streaming kernels' grid (0 = SM count)

edkm_status fail(edkm_status st, const char* fmt, const char* detail = "") {
  snprintf(g_err, sizeof(g_err), fmt, detail);
  return st;
}
edkm_status cuda_fail(cudaError_t e, const char* where) {
  snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
  return EDKM_E_CUDA;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

namespace edkm {
edkm_status set_error(edkm_status st, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return st;
}
void reset_launches() { g_launches = 0; }
void add_launches(int n) { g_launches += n; }
}  // namespace edkm

namespace {

int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return g_max_ctas > 0 && g_max_ctas < n ? g_max_ctas : n;
}

bool params_ok(const edkm_params* p) {
  if (!p) return false;
  if (p->wdtype != EDKM_BF16 && p->wdtype != EDKM_FP16) return false;
  if (p->bits < 1 || p->bits > 8) return false;
  if (!(p->tau > 0.0) || !isfinite(p->tau)) return false;
  if (p->max_iter < 0 || p->max_iter > 100000) return false;
  if (!(p->eps >= 0.0) || !isfinite(p->eps)) return false;
  return true;
}

edkm_status check_params(const edkm_params* p) {
  if (!p) return fail(EDKM_E_ARG, "params is NULL");
  if (p->wdtype != EDKM_BF16 && p->wdtype != EDKM_FP16) return fail(EDKM_E_DTYPE, "wdtype must be BF16 or FP16");
  if (p->bits < 1 || p->bits > 8) return fail(EDKM_E_UNSUPPORTED, "bits must be in 1..8");
  if (!params_ok(p)) return fail(EDKM_E_ARG, "tau must be > 0 and finite, max_iter in [0, 1e5], eps >= 0 and finite");
  return EDKM_OK;
}

edkm_status check_tensors(const edkm_tensor* t, int nt) {
  if (nt < 0) return fail(EDKM_E_ARG, "nt < 0");
  if (nt > 0 && !t) return fail(EDKM_E_ARG, "tensors is NULL");
  for (int i = 0; i < nt; ++i) {
    if (t[i].n < 0) return fail(EDKM_E_ARG, "tensor with n < 0");
    if (t[i].n > 0 && !t[i].w) return fail(EDKM_E_ARG, "tensor with n > 0 and NULL data");
    if (((uintptr_t)t[i].w & 1u) != 0) return fail(EDKM_E_ARG, "weights must be 2-byte aligned");
  }
  return EDKM_OK;
}

edkm_status check_ptrs(const void* const* ptrs, const edkm_tensor* t, int nt, const char* what) {
  if (nt > 0 && !ptrs) return fail(EDKM_E_ARG, "%s array is NULL", what);
  for (int i = 0; i < nt; ++i)
    if (t[i].n > 0 && !ptrs[i]) return fail(EDKM_E_ARG, "%s pointer is NULL for a non-empty tensor", what);
  return EDKM_OK;
}

// Build per-launch tensor groups of <= kMaxTensorsPerLaunch and run `fn` on each.
template <class Fn>
cudaError_t for_groups(const edkm_tensor* t, int nt, const void* const* g, void* const* out, StreamArgs& A, Fn fn) {
  for (int t0 = 0; t0 < nt; t0 += kMaxTensorsPerLaunch) {
    const int n = nt - t0 < kMaxTensorsPerLaunch ? nt - t0 : kMaxTensorsPerLaunch;
    A.nt = n;
    A.t0 = t0;
    A.offs[0] = 0;
    for (int i = 0; i < n; ++i) {
      A.w[i] = reinterpret_cast<const uint16_t*>(t[t0 + i].w);
      A.g[i] = g ? g[t0 + i] : nullptr;
      A.out[i] = out ? out[t0 + i] : nullptr;
      A.offs[i + 1] = A.offs[i] + t[t0 + i].n;
    }
    A.total = A.offs[n];
    cudaError_t e = fn(A);
    if (e != cudaSuccess) return e;
    if (A.total > 0) ++g_launches;
  }
  return cudaSuccess;
}

TableArgs table_args(int nt, const edkm_params* p, const void* saved) {
  TableArgs P = {};
  P.nt = nt;
  P.k = 1 << p->bits;
  P.wdtype = p->wdtype;
  P.max_iter = p->max_iter;
  P.cl = table_cluster_size(nt, p->wdtype);
  P.tau = p->tau;
  P.inv_tau = 1.0 / p->tau;
  P.eps = p->eps;
  const SavedLayout L = saved_layout(nt, P.k, p->max_iter);
  unsigned char* b = (unsigned char*)saved;
  P.state = reinterpret_cast<TensorState*>(b + L.state);
  P.ctraj = reinterpret_cast<double*>(b + L.ctraj);
  P.straj = reinterpret_cast<double*>(b + L.straj);
  P.rows = reinterpret_cast<uint16_t*>(b + L.rows);
  P.table16 = reinterpret_cast<uint16_t*>(b + L.table16);
  P.idx8 = reinterpret_cast<uint8_t*>(b + L.idx8);
  P.page_cnt = reinterpret_cast<int64_t*>(b + L.page_cnt);
  return P;
}

void ws_args(TableArgs& P, void* ws) {
  const WsLayout L = ws_layout(P.nt, P.k);
  unsigned char* b = (unsigned char*)ws;
  P.B = reinterpret_cast<double*>(b + L.B);
  P.psi = reinterpret_cast<double*>(b + L.psi);
  P.phipsi = reinterpret_cast<float2*>(b + L.phipsi);
}

template <class T>
T* off(T* p, int64_t n) { return p ? p + n : p; }

// TableArgs built for nt tensors restricted to tensors [t0, t1): every per-tensor array pointer
// advanced by t0 entries of the full-nt layout; the cluster size follows the range's count.
TableArgs table_range(const TableArgs& P, int t0, int t1) {
  TableArgs R = P;
  const int64_t k = P.k, sc = (int64_t)(P.max_iter + 1) * k, ss = (int64_t)(P.max_iter > 0 ? P.max_iter : 1) * k;
  const int64_t u = (int64_t)t0 * kPatterns;
  R.nt = t1 - t0;
  R.cl = table_cluster_size(R.nt, P.wdtype);
  R.counts = off(P.counts, u);
  R.C0 = off(P.C0, t0 * k);
  R.C_out = off(P.C_out, t0 * k);
  R.table = off(P.table, u);
  R.state = off(P.state, t0);
  R.ctraj = off(P.ctraj, t0 * sc);
  R.straj = off(P.straj, t0 * ss);
  R.rows = off(P.rows, u);
  R.table16 = off(P.table16, u);
  R.idx8 = off(P.idx8, u);
  R.page_cnt = off(P.page_cnt, (int64_t)t0 * 256);
  R.B = off(P.B, u);
  R.psi = off(P.psi, u);
  R.phipsi = off(P.phipsi, u);
  R.gamma = off(P.gamma, t0 * k);
  R.dC0 = off(P.dC0, t0 * k);
  return R;
}

}  // namespace

namespace edkm {
SavedLayout saved_layout(int nt, int k, int max_iter) {
  SavedLayout L;
  size_t o = 0;
  const size_t n = (size_t)nt;
  L.state = o; o = align256(o + n * sizeof(TensorState));
  L.ctraj = o; o = align256(o + n * (size_t)(max_iter + 1) * k * 8);
  L.straj = o; o = align256(o + n * (size_t)(max_iter > 0 ? max_iter : 1) * k * 8);
  L.rows = o; o = align256(o + n * kPatterns * 2);
  L.table16 = o; o = align256(o + n * kPatterns * 2);
  L.idx8 = o; o = align256(o + n * kPatterns);
  L.page_cnt = o; o = align256(o + n * 256 * 8);
  L.total = o;
  return L;
}
WsLayout ws_layout(int nt, int k) {
  WsLayout L;
  size_t o = 0;
  const size_t n = (size_t)nt;
  L.B = o; o = align256(o + n * kPatterns * 8);
  L.psi = o; o = align256(o + n * kPatterns * 8);
  L.phipsi = o; o = align256(o + n * kPatterns * 8);
  L.gamma = o; o = align256(o + n * k * 8);
  L.total = o;
  return L;
}
}  // namespace edkm

extern "C" {

size_t edkm_saved_bytes(int nt, const edkm_params* p) {
  if (nt < 0 || !params_ok(p)) return 0;
  return saved_layout(nt, 1 << p->bits, p->max_iter).total;
}

size_t edkm_workspace_bytes(int nt, const edkm_params* p) {
  if (nt < 0 || !params_ok(p)) return 0;
  return ws_layout(nt, 1 << p->bits).total;
}

edkm_status edkm_uniquify(const edkm_tensor* tensors, int nt, int wdtype, int32_t* counts, edkm_comm* comm,
                          void* stream) {
  EDKM_NVTX("edkm F1 uniquify");
  g_launches = 0;
  if (wdtype != EDKM_BF16 && wdtype != EDKM_FP16) return fail(EDKM_E_DTYPE, "wdtype must be BF16 or FP16");
  edkm_status st = check_tensors(tensors, nt);
  if (st != EDKM_OK) return st;
  if (nt > 0 && !counts) return fail(EDKM_E_ARG, "counts is NULL");
  if (nt == 0) return EDKM_OK;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)nt * kPatterns * sizeof(int32_t), s);
  if (e != cudaSuccess) return cuda_fail(e, "memset counts");
  static thread_local StreamArgs A;
  A.wdtype = wdtype;
  const int sms = sm_count();
  e = for_groups(tensors, nt, nullptr, nullptr, A, [&](const StreamArgs& a) { return launch_f1(a, counts, sms, s); });
  if (e != cudaSuccess) return cuda_fail(e, "F1 histogram launch");
  return comm_allreduce_sum(comm, counts, (size_t)nt * kPatterns, 0, s);  // global counts on every rank
}

edkm_status edkm_nvls_set_timeout(double seconds, int trap) {
  if (!(seconds > 0.0)) return fail(EDKM_E_ARG, "NVLS timeout must be > 0");
  nvls_set_timeout(seconds, trap);
  return EDKM_OK;
}

edkm_status edkm_nvls_failed(int* failed) {
  if (!failed) return fail(EDKM_E_ARG, "NULL failed");
  cudaError_t e = nvls_failed(failed);
  if (e != cudaSuccess) return cuda_fail(e, "read NVLS status");
  return EDKM_OK;
}

edkm_status edkm_uniquify_nvls(const edkm_tensor* tensors, int nt, int wdtype, const edkm_nvls* x, void* stream) {
  EDKM_NVTX("edkm F1 uniquify (NVLS)");
  g_launches = 0;
  if (wdtype != EDKM_BF16 && wdtype != EDKM_FP16) return fail(EDKM_E_DTYPE, "wdtype must be BF16 or FP16");
  edkm_status st = check_tensors(tensors, nt);
  if (st != EDKM_OK) return st;
  if (!x || !x->counts_mc || !x->flags_mc || !x->flags || !x->epoch) return fail(EDKM_E_ARG, "NULL NVLS buffer");
  if (x->nranks < 1) return fail(EDKM_E_ARG, "nranks < 1");
  if (x->emulate && !(x->nranks == 1 || (x->nranks == 2 && x->peer_delta != 0)))
    return fail(EDKM_E_ARG, "emulate requires nranks == 1, or nranks == 2 with a peer buffer");
  if (nt > kMaxTensorsPerLaunch) return fail(EDKM_E_UNSUPPORTED, "NVLS uniquify takes at most 512 tensors per call");
  const int sms = sm_count();
  if (sms > EDKM_NVLS_FLAGS) return fail(EDKM_E_UNSUPPORTED, "more SMs than NVLS arrival counters");
  static thread_local StreamArgs A;
  A.wdtype = wdtype;
  A.nt = nt;
  A.t0 = 0;
  A.offs[0] = 0;
  for (int i = 0; i < nt; ++i) {
    A.w[i] = reinterpret_cast<const uint16_t*>(tensors[i].w);
    A.g[i] = nullptr;
    A.out[i] = nullptr;
    A.offs[i + 1] = A.offs[i] + tensors[i].n;
  }
  A.total = A.offs[nt];
  A.peer_delta = x->emulate ? x->peer_delta : 0;
  cudaError_t e = launch_f1_nvls(A, x->counts_mc, x->flags_mc, x->flags, x->epoch, x->nranks, x->emulate, sms,
                                 (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "F1 NVLS histogram launch");
  g_launches = 2;
  return EDKM_OK;
}

edkm_status edkm_forward_range(const int32_t* counts, int nt, int t0, int t1, const edkm_params* p, const float* C0,
                               float* C_out, float* table, void* saved, void* stream) {
  EDKM_NVTX("edkm TF forward");
  g_launches = 0;
  edkm_status st = check_params(p);
  if (st != EDKM_OK) return st;
  if (nt < 0) return fail(EDKM_E_ARG, "nt < 0");
  if (t0 < 0 || t1 < t0 || t1 > nt) return fail(EDKM_E_ARG, "tensor range outside [0, nt]");
  if (t1 == t0) return EDKM_OK;
  if (!counts || !C0 || !C_out || !table || !saved) return fail(EDKM_E_ARG, "NULL buffer");
  TableArgs P = table_args(nt, p, saved);
  P.counts = counts;
  P.C0 = C0;
  P.C_out = C_out;
  P.table = table;
  const TableArgs R = table_range(P, t0, t1);
  cudaError_t e = R.k >= 32 ? launch_tf_wide(R, (cudaStream_t)stream) : launch_tf(R, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "TF table-forward launch");
  g_launches = 1;
  return EDKM_OK;
}

edkm_status edkm_forward_layout_range(const int32_t* counts, int nt, int t0, int t1, const edkm_params* p,
                                      float* table, void* saved, void* stream) {
  EDKM_NVTX("edkm TF layout");
  g_launches = 0;
  edkm_status st = check_params(p);
  if (st != EDKM_OK) return st;
  if (nt < 0) return fail(EDKM_E_ARG, "nt < 0");
  if (t0 < 0 || t1 < t0 || t1 > nt) return fail(EDKM_E_ARG, "tensor range outside [0, nt]");
  if (t1 == t0) return EDKM_OK;
  if (!counts || !table || !saved) return fail(EDKM_E_ARG, "NULL buffer");
  TableArgs P = table_args(nt, p, saved);
  P.counts = counts;
  P.table = table;
  P.layout_only = 1;
  const TableArgs R = table_range(P, t0, t1);
  cudaError_t e = R.k >= 32 ? launch_tf_wide(R, (cudaStream_t)stream) : launch_tf(R, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "TF layout launch");
  g_launches = 1;
  return EDKM_OK;
}

edkm_status edkm_forward(const int32_t* counts, int nt, const edkm_params* p, const float* C0, float* C_out,
                         float* table, void* saved, void* stream) {
  if (nt < 0) {
    g_launches = 0;
    return fail(EDKM_E_ARG, "nt < 0");
  }
  return edkm_forward_range(counts, nt, 0, nt, p, C0, C_out, table, saved, stream);
}

edkm_status edkm_reconstruct(const edkm_tensor* tensors, int nt, const edkm_params* p, const float* table,
                             const float* C_out, const void* saved, int mode, int out_dtype, void* const* out,
                             void* stream) {
  EDKM_NVTX("edkm F2 reconstruct");
  g_launches = 0;
  edkm_status st = check_params(p);
  if (st != EDKM_OK) return st;
  st = check_tensors(tensors, nt);
  if (st != EDKM_OK) return st;
  st = check_ptrs(out, tensors, nt, "out");
  if (st != EDKM_OK) return st;
  int m;
  if (mode == EDKM_SOFT && out_dtype == p->wdtype) m = 0;
  else if (mode == EDKM_HARD_VALUE && out_dtype == p->wdtype) m = 1;
  else if (mode == EDKM_SOFT && out_dtype == EDKM_FP32) m = 2;
  else if (mode == EDKM_HARD_VALUE && out_dtype == EDKM_FP32) m = 3;
  else if (mode == EDKM_HARD_INDEX && out_dtype == EDKM_U8) m = 4;
  else return fail(EDKM_E_DTYPE, "unsupported (mode, out_dtype) combination");
  if (nt == 0) return EDKM_OK;
  if (!saved || (m == 2 && !table) || ((m == 1 || m == 3) && !C_out)) return fail(EDKM_E_ARG, "NULL buffer");
  const int k = 1 << p->bits;
  const SavedLayout L = saved_layout(nt, k, p->max_iter);
  const unsigned char* b = (const unsigned char*)saved;
  F2Args F;
  F.table = table;
  F.table16 = reinterpret_cast<const uint16_t*>(b + L.table16);
  F.idx8 = b + L.idx8;
  F.C = C_out;
  F.state = reinterpret_cast<const TensorState*>(b + L.state);
  F.k = k;
  static thread_local StreamArgs A;
  A.wdtype = p->wdtype;
  A.odtype = out_dtype;
  A.mode = m;
  const int sms = sm_count();
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = for_groups(tensors, nt, nullptr, out, A, [&](const StreamArgs& a) { return launch_f2(a, F, m, sms, s); });
  if (e != cudaSuccess) return cuda_fail(e, "F2 reconstruct launch");
  return EDKM_OK;
}

static edkm_status check_backward(const edkm_tensor* tensors, int nt, const edkm_params* p, const void* const* grads,
                                  int gdtype) {
  edkm_status st = check_params(p);
  if (st != EDKM_OK) return st;
  st = check_tensors(tensors, nt);
  if (st != EDKM_OK) return st;
  st = check_ptrs(grads, tensors, nt, "grads");
  if (st != EDKM_OK) return st;
  if (gdtype != p->wdtype && gdtype != EDKM_FP32) return fail(EDKM_E_DTYPE, "grads must be the weights' dtype or FP32");
  return EDKM_OK;
}

edkm_status edkm_backward_buckets(const edkm_tensor* tensors, int nt, const edkm_params* p, const void* const* grads,
                                  int gdtype, const void* saved, void* ws, void* stream) {
  EDKM_NVTX("edkm B1 buckets");
  g_launches = 0;
  edkm_status st = check_backward(tensors, nt, p, grads, gdtype);
  if (st != EDKM_OK) return st;
  if (nt == 0) return EDKM_OK;
  if (!saved || !ws) return fail(EDKM_E_ARG, "NULL buffer");
  cudaStream_t s = (cudaStream_t)stream;
  TableArgs P = table_args(nt, p, saved);
  ws_args(P, ws);
  cudaError_t e = cudaMemsetAsync((void*)P.B, 0, (size_t)nt * kPatterns * sizeof(double), s);
  if (e != cudaSuccess) return cuda_fail(e, "memset buckets");
  B1Args Bq;
  Bq.B = const_cast<double*>(P.B);
  Bq.state = P.state;
  static thread_local StreamArgs A;
  A.wdtype = p->wdtype;
  A.gdtype = gdtype;
  const int sms = sm_count();
  e = for_groups(tensors, nt, grads, nullptr, A, [&](const StreamArgs& a) { return launch_b1(a, Bq, sms, s); });
  if (e != cudaSuccess) return cuda_fail(e, "B1 bucket launch");
  return EDKM_OK;
}

edkm_status edkm_backward_gamma(int nt, const edkm_params* p, const int32_t* counts, const void* saved, void* ws,
                                double* gamma, void* stream) {
  EDKM_NVTX("edkm TGAMMA");
  g_launches = 0;
  edkm_status st = check_params(p);
  if (st != EDKM_OK) return st;
  if (nt < 0) return fail(EDKM_E_ARG, "nt < 0");
  if (nt == 0) return EDKM_OK;
  if (!counts || !saved || !ws || !gamma) return fail(EDKM_E_ARG, "NULL buffer");
  TableArgs P = table_args(nt, p, saved);
  ws_args(P, ws);
  P.counts = counts;
  P.gamma = gamma;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = P.k >= 32 ? launch_tgamma_wide(P, s) : launch_tgamma(P, s);
  if (e != cudaSuccess) return cuda_fail(e, "TGAMMA launch");
  g_launches = 1;
  return EDKM_OK;
}

edkm_status edkm_backward_reduce(const edkm_tensor* tensors, int nt, const edkm_params* p, const void* const* grads,
                                 int gdtype, const int32_t* counts, const void* saved, void* ws, double* gamma,
                                 edkm_comm* comm, void* stream) {
  edkm_status st = check_backward(tensors, nt, p, grads, gdtype);
  if (st != EDKM_OK) return st;
  if (nt > 0 && (!counts || !gamma)) return fail(EDKM_E_ARG, "NULL buffer");
  st = edkm_backward_buckets(tensors, nt, p, grads, gdtype, saved, ws, stream);
  if (st != EDKM_OK) return st;
  const int n1 = g_launches;
  st = edkm_backward_gamma(nt, p, counts, saved, ws, gamma, stream);
  if (st != EDKM_OK) return st;
  g_launches += n1;
  // gamma_T is linear in the buckets: the sum of the ranks' partials is the global gamma_T
  return comm_allreduce_sum(comm, gamma, (size_t)nt * (1 << p->bits), 1, (cudaStream_t)stream);
}

edkm_status edkm_backward_table_range(int nt, int t0, int t1, const edkm_params* p, const int32_t* counts,
                                      const void* saved, void* ws, const double* gamma, float* dC0, void* stream) {
  EDKM_NVTX("edkm TB table backward");
  g_launches = 0;
  edkm_status st = check_params(p);
  if (st != EDKM_OK) return st;
  if (nt < 0) return fail(EDKM_E_ARG, "nt < 0");
  if (t0 < 0 || t1 < t0 || t1 > nt) return fail(EDKM_E_ARG, "tensor range outside [0, nt]");
  if (t1 == t0) return EDKM_OK;
  if (!counts || !saved || !ws || !gamma || !dC0) return fail(EDKM_E_ARG, "NULL buffer");
  TableArgs P = table_args(nt, p, saved);
  ws_args(P, ws);
  P.counts = counts;
  P.gamma = const_cast<double*>(gamma);
  P.dC0 = dC0;
  const TableArgs R = table_range(P, t0, t1);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = R.k >= 32 ? launch_tb_wide(R, s) : launch_tb(R, s);
  if (e != cudaSuccess) return cuda_fail(e, "TB table-backward launch");
  g_launches = 1;
  return EDKM_OK;
}

edkm_status edkm_backward_table(int nt, const edkm_params* p, const int32_t* counts, const void* saved, void* ws,
                                const double* gamma, float* dC0, void* stream) {
  if (nt < 0) {
    g_launches = 0;
    return fail(EDKM_E_ARG, "nt < 0");
  }
  return edkm_backward_table_range(nt, 0, nt, p, counts, saved, ws, gamma, dC0, stream);
}

edkm_status edkm_layout(int nt, const edkm_params* p, size_t* saved_offs, size_t* ws_offs) {
  g_launches = 0;
  edkm_status st = check_params(p);
  if (st != EDKM_OK) return st;
  if (nt < 0) return fail(EDKM_E_ARG, "nt < 0");
  const int k = 1 << p->bits;
  if (saved_offs) {
    const SavedLayout L = saved_layout(nt, k, p->max_iter);
    const size_t v[8] = {L.state, L.ctraj, L.straj, L.rows, L.table16, L.idx8, L.page_cnt, L.total};
    memcpy(saved_offs, v, sizeof(v));
  }
  if (ws_offs) {
    const WsLayout L = ws_layout(nt, k);
    const size_t v[5] = {L.B, L.psi, L.phipsi, L.gamma, L.total};
    memcpy(ws_offs, v, sizeof(v));
  }
  return EDKM_OK;
}

edkm_status edkm_backward_dw(const edkm_tensor* tensors, int nt, const edkm_params* p, const void* const* grads,
                             int gdtype, const void* saved, const void* ws, void* const* dW, int dw_dtype,
                             void* stream) {
  EDKM_NVTX("edkm B2 dW");
  g_launches = 0;
  edkm_status st = check_backward(tensors, nt, p, grads, gdtype);
  if (st != EDKM_OK) return st;
  st = check_ptrs(dW, tensors, nt, "dW");
  if (st != EDKM_OK) return st;
  if (dw_dtype != p->wdtype && dw_dtype != EDKM_FP32) return fail(EDKM_E_DTYPE, "dW must be the weights' dtype or FP32");
  if (nt == 0) return EDKM_OK;
  if (!saved || !ws) return fail(EDKM_E_ARG, "NULL buffer");
  TableArgs P = table_args(nt, p, saved);
  ws_args(P, const_cast<void*>(ws));
  B2Args Bq;
  Bq.phipsi = P.phipsi;
  Bq.state = P.state;
  static thread_local StreamArgs A;
  A.wdtype = p->wdtype;
  A.gdtype = gdtype;
  A.odtype = dw_dtype;
  const int sms = sm_count();
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = for_groups(tensors, nt, grads, dW, A, [&](const StreamArgs& a) { return launch_b2(a, Bq, sms, s); });
  if (e != cudaSuccess) return cuda_fail(e, "B2 dW launch");
  return EDKM_OK;
}

edkm_status edkm_backward_apply(const edkm_tensor* tensors, int nt, const edkm_params* p, const void* const* grads,
                                int gdtype, const int32_t* counts, const void* saved, void* ws, const double* gamma,
                                void* const* dW, int dw_dtype, float* dC0, void* stream) {
  edkm_status st = check_backward(tensors, nt, p, grads, gdtype);
  if (st != EDKM_OK) return st;
  st = check_ptrs(dW, tensors, nt, "dW");
  if (st != EDKM_OK) return st;
  if (dw_dtype != p->wdtype && dw_dtype != EDKM_FP32) return fail(EDKM_E_DTYPE, "dW must be the weights' dtype or FP32");
  st = edkm_backward_table(nt, p, counts, saved, ws, gamma, dC0, stream);
  if (st != EDKM_OK) return st;
  const int n1 = g_launches;
  st = edkm_backward_dw(tensors, nt, p, grads, gdtype, saved, ws, dW, dw_dtype, stream);
  if (st == EDKM_OK) g_launches += n1;
  return st;
}

edkm_status edkm_backward(const edkm_tensor* tensors, int nt, const edkm_params* p, const void* const* grads,
                          int gdtype, const int32_t* counts, const void* saved, void* ws, void* const* dW,
                          int dw_dtype, float* dC0, void* stream) {
  edkm_status st = check_params(p);
  if (st != EDKM_OK) return st;
  if (nt < 0) return fail(EDKM_E_ARG, "nt < 0");
  if (nt > 0 && !ws) return fail(EDKM_E_ARG, "NULL workspace");
  double* gamma = nt > 0 ? reinterpret_cast<double*>((unsigned char*)ws + ws_layout(nt, 1 << p->bits).gamma) : nullptr;
  st = edkm_backward_reduce(tensors, nt, p, grads, gdtype, counts, saved, ws, gamma, nullptr, stream);
  if (st != EDKM_OK) return st;
  const int n1 = g_launches;
  st = edkm_backward_apply(tensors, nt, p, grads, gdtype, counts, saved, ws, gamma, dW, dw_dtype, dC0, stream);
  if (st == EDKM_OK) g_launches += n1;
  return st;
}

edkm_status edkm_read_status(const void* saved, int nt, const edkm_params* p, int64_t* nonfinite_host,
                             int32_t* iters_host, void* stream) {
  g_launches = 0;
  edkm_status st = check_params(p);
  if (st != EDKM_OK) return st;
  if (nt < 0) return fail(EDKM_E_ARG, "nt < 0");
  if (nt == 0) return EDKM_OK;
  if (!saved) return fail(EDKM_E_ARG, "NULL saved");
  std::vector<TensorState> h(nt);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(h.data(), saved, (size_t)nt * sizeof(TensorState), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "read status");
  for (int t = 0; t < nt; ++t) {
    if (nonfinite_host) {
      int64_t sum = 0;
      for (int c = 0; c < h[t].cl && c < kMaxCluster; ++c) sum += h[t].nonfinite[c];
      nonfinite_host[t] = sum;
    }
    if (iters_host) iters_host[t] = h[t].T;
  }
  return EDKM_OK;
}

int edkm_last_launch_count(void) { return g_launches; }

int edkm_set_max_ctas(int ctas) {
  const int prev = g_max_ctas;
  g_max_ctas = ctas > 0 ? ctas : 0;
  return prev;
}

const char* edkm_status_string(int status) {
  switch (status) {
    case EDKM_OK: return "EDKM_OK";
    case EDKM_E_ARG: return "EDKM_E_ARG: invalid argument";
    case EDKM_E_DTYPE: return "EDKM_E_DTYPE: unsupported dtype";
    case EDKM_E_CUDA: return "EDKM_E_CUDA: CUDA error";
    case EDKM_E_UNSUPPORTED: return "EDKM_E_UNSUPPORTED: not implemented in this build";
    case EDKM_E_NCCL: return "EDKM_E_NCCL: NCCL error";
    default: return "unknown edkm_status";
  }
}

const char* edkm_last_error(void) { return g_err; }

}  // extern "C"
