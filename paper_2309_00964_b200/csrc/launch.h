// launch.h -- internal launcher declarations shared by the .cu files of libedkm.
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include "../../include/edkm.h"
#include "common.cuh"

typedef struct edkm_comm edkm_comm;

namespace edkm {

// ---- error text / launch count of the calling thread (api.cu), used by every entry point
edkm_status set_error(edkm_status st, const char* msg);
void reset_launches();
void add_launches(int n);
// NVTX range around an entry point's launches (SURVEY S5 tracing): nsys / ncu --nvtx show each
// kernel and collective of the step under its phase name.  Header-only NVTX v3: a no-op unless a
// tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define EDKM_NVTX(name) ::edkm::NvtxRange edkm_nvtx_range_(name)
// in-place sum all-reduce over the library's NCCL communicator (exchange.cu); comm == NULL: no-op
edkm_status comm_allreduce_sum(edkm_comm* comm, void* buf, size_t count, int fp64, cudaStream_t s);

// ---- per-tensor forward state kept in `saved`
constexpr int kMaxCluster = 8;
constexpr int kWinPagesB = 55;    // magnitude pages per sign kept in shared memory by B1 (8 B/pattern) and B2 (float2)
constexpr int kWinPagesF2 = 110;  // F2 with fp32 output (4 B/pattern)
struct TensorState {
  int32_t T;                       // centroid updates run
  int32_t cl;                      // CTAs per tensor in the table phase (row partitions)
  int32_t pbase[kMaxCluster + 1];  // partition p = patterns [pbase[p], pbase[p+1]) (16-aligned, row-balanced)
  int32_t nrows[kMaxCluster];      // populated finite patterns, per partition (stored at rows[pbase[p]...])
  uint8_t win[4];                  // magnitude-page windows of the per-weight kernels (TF, once per
                                   // tensor): B1/B2 (pbase, np), F2 fp32 output (pbase, np)
  int64_t nonfinite[kMaxCluster];  // NaN/Inf weights counted, per partition
};
static_assert(sizeof(TensorState) == 144, "TensorState layout");

struct SavedLayout {
  size_t state, ctraj, straj, rows, table16, idx8, page_cnt, total;
};
struct WsLayout {
  size_t B, psi, phipsi, gamma, total;
};
SavedLayout saved_layout(int nt, int k, int max_iter);
WsLayout ws_layout(int nt, int k);

// F2 mode: 0 soft 16-bit, 1 hard-value 16-bit, 2 soft fp32, 3 hard-value fp32, 4 hard index u8
struct F2Args {
  const float* table;       // [nt][65536] fp32 W~ per pattern
  const uint16_t* table16;  // [nt][65536] W~ rounded to the weights' dtype
  const uint8_t* idx8;      // [nt][65536] hard index per pattern
  const float* C;           // [nt][k] C_out
  const TensorState* state; // [nt]: the magnitude-page windows
  int k;
};
struct B1Args {
  double* B;                // [nt][65536] fp64, zeroed by the caller
  const TensorState* state; // [nt]: the magnitude-page windows
};
struct B2Args {
  const float2* phipsi;     // [nt][65536] (phi, psi) per pattern
  const TensorState* state; // [nt]: the magnitude-page windows
};
cudaError_t launch_f1(const StreamArgs& A, int32_t* counts, int sms, cudaStream_t s);
void nvls_set_timeout(double seconds, int trap);
cudaError_t nvls_failed(int* failed);
cudaError_t launch_f1_nvls(const StreamArgs& A, int32_t* counts_mc, uint32_t* flags_mc, const uint32_t* flags,
                           uint32_t* epoch, int nranks, int emulate, int sms, cudaStream_t s);
cudaError_t launch_f2(const StreamArgs& A, const F2Args& F, int mode, int sms, cudaStream_t s);
cudaError_t launch_b1(const StreamArgs& A, const B1Args& B, int sms, cudaStream_t s);
cudaError_t launch_b2(const StreamArgs& A, const B2Args& B, int sms, cudaStream_t s);

// ---- table phase
struct TableArgs {
  int nt, k, wdtype, max_iter, cl;
  int layout_only;         // TF: rows, partitions, page masses, windows only (no iterations, no tables)
  double tau, inv_tau, eps;
  const int32_t* counts;   // [nt][65536]
  const float* C0;         // [nt][k]
  float* C_out;            // [nt][k]
  float* table;            // [nt][65536]
  TensorState* state;      // [nt]
  double* ctraj;           // [nt][(max_iter+1)*k]
  double* straj;           // [nt][max(max_iter,1)*k]
  uint16_t* rows;          // [nt][65536] populated finite patterns, by partition
  uint16_t* table16;       // [nt][65536]
  uint8_t* idx8;           // [nt][65536]
  int64_t* page_cnt;       // [nt][256]
  const double* B;         // [nt][65536] gradient buckets
  double* psi;             // [nt][65536] per-row psi accumulator
  float2* phipsi;          // [nt][65536]
  double* gamma;           // [nt][k]
  float* dC0;              // [nt][k]
};
int table_cluster_size(int nt, int wdtype);
cudaError_t launch_tf(const TableArgs& P, cudaStream_t s);
cudaError_t launch_tgamma(const TableArgs& P, cudaStream_t s);
cudaError_t launch_tb(const TableArgs& P, cudaStream_t s);
// k = 32..256 (bits 5..8): warp-per-row variants (table_wide.cu)
cudaError_t launch_tf_wide(const TableArgs& P, cudaStream_t s);
cudaError_t launch_tgamma_wide(const TableArgs& P, cudaStream_t s);
cudaError_t launch_tb_wide(const TableArgs& P, cudaStream_t s);

}  // namespace edkm
