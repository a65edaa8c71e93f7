/*
 * edkm.h -- C ABI of libedkm.so: the eDKM hot path (arXiv 2309.00964) on B200.
 *
 * What the path computes (PAPER.md = /root/reference/PAPER.md, "P:<line>"):
 *   DKM weight clustering (P:31-39 S2, Fig. 1; formulas per the north star,
 *   DESIGN.md R1-R6):  attention A[i][j] = softmax_j(-(w_i - C[j])^2 / tau) over
 *   k = 2^b centroids, soft-centroid update C[j] <- sum_i A[i][j] w_i / sum_i A[i][j]
 *   iterated T times, reconstruction W~ = A . C, and the backward pass to dW and
 *   dC_0 through all unrolled iterations.
 *   Every step is evaluated on the <= 65,536 distinct 16-bit patterns of each
 *   weight tensor (uniquification, P:77 S2.2; Fig. 3): the attention map
 *   becomes a table with one row per pattern, and the index of weight i is its
 *   own bit pattern ("the 16bit value ... can serve as an offset"), so the
 *   index list is W's bytes reinterpreted as uint16 -- no copy is made.
 *   Sharding over learners = each rank passes its contiguous slice of each
 *   tensor; the caller sums `counts` (after edkm_uniquify) and `gamma`
 *   (after edkm_backward_reduce) over ranks, see edkm_backward().
 *
 * Conventions for every entry point:
 *   - Device pointers unless stated.  The caller owns every buffer; the library
 *     allocates no device memory (except the edkm_mc_* NVLS buffers, on request) and
 *     keeps no state between calls.
 *   - Asynchronous on `stream` (a cudaStream_t passed as void*, NULL = legacy
 *     default stream).  No call synchronises the host except edkm_read_status.
 *   - Argument errors (null pointers with n > 0, bad dtype, bits outside 1..8,
 *     tau <= 0 or non-finite, max_iter < 0, eps < 0 or NaN, nt < 0, n < 0) are
 *     returned before anything is launched and have no side effects.
 *   - Launch failures return EDKM_E_CUDA; edkm_last_error() gives the text.
 *   - Data errors (NaN/Inf weight patterns) are not returned, since detecting
 *     them needs a host sync: they are counted into `saved` (edkm_read_status),
 *     excluded from clustering, and their outputs are NaN.
 *   - All tensors of one call share dtype, bits, tau, max_iter and eps.
 */
#ifndef EDKM_H_
#define EDKM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    EDKM_OK = 0,
    EDKM_E_ARG = 1,          /* invalid argument (nothing launched)            */
    EDKM_E_DTYPE = 2,        /* unsupported dtype for this argument            */
    EDKM_E_CUDA = 3,         /* a CUDA launch or API call failed               */
    EDKM_E_UNSUPPORTED = 4   /* valid request this build does not implement  */
} edkm_status;

typedef enum { EDKM_BF16 = 0, EDKM_FP16 = 1, EDKM_FP32 = 2, EDKM_U8 = 3 } edkm_dtype;

typedef enum {
    EDKM_SOFT = 0,        /* W~_i = table[bits(w_i)] (Fig. 1)                        */
    EDKM_HARD_VALUE = 1,  /* W^hard_i = C_out[idx(bits(w_i))], the palettised weight  */
    EDKM_HARD_INDEX = 2   /* idx_i as uint8: "a list of low-precision indices"        */
} edkm_recon_mode;

/* One weight tensor, or this rank's contiguous slice of it.  `w` holds n
 * 16-bit weights (bf16 or fp16 per edkm_params.wdtype); its bytes ARE the index
 * list.  n may be 0 (w may then be NULL). */
typedef struct {
    const void* w;
    int64_t n;
} edkm_tensor;

typedef struct {
    int wdtype;    /* EDKM_BF16 or EDKM_FP16: the weights' 16-bit format   */
    int bits;      /* b, 1..8; k = 2^b centroids (8-bit embeddings P:91)    */
    double tau;    /* softmax temperature, > 0 and finite                         */
    int max_iter;  /* >= 0: number of centroid updates when eps == 0 (DESIGN R3)   */
    double eps;    /* >= 0; if > 0 stop once max_j |C_{t+1}[j]-C_t[j]| <= eps (R4) */
} edkm_params;

/* Bytes of the forward state `saved` (centroid/denominator trajectories,
 * compacted pattern rows, 16-bit and index tables, status) for nt tensors.
 * Returns 0 for invalid params. */
size_t edkm_saved_bytes(int nt, const edkm_params* p);

/* Bytes of the backward scratch `ws` (fp64 gradient buckets, per-row state,
 * (phi, psi) table, gamma) for nt tensors.  Returns 0 for invalid params. */
size_t edkm_workspace_bytes(int nt, const edkm_params* p);

/* F1 -- uniquify.  counts[t*65536 + u] = #{i : bits(w_i) = u} over
 * this rank's slice of tensor t.  counts (int32, [nt][65536]) is overwritten.
 * Exact (integer).  With several ranks the caller sums counts over ranks
 * (integer all-reduce) before edkm_forward. */
edkm_status edkm_uniquify(const edkm_tensor* tensors, int nt, int wdtype, int32_t* counts, void* stream);

/* F1 fused with the cross-rank sum of the counts over NVLink SHARP (NVLS) -- the in-kernel
 * form of the integer all-reduce after edkm_uniquify (P:79 learners).
 * Every buffer below is one symmetric allocation mapped on all ranks (e.g. torch symmetric
 * memory); `*_mc` are its multicast addresses: a reduction issued there is applied by the
 * NVSwitch to every rank's copy.
 *   counts_mc : multicast address of an int32 [nt][65536] buffer that is ZERO on every rank
 *               before any rank makes this call (callers alternate two buffers and zero the
 *               one of the next step before this call, so a fast rank cannot add into a copy
 *               that a slow rank has yet to clear).
 *   flags_mc / flags : multicast / local address of EDKM_NVLS_FLAGS uint32 arrival counters,
 *               zero-initialised once; never reset (monotonic).
 *   epoch     : this rank's device step counter (uint32, zero-initialised once, plain memory).
 * F1 runs on exactly the SM count of CTAs on every rank (all ranks: the same GPU model and the
 * same nt), each flushing its counts with multimem.red and then signalling its counter
 * (release, system scope); a one-CTA wait kernel then blocks the stream until every counter
 * reached nranks x epoch (acquire).  After it, the local view of the buffer holds the global
 * counts on every rank -- exact (integer).  No host synchronisation.  Requires NVLS multicast
 * support; callers without it use edkm_uniquify + an all-reduce.
 *   emulate   : 1 = the same protocol on ordinary device memory with plain atomics (nranks
 *               must be 1; `*_mc` are then the buffers themselves) -- for testing the
 *               protocol on a system without multicast.  0 otherwise. */
#define EDKM_NVLS_FLAGS 1024
typedef struct {
    int32_t* counts_mc;
    uint32_t* flags_mc;
    const uint32_t* flags;
    uint32_t* epoch;
    int nranks;
    int emulate;
} edkm_nvls;
edkm_status edkm_uniquify_nvls(const edkm_tensor* tensors, int nt, int wdtype, const edkm_nvls* nvls, void* stream);

/* Timeout of edkm_uniquify_nvls's arrival barrier (host-side setting for later calls; default
 * 20 s with trap = 1: a timed-out wait traps -- the process fails loudly instead of hanging).
 * trap = 0: a timed-out wait records the failure and the stream continues (the counts are then
 * wrong) -- for a first call that checks whether the NVLS exchange works at all and falls back
 * to edkm_uniquify + an all-reduce if not.  EDKM_E_ARG if seconds <= 0 or NaN. */
edkm_status edkm_nvls_set_timeout(double seconds, int trap);

/* *failed = 1 if a non-trapping NVLS wait timed out since the last call (then clears it).
 * Synchronous (reads a device flag of the current device).  EDKM_E_ARG if failed is NULL. */
edkm_status edkm_nvls_failed(int* failed);

/* NVLS multicast buffers backing edkm_nvls (driver-API plumbing; no compute).
 *   edkm_mc_supported : *supported = 1 if the current device supports multicast objects.
 *   edkm_mc_create    : rank 0 -- a multicast object of >= bytes for nranks GPUs (size rounded
 *                       up to the multicast granularity, see edkm_mc_bytes); with export_fd it
 *                       also returns a POSIX file descriptor to pass to the other ranks.
 *   edkm_mc_import    : other ranks -- the object from that descriptor (dup'ed into this
 *                       process), bytes = edkm_mc_bytes of rank 0's object.
 *   edkm_mc_add_device: every rank, for its current device; all ranks must have added their
 *                       device before any rank calls edkm_mc_bind (a barrier in between).
 *   edkm_mc_bind      : backs the object with this rank's device memory and maps the unicast
 *                       (*local_out) and multicast (*mc_out) views, both bytes long.
 *   edkm_mc_destroy   : unmaps and releases (after all use; ranks tear down independently).
 * The library owns nothing else; these are the only calls that allocate device memory. */
typedef struct edkm_mcbuf edkm_mcbuf;
edkm_status edkm_mc_supported(int* supported);
edkm_status edkm_mc_create(size_t bytes, int nranks, int export_fd, int* fd_out, edkm_mcbuf** out);
edkm_status edkm_mc_import(int fd, size_t bytes, edkm_mcbuf** out);
size_t edkm_mc_bytes(const edkm_mcbuf* buf);
edkm_status edkm_mc_add_device(edkm_mcbuf* buf);
edkm_status edkm_mc_bind(edkm_mcbuf* buf, void** local_out, void** mc_out);
edkm_status edkm_mc_destroy(edkm_mcbuf* buf);
const char* edkm_mc_last_error(void);

/* TF -- forward table phase (DKM iterations on the attention table).
 *   counts : [nt][65536] int32, global over ranks.
 *   C0     : [nt][k] fp32 initial centroids.
 *   C_out  : [nt][k] fp32 = C_T, the lookup table of the palettised weight.
 *   table  : [nt][65536] fp32, table[u] = sum_j A(v_u, C_T)[j] C_T[j] (DESIGN R2) for
 *            every pattern with counts > 0; NaN for the others.
 *   saved  : edkm_saved_bytes(nt, p) bytes, consumed by reconstruct/backward.
 * The loop runs in fp64; results are identical on every rank given equal counts. */
edkm_status edkm_forward(const int32_t* counts, int nt, const edkm_params* p, const float* C0, float* C_out,
                         float* table, void* saved, void* stream);

/* TF for tensors [t0, t1) of an nt-tensor call only (same buffers, same layout as edkm_forward,
 * which is the range [0, nt)).  Lets ranks split the table phase by tensor (each rank runs TF
 * for its own block, then the ranks exchange the per-tensor results, see edkm_layout) instead of
 * all running it for every tensor.  Entries of other tensors are not touched. */
edkm_status edkm_forward_range(const int32_t* counts, int nt, int t0, int t1, const edkm_params* p, const float* C0,
                               float* C_out, float* table, void* saved, void* stream);

/* Byte offsets of the arrays inside `saved` and `ws` for nt tensors (for exchanging per-tensor
 * blocks between ranks).  Each array is [nt][per-tensor entries], tensor-major.
 *   saved_offs[8] : TensorState (144 B/tensor), C trajectory (fp64 (max_iter+1)k), S trajectory
 *                   (fp64 max(max_iter,1)k), rows (u16 65536), table16 (u16 65536), idx8 (u8
 *                   65536), page_cnt (i64 256), total.
 *   ws_offs[5]    : B (fp64 65536), psi (fp64 65536), (phi, psi) (float2 65536), gamma (fp64 k),
 *                   total.  Either pointer may be NULL. */
edkm_status edkm_layout(int nt, const edkm_params* p, size_t* saved_offs, size_t* ws_offs);

/* F2 -- reconstruct this rank's slice of each tensor (Fig. 1, "look-up").
 *   table, C_out : the outputs of edkm_forward (table is read only by EDKM_SOFT with
 *                  FP32 output, C_out only by EDKM_HARD_VALUE; the other may be NULL).
 *   out[t] : n_t elements of out_dtype.
 *   EDKM_SOFT:        out_dtype FP32 (table entry), or the weights' own 16-bit dtype
 *                     (round-to-nearest-even from the fp64 value).
 *   EDKM_HARD_VALUE:  out_dtype FP32 or the weights' 16-bit dtype; value C_out[idx].
 *   EDKM_HARD_INDEX:  out_dtype U8; idx = argmin_j (v - C_out[j])^2, lowest j on ties,
 *                     distances in fp64 from the fp32 C_out values (DESIGN R9). */
edkm_status edkm_reconstruct(const edkm_tensor* tensors, int nt, const edkm_params* p, const float* table,
                             const float* C_out, const void* saved, int mode, int out_dtype, void* const* out,
                             void* stream);

/* B1 -- gradient buckets and this rank's partial of gamma_T (DESIGN App. A):
 *   B[u] = sum_{i in slice, bits(w_i)=u} G_i  (64-bit fixed point per CTA, fp64 across CTAs)
 *   gamma[t*k + l] = sum_u B[u] A_T[u][l] (1 + (C_T[l] - W~_u) 2(v_u - C_T[l]) / tau)
 *   grads[t] : n_t elements, gdtype = weights' 16-bit dtype or FP32.
 *   gamma    : [nt][k] fp64, overwritten.  With several ranks the caller sums gamma
 *              over ranks before edkm_backward_apply. */
edkm_status edkm_backward_reduce(const edkm_tensor* tensors, int nt, const edkm_params* p,
                                 const void* const* grads, int gdtype, const int32_t* counts,
                                 const void* saved, void* ws, double* gamma, void* stream);

/* TB + B2 -- reverse loop on the table and dW (DESIGN App. A):
 *   dW_i = G_i phi[u_i] + psi[u_i];  dC0[t*k + l] = dL/dC_0 (fp32, identical on all ranks).
 *   gamma : [nt][k] fp64, global (summed over ranks).
 *   dW[t] : n_t elements of dw_dtype (FP32, or the weights' 16-bit dtype). */
edkm_status edkm_backward_apply(const edkm_tensor* tensors, int nt, const edkm_params* p,
                                const void* const* grads, int gdtype, const int32_t* counts,
                                const void* saved, void* ws, const double* gamma, void* const* dW,
                                int dw_dtype, float* dC0, void* stream);

/* The four kernels of the two calls above, individually (same semantics; for overlap or
 * per-kernel timing):
 *   edkm_backward_buckets : B1     -- ws buckets B[u] of this rank's slice (zeroed first)
 *   edkm_backward_gamma   : TGAMMA -- gamma (this rank's partial) from the buckets
 *   edkm_backward_table   : TB     -- (phi, psi) per pattern into ws, dC0, from the global gamma
 *   edkm_backward_dw      : B2     -- dW from (phi, psi) */
edkm_status edkm_backward_buckets(const edkm_tensor* tensors, int nt, const edkm_params* p,
                                  const void* const* grads, int gdtype, const void* saved, void* ws, void* stream);
edkm_status edkm_backward_gamma(int nt, const edkm_params* p, const int32_t* counts, const void* saved, void* ws,
                                double* gamma, void* stream);
edkm_status edkm_backward_table(int nt, const edkm_params* p, const int32_t* counts, const void* saved, void* ws,
                                const double* gamma, float* dC0, void* stream);
edkm_status edkm_backward_dw(const edkm_tensor* tensors, int nt, const edkm_params* p, const void* const* grads,
                             int gdtype, const void* saved, const void* ws, void* const* dW, int dw_dtype,
                             void* stream);

/* TB for tensors [t0, t1) only (see edkm_forward_range): (phi, psi) and dC0 of those tensors,
 * from the global gamma.  Requires TF to have run for the same range on this rank. */
edkm_status edkm_backward_table_range(int nt, int t0, int t1, const edkm_params* p, const int32_t* counts,
                                      const void* saved, void* ws, const double* gamma, float* dC0, void* stream);

/* Single-process convenience: edkm_backward_reduce then edkm_backward_apply with
 * `gamma` in ws.  Only valid when one process holds every weight of each tensor. */
edkm_status edkm_backward(const edkm_tensor* tensors, int nt, const edkm_params* p, const void* const* grads,
                          int gdtype, const int32_t* counts, const void* saved, void* ws, void* const* dW,
                          int dw_dtype, float* dC0, void* stream);

/* Copies per-tensor status to host and synchronises `stream`:
 *   nonfinite_host[t] = number of weights of tensor t whose pattern is NaN/Inf (global),
 *   iters_host[t]     = T, the number of centroid updates run.  Either may be NULL. */
edkm_status edkm_read_status(const void* saved, int nt, const edkm_params* p, int64_t* nonfinite_host,
                             int32_t* iters_host, void* stream);

/* Caps the grid of the per-weight streaming kernels (F1, F2, B1, B2; one 1024-thread CTA per
 * SM) launched by later calls on the calling thread at `ctas` CTAs, so that two calls on
 * different streams can run side by side on disjoint SMs; ctas <= 0 restores the default
 * (the SM count).  Results do not depend on it.  Returns the previous cap (0 = none). */
int edkm_set_max_ctas(int ctas);

/* Number of kernels the last successful entry point launched on the calling thread. */
int edkm_last_launch_count(void);
const char* edkm_status_string(int status);
const char* edkm_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* EDKM_H_ */
