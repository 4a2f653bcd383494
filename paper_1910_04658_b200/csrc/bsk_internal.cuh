// bsk_internal.cuh — launch interface between the C-ABI host layer (api.cu)
// and the sm_100a kernels (pi.cu, build.cu, pairs.cu). Product code only;
// shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

namespace bsk {

constexpr uint32_t kStatusIndex = 1u;   // latched: bad index / pi value / indptr

// Kernel-launch counter (binsketch_launch_count); every launch site calls count_launch().
void count_launch(uint64_t n = 1);
uint64_t launch_count();

// Device address of the latched status word (defined in build.cu).
unsigned int* status_ptr();

// 64-bit x mod N without a 64-bit division: q = umulhi(x, M), M = floor((2^64-1)/N),
// then at most two corrections. Bit-identical to x % N for 2 <= N < 2^32.
struct ModN {
  uint64_t M;
  uint32_t N;
  uint32_t mask;   // N-1 when N is a power of two (x mod N = x & mask), else 0
};
ModN make_modn(uint32_t N);

int num_sms();

cudaError_t launch_make_pi(uint64_t seed, uint64_t d, uint32_t N, uint32_t* pi, cudaStream_t s);

// pi == nullptr -> seeded (in-kernel pi); else table gather. parity: BCS (XOR) instead of OR.
cudaError_t launch_build(const uint32_t* pi, uint64_t seed, uint64_t d, uint32_t N,
                         const int64_t* indptr, const int32_t* indices, uint64_t n,
                         uint32_t* out, cudaStream_t s, bool parity = false);

cudaError_t launch_popcount(const uint32_t* sk, uint64_t n, uint32_t W, int32_t* out, cudaStream_t s);

// Categorical extension: label codes [n][c] + offsets[c+1] (device) -> one-hot CSR (n*c entries).
cudaError_t launch_onehot(const int32_t* codes, uint64_t n, uint32_t c, const int64_t* offsets, int64_t* indptr,
                          int32_t* indices, cudaStream_t s);

enum PairsMode { kAndPopc = 0, kEstimate = 1 };
// All-pairs kernel: A[na][W] x B[nb][W]. mode kAndPopc writes int32 out[na][nb];
// mode kEstimate reads pa/pb/L (device) and writes float planes.
// Estimate planes from a precomputed AND-popcount table pab[na][nb] (elementwise recipe kernel).
cudaError_t launch_estimate_from_pab(const int32_t* pab, uint64_t na, uint64_t nb, uint32_t N, uint32_t measure,
                                     const int32_t* pa, const int32_t* pb, const double* L, float* out, cudaStream_t s,
                                     bool bcs = false, double dcap = 0.0, double ham_scale = 1.0);
cudaError_t launch_pairs(int mode, const uint32_t* A, uint64_t na, const uint32_t* B, uint64_t nb,
                         uint32_t N, uint32_t measure, const int32_t* pa, const int32_t* pb,
                         const double* L, void* out, cudaStream_t s);

// Top-k: number of db splits chosen for (nq, ndb, k) (pure function).
uint32_t topk_splits(uint64_t nq, uint64_t ndb, uint32_t k);
// Merge `splits` partial top-k lists per query ([nq][splits][k], unsorted ok) into the final lists.
cudaError_t launch_topk_merge(uint64_t nq, uint32_t splits, uint32_t k, uint32_t measure, const double* part_key,
                              const int32_t* part_idx, int32_t* out_idx, float* out_score, cudaStream_t s);
cudaError_t launch_topk(const uint32_t* Q, uint64_t nq, const uint32_t* D, uint64_t ndb, uint32_t N,
                        uint32_t measure, uint32_t k, uint32_t flags, const int32_t* pq,
                        const int32_t* pd, const double* L, double* part_key, int32_t* part_idx,
                        int32_t* out_idx, float* out_score, cudaStream_t s,
                        const int32_t* pab = nullptr);   // pab[nq][ndb] precomputed (tensor cores) or null

// lcnt: [na][ceil(nb / 256)] at least; returns the db chunks (list segments) per row and the
// columns per chunk (segment sp of row r starts at lists[r * nb + sp * seg_cols]).
cudaError_t launch_tc_screen(const uint8_t* A8, uint64_t na, const uint8_t* B8, uint64_t nb, uint32_t N,
                             const int32_t* spb, const int32_t* perm, const uint16_t* tsuf, uint32_t nmp, uint2* lists,
                             uint32_t* lcnt, unsigned long long* ctr, uint32_t& splits, uint32_t& seg_cols,
                             cudaStream_t s);
// Top-k of every measure in `mask` from the pab table: sampled and screened histograms set an
// integer screen pab >= T[pb] (per-query minimum-pab tables), then the survivors are ranked
// exactly (K4c). pd_range: 2 int32 of workspace. Requires topk_pab3_fits and L
// non-decreasing on [0, N) (the keys' monotonicity in pab).
// scratch: topk_pab3_scratch_bytes(mask) of workspace (pass-2 survivors per block slot).
bool topk_pab3_fits(uint32_t N, uint32_t mask, uint32_t k);
size_t topk_pab3_scratch_bytes(uint32_t mask);
cudaError_t launch_topk_pab3(const int32_t* pab, uint64_t nq, uint64_t ndb, uint32_t N, uint32_t mask, uint32_t k,
                             uint32_t flags, const int32_t* pq, const int32_t* pd, const double* L, int32_t* pd_range,
                             void* scratch, int32_t* out_idx, float* out_score, cudaStream_t s);

// Fused-screen top-k (K4d): per query the sample threshold t_s and the suffix-min
// minimum-pab tables tsuf[nq][N + 1][nmp] (nmp = popcount(mask), 4 for 3) from the sample's
// AND-popcounts pab_s[nq][S] (the db rows [0, S) in their own order, popcounts pd[0, S));
// the tensor-core screen (launch_tc_screen) appends survivors to per-row lists; the list
// top-k ranks them exactly.
size_t screen_threshold_smem(uint32_t N, uint32_t nm, uint32_t S);
cudaError_t launch_screen_threshold(const int32_t* pab_s, uint64_t nq, uint32_t S, uint32_t N, uint32_t mask,
                                    uint32_t k, uint32_t flags, const int32_t* pq, const int32_t* pd, const double* L,
                                    const int32_t* pd_range, uint16_t* tsuf, double* ts, cudaStream_t s);
cudaError_t launch_topk_list(const uint2* lists, const uint32_t* lcnt, uint32_t splits, uint32_t seg_cols,
                             uint64_t nq, uint64_t ndb, uint32_t N,
                             uint32_t mask, uint32_t k, uint32_t flags, const int32_t* pq, const double* L,
                             const double* ts, void* scratch, int32_t* out_idx, float* out_score,
                             cudaStream_t s);   // lists: (original db index, |b_s| << 14 | pab); scratch: topk_pab3_scratch_bytes(15)
cudaError_t launch_int_range(const int32_t* x, uint64_t n, int32_t* out, cudaStream_t s);

// Tensor-core pair engine (tc.cu): sketches widened to {0,1} bytes, rows padded to
// tc_kpad(N) bytes (multiple of 128), then tcgen05 kind::i8 all-pairs.
uint32_t tc_kpad(uint32_t N);
// perm (optional): output row r is sketch perm[r].
cudaError_t launch_expand(const uint32_t* sk, uint64_t n, uint32_t N, uint8_t* out, cudaStream_t s,
                          const int32_t* perm = nullptr);
// ctr: one 8-byte device word of workspace (dynamic tile scheduler; reset by the launcher).
cudaError_t launch_tc_andpopc(const uint8_t* A8, uint64_t na, const uint8_t* B8, uint64_t nb, uint32_t N,
                              int32_t* out, unsigned long long* ctr, cudaStream_t s);
// bcs: BCS parity sketches, L = the BCS table, dcap = d (bcs_estimate_pair). ham_scale multiplies
// the fp64 Hamming estimate before rounding (0.5: categorical distance, exact power-of-two scaling).
cudaError_t launch_tc_estimate(const uint8_t* A8, uint64_t na, const uint8_t* B8, uint64_t nb, uint32_t N,
                               uint32_t measure, const int32_t* pa, const int32_t* pb, const double* L, float* out,
                               unsigned long long* ctr, cudaStream_t s, bool bcs = false, double dcap = 0.0,
                               double ham_scale = 1.0);
// Fused top-k on the tensor-core engine for k <= tc_topk_max_k(); partial lists
// [nq][tc_topk_splits][k] in the workspace, then the merge kernel. `prefilter` enables
// the integer L[pab] bound (valid when L is non-decreasing and convex).
uint32_t tc_topk_max_k();
uint32_t tc_topk_max_n();
bool tc_topk_fits(uint32_t N, uint32_t k);   // the fused kernel's shared memory fits (>= 2 stages)
uint32_t tc_topk_splits(uint64_t nq, uint64_t ndb, uint32_t N, uint32_t k);   // partial lists per query
// db order: counting sort by popcount, descending (perm: sorted position -> db row; spb:
// sorted popcounts; bins: N+1 words of scratch). Top-k uses it for N <= 65536 (tc_sortable).
bool tc_sortable(uint32_t N);
cudaError_t launch_sort_by_popcount(const int32_t* pb, uint64_t n, uint32_t N, uint32_t* bins, int32_t* perm,
                                    int32_t* spb, cudaStream_t s, bool descending = true);
// Q8 rows in `qperm` order and D8 rows in `perm` order (nullptr: original order); pq / pd the
// matching popcounts. Results land at the original query indices.
// tc_topk_packed_queries(N): the kernel widens the queries itself from the packed sketches Qsk
// (original order; Q8 is then not read and may be null); else Q8 holds the widened rows.
bool tc_topk_packed_queries(uint32_t N);
cudaError_t launch_tc_topk(const uint8_t* Q8, const uint32_t* Qsk, uint64_t nq, const uint8_t* D8, uint64_t ndb, uint32_t N,
                           uint32_t measure, uint32_t k, uint32_t flags, const int32_t* pq, const int32_t* qperm,
                           const int32_t* pd, const int32_t* perm, const double* L, bool prefilter, double* part_key,
                           int32_t* part_idx, int32_t* out_idx, float* out_score, unsigned long long* ctr,
                           unsigned int* done, int2* meta, cudaStream_t s);   // done: ceil(nq/128) words of workspace

// Threshold join on the tensor-core engine (Exp. 2): bits [nthr][nq][ceil(ndb/32)] (every word
// written by the kernel); tkey descending with tslot[t] its bitmap plane; db rows in their own
// order. exact: L unused, keys from exact_key.
uint32_t tc_join_max_thresholds();
cudaError_t launch_tc_join(const uint8_t* Q8, uint64_t nq, const uint8_t* D8, uint64_t ndb, uint32_t N,
                           uint32_t measure, const double* tkey, const uint32_t* tslot, uint32_t nthr, uint32_t flags,
                           bool exact, const int32_t* pq, const int32_t* pd, const double* L, uint32_t* bits,
                           unsigned long long* ctr, cudaStream_t s);
// join.cu: per-row counts (int32 scratch [nq]) -> row_ptr [nq+1]; list; confusion counts [3][nq].
cudaError_t launch_join_rowptr(const uint32_t* bits, uint64_t nq, uint64_t ndb, int32_t* counts, int64_t* row_ptr,
                               cudaStream_t s);
cudaError_t launch_join_list(const uint32_t* bits, uint64_t nq, uint64_t ndb, const uint32_t* Q, const uint32_t* D,
                             uint32_t N, const int32_t* pq, const int32_t* pd, const double* L, uint32_t measure,
                             bool exact, const int64_t* row_ptr, int32_t* out_j, float* out_score, uint64_t cap,
                             cudaStream_t s);
cudaError_t launch_join_confusion(const uint32_t* est, const uint32_t* tru, uint64_t nq, uint64_t ndb, int64_t* out,
                                  cudaStream_t s);
// Experiment 1: partial sums (mse_partial_bytes() of workspace, zeroed by the caller) over the
// row block [r0, r0 + rows) x all n rows (j > i) from its two AND-popcount tables [rows][n];
// thr: HOST double[nthr], nthr <= 16.
uint32_t mse_partial_bytes();
cudaError_t launch_mse_block(const int32_t* pab_s, const int32_t* pab_x, uint64_t r0, uint64_t rows, uint64_t n,
                             const int32_t* ps, const int32_t* px, const double* L, uint32_t N, double dcap,
                             uint32_t measure, bool bcs, const double* thr, uint32_t nthr, double* part_sse,
                             unsigned long long* part_cnt, cudaStream_t s);
cudaError_t launch_mse_final(const double* part_sse, const unsigned long long* part_cnt, uint32_t nthr, double* sse,
                             unsigned long long* cnt, cudaStream_t s);

}  // namespace bsk
