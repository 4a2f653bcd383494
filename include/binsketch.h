/* binsketch.h — C ABI of the B200-native BinSketch hot path (libbinsketch.so).
 *
 * Method: Pratap, Bera, Revanuru, "Efficient Sketching Algorithm for Sparse
 * Binary Data", arXiv 1910.04658. Line citations are PAPER.md
 * lines; SPEC.md lines where the paper is silent and SPEC's reading is
 * adopted (R-*).
 *
 * Conventions shared by every entry point
 * ----------------------------------------
 *  - Array arguments are DEVICE pointers owned by the caller (e.g. torch
 *    tensors), except where marked HOST. Inputs are read-only; outputs are
 *    fully overwritten (including padding slots).
 *  - Calls enqueue work on `stream` (a cudaStream_t; NULL = legacy default
 *    stream) and return without synchronising, except binsketch_device_status.
 *  - The library keeps no device allocations of its own apart from one
 *    4-byte latched device-status word; scratch memory comes from the caller's
 *    workspace (see binsketch_workspace_bytes). It keeps a host-side cache of
 *    cardinality tables keyed by (N, d), guarded by a mutex. Calls are pure
 *    functions of their inputs and may be issued from many host threads on
 *    different streams.
 *  - Sketch layout (reading R-G10): a sketch of N bits is W = ceil(N/32)
 *    uint32 words, bit j in word j/32 at bit position j%32 (LSB first); tail
 *    bits (j >= N) are 0; row r starts at word r*W (row stride W words).
 *  - Sparse binary rows are CSR: int64 indptr[n+1] (non-decreasing,
 *    indptr[0] arbitrary base), int32 indices[...] in [0,d). Duplicate or
 *    unsorted indices inside a row are allowed (OR is idempotent).
 *  - No exceptions cross the ABI. Host-detectable errors return immediately
 *    (nothing enqueued). Device-detectable input errors (index outside [0,d),
 *    pi value >= N, decreasing indptr) are latched into the device-status
 *    word and reported by binsketch_device_status; output contents are then
 *    unspecified. Zero-sized problems (n = 0, na*nb = 0, k = 0) succeed
 *    without enqueuing anything.
 *  - Determinism: outputs are bit-identical for identical inputs, independent
 *    of launch configuration.
 */
#ifndef BINSKETCH_H
#define BINSKETCH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* binsketch_stream_t; /* == cudaStream_t */

typedef enum {
  BINSKETCH_OK = 0,
  BINSKETCH_EINVAL = 1,     /* bad argument (N < 2, null pointer with nonzero count, bad measure, ...) */
  BINSKETCH_EINDEX = 2,     /* device-detected bad input (latched; see binsketch_device_status) */
  BINSKETCH_ECUDA = 3,      /* a CUDA runtime call failed */
  BINSKETCH_EWORKSPACE = 4, /* workspace too small */
  BINSKETCH_EUNSUPPORTED = 5 /* valid request outside this build's limits (e.g. k > BINSKETCH_MAX_K) */
} binsketch_status;

/* Measures (bit mask). Planes of binsketch_estimate are written in this order. */
enum {
  BINSKETCH_IP = 1,  /* inner product |a ∩ b|, Algorithm 1            */
  BINSKETCH_HAM = 2, /* Hamming |a|+|b|-2|a∩b|, Algorithm 2 (R-G2)      */
  BINSKETCH_JS = 4,  /* Jaccard, Algorithm 3 (R-G3)                    */
  BINSKETCH_COS = 8  /* cosine, Algorithm 4                            */
};

enum { BINSKETCH_TOPK_EXCLUDE_SELF = 1 };  /* topk / join flags: skip db row j == query row i */
enum { BINSKETCH_JOIN_EXCLUDE_SELF = 1,    /* join flags */
       BINSKETCH_JOIN_EXACT = 2 };         /* rows are uncompressed bit vectors: exact similarities */

enum { BINSKETCH_MAX_THRESHOLDS = 16 };    /* thresholds per binsketch_join call */

enum { BINSKETCH_MAX_K = 256 };            /* largest k binsketch_topk accepts */

/* Largest sketch length N accepted (larger values return BINSKETCH_EUNSUPPORTED):
 * construction and popcounts (make_pi, build*, bcs_build*, popcount) take every N >= 2 (their
 * sizes are computed in 64 bits; rows wider than 4096 words use a global-atomic fallback);
 * everything that stages the (N+1)-entry cardinality table (andpopc, estimate, topk, join*,
 * bcs_*, mse, categorical_estimate, card_table, workspace_bytes) up to 2^24 bits. */
#define BINSKETCH_MAX_N_BUILD 0xFFFFFFFFu
#define BINSKETCH_MAX_N_PAIRS 0x01000000u

/* ops for binsketch_workspace_bytes */
enum { BINSKETCH_OP_ANDPOPC = 1, BINSKETCH_OP_ESTIMATE = 2, BINSKETCH_OP_TOPK = 3, BINSKETCH_OP_JOIN = 4,
       BINSKETCH_OP_JOIN_LIST = 5, BINSKETCH_OP_BCS_ESTIMATE = 6,
       BINSKETCH_OP_MSE = 7 /* na = n rows, nb = d */ };

enum { BINSKETCH_MSE_BCS = 1 };            /* mse flags: sketches are BCS parity sketches */

/* W = ceil(N/32), words per sketch row. */
uint32_t binsketch_words(uint32_t N);

/* Theorem 1 sizing rule: N = psi*sqrt(psi/2*ln(2/rho)),
 * made an integer as max(2, ceil(.)) (reading R-G5).
 * Returns 0 on a domain error (psi = 0, rho not in (0,1)). Host only. */
uint32_t binsketch_recommended_N(uint32_t psi, double rho);

/* Random map pi:[d]->[N], generated on the device:
 *   pi[i] = mix64(seed + (i+1)*0x9E3779B97F4A7C15) mod N,   i in [0,d)
 * mix64 = splitmix64 finalizer (reading R-G8).
 * pi: device uint32[d]. EINVAL if N < 2 or (d > 0 and pi == NULL). */
binsketch_status binsketch_make_pi(uint64_t seed, uint64_t d, uint32_t N, uint32_t* pi,
                                   binsketch_stream_t stream);

/* Sketch construction, the BinSketch definition:
 *   out_words[r] bit j = OR over e in [indptr[r], indptr[r+1]) of [pi[indices[e]] == j]
 * pi: device uint32[d] (any table with values in [0,N));
 * indptr: device int64[n+1]; indices: device int32[indptr[n]-indptr[0]] addressed
 * by indptr's values; out_words: device uint32[n][W].
 * EINVAL: N < 2, d == 0 with n > 0, null pointer with n > 0.
 * Latched EINDEX: index outside [0,d), pi value >= N, indptr decreasing. */
binsketch_status binsketch_build(const uint32_t* pi, uint64_t d, uint32_t N, const int64_t* indptr,
                                 const int32_t* indices, uint64_t n, uint32_t* out_words,
                                 binsketch_stream_t stream);

/* Same result as binsketch_make_pi followed by binsketch_build, with pi(i)
 * evaluated in-kernel from (seed, i, N) instead of gathered from a table
 * (removes the random 4-byte gather per nonzero). */
binsketch_status binsketch_build_seeded(uint64_t seed, uint64_t d, uint32_t N, const int64_t* indptr,
                                        const int32_t* indices, uint64_t n, uint32_t* out_words,
                                        binsketch_stream_t stream);

/* Algorithm 1 line 1: out[r] = |sk[r]| (popcount).
 * sk: device uint32[n][W]; out: device int32[n]. */
binsketch_status binsketch_popcount(const uint32_t* sk, uint64_t n, uint32_t N, int32_t* out,
                                    binsketch_stream_t stream);

/* Algorithm 1 line 2: out[i][j] = |A[i] AND B[j]|, computed on the
 * tensor cores as the exact u8 dot product of the sketches widened to {0,1}
 * bytes (tcgen05.mma kind::i8, int32 accumulation; K10). From
 * 128*ceil(N/128) >= 4096 the engine runs CTA pairs (cta_group::2, clusters of
 * two); results are identical either way.
 * A: device uint32[na][W]; B: device uint32[nb][W]; out: device int32[na][nb].
 * ws: device workspace of ws_bytes >= binsketch_workspace_bytes(BINSKETCH_OP_ANDPOPC, ...). */
binsketch_status binsketch_andpopc(const uint32_t* A, uint64_t na, const uint32_t* B, uint64_t nb,
                                   uint32_t N, int32_t* out, void* ws, size_t ws_bytes,
                                   binsketch_stream_t stream);

/* All-pairs estimation from sketches alone (Algorithms 1-4)
 * by the canonical fp64 recipe (DESIGN.md R-C3): with pa = |a_s|, pb = |b_s|,
 * pab = |a_s AND b_s|, pu = pa+pb-pab and L[k] = log1p(-k/N)/log1p(-1/N)
 * (L[N] = d, saturation, R-G12):
 *   IP  = (pu == N && pa < N && pb < N) ? 0 : min(max(L[pa]+L[pb]-L[pu], 0), min(L[pa], L[pb]))
 *   HAM = min(max(S - 2 IP, 0), S),  S = L[pa]+L[pb]
 *   JS  = (pa == pb == 0) ? 1 : clamp(IP/(S-IP), 0, 1)
 *   COS = (pa == 0 || pb == 0) ? 0 : clamp(IP/sqrt(L[pa]L[pb]), 0, 1)
 * The L table is built on the host with the C library's log1p and uploaded.
 * measure: nonzero mask of BINSKETCH_{IP,HAM,JS,COS}; out: device
 * float[popcount(measure)][na][nb], planes in the order IP, HAM, JS, COS, each
 * value the fp64 result rounded to nearest float.
 * d: ambient dimension (saturation cap).
 * Engine (results identical either way): when na*nb*4 bytes fit the 4 GB table
 * budget, the tensor-core AND-popcount writes a pab table into the workspace and
 * an elementwise kernel evaluates the recipe (K10 estimate); otherwise
 * the fused tensor-core estimate (W > 32) or the CUDA-core LOP3+POPC kernel (K3). */
binsketch_status binsketch_estimate(const uint32_t* sketches_a, uint64_t na, const uint32_t* sketches_b,
                                    uint64_t nb, uint32_t N, uint64_t d, uint32_t measure, float* out,
                                    void* ws, size_t ws_bytes, binsketch_stream_t stream);

/* Query x database top-k (ranking; reading R-G17): for each
 * query i, the k database rows with the best estimate under one measure,
 * ordered by (key descending, db index ascending) where key = the estimate
 * (IP, JS, COS) or -HAM; the fp64 key is computed by the recipe above.
 * measure: a nonzero mask of BINSKETCH_* bits; with several bits the lists of each measure are
 * stacked in the order IP, HAM, JS, COS (out_idx / out_score: [popcount(measure)][nq][k]) and the
 * tensor-core AND-popcount table, when that engine is used, is computed once for all of them.
 * 1 <= k <= BINSKETCH_MAX_K (k = 0 is a no-op).
 * flags: BINSKETCH_TOPK_EXCLUDE_SELF skips j == i (self-join, R-G18).
 * out_idx: device int32[nq][k]; out_score: device float[nq][k] per measure (the measure's
 * value, not the key). Slots beyond the number of eligible db rows hold
 * idx = -1 and score = NaN.
 * Engine (results identical either way): k <= 64 and N <= 6143 (and the heaps fit shared
 * memory) — the fused tensor-core top-k (K10; per-row heaps in shared memory, db
 * popcount-sorted for the bound); otherwise, for N <= 16383, the fused tensor-core screen
 * (K4d: sample thresholds, the AND-popcount with an integer screen in its epilogue
 * writing survivor lists into the workspace, an exact list top-k), else the tensor-core
 * AND-popcount into a workspace table + the pab-table top-k (K4c / K4b); small calls (nq * ndb <=
 * 2^25) run the CUDA-core kernels (binsketch_topk_path names the path). The screen path runs
 * two independent branches on an internal stream forked from and joined back to `stream` with
 * events, so the call stays ordered on `stream` like every other call. */
binsketch_status binsketch_topk(const uint32_t* queries, uint64_t nq, const uint32_t* db, uint64_t ndb,
                                uint32_t N, uint64_t d, uint32_t measure, uint32_t k, uint32_t flags,
                                int32_t* out_idx, float* out_score, void* ws, size_t ws_bytes,
                                binsketch_stream_t stream);

/* Which kernel path binsketch_topk takes for these sizes († reporting / measurement: the bench
 * names the dominant kernel and its roofline from it; results are identical on every path).
 * Host-only, no device work. Returns BINSKETCH_PATH_NONE for an empty call,
 * BINSKETCH_PATH_TC_FUSED (the fused tensor-core top-k, K10), BINSKETCH_PATH_TC_SCREEN
 * (K4d), BINSKETCH_PATH_TC_PAB (K4c / K4b) or BINSKETCH_PATH_CUDA (the CUDA-core kernels: small
 * calls, nq * ndb <= 2^25, where the fused kernel has fewer tiles than SMs). */
enum { BINSKETCH_PATH_NONE = 0, BINSKETCH_PATH_TC_FUSED = 1, BINSKETCH_PATH_TC_SCREEN = 2,
       BINSKETCH_PATH_TC_PAB = 3, BINSKETCH_PATH_CUDA = 4 };
int binsketch_topk_path(uint64_t nq, uint64_t ndb, uint32_t N, uint64_t d, uint32_t k);

/* Threshold similarity join — the retrieval step of Experiment 2 (PAPER.md:690-700:
 * "compute the points in the training partition whose similarities are higher than a
 * certain threshold"; thresholds PAPER.md:697; reading R-J1). For each query i, db row j
 * and threshold t, bit j of row i of plane t is set iff key(i,j) >= key(t), where key is
 * the fp64 estimate of binsketch_topk (IP, JS, COS as is; -HAM for Hamming, so a Hamming
 * threshold selects distances <= t) and key(t) = t (-t for Hamming).
 * flags: BINSKETCH_JOIN_EXCLUDE_SELF skips j == i; BINSKETCH_JOIN_EXACT treats the rows as
 *   the UNCOMPRESSED binary vectors (e.g. built by binsketch_build with the identity map,
 *   N = d) and uses the exact similarities |a∩b|, |a|+|b|-2|a∩b|, |a∩b|/|a∪b|,
 *   |a∩b|/sqrt(|a||b|) (JS(∅,∅) = 1, COS with an empty side = 0) — Exp. 2's ground truth O.
 * thresholds: HOST double[nthr], 1 <= nthr <= BINSKETCH_MAX_THRESHOLDS, not NaN, any order.
 * measure: exactly one BINSKETCH_* bit. d: saturation cap (ignored with JOIN_EXACT).
 * out_bits: device uint32[nthr][nq][ceil(ndb/32)] (bit j%32 of word j/32, LSB first; tail
 *   bits 0), fully overwritten. The result is a set, so it is bit-identical run to run.
 * ws: >= binsketch_workspace_bytes(BINSKETCH_OP_JOIN, nq, ndb, N, 0).
 * Runs on the tensor-core engine (K11): AND-popcounts as in binsketch_andpopc,
 * a division-free necessary condition at the lowest threshold screens every pair, the
 * rest are scored exactly, and each output word is written once. */
binsketch_status binsketch_join(const uint32_t* queries, uint64_t nq, const uint32_t* db, uint64_t ndb,
                                uint32_t N, uint64_t d, uint32_t measure, const double* thresholds,
                                uint32_t nthr, uint32_t flags, uint32_t* out_bits, void* ws, size_t ws_bytes,
                                binsketch_stream_t stream);

/* Match list of one join plane (bits: device uint32[nq][ceil(ndb/32)], as written by
 * binsketch_join): row_ptr (device int64[nq+1]) = prefix sums of the per-query match
 * counts; for each query the matches in ascending db index: out_j (device int32[cap]) and
 * out_score (device float[cap]) = the measure's value (estimate, or exact with
 * BINSKETCH_JOIN_EXACT), recomputed from the rows. Entries at positions >= capacity are
 * counted in row_ptr but not written; capacity = 0 (out_j, out_score may be NULL) computes
 * row_ptr only. queries / db / N / d / measure / flags as for the binsketch_join call.
 * ws: >= binsketch_workspace_bytes(BINSKETCH_OP_JOIN_LIST, nq, ndb, N, 0). */
binsketch_status binsketch_join_list(const uint32_t* bits, const uint32_t* queries, uint64_t nq, const uint32_t* db,
                                     uint64_t ndb, uint32_t N, uint64_t d, uint32_t measure, uint32_t flags,
                                     int64_t* row_ptr, int32_t* out_j, float* out_score, uint64_t capacity,
                                     void* ws, size_t ws_bytes, binsketch_stream_t stream);

/* Experiment 2's per-query counts: for two join planes over the same
 * (nq, ndb) — O' = bits_est (from sketches), O = bits_true (exact) — out (device
 * int64[3][nq]) = |O'_i|, |O_i|, |O'_i ∩ O_i|. accuracy, precision, recall and F1 are
 * ratios of these (R-J2). */
binsketch_status binsketch_join_confusion(const uint32_t* bits_est, const uint32_t* bits_true, uint64_t nq,
                                          uint64_t ndb, int64_t* out, binsketch_stream_t stream);

/* BCS parity sketch (Definition 2; the paper's comparison sketch for IP,
 * HAM and JS): out_words[r] bit j = parity of the number of entries e of row r with
 * pi[indices[e]] == j (u_s[j] = sum_{i: b(i) = j} u[i] mod 2). Rows are sets in Definition 2;
 * a repeated index in a CSR row counts twice and cancels (reading R-B1). Arguments, layout,
 * errors and the pi table as for binsketch_build / binsketch_build_seeded (same map b = pi). */
binsketch_status binsketch_bcs_build(const uint32_t* pi, uint64_t d, uint32_t N, const int64_t* indptr,
                                     const int32_t* indices, uint64_t n, uint32_t* out_words,
                                     binsketch_stream_t stream);
binsketch_status binsketch_bcs_build_seeded(uint64_t seed, uint64_t d, uint32_t N, const int64_t* indptr,
                                            const int32_t* indices, uint64_t n, uint32_t* out_words,
                                            binsketch_stream_t stream);

/* All-pairs estimates from BCS sketches (readings R-B2, R-B3 — the paper defines the sketch,
 * not an estimator; SPEC.md:240-243's Hamming inversion, extended to |a| and so to IP/JS/COS):
 * with m = |a_s XOR b_s| = pa + pb - 2 pab and B[x] = log1p(-2x/N)/log1p(-2/N) (B[0] = 0,
 * B[x] = d once 2x >= N; see binsketch_bcs_table):
 *   HAM = min(B[m], d);  n_a = B[pa], n_b = B[pb];  S = n_a + n_b
 *   IP  = min(max((S - HAM)/2, 0), min(n_a, n_b))
 *   JS  = (pa == pb == 0) ? 1 : clamp(IP/(S-IP), 0, 1);  COS = (pa == 0 || pb == 0) ? 0 : clamp(IP/sqrt(n_a n_b), 0, 1)
 * in fp64 in this order, stored as float planes (IP, HAM, JS, COS order) like binsketch_estimate.
 * Tensor-core engine (pab as in binsketch_andpopc).
 * ws: >= binsketch_workspace_bytes(BINSKETCH_OP_BCS_ESTIMATE, na, nb, N, 0). */
binsketch_status binsketch_bcs_estimate(const uint32_t* sketches_a, uint64_t na, const uint32_t* sketches_b,
                                        uint64_t nb, uint32_t N, uint64_t d, uint32_t measure, float* out,
                                        void* ws, size_t ws_bytes, binsketch_stream_t stream);

/* The BCS table B (HOST double[N+1]) binsketch_bcs_estimate uploads. */
binsketch_status binsketch_bcs_table(uint32_t N, uint64_t d, double* host_out);

/* Experiment 1, fidelity of the estimate: over every unordered pair
 * i < j of one corpus whose EXACT similarity reaches threshold t ("pairs whose similarities
 * are higher than" t; reading R-M1: >= t, and for Hamming a distance <= t):
 *   out_count[t] = number of such pairs,  out_sse[t] = sum over them of (est - true)^2
 * so MSE = out_sse / out_count (the paper reports -ln MSE for JS / COS, MSE for IP).
 * est: binsketch_estimate's fp64 recipe from `sketches` (device uint32[n][W(N)]), or with
 *   BINSKETCH_MSE_BCS binsketch_bcs_estimate's from BCS sketches; true: exact similarity of
 *   `exact` (device uint32[n][W(d)], the uncompressed rows, e.g. binsketch_build with the
 *   identity map and N = d).
 * thresholds: HOST double[nthr], 1 <= nthr <= BINSKETCH_MAX_THRESHOLDS, not NaN.
 * out_sse: device double[nthr]; out_count: device uint64[nthr]. Sums are fp64 in a fixed
 * order (fixed grid, independent of the device), so results are bit-identical run to run.
 * Runs two tensor-core AND-popcount tables per block of 4096 rows and a fused reduction.
 * ws: >= binsketch_workspace_bytes(BINSKETCH_OP_MSE, n, d, N, 0). */
binsketch_status binsketch_mse(const uint32_t* sketches, const uint32_t* exact, uint64_t n, uint32_t N, uint64_t d,
                               uint32_t measure, const double* thresholds, uint32_t nthr, uint32_t flags,
                               double* out_sse, uint64_t* out_count, void* ws, size_t ws_bytes,
                               binsketch_stream_t stream);

/* Categorical extension: label-encoded features -> the one-hot binary rows
 * BinSketch compresses ("label-encoding followed by one-hot-encoding").
 * codes: device int32[n][c], codes[r][k] in [0, m_k); offsets: device int64[c+1], offsets[0] = 0,
 * offsets[k+1] - offsets[k] = m_k (so d = offsets[c]). Writes the CSR indptr (device int64[n+1],
 * indptr[r] = r*c) and indices (device int32[n*c], offsets[k] + codes[r][k]) for binsketch_build.
 * Latched EINDEX: a code outside [0, m_k) or an index >= 2^31 (the entry is then offsets[k]). */
binsketch_status binsketch_onehot(const int32_t* codes, uint64_t n, uint32_t c, const int64_t* offsets,
                                  int64_t* indptr, int32_t* indices, binsketch_stream_t stream);

/* Estimated categorical distance D(u,v) = #{k : u[k] != v[k]} from the one-hot
 * rows' sketches: D^ = HAM^/2 with HAM^ the Hamming estimate of binsketch_estimate (the one-hot
 * Hamming distance is exactly 2 D; reading R-C1, SPEC.md:307 — the paper writes "equal").
 * out: device float[na][nb] = (float)(HAM^ * 0.5). ws: >= binsketch_workspace_bytes(
 * BINSKETCH_OP_BCS_ESTIMATE, na, nb, N, 0) (the tensor-core estimate layout). */
binsketch_status binsketch_categorical_estimate(const uint32_t* sketches_a, uint64_t na, const uint32_t* sketches_b,
                                                uint64_t nb, uint32_t N, uint64_t d, float* out, void* ws,
                                                size_t ws_bytes, binsketch_stream_t stream);

/* Workspace bytes needed by op (BINSKETCH_OP_*) for na (queries) x nb (db)
 * rows of N-bit sketches and top-k size k (ignored for other ops). Pure
 * function of its arguments (and of the BINSKETCH_ENGINE=cuda|tc A/B override,
 * which must not change between this call and the op). The tensor-core
 * engine's scratch (K10) dominates: the sketches widened to {0,1}
 * bytes, (na + nb) x 128*ceil(N/128) bytes, plus top-k partial lists and the
 * fused top-k's per-tile db metadata (8 bytes per db row, padded to 256 rows). */
size_t binsketch_workspace_bytes(int op, uint64_t na, uint64_t nb, uint32_t N, uint32_t k);

/* The cardinality table the library uploads (Alg. 1 line 3):
 * host_out[0..N] = L (HOST double[N+1]). For byte-level parity checks. */
binsketch_status binsketch_card_table(uint32_t N, uint64_t d, double* host_out);

/* Synchronises `stream`, returns BINSKETCH_EINDEX if a device-side input
 * error was latched since the last call (and clears it), ECUDA on a CUDA
 * error, else OK. The status word is per device: this reports (and clears)
 * the errors of calls made while the current CUDA device was the same. */
binsketch_status binsketch_device_status(binsketch_stream_t stream);

/* Number of kernels this library has enqueued since it was loaded (all
 * threads, all streams; atomic counter). Used by the bench to report
 * gpu_launches. Host only. */
uint64_t binsketch_launch_count(void);

/* Static string for a status code. */
const char* binsketch_strerror(binsketch_status status);

#ifdef __cplusplus
}
#endif

#endif /* BINSKETCH_H */
