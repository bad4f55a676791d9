/*
 * krp.h — C ABI of the B200-native Khatri-Rao random-projection (KRP) sketch
 * library (libkrp.so) for randomized HOSVD / STHOSVD, arXiv 2507.23207.
 *
 * The hot path is the MTTKRP sketch of a dense d-way tensor against Gaussian
 * factors (Alg. 7 line 3; memoized form P:571-574):
 *
 *     Y_n = X_(n) (Omega_d ⊙ ... ⊙ Omega_{n+1} ⊙ Omega_{n-1} ⊙ ... ⊙ Omega_1)
 *
 * Conventions for every entry point
 * ---------------------------------
 * - X is fp32, first-index-fastest: element (i_1..i_d) (0-based) lives at
 *   offset sum_k i_k * prod_{m<k} I_m (the same bytes as a
 *   C-contiguous array of shape (I_d, ..., I_1)).  The mode-n unfolding X_(n)
 *   takes its columns in that order with mode n removed, which is the
 *   row order of the Khatri-Rao product above (reading R1 in DESIGN.md).
 * - Omega_k is fp32, row-major I_k x R (element (i, r) at i*R + r).
 * - Y_n, Q_n are fp32 row-major I_n x R (resp. I_n x r_n).
 * - The core G is fp32, first-index-fastest, dims (r_1..r_d).
 * - Unless a name ends in _host, every array pointer is a DEVICE pointer owned
 *   by the caller; the library never frees or retains it past the call.  Arrays
 *   of pointers (omega, Y, Q) are HOST arrays of d device pointers.
 * - `stream` is a cudaStream_t (NULL = legacy default stream).  Work is
 *   enqueued on it; results are stream-ordered.  Functions that return a host
 *   scalar (rel_err) synchronize the stream before returning.
 * - `ws`/`ws_bytes`: device workspace of at least krp_workspace_bytes(...)
 *   bytes, 256-byte aligned.  ws == NULL makes the library allocate (and free)
 *   the workspace itself with stream-ordered cudaMallocAsync.
 * - Results are deterministic for a fixed configuration and device: every
 *   cross-block sum is a fixed-order reduction (no floating-point atomics).
 *
 * Errors: every function returns a krp_status.  Arguments are validated before
 * anything is launched; on error, outputs are unspecified.  krp_status_string()
 * gives a description; krp_last_error_message() gives details of the last error
 * on the calling thread.  No C++ exception crosses this boundary.
 */
#ifndef KRP_H_
#define KRP_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__) || defined(__clang__)
#define KRP_API __attribute__((visibility("default")))
#else
#define KRP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum krp_status {
  KRP_OK = 0,
  KRP_EINVAL = 1,       /* null pointer, d not in [2,8], R not in [1,256] (rhosvd/sthosvd: [1,64]), dim < 1,
                           n out of range */
  KRP_ESHAPE = 2,       /* r_n > R, R > min(I_n, N/I_n), inconsistent slab geometry */
  KRP_ECUDA = 3,        /* a CUDA runtime / launch error */
  KRP_ENCCL = 4,        /* NCCL unavailable or a collective failed */
  KRP_ENUMERIC = 5,     /* CholeskyQR failed even after the shifted fallback */
  KRP_ENOMEM = 6,       /* ws_bytes < krp_workspace_bytes(...) or allocation failed */
  KRP_EUNSUPPORTED = 7  /* the device is not sm_100a (B200): the library has no other code path */
} krp_status;

/* op codes for krp_workspace_bytes */
enum {
  KRP_OP_SKETCH_ALL = 0,
  KRP_OP_SKETCH_MODE = 1,
  KRP_OP_RHOSVD = 2,
  KRP_OP_STHOSVD = 3,
  KRP_OP_SKETCH_ALL_HOST = 4, /* krp_sketch_all_modes_host: includes device copies of X, Omega, Y */
  KRP_OP_RHOSVD_ERR = 5,      /* krp_rhosvd with rel_err != NULL */
  KRP_OP_RHOSVD_FRESH = 6,    /* krp_rhosvd_fresh (rel_err buffers included) */
  KRP_OP_RHOSVD_GAUSSIAN = 7, /* krp_rhosvd_gaussian (includes the explicit unfolding buffer) */
  KRP_OP_STHOSVD_GAUSSIAN = 8, /* krp_sthosvd_gaussian */
  KRP_OP_TTM = 9               /* krp_ttm: pass J as R (only mode n = 0 takes workspace) */
};

KRP_API const char* krp_status_string(int status);
KRP_API const char* krp_last_error_message(void);
KRP_API int krp_version(void);

/* Workspace size in bytes for `op` (one of KRP_OP_*).  ranks may be NULL for the sketch ops. */
KRP_API size_t krp_workspace_bytes(int op, int d, const int64_t* dims, int R, const int* ranks);

/* All-mode memoized sketch: one shared set {Omega_k}, every Y_n.
 * omega[k]: I_k x R; Y[n]: I_n x R (outputs).  Algorithmic work 4*N*R flops. */
KRP_API int krp_sketch_all_modes(const float* X, int d, const int64_t* dims, const float* const* omega, int R,
                         float* const* Y, void* ws, size_t ws_bytes, void* stream);

/* Same, with HOST buffers (X, omega[k], Y[n] in host memory, ideally pinned): copies
 * host->device, sketches, copies device->host, all on `stream`, and synchronizes.
 * ws must hold krp_workspace_bytes(KRP_OP_SKETCH_ALL_HOST, ...) bytes (or be NULL). */
KRP_API int krp_sketch_all_modes_host(const float* X_host, int d, const int64_t* dims, const float* const* omega_host,
                              int R, float* const* Y_host, void* ws, size_t ws_bytes, void* stream);

/* Single-mode sketch Y = X_(n) (⊙_{k!=n} Omega_k) (Alg. 7 line 3 / Alg. 8 line 4).
 * n is 0-based; omega[n] is not read (may be NULL).  2*N*R flops. */
KRP_API int krp_sketch_mode(const float* X, int d, const int64_t* dims, int n, const float* const* omega, int R, float* Y,
                    void* ws, size_t ws_bytes, void* stream);

/* Mode-n product Y = X x_n A (the core contractions G = X x_1 Q_1^T ... of Alg. 7 line 5, and
 * B = G x_i Q^T of Alg. 8 line 5; definition of x_n as in S:124-128): A is J x I_n row-major
 * (device), Y has dims with I_n replaced by J (device, first index fastest, written, not accumulated).
 * Mode n = 0 with J <= 64, I_1 % 4 == 0 and X 16-byte aligned runs on the tensor cores (tcgen05,
 * 3xTF32: fp32-level accuracy, fixed summation order); other shapes on fp32 FMA kernels.  ws: at least
 * krp_workspace_bytes(KRP_OP_TTM, d, dims, J, NULL) bytes, or NULL (allocated and freed on the stream).
 * Errors: KRP_EINVAL (null pointers, n out of range, J < 1), KRP_ENOMEM (ws too small). */
KRP_API int krp_ttm(const float* X, int d, const int64_t* dims, int n, const float* A, int J, float* Y, void* ws,
                    size_t ws_bytes, void* stream);

/* RHOSVD-KRP-MEMO (Alg. 7 with memoization):
 *   Y_n = memoized sketch; Q_n = CholeskyQR2(Y_n) (thin QR with diag(R) > 0);
 *   G = X x_1 Q_1^T ... x_d Q_d^T; then, for r_n < R, truncation by HOSVD of the
 *   small core (reading R4): U_n = leading r_n left singular vectors of G_(n),
 *   Q_n <- Q_n U_n, G <- G x_n U_n^T.
 * ranks[n] = r_n in [1, R]; Q[n]: I_n x r_n; core: prod r_n.
 * rel_err (host, nullable): if non-NULL, ||X - [G; Q]||_F / ||X||_F is computed with one more
 * pass over X (needs krp_workspace_bytes(KRP_OP_RHOSVD_ERR, ...)) and the stream is synchronized. */
KRP_API int krp_rhosvd(const float* X, int d, const int64_t* dims, const int* ranks, int R, const float* const* omega,
               float* const* Q, float* core, double* rel_err, void* ws, size_t ws_bytes, void* stream);

/* RSTHOSVD-KRP (Alg. 8), modes in ascending order, per-step truncation (R4):
 *   for i: Y = G_(i) (⊙_{j!=i} Omega^{(i)}_j); Q = CholeskyQR2(Y); B = G x_i Q^T;
 *          U = leading r_i left singular vectors of B_(i); G <- B x_i U^T; Q_i = Q U.
 * omega[i*d + j] (host array of d*d device pointers): step i, mode j, I_j x R; entries with
 * j == i are not read.  For j < i only the leading r_j rows are read (reading R5). */
KRP_API int krp_sthosvd(const float* X, int d, const int64_t* dims, const int* ranks, int R, const float* const* omega,
                float* const* Q, float* core, double* rel_err, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------ the paper's other variants (NEXT-2)
 * RHOSVD-KRP, Alg. 7 read literally ("a fresh sequence ... each time"): mode n is sketched
 * with its own sequence omega_steps[n*d + j] (I_j x R, j != n; layout as krp_sthosvd's omega), 2dNR sketch
 * flops instead of the memoized 4NR; QR, core and truncation as krp_rhosvd. */
KRP_API int krp_rhosvd_fresh(const float* X, int d, const int64_t* dims, const int* ranks, int R,
                             const float* const* omega_steps, float* const* Q, float* core, double* rel_err, void* ws,
                             size_t ws_bytes, void* stream);
/* The dense-Gaussian baselines of Table 1: RHOSVD sketches mode n with omega_dense[n], a dense
 * (N/I_n) x R row-major Gaussian whose rows follow the column order of X_(n); RSTHOSVD sketches step i's
 * current core with omega_dense[i], (prod_{j<i} r_j * prod_{j>i} I_j) x R.  The unfolding is explicit (a
 * batched transpose; the paper's "Unfolding" cost) and the product is an fp32 SGEMM (cuBLAS, loaded at run
 * time; KRP_EUNSUPPORTED if it cannot be loaded).  Baselines for comparison, not the product's hot path. */
KRP_API int krp_rhosvd_gaussian(const float* X, int d, const int64_t* dims, const int* ranks, int R,
                                const float* const* omega_dense, float* const* Q, float* core, double* rel_err,
                                void* ws, size_t ws_bytes, void* stream);
KRP_API int krp_sthosvd_gaussian(const float* X, int d, const int64_t* dims, const int* ranks, int R,
                                 const float* const* omega_dense, float* const* Q, float* core, double* rel_err,
                                 void* ws, size_t ws_bytes, void* stream);

/* Randomized HOSVD of the Hadamard product of two 3-way Tucker tensors (App. C, Alg. 9):
 * X = F x_1 A_1 x_2 A_2 x_3 A_3 (F: q_1 x q_2 x q_3, A_k: n_k x q_k), Y = G x_k U_k (G: s_1 x s_2 x s_3,
 * U_k: n_k x s_k), all fp32 device arrays, cores first-index-fastest, factors row-major.  The product
 * Z = X * Y (n_1 n_2 n_3 entries) is never formed: with H = F (x) G (the Kronecker core, q_k s_k per mode)
 * and the row-wise Kronecker factors A_k (.)^T U_k, mode i's sketch Z_(i)(Omega_{i,k} (.) Omega_{i,j}) is
 * (A_i (.)^T U_i) H_(i) (M_k (.) M_j) with M_j = (A_j^T (.) U_j^T) Omega_{i,j}; H_(i)(...) runs on
 * the KRP sketch kernel.  omega[i*3 + j] (j != i): Omega_{i,j}, n_j x l_i.  ls[i] = l_i in [1, 64] (the sketch
 * width r_i + oversampling), ranks[i] = r_i <= l_i; for r_i < l_i the HOSVD of the l-core truncates (reading
 * R4; equal l_i are then required).  Outputs Q[i] (n_i x r_i, orthonormal) and core (r_1 r_2 r_3), with
 * Z ~= core x_i Q_i.  Synchronizes the stream. */
KRP_API size_t krp_hadamard_workspace_bytes(const int64_t* n, const int64_t* q, const int64_t* s, const int* ranks,
                                            const int* ls);
KRP_API int krp_hadamard_tucker(const float* F, const int64_t* q, const float* const* A, const float* G,
                                const int64_t* s, const float* const* U, const int64_t* n, const int* ranks,
                                const int* ls, const float* const* omega, float* const* Q, float* core, void* ws,
                                size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------ multi-GPU (slab sharding)
 * The tensor is split into contiguous slabs along its LAST mode (contiguous in memory).  Each
 * rank passes its local slab X (dims[d-1] = local slab length) plus the global last-mode size and
 * the slab offset; omega[d-1] is the GLOBAL I_d x R factor.  Outputs are global and replicated on
 * every rank.  Collectives (NCCL over NVLink) are issued on `stream`. */
typedef struct krp_comm_s* krp_comm;

/* Size of the opaque unique id (bytes).  Rank 0 creates it, the caller broadcasts it
 * (e.g. with torch.distributed), every rank passes it to krp_comm_init. */
KRP_API size_t krp_comm_id_bytes(void);
KRP_API int krp_comm_get_unique_id(void* id_out);
KRP_API int krp_comm_init(krp_comm* comm, int nranks, int rank, const void* id);
KRP_API int krp_comm_destroy(krp_comm comm);

KRP_API int krp_sketch_all_modes_dist(const float* X_slab, int d, const int64_t* dims_local, int64_t I_d_global,
                              int64_t slab_begin, const float* const* omega, int R, float* const* Y, void* ws,
                              size_t ws_bytes, krp_comm comm, void* stream);
KRP_API int krp_rhosvd_dist(const float* X_slab, int d, const int64_t* dims_local, int64_t I_d_global, int64_t slab_begin,
                    const int* ranks, int R, const float* const* omega, float* const* Q, float* core,
                    double* rel_err, void* ws, size_t ws_bytes, krp_comm comm, void* stream);
/* RSTHOSVD-KRP (Alg. 8) on a slab-sharded tensor: steps i < d-1 keep the slab
 * layout (the step sketch and the mode Gram of B_(i) are all-reduced, the TTMs are local); the last step
 * gathers the complete rows of Y_d with the zero-padded all-reduce, contracts the sharded mode locally and
 * all-reduces the partial core.  omega[i*d + j] as in krp_sthosvd, with the GLOBAL I_d rows for j = d-1;
 * Q[d-1] is the global I_d x r_d factor; Q, core and rel_err are replicated on every rank. */
KRP_API int krp_sthosvd_dist(const float* X_slab, int d, const int64_t* dims_local, int64_t I_d_global,
                             int64_t slab_begin, const int* ranks, int R, const float* const* omega, float* const* Q,
                             float* core, double* rel_err, void* ws, size_t ws_bytes, krp_comm comm, void* stream);
/* Host-side sharding geometry (pure host functions, no device access; used by the _dist calls and by
 * callers that place the slabs).  SURVEY §8(e): rank g of G owns the contiguous last-mode index range
 * [begin, begin + len) with begin = floor(g * I_d / G) (balanced, ragged when G does not divide I_d).
 * Returns KRP_EINVAL for I_d < 1, nranks < 1 or rank outside [0, nranks). */
KRP_API int krp_slab_range(int64_t I_d, int nranks, int rank, int64_t* begin, int64_t* len);

/* Layout of the packed buffer that the sharded sketch combines with ONE all-reduce(sum):
 * [Y_1 | Y_2 | ... | Y_{d-1} | Y_d], each I_n x R row-major, Y_d with the GLOBAL I_d rows; a rank writes
 * its partial Y_1..Y_{d-1} and only its own slab rows of Y_d (zeros elsewhere), so the sum both adds the
 * partials and gathers the slab rows.  offsets[n] (n = 0..d-1) = float offset of Y_{n+1}; offsets[d] =
 * total floats; *slab_offset = float offset of this rank's first Y_d row.  dims_local[d-1] is the slab
 * length.  Returns KRP_EINVAL / KRP_ESHAPE on bad arguments. */
KRP_API int krp_pack_layout(int d, const int64_t* dims_local, int64_t I_d_global, int64_t slab_begin, int R,
                            int64_t* offsets, int64_t* slab_offset);

/* Workspace for the _dist calls: krp_workspace_bytes(op, d, dims_local, R, ranks) with the global
 * last-mode size passed through this helper. */
KRP_API size_t krp_workspace_bytes_dist(int op, int d, const int64_t* dims_local, int64_t I_d_global, int R,
                                const int* ranks);

/* Kernel-level profiling of the dominant sketch kernel: when enabled, the library records CUDA
 * events around every launch of the main sketch kernel (tcgen05 or SIMT) on the caller's stream.
 * krp_profile_read synchronizes those events and returns the summed duration (ms), the number of
 * launches and the algorithmic bytes/flops those launches processed. */
KRP_API int krp_profile_enable(int on);
KRP_API int krp_profile_read(double* kernel_ms, uint64_t* launches, double* alg_bytes, double* alg_flops);
KRP_API void krp_profile_reset(void);

/* Device-side launch counter (number of kernels this library launched since the last reset),
 * for the bench's gpu_launches field. */
KRP_API uint64_t krp_launch_count(void);
KRP_API void krp_reset_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* KRP_H_ */
