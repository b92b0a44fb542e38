/*
 * sg.h — C ABI of the B200-native 2D (SUMMA) transformer hot path.
 *
 * Every entry point is a per-device ("local") operation of the Optimus 2D
 * partition: plain device pointers, element counts / leading dimensions and
 * a cudaStream_t passed as void*. The row/column collectives between these
 * calls are issued by the host mesh runtime (paper_2104_05343_b200/mesh.py)
 * over NCCL communicators, so nothing here owns communicators or memory.
 *
 * The reference (summagrid, pure numpy) has no FFI; each function below
 * replaces the per-device numpy closure the reference runs inside
 * Mesh.each(...) at the cited file:line of /root/reference/pkg/src/summagrid.
 *
 * Return codes: SG_OK, SG_ERR_SHAPE (-> ShapeError), SG_ERR_CONFIG
 * (-> ConfigError), SG_ERR_CUDA (-> SummaGridError).  Functions validate
 * their arguments before launching any work.
 */
#ifndef SG_H_
#define SG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_OK 0
#define SG_ERR_SHAPE 1
#define SG_ERR_CONFIG 2
#define SG_ERR_CUDA 3

#define SG_DTYPE_BF16 0
#define SG_DTYPE_F32 1

#define SG_ACT_NONE 0
#define SG_ACT_GELU 1  /* D = gelu(x); aux (if set) <- x (bf16 pre-activation) */
#define SG_ACT_DGELU 2 /* D = x * gelu'(aux) with aux the saved pre-activation */

#define SG_EPI_NORMAL 0      /* x = alpha*acc + bias + C; D = act(x) (+ D2, colsum) */
#define SG_EPI_SOFTMAX 1     /* D = softmax_row(alpha*acc), whole row in one tile (N <= 512) */
#define SG_EPI_SOFTMAX_BWD 2 /* D = aux*(acc - rowvec)*alpha, aux = P, rowvec = rowsum(dP*P) = rowsum(dO*O) */

/*
 * Batched local GEMM on the 5th-gen tensor cores (tcgen05, TMEM accumulators,
 * TMA-fed SWIZZLE_128B operand tiles), bf16 operands, fp32 accumulate:
 *
 *   x[z](m,n) = alpha * sum_k opA[z](m,k) * opB[z](k,n) + bias[n] + C[z](m,n)
 *   D[z](m,n) = act(x)
 *
 *   opA(m,k) = A[m*lda + k]   (a_mn_major = 0, "K-major")  or A[k*lda + m] (1)
 *   opB(k,n) = B[n*ldb + k]   (b_mn_major = 0, "K-major")  or B[k*ldb + n] (1)
 *   batch z = z1*nb2 + z2, operand X offset = z1*sx1 + z2*sx2 (elements).
 *
 * It is the local product of every SUMMA step:
 *   summa_ab  C_ij += A_il B_lj     (a: K-major, b: MN-major)  summa.py:114-115 -> mesh.py:349-361
 *   summa_abt c_tmp = A_ij B_lj^T   (a: K-major, b: K-major)   summa.py:135-136
 *   summa_atb c_tmp = A_il^T B_ij   (a: MN-major, b: MN-major) summa.py:159-160
 * and of the per-head attention products (layers.py:409-411, 447-452).
 * The optional C operand implements SUMMA step accumulation (C == D: the
 * product is added in place by TMA reduce-add stores, no epilogue loads)
 * and the fused residual adds (layers.py:706-707, 722-723); colsum fuses the
 * bias gradients (layers.py:238); the softmax modes fuse the attention
 * softmax (dense.py:67-75) and its backward (layers.py:447-450) into the
 * QK^T / dO V^T products.
 */
typedef struct sg_gemm_args {
  int64_t M, N, K;
  int64_t nb1, nb2;
  const void* A; int64_t lda, sa1, sa2; int32_t a_mn_major;
  const void* B; int64_t ldb, sb1, sb2; int32_t b_mn_major;
  void* D; int64_t ldd, sd1, sd2; int32_t d_dtype;
  const void* C; int64_t ldc, sc1, sc2; int32_t c_dtype;
  const float* bias;
  void* aux; int64_t ldx, sx1, sx2;
  int32_t act;
  float alpha;
  /* optional bf16 copy of D (e.g. the GEMM operand twin of an fp32 gradient) */
  void* D2; int64_t ld2, s21, s22;
  /* optional fused column sums: colsum[z1*scs1 + z2*scs2 + n] += sum_m D[z](m, n) */
  float* colsum; int64_t scs1, scs2;
  int32_t mode; /* SG_EPI_* */
  /* SOFTMAX_BWD: D_i = rowsum(dO * O) per output row, rowvec[z1*srv1 + z2*srv2 + m] */
  const float* rowvec; int64_t srv1, srv2;
  /* optional LayerNorm-backward row statistics of the fp32 output dy = D (layers.py:319-326):
   * ln_stats[2m] += sum_n xhat(m,n) * g(m,n), ln_stats[2m+1] += sum_n g(m,n) with
   * g = dy * ln_gamma[n], xhat = (C(m,n) - ln_mean[m]) * ln_rstd[m]; C is then the
   * LayerNorm input x (fp32, read by TMA, not added). Unbatched, fp32 D, no bias / act. */
  const float* ln_gamma; const float* ln_mean; const float* ln_rstd; float* ln_stats;
} sg_gemm_args;

int sg_gemm(const sg_gemm_args* args, void* stream);

/* ---------------------------------------------------------------------------
 * HBM-bound per-device kernels (row kernels: one warp per row, 16-byte
 * vector accesses). dtype arguments are SG_DTYPE_*; leading dimensions are in
 * elements and must keep rows 16-byte aligned.
 * ------------------------------------------------------------------------- */

/* LayerNorm phase 1: stats[r] = (sum_c x, sum_c x^2) — the packed pair the
 * reference all-reduces along the mesh row (layers.py:274-280). */
int sg_ln_stats(const void* x, int xdt, int64_t rows, int64_t cols, int64_t ldx, float* stats, void* stream);
/* LayerNorm phase 2: y = (x-mu)*rstd*gamma + beta over the global hidden size
 * h_total (layers.py:295-303). stats == NULL computes them locally (only valid
 * when cols == h_total, i.e. a 1-column mesh). Saves mean / rstd per row. */
int sg_ln_fwd(const void* x, int xdt, int64_t rows, int64_t cols, int64_t ldx, const float* stats, int64_t h_total,
              float eps, const float* gamma, const float* beta, void* y, int ydt, int64_t ldy, float* mean,
              float* rstd, void* stream);
/* LayerNorm backward phase 1: stats[r] = (sum x^ g, sum g), g = dy*gamma (layers.py:319-326). */
int sg_ln_bwd_stats(const void* dy, int dydt, int64_t lddy, const void* x, int xdt, int64_t ldx, const float* mean,
                    const float* rstd, const float* gamma, int64_t rows, int64_t cols, float* stats, void* stream);
/* LayerNorm backward phase 2: dx = rstd*(g - sum_g/h - x^ sum_xg/h) + resid (fp32),
 * optional bf16 copy dx2, dgamma/dbeta += column sums (layers.py:329-342, 744-753)
 * and dsum += column sums of dx itself (the next bias gradient, layers.py:238). */
int sg_ln_bwd(const void* dy, int dydt, int64_t lddy, const void* x, int xdt, int64_t ldx, const float* mean,
              const float* rstd, const float* gamma, int64_t rows, int64_t cols, const float* stats, int64_t h_total,
              const void* resid, int rdt, int64_t ldr, void* dx, int dxdt, int64_t lddx, void* dx2, int64_t lddx2,
              float* dgamma, float* dbeta, float* dsum, void* stream);
/* out[c] (+)= sum_r x[r,c]: bias gradients before the column reduce (layers.py:238). */
int sg_colsum(const void* x, int xdt, int64_t rows, int64_t cols, int64_t ldx, float* out, int accumulate,
              void* stream);
/* x[r,c] += bias[c] in place (layers.py:228). */
int sg_bias_add(void* x, int xdt, int64_t rows, int64_t cols, int64_t ldx, const float* bias, void* stream);
/* Row softmax with max subtraction (dense.py:67-75) and its backward
 * dS = P*(dP - rowsum(dP*P))*scale (layers.py:447-450). */
int sg_softmax_rows(const void* s, int sdt, int64_t rows, int64_t cols, int64_t lds, void* p, int pdt, int64_t ldp,
                    void* stream);
int sg_softmax_bwd(const void* dp, int dpdt, int64_t lddp, const void* p, int pdt, int64_t ldp, int64_t rows,
                   int64_t cols, float scale, void* ds, int dsdt, int64_t ldds, void* stream);
/* Flash-style attention forward for one mesh position (layers.py:404-416):
 * qkv is the [b*s, 3*nh*d] QKV block (columns [Q heads | K heads | V heads]),
 * out the [b*s, nh*d] context block, lse [b, nh, s] the natural log-sum-exp
 * of the scaled scores; d in {64, 128}. The probabilities are never stored. */
int sg_flash_attn_fwd(const void* qkv, int64_t ldq, int64_t b, int64_t s, int64_t nh, int64_t d, void* out,
                      int64_t ldo, float* lse, void* stream);
/* Flash-style attention backward (d = 64): recomputes P from lse, writes dK, dV
 * (bf16) into the K / V column ranges of the [b*s, 3*nh*d] gradient block dqkv and
 * ADDS dQ into the fp32 accumulator dq_acc [b*s, >= nh*d] (zero it first);
 * drow = rowsum(dO * O) from sg_attn_rowdot. */
int sg_flash_attn_bwd(const void* qkv, int64_t ldq, const void* dout, int64_t lddo, const float* lse,
                      const float* drow, int64_t b, int64_t s, int64_t nh, int64_t d, float* dq_acc, int64_t lddq,
                      void* dqkv, int64_t ldg, float* kv_colsum, void* stream);
/* (kv_colsum, optional: [2*nh*d] += column sums of the bf16 dK, dV written, i.e. the
 * K / V parts of the b_qkv gradient.)
 * After sg_flash_attn_bwd: dqkv[:, 0:hb] = bf16(dq_acc) and colsum[0:cols] += column
 * sums of dQKV columns [0, cols) (cols = 3hb: the whole b_qkv gradient, layers.py:238;
 * cols = hb when the flash backward already summed dK / dV), one pass; hb % 256 == 0. */
int sg_qkv_grad_finish(const float* dq_acc, int64_t lddq, void* dqkv, int64_t ldg, int64_t rows, int64_t hb,
                       float* colsum, int64_t cols, void* stream);
/* D[b, h, t] = rowsum(dO * O) per head and token (= rowsum(dP * P)), the
 * SG_EPI_SOFTMAX_BWD row term; dO / O are [b*s, nh*d] head-interleaved blocks. */
int sg_attn_rowdot(const void* dO, int dt, int64_t ldo, const void* O, int64_t ldO, int64_t rows, int64_t nh,
                   int64_t d, int64_t s, float* out, void* stream);
/* Vocab-parallel cross entropy (layers.py:539-624). Local pass over the device's
 * vocabulary block: lmax, gmax (= lmax, to be max-all-reduced along the row),
 * packed = (sum e^{x-lmax}, x_label). Then sg_xent_rescale re-bases the sums on
 * the row max before the packed sum all-reduce, sg_xent_loss forms per-row
 * losses and their sum, sg_xent_bwd writes dlogits = (softmax - onehot)*scale. */
int sg_xent_local(const void* logits, int ldt, int64_t rows, int64_t ldl, int64_t n_real, const int64_t* labels,
                  int64_t col_lo, float* lmax, float* gmax, float* packed, void* stream);
int sg_xent_rescale(int64_t rows, const float* lmax, const float* gmax, float* packed, void* stream);
int sg_xent_loss(int64_t rows, const float* gmax, const float* packed, float* loss_rows, float* partial,
                 void* stream);
int sg_xent_bwd(const void* logits, int ldt, int64_t rows, int64_t ldl, int64_t n_real, int64_t ncols,
                const int64_t* labels, int64_t col_lo, const float* gmax, const float* packed, float scale, void* dl,
                int dldt, int64_t lddl, void* stream);
/* Embedding gather for ids in [lo, lo+vb) and its scatter-add backward (layers.py:178-205). */
int sg_embed_fwd(const int64_t* ids, int64_t n, int64_t lo, int64_t vb, const void* table, int tdt, int64_t ldt,
                 int64_t hc, void* out, int odt, int64_t ldo, void* stream);
int sg_embed_bwd(const int64_t* ids, int64_t n, int64_t lo, int64_t vb, const void* dout, int ddt, int64_t ldd,
                 int64_t hc, float* grad, int64_t ldg, void* stream);
/* Device-side id range check (layers.py:164-165 tokens, layers.py:552-553 labels):
 * *flag |= 1 when any of the n ids lies outside [0, v). The host reads the flag at
 * its next synchronisation (the loss read-back) and raises ConfigError. */
int sg_check_ids(const int64_t* ids, int64_t n, int64_t v, int* flag, void* stream);

/* ---- Peer memory of the SPMD mesh (replaces the reference's row / column reduce
 * collectives mesh.py:458-482 on the AB^T / A^T B paths, summa.py:128-139, 152-163).
 * sg_sym_alloc: zeroed device arena + its CUDA IPC handle (sg_ipc_handle_size bytes);
 * sg_ipc_open maps a peer's arena into the calling device (peer access enabled
 * lazily); sg_peer_barrier: stream-ordered group barrier over signal pads in such
 * arenas. args = n pad pointers then n member flat ranks (int64, device memory);
 * the epoch counter lives on the device (graph-capturable); on timeout *err |= 1. */
int sg_sym_alloc(int64_t bytes, void** ptr, void* handle);
int sg_sym_free(void* ptr);
int sg_ipc_open(const void* handle, void** ptr);
int sg_ipc_close(void* ptr);
int sg_ipc_handle_size(void);
/* SMs the persistent GEMM grid leaves free (dist meshes: the NCCL kernels moving the
 * next SUMMA step's panels co-reside with the current product); default 0. */
int sg_set_sm_reserve(int n);
int sg_gemm_sm_budget(void);
int sg_peer_barrier(const int64_t* args, int n, int me_idx, int* epoch, int* err, int64_t timeout_cycles,
                    void* stream);
/* Panel broadcasts and small all-reduces over peer memory (replacing the reference's
 * mesh.py:440-456 broadcasts and 484-513 all-reduces on the dist mesh): sg_copy_async is
 * a stream-ordered copy between any two device addresses (copy engines over NVLink
 * for a peer-mapped side); sg_peer_fold folds n fp32 buffers (device array of
 * pointers, member order) into dst, sum or max, optionally accumulating. */
int sg_copy_async(void* dst, const void* src, int64_t bytes, void* stream);
int sg_peer_fold(float* dst, const int64_t* srcs, int n, int64_t count, int accumulate, int op_max, void* stream);
/* SGD on the fp32 master, refreshing the bf16 GEMM copy (layers.py:761-772, model.py:356-364). */
int sg_sgd(float* w, int64_t ldw, void* w_bf16, int64_t ldl, const float* g, int64_t ldg, float lr, int64_t rows,
           int64_t cols, void* stream);
/* Multi-tensor form: every (w, bf16 twin, g) of a layer / model in one launch per
 * 96 tensors (the reference's per-parameter loop, layers.py:761-772). g == NULL:
 * w was already updated (its weight-gradient product reduce-added -lr dW into it),
 * only the bf16 twin is refreshed. */
typedef struct sg_sgd_item {
  float* w; void* w_bf16; const float* g;
  int64_t ldw, ldl, ldg, rows, cols;
} sg_sgd_item;
int sg_sgd_multi(const sg_sgd_item* items, int n, float lr, void* stream);
/* out = dact * gelu'(mid), colsum += column sums of out (GELU backward + b1 gradient,
 * layers.py:502-504); bf16 dact / mid, out may alias dact. */
int sg_dgelu(const void* dact, int64_t lda, const void* mid, int64_t ldm, int64_t rows, int64_t cols, void* out,
             int odt, int64_t ldo, float* colsum, void* stream);
/* out = act(alpha*x + bias + C) on an fp32 partial sum: the sg_gemm epilogue for
 * products whose mesh reduce had to complete first (dist AB^T forms). */
int sg_epilogue(const float* x, int64_t rows, int64_t cols, int64_t ldx, float alpha, const float* bias,
                const void* cin, int cdt, int64_t ldc, int act, void* aux, int64_t ldaux, void* out, int odt,
                int64_t ldo, void* stream);
/* Element-wise cast, memset and ordered fold dst = [dst op] src0 op src1 ...
 * (op: 0 sum, 1 max) — the rank-ordered reduce of mesh.py:458-499. */
int sg_cast(const void* src, int sdt, void* dst, int ddt, int64_t n, void* stream);
int sg_zero(void* ptr, int64_t bytes, void* stream);
int sg_fold(void* dst, int dt, const void* const* srcs, int nsrc, int64_t n, int accumulate, int op_max,
            void* stream);

/* Number of SMs of the current device and library build id (sanity). */
int sg_device_sm_count(void);
const char* sg_build_info(void);
/* Number of kernels this library has launched in the process (instrumentation). */
int64_t sg_launch_count(void);
/* Message of the last failing call on this thread ("" if none). */
const char* sg_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SG_H_ */
