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
 * The optional C operand implements SUMMA step accumulation (C == D allowed)
 * and the fused residual adds (layers.py:706-707, 722-723).
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
} sg_gemm_args;

int sg_gemm(const sg_gemm_args* args, void* stream);

/* Number of SMs of the current device and library build id (sanity). */
int sg_device_sm_count(void);
const char* sg_build_info(void);
/* Message of the last failing call on this thread ("" if none). */
const char* sg_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SG_H_ */
