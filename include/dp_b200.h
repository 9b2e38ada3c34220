/*
 * dp_b200.h — C ABI of the B200-native ShardTensor domain-parallel hot path.
 *
 * Every entry point is `extern "C"`, takes plain pointers / sizes / strides,
 * returns DP_OK (0) or a DP_ERR_* code, never throws, never allocates (the
 * caller passes any workspace), and enqueues its kernels on the caller's
 * `stream` (a cudaStream_t passed as void*).  dp_last_error() returns the
 * calling thread's last message.  There is no CPU implementation behind any
 * of these symbols.
 *
 * Reference interfaces each group replaces (the reference is pure Python;
 * these are the NumPy regions its operator API bottoms out in — SURVEY.md
 * §2.1 / §8(b)):
 *
 *   dp_copy_strided        domainpar/mesh.py:370-386   halo face slicing +
 *                                                     np.concatenate;
 *                          domainpar/sharding.py:375-383 redistribute column
 *                                                     slice; mesh.py:302
 *                                                     varlen concat
 *   dp_accumulate_strided  (no reference function)    reverse-halo gradient
 *                                                     accumulate, SURVEY A9
 *   dp_conv_fwd            domainpar/ops.py:397-413 + dense.py:174-214
 *                                                     trim/pad + dense.conv
 *   dp_conv_dgrad,         (no reference function)    conv backward, A9
 *   dp_conv_wgrad
 *   dp_conv_x3_*           same, fp32 operands split once (bf16x3)
 *   dp_attn_fwd_update     domainpar/ops.py:199-211,272-275  scores +
 *                                                     RingSoftmaxState.update
 *   dp_attn_finalize       domainpar/ops.py:213-214,278   acc / l
 *   dp_attn_bwd_*          (no reference function)    ring attention bwd
 *   dp_norm_stats/_apply   domainpar/ops.py:126-173     sharded_softmax /
 *                                                     sharded_layer_norm
 *   dp_elementwise         domainpar/ops.py:93-104      sharded_elementwise
 */
#ifndef DP_B200_H
#define DP_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DP_ABI_VERSION 1

/* return codes */
#define DP_OK 0
#define DP_ERR_INVALID 1      /* bad argument (shape, stride, null pointer) */
#define DP_ERR_UNSUPPORTED 2  /* configuration outside the kernel envelope  */
#define DP_ERR_CUDA 3         /* CUDA runtime / launch failure              */
#define DP_ERR_COMM 4         /* NCCL failure (synchronous or asynchronous) */
#define DP_ERR_TIMEOUT 5      /* dp_comm_wait deadline passed (comm aborted) */

/* element types */
#define DP_F32 0
#define DP_F64 1
#define DP_BF16 2

/* algorithm selectors for the conv / attention entry points */
#define DP_ALGO_AUTO 0     /* tcgen05 path when eligible, else SIMT          */
#define DP_ALGO_SIMT 1     /* direct CUDA-core kernels (any dtype / stride)  */
#define DP_ALGO_TC 2       /* tcgen05 + TMA path; DP_ERR_UNSUPPORTED if not  */
#define DP_ALGO_STRICT 3   /* tcgen05 for bf16 / fp32 (UNSUPPORTED outside the
                              envelope), CUDA cores only for fp64            */

int dp_abi_version(void);
const char *dp_last_error(void);
/* Kernels this library has launched in this process (monotonic). */
uint64_t dp_launch_count(void);
/* Conv / attention calls routed to the CUDA-core kernels (fp64, or a
 * geometry outside the tcgen05 envelope under DP_ALGO_AUTO) in this process
 * (monotonic).  The hot path asserts it never moves. */
uint64_t dp_simt_count(void);
/* SM count and compute capability of the current device. */
int dp_device_info(int *sm_count, int *cc_major, int *cc_minor);

/* ---- data movement (halo / varlen pack, unpack, accumulate) ------------ */

/* dst[i] = src[i] over an `ndim`-D index space (ndim <= 8); strides are in
 * elements; elem_bytes in {1,2,4,8,16}.  Dimensions are collapsed and the
 * innermost run is moved with 16-byte vectors when alignment allows. */
int dp_copy_strided(int ndim, const int64_t *shape, void *dst, const int64_t *dst_strides,
                    const void *src, const int64_t *src_strides, int elem_bytes, void *stream);

/* dst[i] += src[i] (dtype DP_F32 / DP_F64 / DP_BF16 with fp32 add). */
int dp_accumulate_strided(int ndim, const int64_t *shape, void *dst,
                          const int64_t *dst_strides, const void *src,
                          const int64_t *src_strides, int dtype, void *stream);

/* dst[i] = (dst dtype) src[i]: strided converted copy between DP_F32 /
 * DP_F64 / DP_BF16 (round to nearest even into bf16) — accumulator ->
 * parameter-dtype casts (ring-attention dQ/dK/dV, weight gradients). */
int dp_convert_strided(int ndim, const int64_t *shape, void *dst, const int64_t *dst_strides,
                       int dst_dtype, const void *src, const int64_t *src_strides, int src_dtype,
                       void *stream);

/* dst[i] = max(dst[i], src[i]) (all_reduce "max", domainpar/mesh.py:271-277). */
int dp_max_strided(int ndim, const int64_t *shape, void *dst, const int64_t *dst_strides,
                   const void *src, const int64_t *src_strides, int dtype, void *stream);

/* dst[0..n) = value (contiguous; value 0 is a memset). */
int dp_fill(int64_t n, void *dst, int dtype, double value, void *stream);

/* ---- halo convolution --------------------------------------------------- */

/* Geometry of one rank's share of a (possibly sharded) convolution.
 * The input along spatial dim `shard` is the *virtual* block
 *     [zeros | main (in_ext[shard] rows) | right halo (halo rows) | zeros]
 * and output row o of every spatial dim i reads virtual rows
 *     base[i] + o*stride[i] + t,  t in [0, kernel[i])
 * (unsharded dims: base = -padding; virtual rows outside [0, in_ext) are
 * zero).  This is the reference's trimmed + zero-padded extended block
 * (domainpar/ops.py:397-413) without materialising it. */
typedef struct dp_conv_geom {
    int32_t nsp;            /* spatial dims, 1..3 */
    int32_t shard;          /* spatial index extended by `halo`, or -1 */
    int64_t batch, c_in, c_out;
    int64_t in_ext[3];      /* main-block spatial extents */
    int64_t halo;           /* right-halo rows on `shard` */
    int64_t out_ext[3];     /* this rank's output spatial extents */
    int32_t kernel[3];
    int32_t stride[3];
    int64_t base[3];
    int64_t xs[5];          /* element strides [b, c, s0, s1, s2] of the main block */
    int64_t hs[5];          /* ... of the halo block (ignored when halo == 0) */
    int64_t ys[5];          /* ... of the output */
    int64_t out_org[3];     /* global index of the output's element 0 on each spatial dim
                             * (fwd: y, dgrad: dx) — aligns the tcgen05 kernels'
                             * accumulator ring to global rows so a sharded launch sums
                             * every output in the same order as the unsharded one
                             * (bitwise sharding invariance); 0 when unknown */
} dp_conv_geom;

/* Workspace bytes the conv entry point `which` (DP_CONV_FWD / _DGRAD /
 * _WGRAD) needs for this geometry and algorithm (weight images for the
 * tcgen05 path, split-K partials for wgrad); -1 when `algo` cannot run it. */
#define DP_CONV_FWD 0
#define DP_CONV_DGRAD 1
#define DP_CONV_WGRAD 2
int64_t dp_conv_workspace(const dp_conv_geom *g, int dtype, int algo, int which);

/* y = conv(x_virtual, w); w is contiguous [c_out, c_in, k0(, k1(, k2))] in
 * the activation dtype; accumulation is fp32 (fp64 for DP_F64). */
int dp_conv_fwd(const dp_conv_geom *g, int dtype, int algo, const void *x, const void *x_halo,
                const void *w, void *y, void *workspace, int64_t workspace_bytes,
                void *stream);

/* dx_virtual = conv^T(dy, w) over virtual rows [0, in_ext + halo) of the
 * sharded dim: rows [0, in_ext) land in dx (strides g->xs), rows
 * [in_ext, in_ext + halo) in dx_halo (strides g->hs) — the block that is
 * sent back to the next rank and accumulated there.  dy uses
 * strides g->ys.  Overwrites dx / dx_halo. */
int dp_conv_dgrad(const dp_conv_geom *g, int dtype, int algo, const void *dy, const void *w,
                  void *dx, void *dx_halo, void *workspace, int64_t workspace_bytes,
                  void *stream);

/* dw (fp32 for DP_F32/DP_BF16, fp64 for DP_F64; contiguous [c_out, c_in,
 * k...]) = sum over batch and output positions of dy * x_virtual.  The
 * result is this rank's partial; the caller all-reduces it over the
 * sharding group. */
int dp_conv_wgrad(const dp_conv_geom *g, int dtype, int algo, const void *x, const void *x_halo,
                  const void *dy, void *dw, void *workspace, int64_t workspace_bytes,
                  void *stream);

/* ---- fp32 conv on the tensor cores with operands split once --------------- */
/* The fp32 convs above run as bf16x3 (three exact bf16 parts per value,
 * six part products, fp32 accumulation: the reference's 1e-5 tolerance,
 * domainpar/verify.py:40) and split their fp32 operands inside each call.
 * These entry points let the caller split an operand ONCE and reuse it: x
 * (split in the forward) feeds the forward and the weight gradient, dy
 * (split in the backward) feeds the data and the weight gradient — the
 * tape of domainpar/ops.py:303-422's halo_conv keeps x's parts.  A split
 * operand is [3][batch][s0][s1][c] bf16 channels-last (the parts as batch
 * blocks); operand = DP_X3_X (x main block, strides g->xs), DP_X3_XHALO (the
 * received halo rows, g->hs) or DP_X3_DY (g->ys).  Bytes: 0 for an empty
 * operand, -1 outside the envelope (2-D 3x3, stride 1, c_in/c_out 16|32). */
#define DP_X3_X 0
#define DP_X3_XHALO 1
#define DP_X3_DY 2
int64_t dp_conv_x3_operand_bytes(const dp_conv_geom *g, int operand);
int dp_conv_x3_split(const dp_conv_geom *g, int operand, const void *src, void *parts,
                     void *stream);
/* workspace of the *_parts calls (weight images, wgrad partials); -1 when
 * the geometry is outside the bf16x3 path */
int64_t dp_conv_x3_parts_workspace(const dp_conv_geom *g, int which);
int dp_conv_x3_fwd_parts(const dp_conv_geom *g, const void *x_parts, const void *x_halo_parts,
                         const void *w, void *y, void *workspace, int64_t workspace_bytes,
                         void *stream);
int dp_conv_x3_dgrad_parts(const dp_conv_geom *g, const void *dy_parts, const void *w, void *dx,
                           void *dx_halo, void *workspace, int64_t workspace_bytes, void *stream);
int dp_conv_x3_wgrad_parts(const dp_conv_geom *g, const void *x_parts, const void *x_halo_parts,
                           const void *dy_parts, void *dw, void *workspace,
                           int64_t workspace_bytes, void *stream);

/* ---- ring attention blocks ------------------------------------------------ */

/* Shapes: q [sq, h, d], k/v [sk, h, d] with element strides (row, head)
 * and unit stride on d.  State: m, l [sq, h] and acc [sq, h, d] contiguous,
 * fp32 (fp64 for DP_F64).  One call folds one K/V block into the running
 * online-softmax state exactly as RingSoftmaxState.update
 * (domainpar/ops.py:199-211): m' = max(m, rowmax(s)), c = exp(m - m'),
 * l' = l*c + sum(exp(s - m')), acc' = acc*c + exp(s - m') @ v with
 * s = (q @ k^T) * scale.  sk == 0 is a no-op. */
typedef struct dp_attn_geom {
    int64_t sq, sk, heads, dim;
    int64_t q_rs, q_hs;     /* q row / head strides (elements) */
    int64_t k_rs, k_hs;
    int64_t v_rs, v_hs;
    int64_t o_rs, o_hs;     /* output / dO strides */
    double scale;
} dp_attn_geom;

int dp_attn_fwd_update(const dp_attn_geom *g, int dtype, int algo, const void *q, const void *k,
                       const void *v, void *m, void *l, void *acc, void *stream);

/* out = acc / l cast to dtype; lse = m + log(l) (fp32/fp64) for backward. */
int dp_attn_finalize(const dp_attn_geom *g, int dtype, const void *m, const void *l,
                     const void *acc, void *out, void *lse, void *stream);

/* delta[i,h] = sum_d dO[i,h,d] * O[i,h,d] (fp32/fp64). */
int dp_attn_bwd_preprocess(const dp_attn_geom *g, int dtype, const void *o, const void *dout,
                           void *delta, void *stream);

/* Fold one K/V block into the gradients: with P = exp(s - lse),
 * dV += P^T dO, dS = P * (dO V^T - delta), dQ += scale dS K,
 * dK += scale dS^T Q.  dq [sq,h,d], dk/dv [sk,h,d] are contiguous fp32
 * (fp64) accumulators. */
int dp_attn_bwd_update(const dp_attn_geom *g, int dtype, int algo, const void *q, const void *k,
                       const void *v, const void *dout, const void *lse, const void *delta,
                       void *dq, void *dk, void *dv, void *stream);

/* ---- sharded normalisations and pointwise ops -------- */

/* The reduced dim is the middle of an [outer, n, inner] view with element
 * strides xs = {outer, n, inner}.  Statistics are fp64 and laid out
 * [nstat][outer * inner] (cell = o * inner + i):
 *   kind 0  layer-norm moments: stats[0] = sum x, stats[1] = sum x^2
 *           (domainpar/ops.py:165-168: both ride ONE all_reduce)
 *   kind 1  softmax local max (-inf for n == 0)          (ops.py:141-145)
 *   kind 2  softmax local sum exp(x - aux), aux = global max  (ops.py:146-148)
 * Deterministic (fixed-order split + combine, no atomics). */
#define DP_NORM_MOMENTS 0
#define DP_NORM_MAX 1
#define DP_NORM_EXPSUM 2
int64_t dp_norm_workspace(int kind, int64_t outer, int64_t n, int64_t inner);
int dp_norm_stats(int kind, int64_t outer, int64_t n, int64_t inner, const void *x,
                  const int64_t *xs, int dtype, const void *aux, void *stats, void *workspace,
                  int64_t workspace_bytes, void *stream);

/* y = normalised x (y strides ys), from the GLOBAL statistics:
 *   kind 0  layer norm: mean = s1/count, var = max(s2/count - mean^2, 0),
 *           y = (x - mean) / sqrt(var + eps)           (domainpar/ops.py:169-172)
 *   kind 1  softmax: y = exp(x - aux) / stats (aux = global max, stats =
 *           global denominator)                         (ops.py:146-149) */
int dp_norm_apply(int kind, int64_t outer, int64_t n, int64_t inner, const void *x,
                  const int64_t *xs, void *y, const int64_t *ys, int dtype, const void *stats,
                  const void *aux, double count, double eps, void *stream);

/* out = a (op) b over n contiguous elements: op 0 add, 1 mul (b array, or
 * the scalar when b is NULL), 2 scale (out = a * scalar) — domainpar/dense.py:65-98; fp32 math for
 * DP_F32/DP_BF16, fp64 for DP_F64. */
#define DP_EW_ADD 0
#define DP_EW_MUL 1
#define DP_EW_SCALE 2
int dp_elementwise(int op, int64_t n, const void *a, const void *b, double scalar, void *out,
                   int dtype, void *stream);

/* ---- communicators and exchanges (NCCL over NVLink / NVSwitch) ------------
 *
 * Replace domainpar/mesh.py:252-403 (all_reduce, all_gather_varlen,
 * ring_shift, halo_exchange, barrier over per-pair queues).  NCCL is loaded
 * at run time (dlopen; dp_comm_load(NULL) = "libnccl.so.2", normally the copy
 * the host process already has); without it these return DP_ERR_UNSUPPORTED
 * and every other entry point still works.  A communicator is an opaque
 * handle; one per mesh-axis line (dp_comm_split of the world communicator,
 * color = line, key = position on the line).  Every exchange is ONE
 * ncclGroupStart/End of byte sends / receives enqueued on `stream`: buffers
 * are sent in their memory order (a dense channels-last face goes as-is).
 * Byte counts of 0 post nothing.  The caller keeps buffers alive until the
 * stream passes the exchange. */
#define DP_NCCL_UNIQUE_ID_BYTES 128
#define DP_REDUCE_SUM 0
#define DP_REDUCE_MAX 1
int dp_comm_load(const char *nccl_path);
int dp_comm_version(int *version);
/* rank 0 creates the id and ships it to the others out of band */
int dp_comm_unique_id(void *id_out /* DP_NCCL_UNIQUE_ID_BYTES */);
/* collective over `world` ranks; the current CUDA device is this rank's */
int dp_comm_init(void **comm_out, int world, int rank, const void *unique_id);
/* collective over the parent: ranks with the same color form one
 * communicator ranked by key; color < 0 -> *comm_out = NULL */
int dp_comm_split(void *parent, int color, int key, void **comm_out);
int dp_comm_info(void *comm, int *rank, int *size);
int dp_comm_destroy(void *comm);
int dp_comm_abort(void *comm);
/* generic grouped point-to-point: op i sends (is_recv[i] == 0) or receives
 * bytes[i] bytes of bufs[i] to / from peers[i] */
int dp_comm_exchange(void *comm, int n, const int *peers, const int *is_recv, void *const *bufs,
                     const int64_t *bytes, void *stream);
/* halo round (domainpar/mesh.py:318-386): send my first / last rows to the
 * left / right neighbour, receive their faces; peer -1 = no neighbour */
int dp_halo_sendrecv(void *comm, int left, int right, const void *send_left,
                     int64_t send_left_bytes, const void *send_right, int64_t send_right_bytes,
                     void *recv_left, int64_t recv_left_bytes, void *recv_right,
                     int64_t recv_right_bytes, void *stream);
/* ring hop (domainpar/mesh.py:305-315): send to rank+1, receive from rank-1 */
int dp_ring_step(void *comm, const void *send, int64_t send_bytes, void *recv, int64_t recv_bytes,
                 void *stream);
/* varlen all-gather (domainpar/mesh.py:280-302): every rank's `local` lands
 * at out + offsets[rank] (bytes[rank] bytes; this rank's own block is the
 * caller's copy) */
int dp_varlen_allgather(void *comm, const void *local, int64_t local_bytes, void *out,
                        const int64_t *offsets, const int64_t *bytes, void *stream);
/* variable-count all-to-all (Shard(i) -> Shard(j) redistribute): send[j] /
 * recv[j] per peer j (entries for this rank are ignored) */
int dp_varlen_alltoall(void *comm, const void *const *send, const int64_t *send_bytes,
                       void *const *recv, const int64_t *recv_bytes, void *stream);
/* recv = reduce(send) over the communicator, DP_REDUCE_SUM / _MAX
 * (domainpar/mesh.py:252-277) */
int dp_allreduce(void *comm, const void *send, void *recv, int64_t count, int dtype, int op,
                 void *stream);
/* watchdog: block until `stream` drains; an asynchronous NCCL error or the
 * deadline (timeout_s > 0) aborts the communicator -> DP_ERR_COMM /
 * DP_ERR_TIMEOUT */
int dp_comm_wait(void *comm, void *stream, double timeout_s);

#ifdef __cplusplus
}
#endif
#endif /* DP_B200_H */
