/* apt.h — C ABI of the B200-native APT arbitrary-precision W_p x A_q integer MatMul.
 *
 * The operation (arXiv 2508.19087, PAPER.md = "P:<line>"):
 *   signed n-bit integer codes are converted losslessly to bipolar-INT by flipping
 *   the sign bit (§3.1: x' = 2x + 1), decomposed into n bit-planes and
 *   packed into 32-bit words concatenated into one "unified matrix" (§4.1);
 *   the GEMM multiplies the planes and reassembles the exact result by shift-add
 *   (§3.2: Y = sum_{i,j} 2^(i+j) Y^(i,j)), with the reassembly kept on chip
 *   (§4.2).  An optional epilogue scales the exact int32 result by
 *   per-channel / per-token fp32 scales (linear quantization W = s*W_hat)
 *   and rounds once to fp16.
 *
 * Orientation (reading Q2): A = activations [M, K] (abits = p_a bits),
 * W = weights [N, K] (wbits = p_w bits), both K-contiguous;
 *     Y[m][n] = sum_{k<K} A[m][k] * W[n][k]             (signed codes, exact)
 *     Y'[m][n] = sum_{k<K} (2A+1)[m][k] * (2W+1)[n][k]  (bipolar product)
 *
 * General contract
 *   - Every pointer is a DEVICE pointer unless marked "host".
 *   - All calls taking a stream are stream-ordered and asynchronous; the library never
 *     synchronizes, never allocates device memory, and keeps no per-call state.
 *     Argument errors are returned synchronously before anything is launched.
 *   - Stream order and programmatic dependent launch (PDL): every kernel is launched with
 *     programmatic stream serialization.  apt_gemm's kernels read the WEIGHT-side operands
 *     (W planes, W row sums, w_scale) before waiting for their stream predecessor, so that the next
 *     GEMM's weights stream from HBM while the previous kernel finishes; activation-side operands
 *     and the output are touched only after the wait.  This is safe whenever the kernel that wrote the
 *     weight-side buffers did not release its dependents early: apt_pack_bipolar / apt_quantize_pack
 *     without a digit view never do (their dependents start after every CTA has exited, stores
 *     fenced at GPU scope), and ordinary kernels (torch, cuBLAS, memcpy) never do.  A pack WITH a
 *     digit view produces an activation operand and releases its dependents at entry (activations
 *     are read after the wait); apt_gemm therefore rejects a W that carries a digit view.  Only a caller kernel that itself executes
 *     griddepcontrol.launch_dependents / cudaTriggerProgrammaticLaunchCompletion BEFORE writing the
 *     weights of the apt_gemm that follows it on the same stream breaks this; insert an event or
 *     any non-PDL kernel between them.
 *   - The caller owns every buffer (in practice torch tensors).
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *   - Thread-safe: the only global state is the per-device SM count (queried once under a mutex), the
 *     driver entry point of cuTensorMapEncodeTiled (resolved once) and per-kernel "max dynamic shared
 *     memory set" flags (atomics).  Tensor maps are encoded per call on the host (no cache).
 *   - There is no CPU fallback: with no CUDA device every launching call returns APT_ERR_CUDA.
 */
#ifndef APT_H_
#define APT_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define APT_API __attribute__((visibility("default")))
#else
#define APT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define APT_ABI_VERSION 8
#define APT_KPAD_QUANTUM 256 /* packed rows are padded to Kpad = round_up(K, 256) elements */
#define APT_GROUP_MAX 64     /* problems per grouped call (apt_pack_grouped, apt_gemm_grouped) */

typedef enum {
  APT_OK = 0,
  APT_ERR_INVALID_ARGUMENT = 1, /* null pointer, bits outside [1,8], dim <= 0, ld < K, misalignment,
                                   shape mismatch between the packed operands and M/N/K           */
  APT_ERR_UNSUPPORTED = 2,      /* int32 overflow bound exceeded (reading Q8) or a config that is
                                   illegal for the shape                                            */
  APT_ERR_WORKSPACE = 3,        /* workspace missing or smaller than apt_gemm_workspace_bytes()      */
  APT_ERR_CUDA = 4              /* a CUDA launch/runtime error (cudaGetLastError) or no device        */
} apt_status;

typedef enum {
  APT_ENC_SIGNED = 0, /* codes are signed n-bit integers x in [-2^(n-1), 2^(n-1)-1]; n = 1 -> {-1, 0}
                         (reading Q4)                                                 */
  APT_ENC_BIPOLAR = 1 /* codes are bipolar values x' (odd, |x'| <= 2^n - 1); converted by
                         x = (x' - 1) / 2.  int8 storage limits this encoding to n <= 7.     */
} apt_encoding;

typedef enum {
  APT_PACK_ROWS = 0,  /* planes[i][r][w]: plane-major, row-major words (the canonical layout)            */
  APT_PACK_TILED = 1  /* planes[i][r/128][w/8][(w%8)/4][r%128][w%4]: every 128-row x 256-element slab of a
                         plane is 4 KB contiguous (so the GEMM streams weight tiles with few large bulk
                         copies), split into two 2 KB halves of 128 rows x 4 words (one 128-element K
                         step each, read bank-conflict-free on chip).  Rows padded to a multiple of 128;
                         pad-row words are unspecified and never reach a result.  Accepted for weights
                         by the tcgen05 kernel.                                                           */
} apt_pack_layout;

/* The packed "unified matrix" (SPEC PackedPlanes S:35-41, with 32-bit words per P:252).
 *   planes  : uint32 [bits][rows][k_words] (layout APT_PACK_ROWS), plane-major, one contiguous buffer,
 *             or the same words tile-major (APT_PACK_TILED, see apt_pack_layout).
 *             Plane i holds bit i of the bipolar pattern u = x + 2^(n-1) (the sign-bit-flipped
 *             two's-complement code).  Element c of a row is bit (c % 32) of word (c / 32),
 *             LSB first (reading Q5).  Pad elements c in [k, Kpad) hold the signed code 0,
 *             i.e. u = 2^(n-1) (reading Q6), so they contribute exactly 0 to signed products.
 *             NOTE: this differs from the SPEC's zero-bit padding (pads = bipolar -1): planes
 *             padded with zero bits are NOT valid input to apt_gemm (the epilogue assumes signed-0
 *             pads); produce packed operands with apt_pack_bipolar / apt_quantize_pack only.
 *             Must be 16-byte aligned.
 *   row_sum : int32 [rows], sum_{c<k} of the signed codes of the row (used by the rank-1 terms of
 *             the epilogue; SURVEY §8c identities I2/I3).
 *   rows, k : logical shape; k_words = Kpad / 32; bits = n in [1, 8].
 *   digits  : OPTIONAL (may be NULL) uint8 [rows][Kpad], 16-byte aligned: the same codes as unsigned
 *             digits u in the GEMM kernels' internal K order (within every 32-element word the
 *             element order of the on-chip operand rebuild; word order unchanged).  When non-NULL,
 *             apt_pack_bipolar fills it in the same pass, and apt_gemm reads the ACTIVATION operand
 *             from it instead of rebuilding the activation planes (the weight operand is always read
 *             as planes).  Intended for the small per-call activation matrix.                       */
typedef struct {
  int32_t rows;
  int32_t k;
  int32_t k_words;
  int32_t bits;
  uint32_t* planes;
  int32_t* row_sum;
  uint8_t* digits;
  int32_t layout; /* apt_pack_layout of `planes`; set by the caller before apt_pack_bipolar */
} apt_packed;

/* Host.  Bytes of the `planes` buffer for a rows x k matrix of n-bit codes in `layout`:
 * APT_PACK_ROWS bits * rows * round_up(k,256)/32 * 4; APT_PACK_TILED the same with rows rounded up to 128.
 * Returns 0 for invalid arguments. */
APT_API size_t apt_packed_plane_bytes(int32_t rows, int32_t k, int32_t bits, int32_t layout);

/* Decomposition & reassembly (§4.1 Steps 1-3) on the device.
 *   codes       : int8 [rows][ld] row-major, element (r, c) at codes[r*ld + c], c < k.
 *   out         : host struct; out->planes (apt_packed_plane_bytes) and out->row_sum (rows int32)
 *                 must point to caller-allocated device buffers and out->layout must be set.  The call
 *                 fills rows/k/k_words/bits and writes both buffers (every word, including padding).
 *   range_error : nullable device int32.  If some code is outside the declared range, the kernel
 *                 stores 1 + (linear index r*k + c of one such code) there (first writer wins; the
 *                 caller zeroes it beforehand and reads it after its own synchronization).
 *                 Out-of-range codes are packed as u = (x + 2^(n-1)) mod 2^n.
 * Errors: APT_ERR_INVALID_ARGUMENT (null codes/out/buffers, rows <= 0, k <= 0, ld < k,
 *         bits outside [1,8], bipolar with bits > 7, misaligned planes), APT_ERR_CUDA. */
APT_API apt_status apt_pack_bipolar(const int8_t* codes, int32_t rows, int32_t k, int64_t ld, int32_t bits,
                            apt_encoding enc, apt_packed* out, int32_t* range_error, void* stream);

/* Fused activation quantize + pack (reading R-Q).  Linear quantization
 * x = s * x_hat + z with z = 0 and one scale per row (per token), then the same
 * decomposition as apt_pack_bipolar, in one kernel:
 *   s[r]        = RN_f32( max_{c<k} |x[r][c]| / (2^(bits-1) - 1) )
 *   x_hat[r][c] = clamp( rint( RN_f32(x[r][c] / s[r]) ), -2^(bits-1), 2^(bits-1) - 1 ), 0 if s[r] == 0
 * IEEE fp32 arithmetic (division rounded to nearest even, rint half-to-even); the codes are the
 * signed encoding (APT_ENC_SIGNED).  Pass `scale` as apt_scales.a_scale of the following apt_gemm.
 *   x     : fp16 (IEEE binary16, as uint16 bits) [rows][ld] row-major, finite values.
 *   out   : as apt_pack_bipolar (caller-allocated planes / row_sum / optional digits, layout set).
 *   scale : device fp32 [rows], written.
 * Errors: APT_ERR_INVALID_ARGUMENT (null pointers, rows <= 0, k <= 0, ld < k, bits outside [2,8] —
 *         a 1-bit symmetric grid has no positive level —, misaligned planes/digits), APT_ERR_CUDA. */
APT_API apt_status apt_quantize_pack(const uint16_t* x, int32_t rows, int32_t k, int64_t ld, int32_t bits,
                                     apt_packed* out, float* scale, void* stream);

/* Grouped activation packs: `count` independent apt_pack_bipolar (quantize == 0) / apt_quantize_pack
 * (quantize == 1) calls in ONE launch (the activations of several decode GEMMs), each with exactly the
 * semantics and outputs of its single call (§4.1 Steps 1-3; the quantization of P:199-201,
 * reading R-Q).  Per problem:
 *   src         : int8 codes (quantize == 0, signed encoding) or fp16 activations (quantize == 1), [rows][ld];
 *   rows        : 1 .. APT_PACK_GROUP_MAX_ROWS (activation matrices: the one-word-per-thread pack);
 *   bits        : 1..8 (2..8 with quantize);
 *   out         : host struct as for apt_pack_bipolar, APT_PACK_ROWS layout, digit view REQUIRED (the
 *                 packs are activation operands and release their dependents early, see "General contract");
 *   scale       : quantize: device fp32 [rows] written (pass it as the GEMM's a_scale); else NULL;
 *   range_error : codes only, nullable device int32 (as apt_pack_bipolar).
 * Errors: APT_ERR_INVALID_ARGUMENT (count outside [1, APT_GROUP_MAX], a problem violating the above),
 *         APT_ERR_CUDA. */
#define APT_PACK_GROUP_MAX_ROWS 64
typedef struct {
  const void* src;
  int32_t quantize;
  int32_t rows;
  int32_t k;
  int32_t bits;
  int64_t ld;
  apt_packed* out;
  float* scale;
  int32_t* range_error;
} apt_pack_problem;
APT_API apt_status apt_pack_grouped(int32_t count, const apt_pack_problem* problems /* host */, void* stream);

/* Per-channel / per-token fp32 scales for APT_OUT_F16_SCALED (reading Q10):
 *   out[m][n] = RN_fp16( ((float)Y[m][n] * w_scale[n]) * a_scale[m] ), fp32 arithmetic,
 *   one final round-to-nearest-even to fp16 (overflow -> +-inf).
 * Optional zero points (linear quantization x = s x_hat + z of P:199-201 on both
 * operands: activations a_scale[m] x_hat + a_zero[m], weights w_scale[n] w_hat + w_zero[n]):
 *   v = ((float)Y * w_scale[n]) * a_scale[m];  v += ((float)RW[n] * w_scale[n]) * az;
 *   v += ((float)RA[m] * as) * wz;  v += ((float)K * az) * wz;  out = RN_fp16(v)
 * (az, wz = 0 where NULL; RW / RA the packed row sums).  With zero points the GEMM writes the exact
 * int32 Y into the workspace and a second elementwise pass applies the formula, so the workspace
 * must hold apt_gemm_zp_workspace_bytes(); without them nothing changes.  Zero points are ignored
 * for the int32 output kinds. */
/* Group-wise scales (the 128-group configurations of the paper's PPL table, P:655-656,
 * i.e. the linear quantization of P:199-201 applied per K-group g = k / 128), APT_OUT_F16_SCALED only:
 *   out[m][n] = RN_fp16( sum_g ((float)Y_g[m][n] * w_gscale[g][n]) * a_g[m] ),  Y_g = sum_{k in g} A W exact,
 *   a_g[m] = a_gscale[g][m] (or a_scale[m] / 1 when a_gscale is NULL), fp32 sums over g in order.
 * group_size = 128 selects it (0 = per-channel scales as above; w_scale is then ignored); zero points are
 * not combined with group scales.  w_gscale: fp32 [Kpad/128][N] (group-major, the GPTQ layout), a_gscale:
 * fp32 [Kpad/128][M] or NULL.  The GEMM computes every group's exact product on signed digits in the
 * grouped decode kernel (gemm_grp.cu; any M, in chunks of 16 tokens): W in the APT_PACK_TILED layout and A
 * with its digit view are required (else APT_ERR_UNSUPPORTED), and the workspace must hold
 * apt_gemm_grouped_workspace_bytes(1) (else APT_ERR_WORKSPACE).
 * Zero points at M <= 16 with a tiled W, a digit-view A, no forced config and such a workspace are fused
 * into the same kernel's epilogue (one launch, the formula above evaluated identically). */
typedef struct {
  const float* w_scale;  /* [N], required for APT_OUT_F16_SCALED unless group_size != 0 */
  const float* a_scale;  /* [M] per token, or NULL (== 1)        */
  const float* w_zero;   /* [N] per output channel, or NULL (== 0) */
  const float* a_zero;   /* [M] per token, or NULL (== 0)          */
  const float* w_gscale; /* [Kpad/128][N] group scales (group_size == 128), else NULL */
  const float* a_gscale; /* [Kpad/128][M] or NULL                  */
  int32_t group_size;    /* 0 (per channel) or 128                 */
} apt_scales;

typedef enum {
  APT_OUT_I32_SIGNED = 0,  /* int32 Y  = A . W^T over signed codes (reading Q1, default)        */
  APT_OUT_I32_BIPOLAR = 1, /* int32 Y' = A' . W'^T over bipolar values (Fig. 4)          */
  APT_OUT_F16_SCALED = 2   /* fp16 scaled Y (needs scales->w_scale)                             */
} apt_out_kind;

typedef enum {
  APT_LAYOUT_ROW = 0, /* out[m * ldo + n], ldo >= N                                       */
  APT_LAYOUT_COL = 1  /* out[n * ldo + m] = Y^T, ldo >= M (contiguous N-slices for the TP gather) */
} apt_layout;

typedef enum {
  APT_KERNEL_AUTO = 0,
  /* 1 was APT_KERNEL_MMA_SPLITK (ABI <= 2, removed: never selected, superseded by APT_KERNEL_SKINNY) */
  APT_KERNEL_TC = 2,         /* tcgen05 kind::i8 kernel: weights rebuilt in registers -> TMEM (A operand),
                                tokens via TMA from the int8 token workspace, s32 accumulator in TMEM */
  APT_KERNEL_GEMV = 3,       /* M <= 4: SIMT GEMV, weights rebuilt in registers (same u8 digits), dp4a
                                against the activation digit view; 32 weight rows x all of K per CTA
                                (bm = 32, bn = M, bk = 128, split_k = 8 or 16 warps, stages = 1)  */
  APT_KERNEL_SKINNY = 4,     /* M <= 16 per token tile: mma.sync m16n8k32 u8 fed from registers (weights
                                rebuilt in registers, tokens from the digit view), 16 weight rows x
                                bn (8 or 16) tokens x all of K per CTA (bm = 16, bk = 256,
                                split_k = 4, 8 or 16 warps splitting K, stages = 1)                */
  APT_KERNEL_DEC = 5,        /* M <= 16: mma.sync m16n8k32 u8 with the WEIGHTS as the streamed B operand
                                (8 rows x 32 K per instruction) and the tokens as the A operand (held in
                                registers, loaded from a per-CTA shared-memory slab); weights copied into a
                                per-lane shared-memory ring with cp.async.  bm = 128 weight rows per CTA of
                                4 warps, bn = 8 (M <= 8) or 16, bk = 256, stages = ring depth (16 for
                                wbits <= 2, 8 for 3-4, 4 above), split_k = CTAs along K (1..32, at most
                                16 blocks of 256 K per CTA; > 1 uses the workspace: int32 partials + one
                                ticket per row tile, see apt_gemm_workspace_bytes).  Needs
                                Kpad * 255 * 255 < 2^32 (digits are rebuilt as u * 2^s). */
  APT_KERNEL_PF = 6          /* persistent tcgen05 GEMM for token-rich shapes: one CTA per SM walks the 128 x bn
                                tiles, every ring continues across tiles, the TMEM accumulator is double-buffered
                                so dedicated epilogue warps overlap the next tile's MMAs.  bm 128, bk 128,
                                split_k 1, cluster_n 1; bn 128 (stages 6; mma_kind i8 or mxf4 with wbits,
                                abits <= 3), bn 192 (stages 4, i8) or bn 256 (stages 3, i8: weight digits staged
                                in shared memory).  i8 needs Kpad * 255 * 255 < 2^31.  The analytic choice for
                                M > 64.                                                                         */
} apt_kernel;

/* Kernel configuration (the B200 analogue of the paper's tunable hyperparameters, §5.1).
 *   kernel   : apt_kernel
 *   w_digit, a_digit : digit widths of the operand rebuild; this build uses full width (= bits),
 *                      one MMA pass for every p, q <= 8
 *   bm       : weight rows per CTA tile (MMA M side)
 *   bn       : tokens per CTA tile (MMA N side)
 *   bk       : K elements per pipeline step
 *   stages   : pipeline depth (TC kernel)
 *   split_k  : K splits (TC kernel: CTAs of a (1,1,S) cluster, 1..8; GEMV / SKINNY: warps per CTA)
 *   cta_pair : 1 = cta_group::2 pairs (TC kernel), 0 = single CTA (this build: 0)
 *   cluster_n: TC kernel: CTAs along N (weight tiles) sharing one token tile; the token tile is loaded
 *              once per cluster with TMA multicast (1, 2 or 4)
 *   mma_kind : tensor-core operand kind (apt_mma_kind)                                                  */
typedef enum {
  APT_MMA_I8 = 0,   /* u8 x u8 -> s32 digits (tcgen05 kind::i8 / mma.sync u8 / dp4a)                  */
  APT_MMA_MXF4 = 1  /* signed codes as e2m1 (fp4) digits, tcgen05 kind::mxf4 with unit UE8M0 block scales,
                       f32 accumulator (exact: every partial sum is an integer below 2^24), twice the i8
                       MMA rate.  wbits, abits <= 3 (signed {-4..3} is a subset of e2m1); APT_KERNEL_TC
                       only, bn 128 / 256, split_k 1, cluster_n 1, Kpad * 16 < 2^24.  Tokens are expanded
                       from the activation planes into the workspace's expansion area (the digit view is
                       not used), so the workspace is required (apt_gemm_workspace_bytes).           */
} apt_mma_kind;

typedef struct {
  int32_t kernel, w_digit, a_digit, bm, bn, bk, stages, split_k, cta_pair, cluster_n, mma_kind;
} apt_config;

/* Host, deterministic for a given loaded table (see apt_table_load; the analytic rules below when no
 * legal table row applies).
 * p = wbits, q = abits as in the north_star's "W_p x A_q".  Analytic rules (measured on B200):
 *   M <= 2       -> APT_KERNEL_GEMV, 16 warps per CTA if ceil(N/32) <= 148 else 8;
 *   M <= 8, K <= 4096 -> APT_KERNEL_SKINNY, bn 8, 8 warps per CTA if ceil(N/16) <= 296 else 4;
 *   M <= 64      -> APT_KERNEL_TC decode tile (bn 16 for M <= 16 else 64), K split over a cluster so that
 *                   about two CTAs per SM stream weights (<= 16 K steps per CTA at bn 16);
 *   M > 64       -> APT_KERNEL_TC, bn 256, one CTA per SM, no cluster.
 * Errors: APT_ERR_INVALID_ARGUMENT (dims <= 0, bits outside [1,8], null out),
 *         APT_ERR_UNSUPPORTED (int32 bound, reading Q8). */
APT_API apt_status apt_select_config(int32_t M, int32_t N, int32_t K, int32_t wbits, int32_t abits,
                             apt_config* out /* host */);

/* Autotuned configuration table (the paper's lookup table, Best Kernel Search and
 * Approximate Matching, §5.2).  Host-only, thread-safe (one mutex-guarded table per process).
 * File format: text, '#' comments, one row per key:
 *   M N K wbits abits  kernel w_digit a_digit bm bn bk stages split_k cta_pair cluster_n mma_kind  us
 * (the apt_config fields in declaration order, then the measured time in microseconds).  tools/tune.py
 * writes it by timing every config apt_enumerate_configs returns.
 * apt_select_config consults the table first: the exact key, else the nearest key by
 *   d = |log2 M - log2 M'| + |log2 N - log2 N'| + |log2 K - log2 K'|
 * among rows of the same token regime (M <= 16, M <= 64, M > 64) with the same (wbits, abits) (any row of
 * that regime if none has them; no match if the regime has no row), ties -> smaller measured time, then
 * smaller key; the row's config is returned only if it is legal for the queried shape, else the analytic
 * rules decide.  Rows loaded later replace earlier rows with the same key.
 * apt_table_load: APT_ERR_INVALID_ARGUMENT for a missing file or a malformed row (nothing is loaded then).
 * apt_table_lookup: the nearest row's stored config and its distance (0 = exact);
 *   APT_ERR_UNSUPPORTED if the table is empty. */
APT_API apt_status apt_table_load(const char* path /* host */);
APT_API void apt_table_clear(void);
APT_API int32_t apt_table_size(void);
APT_API apt_status apt_table_lookup(int32_t M, int32_t N, int32_t K, int32_t wbits, int32_t abits,
                                    apt_config* out /* host */, double* distance /* host, nullable */);
/* Host.  The search space of the Best Kernel Search: every config legal for (M, N, K, wbits, abits)
 * (GEMV warps 8/16; SKINNY bn 8/16 x warps 4/8/16; DEC warps 4/8 x split 1,2,3,4,6,8; TC bn 16/64/128/256 x
 * cluster 1/2/4 x split 1..8; TC kind::mxf4 bn 128/256 when wbits, abits <= 3), in that order.  Writes up to `cap` of them to `out` (nullable) and returns
 * how many exist (0 for invalid arguments or the int32 bound). */
APT_API int32_t apt_enumerate_configs(int32_t M, int32_t N, int32_t K, int32_t wbits, int32_t abits,
                                      apt_config* out /* host */, int32_t cap);

/* Host.  Device workspace bytes apt_gemm needs for (cfg, M, N, K).
 * Layout: [APT_WS_TICKET_BYTES of split-K tickets at offset 0 — the same place for every call]
 * [token digit expansion, M * Kpad bytes, used when the activation operand has no digit view]
 * [APT_KERNEL_DEC split-K int32 partials].  The ticket area must be ZERO before a workspace is first used
 * (e.g. one cudaMemsetAsync after allocation); every apt_gemm call leaves it zero again, so one workspace
 * serves any sequence of calls on a stream.  Calls that may run concurrently (different streams) need
 * distinct workspaces.  A call that needs no workspace (digit-view activations, no split-K, no zero
 * points) accepts NULL. */
#define APT_WS_TICKETS 4096
#define APT_WS_TICKET_BYTES (APT_WS_TICKETS * 4)
APT_API size_t apt_gemm_workspace_bytes(const apt_config* cfg, int32_t M, int32_t N, int32_t K);

/* Host.  Device workspace bytes apt_gemm needs for (cfg, M, N, K) when the scales carry zero points
 * (fp16 output): the apt_gemm_workspace_bytes area rounded up to 16 bytes, then int32 Y [M][N]. */
APT_API size_t apt_gemm_zp_workspace_bytes(const apt_config* cfg, int32_t M, int32_t N, int32_t K);

/* The W_p x A_q GEMM (§3.2 + §4.2): out = epilogue(A . W^T), exact in int32.
 *   W, A      : host structs describing device buffers produced by apt_pack_bipolar
 *               (W->rows == N, A->rows == M, W->k == A->k == K, W->bits == wbits, A->bits == abits).
 *   scales    : host struct (nullable unless kind == APT_OUT_F16_SCALED).
 *   out       : int32 (I32 kinds) or fp16 (F16 kind) buffer in `layout` with leading dimension ldo.
 *   cfg       : host, NULL -> apt_select_config.
 *   workspace : device scratch of apt_gemm_workspace_bytes(cfg, M, N, K) bytes (nullable if 0).
 * Bound (reading Q8): requires Kpad * (2^abits - 1) * (2^wbits - 1) < 2^31, else APT_ERR_UNSUPPORTED.
 * Errors: APT_ERR_INVALID_ARGUMENT (also: W->digits != NULL, see "General contract"),
 *         APT_ERR_UNSUPPORTED, APT_ERR_WORKSPACE, APT_ERR_CUDA. */
APT_API apt_status apt_gemm(int32_t M, int32_t N, int32_t K, int32_t wbits, int32_t abits, const apt_packed* W,
                    const apt_packed* A, const apt_scales* scales, apt_out_kind kind, apt_layout layout,
                    void* out, int64_t ldo, const apt_config* cfg, void* workspace, size_t ws_bytes,
                    void* stream);

/* Grouped decode GEMM: `count` INDEPENDENT W_p x A_q products in one persistent launch (the projections
 * of a decoder layer that share no data dependency, the experts of a mixture-of-experts layer, a batch of
 * decode linears).  Each problem's result is bit-identical to apt_gemm on the same arguments (same
 * digit rebuild, products and epilogue as APT_KERNEL_DEC; P:223-228 for the product, P:201 for the
 * scales); what differs is the schedule: the warps of one grid split the SUM of all problems' packed
 * weight blocks (32 rows x 256 K) into equal-cost contiguous ranges (stream-K), so weights stream
 * through one continuous pipeline with no launch boundary between problems (DESIGN.md §7 "Grouped").
 * Per problem (apt_gemm_problem, host array):
 *   M in [1, 16]; W = apt_pack_bipolar output in APT_PACK_TILED layout without a digit view; A = an
 *   APT_PACK_ROWS activation WITH its digit view; kind / layout / out / ldo / scales as apt_gemm
 *   (zero points fused into the epilogue; group-wise scales: every problem of the call with
 *   group_size 128, or none); 1 <= wbits, abits <= 8 and
 *   Kpad * 255 * 255 < 2^32 (the digits are u * 2^s).
 * The problems must not overlap: no problem's `out` may alias another problem's inputs or output.
 *   workspace : device, >= apt_gemm_grouped_workspace_bytes(count), 16-byte aligned; its first
 *               APT_WS_TICKET_BYTES are the same zero-initialised ticket area as apt_gemm's (one
 *               workspace serves both kinds of call on one stream).
 * Errors: APT_ERR_INVALID_ARGUMENT (count outside [1, APT_GROUP_MAX], a problem violating the above),
 *         APT_ERR_UNSUPPORTED (int32 bound), APT_ERR_WORKSPACE, APT_ERR_CUDA. */
/* Epilogue-direct peer stores (SURVEY §8f NEXT-4 ii): every output element is also written, at the same
 * byte offset, to out_peers[0 .. n_peers-1] (device pointers valid on the calling device, e.g. NVLink
 * peer mappings of a symmetric-memory buffer).  With out pointing at a rank's own slice of a gathered
 * tensor parallel output, the GEMM itself is the all-gather: no staging copy, no collective launch.  The
 * stores are plain weak global stores; the caller makes them visible to the peers (e.g. a symmetric-
 * memory barrier after the call, stream-ordered). */
#define APT_MAX_PEERS 7
typedef struct {
  int32_t M, N, K, wbits, abits;
  apt_packed W;
  apt_packed A;
  apt_scales scales;
  int32_t kind;   /* apt_out_kind */
  int32_t layout; /* apt_layout   */
  void* out;
  int64_t ldo;
  void* out_peers[APT_MAX_PEERS];
  int32_t n_peers; /* 0 .. APT_MAX_PEERS */
} apt_gemm_problem;
APT_API size_t apt_gemm_grouped_workspace_bytes(int32_t count);
APT_API apt_status apt_gemm_grouped(int32_t count, const apt_gemm_problem* problems /* host */, void* workspace,
                                    size_t ws_bytes, void* stream);

/* Ablation only (the paper's "Basic" design, §6.5): recovery in global
 * memory.  parts: int32 [abits * wbits][part_stride], part (i, j) at offset (i * wbits + j) * part_stride
 * holds the plane-pair product Y^(i,j) = sum_k (2 a_i - 1)(2 w_j - 1) of activation plane i and weight
 * plane j (e.g. apt_gemm of the 1-bit planes with APT_OUT_I32_BIPOLAR); writes
 *   out[e] = sum_{i, j} 2^(i + j) parts[(i * wbits + j) * part_stride + e]   (mod 2^32)
 * for e < count, i.e. the bipolar product Y' of the full codes.  The product path never uses this (its
 * shift-add is folded into the operand rebuild); it exists to measure what the folding saves.
 * Errors: APT_ERR_INVALID_ARGUMENT, APT_ERR_CUDA. */
APT_API apt_status apt_recombine_plane_products(const int32_t* parts, int32_t abits, int32_t wbits, int64_t part_stride,
                                                int64_t count, int32_t* out, void* stream);

/* Host.  Human-readable name of a status code (static storage). */
APT_API const char* apt_status_string(apt_status s);

/* Host.  ABI version (APT_ABI_VERSION) of the loaded library. */
APT_API int32_t apt_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* APT_H_ */
