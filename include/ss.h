/*
 * ss.h -- C ABI of the B200 (sm_100a) sliding-window-sum library `libss.so`,
 * the data-parallel hot path of arXiv 2305.16513 ("sliding window sums" for
 * DNN pooling and convolution).  Implementation: paper_2305_16513_b200/csrc/.
 *
 * The operation (Sec. 2.2, Eq. 3):
 *     y_i = x_i (+) x_{i+1} (+) ... (+) x_{i+w-1}      ("exactly w addends")
 * for (+) in {+, max} (Sec. 2.3: average / max pooling) and
 * the sliding dot product (Sec. 2.4-2.5: convolution with a
 * length-k filter), evaluated directly on the unmodified input (no im2col,
 * PAPER.md l.17-19).  2-D pooling is the multi-dimensional extension named in
 * the Conclusion, computed separably (row pass, then column
 * pass).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  Pointers   x, y are DEVICE pointers (cudaMalloc / torch CUDA memory) on the
 *             current CUDA device; `filter_host` is a HOST pointer.  The
 *             caller owns all memory.  x and y must not overlap.  Any
 *             element-aligned pointer is accepted (16-byte-aligned buffers
 *             take the fastest path).  Reads may touch the bytes of the
 *             16-byte granules that contain x's first and last element; they
 *             are never written.
 *  Layout     1-D: x is [batch][N] row-major contiguous (row pitch N);
 *             y is [batch][out_len] contiguous, out_len = ss_out_len(N,w,s).
 *             2-D: x is [planes][H][W], y is [planes][OH][OW], contiguous.
 *             Valid padding: output i covers x[i*s .. i*s+w-1] (DESIGN.md
 *             readings R1-R4); the *_ex calls below add dilation and zero
 *             padding.
 *  Sizes      int64_t throughout (N = 2^32 is supported).
 *  Stream     `stream` is a cudaStream_t passed as void* (NULL = the legacy
 *             default stream).  Every call only ENQUEUES work on `stream`
 *             and returns; there is no implicit synchronisation.  Calls on
 *             different streams may run concurrently (no global mutable
 *             device state; no __constant__ writes).
 *  Errors     A non-OK status means NOTHING was enqueued: all arguments are
 *             validated before any launch.  SS_ERR_CUDA reports a launch
 *             failure (detail in ss_last_error()).  Asynchronous faults
 *             surface at the caller's next synchronisation.  The library
 *             never aborts, throws or prints.
 *  Memory     The library allocates no device memory and keeps no per-call
 *             or cross-call device state; it caches per-device attributes
 *             (SM count, kernel smem attributes) only.  The persistent
 *             kernels distribute their tiles dynamically by cluster launch
 *             control (the grid has one CTA per tile; running CTAs cancel
 *             pending CTAs and take their tiles), so the claim state lives
 *             in the hardware scheduler of each launch: concurrent calls,
 *             CUDA-graph captures (including a first call made inside a
 *             capture) and concurrent graph replays are independent.  Calls
 *             that need scratch (the filter gradients) take a caller-owned
 *             workspace.
 *  Numerics   int32 + wraps modulo 2^32.  fp32 uses IEEE round-to-nearest
 *             FMA/adds (no fast-math, no flush-to-zero), except the
 *             tensor-core conv1d path (see ss_conv1d).  max equals
 *             `a > b ? a : b` for finite inputs (NaN unsupported; the sign of
 *             a zero maximum is unspecified).  Results are bitwise
 *             deterministic run to run; max results and conv1d results
 *             with k <= 32 are also independent of tiling and sharding.
 *             fp32 results
 *             satisfy |y - y_exact| <= 1e-5 * sum_j |x_j f_j| + 1e-6
 *             (BASELINE.json north_star; f = 1 for sums, 1/(kh*kw) for avg).
 */
#ifndef SS_H
#define SS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_ABI_VERSION 13

typedef enum { SS_F32 = 0, SS_I32 = 1 } ss_dtype_t;
typedef enum { SS_POOL_MAX = 0, SS_POOL_AVG = 1 } ss_pool_mode_t;
/* Boundary extension of the window spec ("padding, mirroring,
 * or periodicity"): SS_PAD_ZEROS pads with the operator's identity (0 for sums
 * and dot products; never wins a max / min), SS_PAD_REFLECT mirrors about the
 * end elements without repeating them (x[-u] = x[u], x[N-1+u] = x[N-1-u]),
 * SS_PAD_CIRCULAR wraps (x[u mod N]), SS_PAD_REPLICATE repeats the end element. */
typedef enum { SS_PAD_ZEROS = 0, SS_PAD_REFLECT = 1, SS_PAD_CIRCULAR = 2, SS_PAD_REPLICATE = 3 } ss_pad_mode_t;

typedef enum {
  SS_OK = 0,
  SS_ERR_NULL = 1,                  /* a required pointer is NULL              */
  SS_ERR_BAD_SIZE = 2,              /* N/batch/w/k/stride/planes/H/W < 1, or a  */
                                    /* size whose byte count overflows int64    */
  SS_ERR_WINDOW_EXCEEDS_INPUT = 3,  /* w > N ("window exceeds"); */
                                    /* _ex: (w-1)*dilation+1 > N+pads           */
  SS_ERR_UNSUPPORTED = 4,           /* dtype/op combination not provided,      */
                                    /* or k > SS_K_MAX                          */
  SS_ERR_CUDA = 5,                  /* CUDA launch/attribute failure           */
  SS_ERR_OVERLAP = 6                /* x and y byte ranges overlap             */
} ss_status_t;

/* Largest conv1d filter length accepted. */
#define SS_K_MAX 1024

/* ABI version of the loaded library (== SS_ABI_VERSION it was built with). */
int ss_abi_version(void);

/* Valid-padding output length (N - w) / stride + 1 (Eq. 3 at stride 1 gives
 * N - w + 1); -1 if N < 1, w < 1, stride < 1 or w > N.  Pure host function. */
int64_t ss_out_len(int64_t N, int64_t w, int64_t stride);

/* Eq. 3 with (+) = + (average pooling is the sliding sum with
 * +).  Returns the RAW window sum (divide by w for the average; reading R5).
 * y[b][i] = sum_{j<w} x[b][i*stride + j].  dtype SS_I32 (wrapping) or SS_F32. */
ss_status_t ss_pool_sum(const void* x, void* y, int64_t N, int64_t batch,
                        int64_t w, int64_t stride, ss_dtype_t dtype, void* stream);

/* Eq. 3 with (+) = max (max pooling).
 * y[b][i] = max_{j<w} x[b][i*stride + j].  dtype SS_I32 or SS_F32. */
ss_status_t ss_pool_max(const void* x, void* y, int64_t N, int64_t batch,
                        int64_t w, int64_t stride, ss_dtype_t dtype, void* stream);

/* Eq. 3 with (+) = min ("min is associative", the sliding min
 * example).  y[b][i] = min_{j<w} x[b][i*stride + j].
 * dtype SS_I32 or SS_F32; exact (bitwise), same kernels as ss_pool_max. */
ss_status_t ss_pool_min(const void* x, void* y, int64_t N, int64_t batch,
                        int64_t w, int64_t stride, ss_dtype_t dtype, void* stream);

/* Sliding dot product = 1-D convolution with a length-k filter (PAPER.md
 * l.86-87, Sec. 2.5; Eq. 4 per window), cross-correlation orientation
 * (reading R2): y[b][i] = sum_{j<k} filter[j] * x[b][i*stride + j].
 * Accumulation (fp32):
 *   otherwise (k <= 32, strides > 1, longer dilated extents): fl(S_even + S_odd), S_even / S_odd FMA
 *     chains over the even / odd taps in increasing j from 0 -- fixed by the
 *     tap index alone, so every output is independent of tiling and sharding.
 *   33 <= k <= 64 at stride 1, and (conv1d_ex) dilated filters with
 *     (k-1)*dilation + 1 <= 64 at stride 1: tensor cores (Toeplitz matrix
 *     product): x f ~ xh fh (TF32, xh / fh = fp32 truncated to
 *     TF32) + bf16(xh) bf16(fl) + bf16(xl) bf16(fh) (one bf16 MMA), fp32
 *     accumulation; per-product error <= ~2^-18 |x f|, within the bound below
 *     (measured worst error / bound 0.27; environment SS_CONV_TC_MIXED=0 selects
 *     3xTF32, 0.08).  Bitwise deterministic run to run, but an output's
 *     rounding depends on its position modulo 8 in the 16-B-aligned view of x
 *     (tensor-core conv).
 * One filter shared by all rows.  `filter_host` (k floats, HOST memory) is read
 * before the call returns and may be freed immediately.  dtype must be SS_F32;
 * 1 <= k <= SS_K_MAX. */
ss_status_t ss_conv1d(const void* x, void* y, int64_t N, int64_t batch,
                      const float* filter_host, int64_t k, int64_t stride,
                      ss_dtype_t dtype, void* stream);

/* 2-D pooling, computed separably: a row sliding (+) over kw at stride sw,
 * then a column sliding (+) over kh at stride sh (PAPER.md l.53 operators,
 * l.226 multi-dimensional extension).  mode SS_POOL_MAX: max; SS_POOL_AVG:
 * window sum times 1/(kh*kw) (no padding, so every window has kh*kw terms).
 * x is [planes][H][W] (planes = N*C of an NCHW tensor), y is
 * [planes][(H-kh)/sh+1][(W-kw)/sw+1].  dtype must be SS_F32. */
ss_status_t ss_pool2d(const void* x, void* y, int64_t planes, int64_t H, int64_t W,
                      int64_t kh, int64_t kw, int64_t sh, int64_t sw,
                      ss_pool_mode_t mode, ss_dtype_t dtype, void* stream);

/* ---- window spec: stride, dilation, padding -------------
 * The input is logically extended by pad_left / pad_right positions:
 * xp[t] = x[t - pad_left] for 0 <= t - pad_left < N, otherwise by pad_mode
 * (ss_pad_mode_t above).  Output i of a row covers xp[i*stride + j*dilation],
 * j < w (or k), so
 *   out_len = (N + pad_left + pad_right - ((w-1)*dilation + 1)) / stride + 1
 * (SPEC.md l.263-268 WindowSpec).  SS_PAD_ZEROS: padding adds 0 to sums and dot
 * products and never wins a max or a min; a window made only of
 * padding yields the identity (0, -inf / INT32_MIN, +inf / INT32_MAX).
 * SS_PAD_REFLECT needs pad_left, pad_right <= N-1 and SS_PAD_CIRCULAR <= N
 * (one reflection / one period; else SS_ERR_BAD_SIZE); an unknown pad_mode is
 * SS_ERR_UNSUPPORTED.  dilation >= 1, pads >= 0; everything else, layout (y is
 * [batch][out_len]), errors, streams and numerics as for the valid-padding
 * calls above (which equal these with dilation 1, pads 0).  Stride 1 runs the
 * tile kernels (TMA tile kernel, dilated phase kernel or tensor cores) on the
 * interior outputs -- whose windows never touch padding, so they are the same
 * for every mode -- and a direct kernel on the pad_left + pad_right edge
 * outputs of each row. */
int64_t ss_out_len_ex(int64_t N, int64_t w, int64_t stride, int64_t dilation,
                      int64_t pad_left, int64_t pad_right);
ss_status_t ss_pool_sum_ex(const void* x, void* y, int64_t N, int64_t batch, int64_t w,
                           int64_t stride, int64_t dilation, int64_t pad_left,
                           int64_t pad_right, ss_pad_mode_t pad_mode, ss_dtype_t dtype, void* stream);
ss_status_t ss_pool_max_ex(const void* x, void* y, int64_t N, int64_t batch, int64_t w,
                           int64_t stride, int64_t dilation, int64_t pad_left,
                           int64_t pad_right, ss_pad_mode_t pad_mode, ss_dtype_t dtype, void* stream);
ss_status_t ss_pool_min_ex(const void* x, void* y, int64_t N, int64_t batch, int64_t w,
                           int64_t stride, int64_t dilation, int64_t pad_left,
                           int64_t pad_right, ss_pad_mode_t pad_mode, ss_dtype_t dtype, void* stream);
ss_status_t ss_conv1d_ex(const void* x, void* y, int64_t N, int64_t batch,
                         const float* filter_host, int64_t k, int64_t stride,
                         int64_t dilation, int64_t pad_left, int64_t pad_right,
                         ss_pad_mode_t pad_mode, ss_dtype_t dtype, void* stream);

/* ---- sliding window of gamma pairs --------------------
 * The paper's pair operator (Eq. 8)
 *     (u_i, v_i) (+) (u_j, v_j) = (u_i u_j, u_j v_i + v_j)
 * is associative and NOT commutative; slid over a sequence of pairs with
 * window w (Eq. 3) it gives, for output i of a row,
 *     (U_i, V_i) = gamma_{i*s} (+) gamma_{i*s+1} (+) ... (+) gamma_{i*s+w-1},
 *     U_i = prod_j u_j,   V_i = sum_j v_j prod_{l > j in the window} u_l,
 * the recurrence s_t = u_t s_{t-1} + v_t run over each window from s = 0 (V)
 * and its gain (U): exponentially weighted / decaying windowed sums,
 * windowed first-order IIR filters, and Eq. 9's dot product when u, v come
 * from Eq. 7.  u, v are DEVICE [batch][N] fp32 (planar: one array per pair
 * component); U, V are DEVICE [batch][L], L = ss_out_len(N, w, stride).
 * U may be NULL (V only).  No argument may overlap another output.
 * Numerics: fp32 with one rounding per product and one per FMA; the
 * evaluation order is a fixed tree of (+) (left-to-right order preserved), so
 *     |V - V_exact| <= 2 w 2^-24 sum_j |v_j| prod_{l>j} |u_l| + 1e-6
 *     |U - U_exact| <= 2 w 2^-24 |U_exact| + 1e-30   (reading R15).
 * Stride 1 costs O(1) (+) per output for any w (two-level P-block pivot);
 * stride > 1 folds each window directly (O(w) per output).
 * Statuses as above; w > SS_AFFINE_W_MAX -> SS_ERR_UNSUPPORTED. */
#define SS_AFFINE_W_MAX 65536
ss_status_t ss_affine_window(const float* u, const float* v, float* U, float* V, int64_t N,
                             int64_t batch, int64_t w, int64_t stride, void* stream);

/* ---- 2-D convolution (multi-dimensional extension, l.226) --
 * Single-channel 2-D sliding dot product (cross-correlation, valid padding,
 * DESIGN.md reading R17):
 *   y[p][r][c] = sum_{a<kh} sum_{b<kw} filter[a*kw + b] * x[p][r*sh + a][c*sw + b]
 * x is [planes][H][W], y is [planes][(H-kh)/sh+1][(W-kw)/sw+1] (DEVICE, 4-byte
 * aligned); filter_host is kh*kw floats in HOST memory (row-major), read before
 * the call returns; kh*kw <= SS_K_MAX.  fp32, each output's products
 * accumulated with FMA in row-major tap order (deterministic, tiling-
 * independent).  Statuses as ss_pool2d. */
ss_status_t ss_conv2d(const void* x, void* y, int64_t planes, int64_t H, int64_t W,
                      const float* filter_host, int64_t kh, int64_t kw, int64_t sh, int64_t sw,
                      ss_dtype_t dtype, void* stream);

/* Gradients of ss_conv2d (SURVEY 8f NEXT #4 "2-D convolution and backward
 * passes"; the vector-Jacobian products, reading R21).  Shapes as
 * ss_conv2d: x / dx [planes][H][W], dy [planes][OH][OW], all DEVICE fp32
 * (SS_F32 only), 4-byte aligned, dx / df must not overlap an input.
 *   ss_conv2d_backward_input   dx[p][h][w] = sum over windows (r, c) and taps
 *                              (a, b) with r*sh + a = h, c*sw + b = w of
 *                              filter[a*kw + b] * dy[p][r][c]; elements no
 *                              window covers are written 0.  filter_host: HOST,
 *                              kh*kw <= SS_K_MAX floats, read before return.
 *   ss_conv2d_backward_filter  df[a*kw + b] = sum_p sum_r sum_c dy[p][r][c] *
 *                              x[p][r*sh + a][c*sw + b]  (df: DEVICE, kh*kw
 *                              floats; fp32 products summed in fp32 runs of one
 *                              tile, then fp64, deterministic).  `workspace`
 *                              (DEVICE, caller-owned, >= ss_conv2d_backward_
 *                              filter_workspace(kh, kw) bytes on the current
 *                              device) holds per-CTA fp64 partials.
 * Accuracy: |g - g_exact| <= 1e-5 * sum of |term| + 1e-6 per element (BJ bound).
 * Statuses as ss_conv2d; a short workspace -> SS_ERR_BAD_SIZE. */
ss_status_t ss_conv2d_backward_input(const void* dy, void* dx, int64_t planes, int64_t H, int64_t W,
                                     const float* filter_host, int64_t kh, int64_t kw, int64_t sh,
                                     int64_t sw, ss_dtype_t dtype, void* stream);
size_t ss_conv2d_backward_filter_workspace(int64_t kh, int64_t kw);
ss_status_t ss_conv2d_backward_filter(const void* x, const void* dy, float* df, int64_t planes, int64_t H,
                                      int64_t W, int64_t kh, int64_t kw, int64_t sh, int64_t sw,
                                      void* workspace, size_t workspace_bytes, void* stream);

/* ---- multi-channel convolution (a real contraction) -------
 * y[b][i][co] = sum_{j<k} sum_{ci<cin} w[co][ci][j] * x[b][i+j][ci],  i < N-k+1
 * (the Sec. 2.5 sliding dot product summed over input channels; DESIGN.md
 * reading R18).  Channels-last: x is [batch][N][cin] bfloat16, w is
 * [cout][cin][k] bfloat16 (torch conv1d weight order), y is [batch][N-k+1][cout]
 * fp32, all DEVICE memory.  bf16 products are exact; accumulation is fp32.
 * cin, cout in {64, 128}, k <= 9 with 16-B aligned x / y run on the tensor cores
 * (kind::f16 MMAs, the tap shift is an operand start-address offset); other
 * shapes run a direct kernel (same definition).  Statuses as above. */
ss_status_t ss_conv1d_mc(const void* x, const void* w, float* y, int64_t batch, int64_t N,
                         int64_t cin, int64_t cout, int64_t k, void* stream);

/* Multi-channel 2-D convolution (the Conclusion's multi-dimensional extension,
 * PAPER.md l.226, of the channel-summed dot product above; reading R22):
 *   y[b][r][c][co] = sum_{a<kh} sum_{e<kw} sum_{ci<cin} w[co][ci][a][e] * x[b][r+a][c+e][ci]
 * for r < H-kh+1, c < W-kw+1 (valid padding, stride 1).  NHWC: x is
 * [batch][H][W][cin] bfloat16, w is [cout][cin][kh][kw] bfloat16 (torch conv2d
 * weight order), y is [batch][H-kh+1][W-kw+1][cout] fp32, all DEVICE memory.
 * bf16 products are exact; accumulation is fp32.  cin, cout in {64, 128},
 * kh*kw <= 64, (kh-1)*W + kw - 1 <= 1024 and 16-B aligned x / y run on the
 * tensor cores: positions are flat over the image rows, so tap (a, e) is the
 * staged tile shifted by a*W + e positions (no im2col); other shapes run a
 * direct kernel (same definition).  Statuses as above (kh > H or kw > W ->
 * SS_ERR_WINDOW_EXCEEDS_INPUT). */
ss_status_t ss_conv2d_mc(const void* x, const void* w, float* y, int64_t batch, int64_t H, int64_t W,
                         int64_t cin, int64_t cout, int64_t kh, int64_t kw, void* stream);

/* Input gradient of ss_conv2d_mc (reading R26):
 *   dx[b][r][c][ci] = sum_{a<kh} sum_{e<kw} sum_{co<cout} w[co][ci][a][e] * dy[b][r-a][c-e][co]
 * for r < H, c < W, terms with (r-a, c-e) outside the H-kh+1 x W-kw+1 output
 * absent.  dy is [batch][H-kh+1][W-kw+1][cout] bfloat16, w the forward's
 * [cout][cin][kh][kw] bfloat16, dx [batch][H][W][cin] fp32, fully overwritten;
 * all DEVICE memory, dx must not overlap dy or w.  It is the forward contraction
 * on dy zero-padded by kh-1 rows and kw-1 columns on each side with the weights
 * transposed and flipped: cin, cout in {64, 128}, kh*kw <= 64 and 16-B aligned
 * dy / dx run on the tensor cores (tiles of R dx rows x Cw columns, staged as one
 * 5-D TMA box per 64 channels whose zero fill is the padding, no padded copy);
 * other shapes (or tilings that do not fit shared memory) run a direct kernel.
 * bf16 products are exact, accumulation is fp32.  Statuses as ss_conv2d_mc
 * (kh > H or kw > W -> SS_ERR_WINDOW_EXCEEDS_INPUT). */
ss_status_t ss_conv2d_mc_backward_input(const void* dy, const void* w, float* dx, int64_t batch, int64_t H,
                                        int64_t W, int64_t cin, int64_t cout, int64_t kh, int64_t kw, void* stream);

/* Filter gradient of ss_conv2d_mc (reading R27):
 *   dw[co][ci][a][e] = sum_b sum_{r < H-kh+1} sum_{c < W-kw+1} dy[b][r][c][co] * x[b][r+a][c+e][ci].
 * dy is [batch][H-kh+1][W-kw+1][cout] bfloat16, x the forward's [batch][H][W][cin]
 * bfloat16, dw [cout][cin][kh][kw] fp32 (torch weight order), fully overwritten; all
 * DEVICE memory.  workspace: caller-owned device memory of at least
 * ss_conv2d_mc_backward_filter_workspace(cin, cout, kh, kw) bytes (8-byte aligned;
 * may be NULL when that is 0), not overlapping dy, x or dw; its contents are
 * scratch.  cin = 64 with cout = 64 (kw <= 4) or 128 (kw <= 2), kh <= 64, W <= 128
 * and 16-B aligned dy / x run on the tensor cores: a tile is R = floor(128 / W) dy
 * rows staged with pitch W (the 5-D TMA box runs past the row's W-kw+1 outputs and
 * zero-fills) against the x rows the tap row reads, as the 1-D filter gradient
 * below, with the CTAs split over the kh tap rows (cout = 64: tap rows a, a-1
 * share one M = 128 accumulator whose second dy atom is one image row down);
 * numerics as that function
 * (fp32 per 128-position tile and 32-tile run, fp64 across runs and CTAs, a
 * fixed order: deterministic).  Other shapes run a direct kernel (double).
 * Statuses as ss_conv2d_mc; workspace too small -> SS_ERR_BAD_SIZE. */
size_t ss_conv2d_mc_backward_filter_workspace(int64_t cin, int64_t cout, int64_t kh, int64_t kw);
ss_status_t ss_conv2d_mc_backward_filter(const void* dy, const void* x, float* dw, int64_t batch, int64_t H,
                                         int64_t W, int64_t cin, int64_t cout, int64_t kh, int64_t kw,
                                         void* workspace, size_t workspace_bytes, void* stream);

/* Input gradient of ss_conv1d_mc (the vector-Jacobian product of the channel-summed
 * sliding dot product; reading R23):
 *   dx[b][t][ci] = sum_{j<k} sum_{co<cout} w[co][ci][j] * dy[b][t-j][co],  t < N,
 * terms with t-j outside [0, N-k+1) absent.  dy is [batch][N-k+1][cout] bfloat16
 * (the forward output's gradient, rounded to bf16 like the forward's operands),
 * w is the forward's [cout][cin][k] bfloat16, dx is [batch][N][cin] fp32 and fully
 * overwritten; all DEVICE memory, dx must not overlap dy or w.  It is the forward
 * contraction on dy with the weights transposed and flipped, w'[ci][co][j] =
 * w[co][ci][k-1-j], over each row padded by k-1 zeros on both sides: cin, cout in
 * {64, 128}, k <= 9 and 16-B aligned dy / dx run on the tensor cores (the
 * padding is the TMA's zero fill of a 4-D box per row, no padded copy); other
 * shapes run a direct kernel.  bf16 products are exact, accumulation is fp32.
 * Statuses as ss_conv1d_mc (k > N -> SS_ERR_WINDOW_EXCEEDS_INPUT). */
ss_status_t ss_conv1d_mc_backward_input(const void* dy, const void* w, float* dx, int64_t batch, int64_t N,
                                        int64_t cin, int64_t cout, int64_t k, void* stream);

/* Filter gradient of ss_conv1d_mc (reading R25):
 *   dw[co][ci][j] = sum_b sum_{i < N-k+1} dy[b][i][co] * x[b][i+j][ci].
 * dy is [batch][N-k+1][cout] bfloat16, x the forward's [batch][N][cin] bfloat16, dw
 * [cout][cin][k] fp32 (torch weight order), fully overwritten; all DEVICE memory.
 * cin = 64 with cout = 64 (k <= 4) or 128 (k <= 2) and 16-B aligned dy / x run on the
 * tensor cores: per tile of 128 positions D[co][(j, ci)] += dy^T . x shifted by j rows
 * (both operands read MN-major straight from the activations), fp32 per tile, fp32 runs
 * of 32 tiles, fp64 beyond; `workspace` (DEVICE, caller-owned, 8-B aligned, >=
 * ss_conv1d_mc_backward_filter_workspace(cin, cout, k) bytes on the current device)
 * holds per-CTA fp64 partials summed in a fixed order -- deterministic.  Other shapes run
 * a direct kernel (products and sums in double; the workspace size is then 0 and
 * `workspace` may be NULL).  Tolerance 1e-5 * sum|terms| + 1e-6.  Statuses as
 * ss_conv1d_mc; a short workspace -> SS_ERR_BAD_SIZE. */
size_t ss_conv1d_mc_backward_filter_workspace(int64_t cin, int64_t cout, int64_t k);
ss_status_t ss_conv1d_mc_backward_filter(const void* dy, const void* x, float* dw, int64_t batch, int64_t N,
                                         int64_t cin, int64_t cout, int64_t k, void* workspace,
                                         size_t workspace_bytes, void* stream);

/* ---- backward passes (training) ----------
 * Vector-Jacobian products of the forward calls above (DESIGN.md reading
 * R16): given dy = dLoss/dy (the forward output's shape, [batch][L] with
 * L = ss_out_len(N, w or k, stride)), write dx = dLoss/dx ([batch][N], fully
 * overwritten: positions no window touches get 0) or df.  Each result is a
 * gather over the windows touching an output position in increasing window
 * order (no atomics): bitwise deterministic.  Errors, streams and ownership
 * as above; dx / df must not overlap any input.  Stride-1 sum and conv input
 * gradients run the forward kernels on dy zero-padded by w-1 (k-1) with the
 * filter flipped, so their numerics are the forward ones.
 *
 *   ss_pool_sum_backward   dx_t = sum_{i: i*s <= t < i*s+w} dy_i.  SS_F32 or SS_I32 (wraps).
 *   ss_pool_max_backward   dx_t = sum of dy_i over the windows whose FIRST maximum
 *                          (left-to-right, replaced on strictly greater) is x_t.
 *                          x = the forward input.  SS_F32 only.
 *   ss_conv1d_backward_input   dx_t = sum_{(i,j): i*s+j = t} f_j dy_i.  SS_F32.
 *   ss_conv1d_backward_filter  df_j = sum_b sum_i dy[b][i] x[b][i*s+j]  (df: DEVICE,
 *                          k floats; fp32 products summed in fp32 runs of 64, then
 *                          fp64.  Stride 1, k <= 64, N % 128 == 0 and 16-B aligned x
 *                          run on the tensor cores (reading R24): the same
 *                          products regrouped by chunks of 128 dy positions, 3xTF32
 *                          (~2^-21 relative each), fp32 over <= 128 chunks, then fp64;
 *                          also deterministic, within the same bound).  `workspace` (DEVICE, caller-owned,
 *                          >= ss_conv1d_backward_filter_workspace(k) bytes on the
 *                          current device) holds per-CTA fp64 partials.
 *   ss_pool2d_backward     [planes][H][W] gradient of ss_pool2d: avg spreads
 *                          dy/(kh*kw) over each window; max routes dy to the window's
 *                          first maximum in row-major order (x may be NULL for avg).
 */
ss_status_t ss_pool_sum_backward(const void* dy, void* dx, int64_t N, int64_t batch, int64_t w,
                                 int64_t stride, ss_dtype_t dtype, void* stream);
ss_status_t ss_pool_max_backward(const void* x, const void* dy, void* dx, int64_t N, int64_t batch,
                                 int64_t w, int64_t stride, ss_dtype_t dtype, void* stream);
ss_status_t ss_conv1d_backward_input(const void* dy, void* dx, int64_t N, int64_t batch,
                                     const float* filter_host, int64_t k, int64_t stride,
                                     ss_dtype_t dtype, void* stream);
size_t ss_conv1d_backward_filter_workspace(int64_t k);
ss_status_t ss_conv1d_backward_filter(const void* x, const void* dy, float* df, int64_t N,
                                      int64_t batch, int64_t k, int64_t stride, void* workspace,
                                      size_t workspace_bytes, void* stream);
ss_status_t ss_pool2d_backward(const void* x, const void* dy, void* dx, int64_t planes, int64_t H,
                               int64_t W, int64_t kh, int64_t kw, int64_t sh, int64_t sw,
                               ss_pool_mode_t mode, ss_dtype_t dtype, void* stream);

/* Static description of a status code. */
const char* ss_status_string(ss_status_t s);
/* Thread-local detail for the last non-OK status returned on this thread
 * ("" if none).  Valid until the next ss_* call on the same thread. */
const char* ss_last_error(void);

/* Number of kernel launches the library has enqueued in this process (all
 * threads).  Used by bench.py to report `gpu_launches`. */
uint64_t ss_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SS_H */
