/*
 * oracle.h -- plain, slow, obviously-correct CPU oracle for the sliding-window
 * sum hot path of arXiv 2305.16513 ("sliding window sums" for DNN pooling and
 * convolution).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (include/ss.h, paper_2305_16513_b200/) never links, imports or
 * calls it, and this file shares no code, header, table or helper with it.
 *
 * Every routine is the plain definition from the paper written out as loops,
 * accumulating in int64 (integer inputs) or double (float inputs), with no
 * blocking, fusion or reordering:
 *
 *   Eq. 3 (Sec. 2.2):  y_i = x_i (+) x_{i+1} (+) ... (+) x_{i+w-1}
 *       "each sum ... contains exactly w addends"; naive O(wN).
 *   Sec. 2.3: average pooling = sliding sum with +,
 *       max pooling = sliding sum with max.
 *   Eq. 4 + Sec. 2.5: convolution is a
 *       sliding dot product: y_i = sum_{j<k} f_j x_{i+j}.
 *   Eq. 5-9: dot product as a prefix sum of gamma pairs.
 *   Conclusion: multi-dimensional extension -> 2-D pooling.
 *
 * Readings where the paper is silent (DESIGN.md "Readings" R1-R8):
 *   - stride s (R4): output i covers x[i*s .. i*s+w-1]; out_len = (N-w)/s + 1.
 *   - valid padding only (R3); cross-correlation orientation (R2).
 *   - pool2d avg divides the window sum by kh*kw (R5); pool_sum returns the raw sum.
 *
 * Layout: x is [batch][N] row-major contiguous; y is [batch][out_len].
 *         pool2d: x is [planes][H][W], y is [planes][OH][OW].
 * absmag[o] = sum over the window of |x_j * f_j| (f = 1 for sums,
 *         f = 1/(kh*kw) for avg) -- the scale of the fp32 error bound in
 *         BASELINE.json north_star: |y - y_ref| <= 1e-5 * absmag + 1e-6.
 *         absmag may be NULL.
 * Return value: 0 on success, -1 on invalid arguments (nothing written).
 *
 * parity pins: tests/test_oracle_pins.py (every function below is pinned).
 */
#ifndef SS_ORACLE_H
#define SS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int64_t oracle_out_len(int64_t N, int64_t w, int64_t s);

/* Eq. 3 with (+) = +, int32 input, exact int64 window sums. */
int oracle_pool_sum_i32(const int32_t* x, int64_t N, int64_t batch, int64_t w,
                        int64_t s, int64_t* y);
/* Eq. 3 with (+) = +, fp32 input, double accumulation. */
int oracle_pool_sum_f32(const float* x, int64_t N, int64_t batch, int64_t w,
                        int64_t s, double* y, double* absmag);
/* Eq. 3 with (+) = max. */
int oracle_pool_max_i32(const int32_t* x, int64_t N, int64_t batch, int64_t w,
                        int64_t s, int32_t* y);
int oracle_pool_max_f32(const float* x, int64_t N, int64_t batch, int64_t w,
                        int64_t s, float* y);
/* Sec. 2.5: y[b][i] = sum_{j<k} f_j * x[b][i*s + j]  (double accumulation). */
int oracle_conv1d_f32(const float* x, int64_t N, int64_t batch, const float* f,
                      int64_t k, int64_t s, double* y, double* absmag);
/* 2-D pooling over a kh x kw window, stride (sh, sw); mode 0 = max, 1 = avg.
 * Direct 2-D window (NOT separable), so it is independent of the GPU design. */
int oracle_pool2d_f32(const float* x, int64_t planes, int64_t H, int64_t W,
                      int64_t kh, int64_t kw, int64_t sh, int64_t sw, int mode,
                      double* y, double* absmag);

/* Window spec with dilation and padding (SPEC.md l.263-268
 * WindowSpec, l.282 / l.332 pad semantics; PAPER.md l.158 names "padding,
 * mirroring, or periodicity" as the boundary conditions):
 *   xp[t] = x[t - pl] for 0 <= t - pl < N, else padding by `mode`:
 *     0 zeros (contributes 0 to sums and dot products, never wins a max or a
 *       min: a window made only of padding gives the identity),
 *     1 reflect (x[-u] = x[u], x[N-1+u] = x[N-1-u]; requires pl, pr <= N-1),
 *     2 circular (x[u mod N]; requires pl, pr <= N),
 *     3 replicate (the end element);
 *   output i covers xp[i*s + j*d], j < w;  extent E = (w-1)*d + 1;
 *   out_len = (N + pl + pr - E) / s + 1  (-1 if invalid or E > N + pl + pr).
 * Min is Sec. 2.3's other extremum ("min is associative"). */
int64_t oracle_out_len_ex(int64_t N, int64_t w, int64_t s, int64_t d, int64_t pl, int64_t pr);
int oracle_pool_sum_ex_i32(const int32_t* x, int64_t N, int64_t batch, int64_t w, int64_t s,
                           int64_t d, int64_t pl, int64_t pr, int mode, int64_t* y);
int oracle_pool_sum_ex_f32(const float* x, int64_t N, int64_t batch, int64_t w, int64_t s,
                           int64_t d, int64_t pl, int64_t pr, int mode, double* y, double* absmag);
int oracle_pool_max_ex_i32(const int32_t* x, int64_t N, int64_t batch, int64_t w, int64_t s,
                           int64_t d, int64_t pl, int64_t pr, int mode, int32_t* y);
int oracle_pool_max_ex_f32(const float* x, int64_t N, int64_t batch, int64_t w, int64_t s,
                           int64_t d, int64_t pl, int64_t pr, int mode, float* y);
int oracle_pool_min_ex_i32(const int32_t* x, int64_t N, int64_t batch, int64_t w, int64_t s,
                           int64_t d, int64_t pl, int64_t pr, int mode, int32_t* y);
int oracle_pool_min_ex_f32(const float* x, int64_t N, int64_t batch, int64_t w, int64_t s,
                           int64_t d, int64_t pl, int64_t pr, int mode, float* y);
int oracle_conv1d_ex_f32(const float* x, int64_t N, int64_t batch, const float* f, int64_t k,
                         int64_t s, int64_t d, int64_t pl, int64_t pr, int mode, double* y, double* absmag);

/* Sliding window of gamma pairs (Eq. 3 with the pair operator of Eq. 8; the
 * windowed linear recurrence s_t = u_t s_{t-1} + v_t):
 *   (U_i, V_i) = gamma_{i*s} (+) gamma_{i*s+1} (+) ... (+) gamma_{i*s+w-1},
 * folded left to right in double (Eq. 9's recurrence restricted to a window):
 *   U_i = prod_j u_j,  V_i = sum_j v_j prod_{l>j, l in window} u_l.
 * magV_i = sum_j |v_j| prod_{l>j} |u_l| (error-bound scale).  U and magV may be NULL. */
int oracle_affine_window(const float* u, const float* v, int64_t N, int64_t batch, int64_t w,
                         int64_t s, double* U, double* V, double* magV);

/* Eq. 8: gamma_i (+) gamma_j = (u_i*u_j, u_j*v_i + v_j). */
void oracle_gamma_combine(double ui, double vi, double uj, double vj,
                          double* u_out, double* v_out);
/* Eq. 5 + Eq. 7: build gamma_0..gamma_M (M+1 pairs) from a, b (length M). */
int oracle_gamma_sequence(const double* a, const double* b, int64_t M,
                          double* u, double* v);
/* Eq. 9: delta_M = gamma_0 (+) ... (+) gamma_M by the recurrence
 * delta_i = delta_{i-1} (+) gamma_i; returns v(delta_M) (the dot product),
 * and u(delta_M) in *u_out. */
double oracle_gamma_dot(const double* a, const double* b, int64_t M, double* u_out);

/* Backward passes (vector-Jacobian products of the forward definitions; SURVEY
 * 8f NEXT #4).  dy is [batch][L] (L = oracle_out_len), dx is [batch][N]; for
 * 2-D, dy is [planes][OH][OW] and dx [planes][H][W].  Results in double;
 * absmag (optional) = per-output sum of term magnitudes. */
int oracle_pool_sum_backward_f32(const float* dy, int64_t N, int64_t batch, int64_t w,
                                 int64_t s, double* dx, double* absmag);
int oracle_pool_max_backward_f32(const float* x, const float* dy, int64_t N, int64_t batch,
                                 int64_t w, int64_t s, double* dx);
int oracle_conv1d_backward_input_f32(const float* dy, int64_t N, int64_t batch, const float* f,
                                     int64_t k, int64_t s, double* dx, double* absmag);
int oracle_conv1d_backward_filter_f32(const float* x, const float* dy, int64_t N, int64_t batch,
                                      int64_t k, int64_t s, double* df, double* absmag);
int oracle_pool2d_backward_f32(const float* x, const float* dy, int64_t planes, int64_t H,
                               int64_t W, int64_t kh, int64_t kw, int64_t sh, int64_t sw,
                               int mode, double* dx, double* absmag);

/* 2-D single-channel sliding dot product (multi-dimensional extension,
 * PAPER.md l.226): y [planes][OH][OW] in double, absmag optional. */
int oracle_conv2d_f32(const float* x, int64_t planes, int64_t H, int64_t W, const float* f,
                      int64_t kh, int64_t kw, int64_t sh, int64_t sw, double* y, double* absmag);

/* Gradients of oracle_conv2d_f32 (reading R21): dx [planes][H][W] (scatter of
 * f[a][b] dy[p][r][c] to x[p][r*sh+a][c*sw+b]; elements no window covers get 0)
 * and df [kh][kw] = sum over planes and outputs of dy * x, both in double. */
int oracle_conv2d_backward_input_f32(const float* dy, int64_t planes, int64_t H, int64_t W, const float* f,
                                     int64_t kh, int64_t kw, int64_t sh, int64_t sw, double* dx, double* absmag);
int oracle_conv2d_backward_filter_f32(const float* x, const float* dy, int64_t planes, int64_t H, int64_t W,
                                      int64_t kh, int64_t kw, int64_t sh, int64_t sw, double* df, double* absmag);

/* Multi-channel 1-D convolution, channels-last, bfloat16 inputs (bit patterns),
 * double result: y[b][i][co] = sum_j sum_ci w[co][ci][j] x[b][i+j][ci]. */
int oracle_conv1d_mc_bf16(const uint16_t* x, const uint16_t* w, int64_t batch, int64_t N, int64_t cin,
                          int64_t cout, int64_t k, double* y, double* absmag);
/* Multi-channel 2-D convolution, NHWC bf16 activations, [cout][cin][kh][kw] bf16
 * weights, valid padding, stride 1 (reading R22); y [batch][H-kh+1][W-kw+1][cout]. */
int oracle_conv2d_mc_bf16(const uint16_t* x, const uint16_t* w, int64_t batch, int64_t H, int64_t W, int64_t cin,
                          int64_t cout, int64_t kh, int64_t kw, double* y, double* absmag);
/* Input gradient of the multi-channel 1-D convolution (reading R23): dy [batch][N-k+1][cout] and
 * w [cout][cin][k] as bf16 bits; dx [batch][N][cin] = the scatter of w * dy, in double. */
int oracle_conv1d_mc_backward_input_bf16(const uint16_t* dy, const uint16_t* w, int64_t batch, int64_t N,
                                         int64_t cin, int64_t cout, int64_t k, double* dx, double* absmag);
int oracle_conv1d_mc_backward_filter_bf16(const uint16_t* dy, const uint16_t* x, int64_t batch, int64_t N,
                                          int64_t cin, int64_t cout, int64_t k, double* dw, double* absmag);
int oracle_conv2d_mc_backward_input_bf16(const uint16_t* dy, const uint16_t* w, int64_t batch, int64_t H, int64_t W,
                                         int64_t cin, int64_t cout, int64_t kh, int64_t kw, double* dx,
                                         double* absmag);
int oracle_conv2d_mc_backward_filter_bf16(const uint16_t* dy, const uint16_t* x, int64_t batch, int64_t H, int64_t W,
                                          int64_t cin, int64_t cout, int64_t kh, int64_t kw, double* dw,
                                          double* absmag);

#ifdef __cplusplus
}
#endif
#endif
