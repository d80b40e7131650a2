/*
 * oracle.c -- plain CPU oracle (TEST INFRASTRUCTURE ONLY; see oracle.h).
 *
 * Each function is the definition it cites, written as the obvious loop.
 * Compiled with -O2 and no fast-math (IEEE double).  Single-threaded.
 */
#include "oracle.h"

#include <math.h>
#include <stddef.h>
#include <stdint.h>

/* Output length of a valid-padding window of w addends at stride s
 * (Eq. 3 gives N-w+1 at s=1; stride reading R4 in DESIGN.md). */
int64_t oracle_out_len(int64_t N, int64_t w, int64_t s) {
  if (N < 1 || w < 1 || s < 1 || w > N) return -1;
  return (N - w) / s + 1;
}

static int bad_1d(const void* x, const void* y, int64_t N, int64_t batch,
                  int64_t w, int64_t s) {
  return x == NULL || y == NULL || batch < 1 || oracle_out_len(N, w, s) < 0;
}

/* Eq. 3, (+) = +: y_i = x_{is} + ... + x_{is+w-1}, left to right, in int64. */
int oracle_pool_sum_i32(const int32_t* x, int64_t N, int64_t batch, int64_t w,
                        int64_t s, int64_t* y) {
  if (bad_1d(x, y, N, batch, w, s)) return -1;
  int64_t L = oracle_out_len(N, w, s);
  for (int64_t b = 0; b < batch; ++b) {
    const int32_t* xr = x + b * N;
    for (int64_t i = 0; i < L; ++i) {
      int64_t acc = 0;
      for (int64_t j = 0; j < w; ++j) acc += (int64_t)xr[i * s + j];
      y[b * L + i] = acc;
    }
  }
  return 0;
}

/* Eq. 3, (+) = +, fp32 input summed in double. */
int oracle_pool_sum_f32(const float* x, int64_t N, int64_t batch, int64_t w,
                        int64_t s, double* y, double* absmag) {
  if (bad_1d(x, y, N, batch, w, s)) return -1;
  int64_t L = oracle_out_len(N, w, s);
  for (int64_t b = 0; b < batch; ++b) {
    const float* xr = x + b * N;
    for (int64_t i = 0; i < L; ++i) {
      double acc = 0.0, mag = 0.0;
      for (int64_t j = 0; j < w; ++j) {
        double v = (double)xr[i * s + j];
        acc += v;
        mag += fabs(v);
      }
      y[b * L + i] = acc;
      if (absmag) absmag[b * L + i] = mag;
    }
  }
  return 0;
}

/* Eq. 3, (+) = max (Sec. 2.3): m = x_{is}; m = (v > m ? v : m) left to right. */
int oracle_pool_max_i32(const int32_t* x, int64_t N, int64_t batch, int64_t w,
                        int64_t s, int32_t* y) {
  if (bad_1d(x, y, N, batch, w, s)) return -1;
  int64_t L = oracle_out_len(N, w, s);
  for (int64_t b = 0; b < batch; ++b) {
    const int32_t* xr = x + b * N;
    for (int64_t i = 0; i < L; ++i) {
      int32_t m = xr[i * s];
      for (int64_t j = 1; j < w; ++j) {
        int32_t v = xr[i * s + j];
        m = v > m ? v : m;
      }
      y[b * L + i] = m;
    }
  }
  return 0;
}

int oracle_pool_max_f32(const float* x, int64_t N, int64_t batch, int64_t w,
                        int64_t s, float* y) {
  if (bad_1d(x, y, N, batch, w, s)) return -1;
  int64_t L = oracle_out_len(N, w, s);
  for (int64_t b = 0; b < batch; ++b) {
    const float* xr = x + b * N;
    for (int64_t i = 0; i < L; ++i) {
      float m = xr[i * s];
      for (int64_t j = 1; j < w; ++j) {
        float v = xr[i * s + j];
        m = v > m ? v : m;
      }
      y[b * L + i] = m;
    }
  }
  return 0;
}

/* Sec. 2.4-2.5: convolution = sliding dot product (Eq. 4 per window),
 * cross-correlation orientation (reading R2): y_i = sum_j f_j * x_{is+j}. */
int oracle_conv1d_f32(const float* x, int64_t N, int64_t batch, const float* f,
                      int64_t k, int64_t s, double* y, double* absmag) {
  if (bad_1d(x, y, N, batch, k, s) || f == NULL) return -1;
  int64_t L = oracle_out_len(N, k, s);
  for (int64_t b = 0; b < batch; ++b) {
    const float* xr = x + b * N;
    for (int64_t i = 0; i < L; ++i) {
      double acc = 0.0, mag = 0.0;
      for (int64_t j = 0; j < k; ++j) {
        double p = (double)f[j] * (double)xr[i * s + j];
        acc += p;
        mag += fabs(p);
      }
      y[b * L + i] = acc;
      if (absmag) absmag[b * L + i] = mag;
    }
  }
  return 0;
}

/* 2-D pooling (Sec. 2.3 operators over the multi-dimensional window of the
 * Conclusion): out[p][r][c] = (+)_{dr<kh, dc<kw} x[p][r*sh+dr][c*sw+dc].
 * mode 0: max; mode 1: average = (double sum) / (kh*kw). */
int oracle_pool2d_f32(const float* x, int64_t planes, int64_t H, int64_t W,
                      int64_t kh, int64_t kw, int64_t sh, int64_t sw, int mode,
                      double* y, double* absmag) {
  if (x == NULL || y == NULL || planes < 1 || (mode != 0 && mode != 1)) return -1;
  int64_t OH = oracle_out_len(H, kh, sh), OW = oracle_out_len(W, kw, sw);
  if (OH < 0 || OW < 0) return -1;
  double cnt = (double)(kh * kw);
  for (int64_t p = 0; p < planes; ++p) {
    const float* xp = x + p * H * W;
    for (int64_t r = 0; r < OH; ++r) {
      for (int64_t c = 0; c < OW; ++c) {
        double acc = 0.0, mag = 0.0;
        float m = xp[(r * sh) * W + c * sw];
        for (int64_t dr = 0; dr < kh; ++dr) {
          for (int64_t dc = 0; dc < kw; ++dc) {
            float v = xp[(r * sh + dr) * W + (c * sw + dc)];
            acc += (double)v;
            mag += fabs((double)v);
            m = v > m ? v : m;
          }
        }
        int64_t o = (p * OH + r) * OW + c;
        if (mode == 0) {
          y[o] = (double)m;
          if (absmag) absmag[o] = 0.0;
        } else {
          y[o] = acc / cnt;
          if (absmag) absmag[o] = mag / cnt;
        }
      }
    }
  }
  return 0;
}

/* ---- window spec with dilation d and padding (pl, pr, mode): see oracle.h ---- */
int64_t oracle_out_len_ex(int64_t N, int64_t w, int64_t s, int64_t d, int64_t pl, int64_t pr) {
  if (N < 1 || w < 1 || s < 1 || d < 1 || pl < 0 || pr < 0) return -1;
  int64_t E = (w - 1) * d + 1, Np = N + pl + pr;
  if (E > Np) return -1;
  return (Np - E) / s + 1;
}

/* x index of padded position t - pl =: u (u may be outside [0, N)), or -1 for
 * zero padding (the identity).  Modes: 0 zeros, 1 reflect (mirror about the end
 * elements, which are not repeated), 2 circular (periodic), 3 replicate. */
static int64_t pad_source(int64_t u, int64_t N, int mode) {
  if (u >= 0 && u < N) return u;
  switch (mode) {
    case 1: return u < 0 ? -u : 2 * (N - 1) - u;
    case 2: return ((u % N) + N) % N;
    case 3: return u < 0 ? 0 : N - 1;
    default: return -1;
  }
}

static int bad_ex(const void* x, const void* y, int64_t N, int64_t batch, int64_t w, int64_t s,
                  int64_t d, int64_t pl, int64_t pr, int mode) {
  if (x == NULL || y == NULL || batch < 1 || oracle_out_len_ex(N, w, s, d, pl, pr) < 0) return 1;
  if (mode < 0 || mode > 3) return 1;
  if (mode == 1 && (pl > N - 1 || pr > N - 1)) return 1; /* one reflection only */
  if (mode == 2 && (pl > N || pr > N)) return 1;         /* one period only */
  return 0;
}

int oracle_pool_sum_ex_i32(const int32_t* x, int64_t N, int64_t batch, int64_t w, int64_t s,
                           int64_t d, int64_t pl, int64_t pr, int mode, int64_t* y) {
  if (bad_ex(x, y, N, batch, w, s, d, pl, pr, mode)) return -1;
  int64_t L = oracle_out_len_ex(N, w, s, d, pl, pr);
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t i = 0; i < L; ++i) {
      int64_t acc = 0;
      for (int64_t j = 0; j < w; ++j) {
        int64_t t = pad_source(i * s + j * d - pl, N, mode);
        if (t >= 0) acc += (int64_t)x[b * N + t];
      }
      y[b * L + i] = acc;
    }
  return 0;
}

int oracle_pool_sum_ex_f32(const float* x, int64_t N, int64_t batch, int64_t w, int64_t s,
                           int64_t d, int64_t pl, int64_t pr, int mode, double* y, double* absmag) {
  if (bad_ex(x, y, N, batch, w, s, d, pl, pr, mode)) return -1;
  int64_t L = oracle_out_len_ex(N, w, s, d, pl, pr);
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t i = 0; i < L; ++i) {
      double acc = 0.0, mag = 0.0;
      for (int64_t j = 0; j < w; ++j) {
        int64_t t = pad_source(i * s + j * d - pl, N, mode);
        if (t >= 0) {
          acc += (double)x[b * N + t];
          mag += fabs((double)x[b * N + t]);
        }
      }
      y[b * L + i] = acc;
      if (absmag) absmag[b * L + i] = mag;
    }
  return 0;
}

/* max (sign = +1) or min (sign = -1) of each window; padding in zeros mode is
 * skipped (the identity: -inf / INT32_MIN for max, +inf / INT32_MAX for min) */
static int extremum_ex_i32(const int32_t* x, int64_t N, int64_t batch, int64_t w, int64_t s, int64_t d,
                           int64_t pl, int64_t pr, int mode, int sign, int32_t* y) {
  if (bad_ex(x, y, N, batch, w, s, d, pl, pr, mode)) return -1;
  int64_t L = oracle_out_len_ex(N, w, s, d, pl, pr);
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t i = 0; i < L; ++i) {
      int32_t m = sign > 0 ? INT32_MIN : INT32_MAX;
      for (int64_t j = 0; j < w; ++j) {
        int64_t t = pad_source(i * s + j * d - pl, N, mode);
        if (t >= 0) {
          int32_t v = x[b * N + t];
          if (sign > 0 ? v > m : v < m) m = v;
        }
      }
      y[b * L + i] = m;
    }
  return 0;
}

static int extremum_ex_f32(const float* x, int64_t N, int64_t batch, int64_t w, int64_t s, int64_t d,
                           int64_t pl, int64_t pr, int mode, int sign, float* y) {
  if (bad_ex(x, y, N, batch, w, s, d, pl, pr, mode)) return -1;
  int64_t L = oracle_out_len_ex(N, w, s, d, pl, pr);
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t i = 0; i < L; ++i) {
      float m = sign > 0 ? -INFINITY : INFINITY;
      for (int64_t j = 0; j < w; ++j) {
        int64_t t = pad_source(i * s + j * d - pl, N, mode);
        if (t >= 0) {
          float v = x[b * N + t];
          if (sign > 0 ? v > m : v < m) m = v;
        }
      }
      y[b * L + i] = m;
    }
  return 0;
}

int oracle_pool_max_ex_i32(const int32_t* x, int64_t N, int64_t batch, int64_t w, int64_t s,
                           int64_t d, int64_t pl, int64_t pr, int mode, int32_t* y) {
  return extremum_ex_i32(x, N, batch, w, s, d, pl, pr, mode, +1, y);
}
int oracle_pool_max_ex_f32(const float* x, int64_t N, int64_t batch, int64_t w, int64_t s,
                           int64_t d, int64_t pl, int64_t pr, int mode, float* y) {
  return extremum_ex_f32(x, N, batch, w, s, d, pl, pr, mode, +1, y);
}
int oracle_pool_min_ex_i32(const int32_t* x, int64_t N, int64_t batch, int64_t w, int64_t s,
                           int64_t d, int64_t pl, int64_t pr, int mode, int32_t* y) {
  return extremum_ex_i32(x, N, batch, w, s, d, pl, pr, mode, -1, y);
}
int oracle_pool_min_ex_f32(const float* x, int64_t N, int64_t batch, int64_t w, int64_t s,
                           int64_t d, int64_t pl, int64_t pr, int mode, float* y) {
  return extremum_ex_f32(x, N, batch, w, s, d, pl, pr, mode, -1, y);
}

int oracle_conv1d_ex_f32(const float* x, int64_t N, int64_t batch, const float* f, int64_t k,
                         int64_t s, int64_t d, int64_t pl, int64_t pr, int mode, double* y, double* absmag) {
  if (bad_ex(x, y, N, batch, k, s, d, pl, pr, mode) || f == NULL) return -1;
  int64_t L = oracle_out_len_ex(N, k, s, d, pl, pr);
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t i = 0; i < L; ++i) {
      double acc = 0.0, mag = 0.0;
      for (int64_t j = 0; j < k; ++j) {
        int64_t t = pad_source(i * s + j * d - pl, N, mode);
        if (t >= 0) {
          double p = (double)f[j] * (double)x[b * N + t];
          acc += p;
          mag += fabs(p);
        }
      }
      y[b * L + i] = acc;
      if (absmag) absmag[b * L + i] = mag;
    }
  return 0;
}

/* Sliding window of gamma pairs: Eq. 3's window with Eq. 8's operator, each
 * window folded left to right (delta = delta (+) gamma, Eq. 9). */
int oracle_affine_window(const float* u, const float* v, int64_t N, int64_t batch, int64_t w,
                         int64_t s, double* U, double* V, double* magV) {
  if (u == NULL || v == NULL || V == NULL || batch < 1 || oracle_out_len(N, w, s) < 0) return -1;
  int64_t L = oracle_out_len(N, w, s);
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t i = 0; i < L; ++i) {
      int64_t t0 = b * N + i * s;
      double du = (double)u[t0], dv = (double)v[t0];
      double au = fabs((double)u[t0]), av = fabs((double)v[t0]);
      for (int64_t j = 1; j < w; ++j) {
        double nu, nv;
        oracle_gamma_combine(du, dv, (double)u[t0 + j], (double)v[t0 + j], &nu, &nv);
        du = nu;
        dv = nv;
        double anu, anv;
        oracle_gamma_combine(au, av, fabs((double)u[t0 + j]), fabs((double)v[t0 + j]), &anu, &anv);
        au = anu;
        av = anv;
      }
      if (U) U[b * L + i] = du;
      V[b * L + i] = dv;
      if (magV) magV[b * L + i] = av;
    }
  return 0;
}

/* Eq. 8. */
void oracle_gamma_combine(double ui, double vi, double uj, double vj,
                          double* u_out, double* v_out) {
  *u_out = ui * uj;
  *v_out = uj * vi + vj;
}

/* Eq. 5 (masking) then Eq. 7:
 *   alpha_i = 1 if a_i == 0 else a_i;   beta_i = 0 if a_i == 0 else b_i
 *   u_0 = 1;  u_i = alpha_{i-1} / alpha_i (0 < i < M);  u_M = alpha_{M-1}
 *   v_i = beta_i (i < M);  v_M = 0.                                          */
int oracle_gamma_sequence(const double* a, const double* b, int64_t M,
                          double* u, double* v) {
  if (a == NULL || b == NULL || u == NULL || v == NULL || M < 1) return -1;
  for (int64_t i = 0; i <= M; ++i) {
    if (i == 0) {
      u[i] = 1.0;
    } else if (i < M) {
      double alpha_prev = a[i - 1] == 0.0 ? 1.0 : a[i - 1];
      double alpha_i = a[i] == 0.0 ? 1.0 : a[i];
      u[i] = alpha_prev / alpha_i;
    } else {
      u[i] = a[M - 1] == 0.0 ? 1.0 : a[M - 1];
    }
    if (i < M) {
      v[i] = a[i] == 0.0 ? 0.0 : b[i];
    } else {
      v[i] = 0.0;
    }
  }
  return 0;
}

/* Eq. 9: delta_0 = gamma_0, delta_i = delta_{i-1} (+) gamma_i;
 * the bottom element of delta_M is the dot product. */
double oracle_gamma_dot(const double* a, const double* b, int64_t M, double* u_out) {
  if (a == NULL || b == NULL || M < 1) return NAN;
  double du = 1.0, dv = 0.0;
  for (int64_t i = 0; i <= M; ++i) {
    double ui, vi;
    if (i == 0) {
      ui = 1.0;
    } else if (i < M) {
      double alpha_prev = a[i - 1] == 0.0 ? 1.0 : a[i - 1];
      double alpha_i = a[i] == 0.0 ? 1.0 : a[i];
      ui = alpha_prev / alpha_i;
    } else {
      ui = a[M - 1] == 0.0 ? 1.0 : a[M - 1];
    }
    vi = (i < M) ? (a[i] == 0.0 ? 0.0 : b[i]) : 0.0;
    if (i == 0) {
      du = ui;
      dv = vi;
    } else {
      double nu, nv;
      oracle_gamma_combine(du, dv, ui, vi, &nu, &nv);
      du = nu;
      dv = nv;
    }
  }
  if (u_out) *u_out = du;
  return dv;
}

/* ---- backward passes (the abstract's "training", PAPER.md
 * l.7).  Each is the vector-Jacobian product of the forward definition above,
 * written as the scatter J^T dy: every forward term y_i <- x_t sends dy_i back
 * to dx_t (times its coefficient).  Accumulation in double; absmag = the sum of
 * the magnitudes of the terms (BASELINE.json tolerance form). */

/* Eq. 3 with +:  y_i = sum_{j<w} x_{is+j}  =>  dx_t = sum_{i: is <= t < is+w} dy_i. */
int oracle_pool_sum_backward_f32(const float* dy, int64_t N, int64_t batch, int64_t w,
                                 int64_t s, double* dx, double* absmag) {
  if (bad_1d(dy, dx, N, batch, w, s)) return -1;
  int64_t L = oracle_out_len(N, w, s);
  for (int64_t t = 0; t < batch * N; ++t) {
    dx[t] = 0.0;
    if (absmag) absmag[t] = 0.0;
  }
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t i = 0; i < L; ++i)
      for (int64_t j = 0; j < w; ++j) {
        double g = (double)dy[b * L + i];
        dx[b * N + i * s + j] += g;
        if (absmag) absmag[b * N + i * s + j] += fabs(g);
      }
  return 0;
}

/* Eq. 3 with max:  y_i = x_{a_i}, a_i = the FIRST index of the maximum of
 * window i (scan left to right, replace on strictly greater)  =>
 * dx_t = sum_{i: a_i = t} dy_i  (the subgradient that routes each window's
 * gradient to its first maximum; reading R16). */
int oracle_pool_max_backward_f32(const float* x, const float* dy, int64_t N, int64_t batch,
                                 int64_t w, int64_t s, double* dx) {
  if (bad_1d(x, dx, N, batch, w, s) || dy == NULL) return -1;
  int64_t L = oracle_out_len(N, w, s);
  for (int64_t t = 0; t < batch * N; ++t) dx[t] = 0.0;
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t i = 0; i < L; ++i) {
      const float* xw = x + b * N + i * s;
      int64_t a = 0;
      float m = xw[0];
      for (int64_t j = 1; j < w; ++j)
        if (xw[j] > m) {
          m = xw[j];
          a = j;
        }
      dx[b * N + i * s + a] += (double)dy[b * L + i];
    }
  return 0;
}

/* Sec. 2.5:  y_i = sum_j f_j x_{is+j}  =>  dx_t = sum_{(i,j): is+j = t} f_j dy_i. */
int oracle_conv1d_backward_input_f32(const float* dy, int64_t N, int64_t batch, const float* f,
                                     int64_t k, int64_t s, double* dx, double* absmag) {
  if (bad_1d(dy, dx, N, batch, k, s) || f == NULL) return -1;
  int64_t L = oracle_out_len(N, k, s);
  for (int64_t t = 0; t < batch * N; ++t) {
    dx[t] = 0.0;
    if (absmag) absmag[t] = 0.0;
  }
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t i = 0; i < L; ++i)
      for (int64_t j = 0; j < k; ++j) {
        double p = (double)f[j] * (double)dy[b * L + i];
        dx[b * N + i * s + j] += p;
        if (absmag) absmag[b * N + i * s + j] += fabs(p);
      }
  return 0;
}

/* Sec. 2.5:  y_i = sum_j f_j x_{is+j}  =>  df_j = sum_b sum_i dy_i x_{is+j}. */
int oracle_conv1d_backward_filter_f32(const float* x, const float* dy, int64_t N, int64_t batch,
                                      int64_t k, int64_t s, double* df, double* absmag) {
  if (bad_1d(x, df, N, batch, k, s) || dy == NULL) return -1;
  int64_t L = oracle_out_len(N, k, s);
  for (int64_t j = 0; j < k; ++j) {
    df[j] = 0.0;
    if (absmag) absmag[j] = 0.0;
  }
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t i = 0; i < L; ++i)
      for (int64_t j = 0; j < k; ++j) {
        double p = (double)dy[b * L + i] * (double)x[b * N + i * s + j];
        df[j] += p;
        if (absmag) absmag[j] += fabs(p);
      }
  return 0;
}

/* 2-D pooling (direct window, as oracle_pool2d_f32):  avg: y = (1/(kh kw)) sum of
 * the window => dx gets dy/(kh kw) at every window position; max: y = x at the
 * first maximum in row-major scan order => dx gets dy there. */
int oracle_pool2d_backward_f32(const float* x, const float* dy, int64_t planes, int64_t H,
                               int64_t W, int64_t kh, int64_t kw, int64_t sh, int64_t sw,
                               int mode, double* dx, double* absmag) {
  int64_t OH = oracle_out_len(H, kh, sh), OW = oracle_out_len(W, kw, sw);
  if (dy == NULL || dx == NULL || planes < 1 || OH < 0 || OW < 0) return -1;
  if (mode == 0 && x == NULL) return -1;
  for (int64_t t = 0; t < planes * H * W; ++t) {
    dx[t] = 0.0;
    if (absmag) absmag[t] = 0.0;
  }
  double inv = 1.0 / (double)(kh * kw);
  for (int64_t p = 0; p < planes; ++p)
    for (int64_t r = 0; r < OH; ++r)
      for (int64_t c = 0; c < OW; ++c) {
        double g = (double)dy[(p * OH + r) * OW + c];
        if (mode == 1) {
          for (int64_t a = 0; a < kh; ++a)
            for (int64_t e = 0; e < kw; ++e) {
              int64_t t = (p * H + r * sh + a) * W + c * sw + e;
              dx[t] += g * inv;
              if (absmag) absmag[t] += fabs(g * inv);
            }
        } else {
          int64_t best = (p * H + r * sh) * W + c * sw;
          float m = x[best];
          for (int64_t a = 0; a < kh; ++a)
            for (int64_t e = 0; e < kw; ++e) {
              int64_t t = (p * H + r * sh + a) * W + c * sw + e;
              if (x[t] > m) {
                m = x[t];
                best = t;
              }
            }
          dx[best] += g;
          if (absmag) absmag[best] += fabs(g);
        }
      }
  return 0;
}

/* Multi-dimensional extension of the sliding dot product
 * (Sec. 2.5) to a single-channel 2-D filter: cross-correlation of each plane
 * with f [kh][kw] at stride (sh, sw), valid padding, taps summed in row-major
 * order in double:  y[p][r][c] = sum_{a<kh} sum_{b<kw} f[a][b] x[p][r sh + a][c sw + b]. */
int oracle_conv2d_f32(const float* x, int64_t planes, int64_t H, int64_t W, const float* f,
                      int64_t kh, int64_t kw, int64_t sh, int64_t sw, double* y, double* absmag) {
  int64_t OH = oracle_out_len(H, kh, sh), OW = oracle_out_len(W, kw, sw);
  if (x == NULL || f == NULL || y == NULL || planes < 1 || OH < 0 || OW < 0) return -1;
  for (int64_t p = 0; p < planes; ++p)
    for (int64_t r = 0; r < OH; ++r)
      for (int64_t c = 0; c < OW; ++c) {
        double acc = 0.0, mag = 0.0;
        for (int64_t a = 0; a < kh; ++a)
          for (int64_t b = 0; b < kw; ++b) {
            double t = (double)f[a * kw + b] * (double)x[(p * H + r * sh + a) * W + c * sw + b];
            acc += t;
            mag += fabs(t);
          }
        y[(p * OH + r) * OW + c] = acc;
        if (absmag) absmag[(p * OH + r) * OW + c] = mag;
      }
  return 0;
}

/* Backward passes of the 2-D sliding dot product (SURVEY 8f NEXT #4 "2-D
 * convolution and backward passes"; reading R21), the vector-Jacobian
 * products of y[p][r][c] = sum_a sum_b f[a][b] x[p][r*sh+a][c*sw+b]:
 *   dx[p][r*sh+a][c*sw+b] += f[a][b] dy[p][r][c]   (scatter form, every (r, c, a, b))
 *   df[a][b] = sum_p sum_r sum_c dy[p][r][c] x[p][r*sh+a][c*sw+b]
 * accumulated in double; absmag = per-element sum of term magnitudes. */
int oracle_conv2d_backward_input_f32(const float* dy, int64_t planes, int64_t H, int64_t W, const float* f,
                                     int64_t kh, int64_t kw, int64_t sh, int64_t sw, double* dx, double* absmag) {
  int64_t OH = oracle_out_len(H, kh, sh), OW = oracle_out_len(W, kw, sw);
  if (dy == NULL || f == NULL || dx == NULL || planes < 1 || OH < 0 || OW < 0) return -1;
  for (int64_t t = 0; t < planes * H * W; ++t) {
    dx[t] = 0.0;
    if (absmag) absmag[t] = 0.0;
  }
  for (int64_t p = 0; p < planes; ++p)
    for (int64_t r = 0; r < OH; ++r)
      for (int64_t c = 0; c < OW; ++c)
        for (int64_t a = 0; a < kh; ++a)
          for (int64_t b = 0; b < kw; ++b) {
            double t = (double)f[a * kw + b] * (double)dy[(p * OH + r) * OW + c];
            int64_t e = (p * H + r * sh + a) * W + c * sw + b;
            dx[e] += t;
            if (absmag) absmag[e] += fabs(t);
          }
  return 0;
}

int oracle_conv2d_backward_filter_f32(const float* x, const float* dy, int64_t planes, int64_t H, int64_t W,
                                      int64_t kh, int64_t kw, int64_t sh, int64_t sw, double* df, double* absmag) {
  int64_t OH = oracle_out_len(H, kh, sh), OW = oracle_out_len(W, kw, sw);
  if (x == NULL || dy == NULL || df == NULL || planes < 1 || OH < 0 || OW < 0) return -1;
  for (int64_t a = 0; a < kh; ++a)
    for (int64_t b = 0; b < kw; ++b) {
      double acc = 0.0, mag = 0.0;
      for (int64_t p = 0; p < planes; ++p)
        for (int64_t r = 0; r < OH; ++r)
          for (int64_t c = 0; c < OW; ++c) {
            double t = (double)dy[(p * OH + r) * OW + c] * (double)x[(p * H + r * sh + a) * W + c * sw + b];
            acc += t;
            mag += fabs(t);
          }
      df[a * kw + b] = acc;
      if (absmag) absmag[a * kw + b] = mag;
    }
  return 0;
}

/* Multi-channel 1-D convolution ("with C_in > 1 it becomes a
 * real contraction"): the sliding dot product of Sec. 2.5 summed over input
 * channels, channels-last layout, inputs given as bfloat16 bit patterns
 * (reading R18):
 *   y[b][i][co] = sum_{j<k} sum_{ci<cin} w[co][ci][j] * x[b][i+j][ci],  i < N-k+1
 * x [batch][N][cin], w [cout][cin][k] (torch conv1d weight order), y [batch][L][cout],
 * accumulated in double (terms taken in j, ci order). */
static double bf16_to_double(uint16_t h) {
  union { uint32_t u; float f; } c;
  c.u = (uint32_t)h << 16;
  return (double)c.f;
}

int oracle_conv1d_mc_bf16(const uint16_t* x, const uint16_t* w, int64_t batch, int64_t N, int64_t cin,
                          int64_t cout, int64_t k, double* y, double* absmag) {
  if (x == NULL || w == NULL || y == NULL || batch < 1 || cin < 1 || cout < 1 || k < 1 || k > N) return -1;
  int64_t L = N - k + 1;
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t i = 0; i < L; ++i)
      for (int64_t co = 0; co < cout; ++co) {
        double acc = 0.0, mag = 0.0;
        for (int64_t j = 0; j < k; ++j)
          for (int64_t ci = 0; ci < cin; ++ci) {
            double t = bf16_to_double(w[(co * cin + ci) * k + j]) * bf16_to_double(x[(b * N + i + j) * cin + ci]);
            acc += t;
            mag += fabs(t);
          }
        y[(b * L + i) * cout + co] = acc;
        if (absmag) absmag[(b * L + i) * cout + co] = mag;
      }
  return 0;
}

/* Multi-channel 2-D convolution (the Conclusion's
 * multi-dimensional extension, of the channel-summed sliding dot
 * product of reading R18; reading R22): channels-last (NHWC) bf16
 * activations, weights in torch conv2d order [cout][cin][kh][kw], valid padding,
 * stride 1:
 *   y[b][r][c][co] = sum_{a<kh} sum_{e<kw} sum_{ci<cin} w[co][ci][a][e] * x[b][r+a][c+e][ci]
 * x [batch][H][W][cin], y [batch][H-kh+1][W-kw+1][cout]; accumulated in double
 * (terms taken in a, e, ci order). */
int oracle_conv2d_mc_bf16(const uint16_t* x, const uint16_t* w, int64_t batch, int64_t H, int64_t W, int64_t cin,
                          int64_t cout, int64_t kh, int64_t kw, double* y, double* absmag) {
  if (x == NULL || w == NULL || y == NULL || batch < 1 || cin < 1 || cout < 1 || kh < 1 || kw < 1 || kh > H ||
      kw > W)
    return -1;
  int64_t OH = H - kh + 1, OW = W - kw + 1;
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t r = 0; r < OH; ++r)
      for (int64_t c = 0; c < OW; ++c)
        for (int64_t co = 0; co < cout; ++co) {
          double acc = 0.0, mag = 0.0;
          for (int64_t a = 0; a < kh; ++a)
            for (int64_t e = 0; e < kw; ++e)
              for (int64_t ci = 0; ci < cin; ++ci) {
                double t = bf16_to_double(w[((co * cin + ci) * kh + a) * kw + e]) *
                           bf16_to_double(x[((b * H + r + a) * W + c + e) * cin + ci]);
                acc += t;
                mag += fabs(t);
              }
          int64_t o = ((b * OH + r) * OW + c) * cout + co;
          y[o] = acc;
          if (absmag) absmag[o] = mag;
        }
  return 0;
}

/* Input gradient of the multi-channel 1-D convolution (reading R23: the
 * vector-Jacobian product of reading R18), bf16 dy and weights:
 *   y[b][i][co] = sum_j sum_ci w[co][ci][j] x[b][i+j][ci]
 *   =>  dx[b][i+j][ci] += w[co][ci][j] * dy[b][i][co]   for every (b, i, j, co, ci)
 * dy [batch][N-k+1][cout], w [cout][cin][k], dx [batch][N][cin] (elements no window
 * covers get 0); the scatter is accumulated in double in (i, j, co) order. */
int oracle_conv1d_mc_backward_input_bf16(const uint16_t* dy, const uint16_t* w, int64_t batch, int64_t N,
                                         int64_t cin, int64_t cout, int64_t k, double* dx, double* absmag) {
  if (dy == NULL || w == NULL || dx == NULL || batch < 1 || cin < 1 || cout < 1 || k < 1 || k > N) return -1;
  int64_t L = N - k + 1;
  for (int64_t t = 0; t < batch * N * cin; ++t) {
    dx[t] = 0.0;
    if (absmag) absmag[t] = 0.0;
  }
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t i = 0; i < L; ++i)
      for (int64_t j = 0; j < k; ++j)
        for (int64_t co = 0; co < cout; ++co) {
          double g = bf16_to_double(dy[(b * L + i) * cout + co]);
          for (int64_t ci = 0; ci < cin; ++ci) {
            double p = bf16_to_double(w[(co * cin + ci) * k + j]) * g;
            dx[(b * N + i + j) * cin + ci] += p;
            if (absmag) absmag[(b * N + i + j) * cin + ci] += fabs(p);
          }
        }
  return 0;
}

/* Filter gradient of the multi-channel 1-D convolution (reading R25: the
 * vector-Jacobian product of reading R18 with respect to the weights), bf16 dy and x:
 *   y[b][i][co] = sum_j sum_ci w[co][ci][j] x[b][i+j][ci]
 *   =>  dw[co][ci][j] = sum_b sum_{i < N-k+1} dy[b][i][co] * x[b][i+j][ci]
 * dy [batch][N-k+1][cout], x [batch][N][cin], dw [cout][cin][k]; accumulated in
 * double in (b, i) order. */
int oracle_conv1d_mc_backward_filter_bf16(const uint16_t* dy, const uint16_t* x, int64_t batch, int64_t N,
                                          int64_t cin, int64_t cout, int64_t k, double* dw, double* absmag) {
  if (dy == NULL || x == NULL || dw == NULL || batch < 1 || cin < 1 || cout < 1 || k < 1 || k > N) return -1;
  int64_t L = N - k + 1;
  for (int64_t co = 0; co < cout; ++co)
    for (int64_t ci = 0; ci < cin; ++ci)
      for (int64_t j = 0; j < k; ++j) {
        double acc = 0.0, mag = 0.0;
        for (int64_t b = 0; b < batch; ++b)
          for (int64_t i = 0; i < L; ++i) {
            double t = bf16_to_double(dy[(b * L + i) * cout + co]) * bf16_to_double(x[(b * N + i + j) * cin + ci]);
            acc += t;
            mag += fabs(t);
          }
        dw[(co * cin + ci) * k + j] = acc;
        if (absmag) absmag[(co * cin + ci) * k + j] = mag;
      }
  return 0;
}

/* Input gradient of the multi-channel 2-D convolution (reading R26: the
 * vector-Jacobian product of reading R22), bf16 dy and weights, NHWC:
 *   y[b][r][c][co] = sum_{a,e,ci} w[co][ci][a][e] x[b][r+a][c+e][ci]
 *   =>  dx[b][r+a][c+e][ci] += w[co][ci][a][e] * dy[b][r][c][co]
 * dy [batch][H-kh+1][W-kw+1][cout], w [cout][cin][kh][kw], dx [batch][H][W][cin]
 * (elements no window covers get 0); the scatter is accumulated in double in
 * (r, c, a, e, co) order. */
int oracle_conv2d_mc_backward_input_bf16(const uint16_t* dy, const uint16_t* w, int64_t batch, int64_t H, int64_t W,
                                         int64_t cin, int64_t cout, int64_t kh, int64_t kw, double* dx,
                                         double* absmag) {
  if (dy == NULL || w == NULL || dx == NULL || batch < 1 || cin < 1 || cout < 1 || kh < 1 || kw < 1 || kh > H ||
      kw > W)
    return -1;
  int64_t OH = H - kh + 1, OW = W - kw + 1;
  for (int64_t t = 0; t < batch * H * W * cin; ++t) {
    dx[t] = 0.0;
    if (absmag) absmag[t] = 0.0;
  }
  for (int64_t b = 0; b < batch; ++b)
    for (int64_t r = 0; r < OH; ++r)
      for (int64_t c = 0; c < OW; ++c)
        for (int64_t a = 0; a < kh; ++a)
          for (int64_t e = 0; e < kw; ++e)
            for (int64_t co = 0; co < cout; ++co) {
              double g = bf16_to_double(dy[((b * OH + r) * OW + c) * cout + co]);
              for (int64_t ci = 0; ci < cin; ++ci) {
                double p = bf16_to_double(w[((co * cin + ci) * kh + a) * kw + e]) * g;
                int64_t o = ((b * H + r + a) * W + c + e) * cin + ci;
                dx[o] += p;
                if (absmag) absmag[o] += fabs(p);
              }
            }
  return 0;
}

/* Filter gradient of the multi-channel 2-D convolution (reading R27: the weight
 * vector-Jacobian product of reading R22), bf16 dy and x, NHWC:
 *   dw[co][ci][a][e] = sum_b sum_{r < H-kh+1} sum_{c < W-kw+1} dy[b][r][c][co] x[b][r+a][c+e][ci]
 * dy [batch][H-kh+1][W-kw+1][cout], x [batch][H][W][cin], dw [cout][cin][kh][kw];
 * each sum in double in (b, r, c) order. */
int oracle_conv2d_mc_backward_filter_bf16(const uint16_t* dy, const uint16_t* x, int64_t batch, int64_t H, int64_t W,
                                          int64_t cin, int64_t cout, int64_t kh, int64_t kw, double* dw,
                                          double* absmag) {
  if (dy == NULL || x == NULL || dw == NULL || batch < 1 || cin < 1 || cout < 1 || kh < 1 || kw < 1 || kh > H ||
      kw > W)
    return -1;
  int64_t OH = H - kh + 1, OW = W - kw + 1;
  for (int64_t co = 0; co < cout; ++co)
    for (int64_t ci = 0; ci < cin; ++ci)
      for (int64_t a = 0; a < kh; ++a)
        for (int64_t e = 0; e < kw; ++e) {
          double acc = 0.0, mag = 0.0;
          for (int64_t b = 0; b < batch; ++b)
            for (int64_t r = 0; r < OH; ++r)
              for (int64_t c = 0; c < OW; ++c) {
                double t = bf16_to_double(dy[((b * OH + r) * OW + c) * cout + co]) *
                           bf16_to_double(x[((b * H + r + a) * W + c + e) * cin + ci]);
                acc += t;
                mag += fabs(t);
              }
          int64_t o = ((co * cin + ci) * kh + a) * kw + e;
          dw[o] = acc;
          if (absmag) absmag[o] = mag;
        }
  return 0;
}
