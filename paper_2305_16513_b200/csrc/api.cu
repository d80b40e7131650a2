// api.cu -- the C ABI of libss (include/ss.h): argument validation, kernel
// selection and launch.  No device memory is allocated here; every entry point
// validates all arguments before enqueuing anything on the caller's stream.
#include <atomic>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "../../include/ss.h"
#include "ss_internal.h"

namespace ss {

static std::atomic<uint64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static thread_local std::string g_last_error;

cudaError_t ensure_smem_attr(const void* kfn) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, cudaError_t>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  for (auto& d : done)
    if (d.first.first == kfn && d.first.second == dev) return d.second;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
  done.push_back({{kfn, dev}, e});
  return e;
}

static ss_status_t fail(ss_status_t st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}
static ss_status_t cuda_fail(cudaError_t e, const char* where) {
  return fail(SS_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

int num_sms(int device) {
  static std::mutex mu;
  static int cache[128] = {0};
  if (device < 0 || device >= 128) return 148;
  std::lock_guard<std::mutex> lk(mu);
  if (cache[device] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0)
      n = 148;
    cache[device] = n;
  }
  return cache[device];
}

static int current_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  return num_sms(dev);
}

// cuTensorMapEncodeTiled from the driver, without linking libcuda.
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D view [rows][32] of 4-byte elements starting at `base` (16-B aligned),
// 128-B swizzled boxes of {32, box_rows}.
static bool make_map(CUtensorMap* m, const void* base, int64_t rows, int box_rows) {
  auto enc = encode_fn();
  if (!enc || rows < 1) return false;
  cuuint64_t dims[2] = {32, (cuuint64_t)rows};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool encode_rows_map(CUtensorMap* m, const void* base, int64_t rows, int box_rows) {
  return make_map(m, base, rows, box_rows);
}

// Fill the TMA-kernel geometry; false if this problem cannot take that path.
static bool make_slide_params(Slide1DParams& p, const void* x, void* y, int64_t N, int64_t batch,
                              int64_t L) {
  memset(&p, 0, sizeof p);
  const uintptr_t xa = reinterpret_cast<uintptr_t>(x), ya = reinterpret_cast<uintptr_t>(y);
  if ((xa & 3) || (ya & 3)) return false;
  p.x_view = reinterpret_cast<const void*>(xa & ~uintptr_t(15));
  p.y_view = reinterpret_cast<void*>(ya & ~uintptr_t(15));
  p.shift_x = (int64_t)((xa & 15) >> 2);
  p.shift_y = (int64_t)((ya & 15) >> 2);
  p.N = N;
  p.L = L;
  p.batch = batch;
  p.x_total_elems = p.shift_x + batch * N;
  const int64_t x_rows = p.x_total_elems / 32;
  if (x_rows < 8 || x_rows >= (int64_t(1) << 31) - 1024) return false;
  p.x_full_elems = 32 * x_rows;
  const int64_t y_rows = (p.shift_y + batch * L) / 32;
  if (y_rows >= (int64_t(1) << 31) - 1024) return false;
  if (!make_map(&p.tm_x_main, p.x_view, x_rows, kSlideTileRows)) return false;
  if (!make_map(&p.tm_x_halo, p.x_view, x_rows, 8)) return false;
  p.y_rows = y_rows;
  p.has_y_map = y_rows >= 1 && make_map(&p.tm_y, p.y_view, y_rows, 16);
  return true;
}

static bool overlaps(const void* a, int64_t abytes, const void* b, int64_t bbytes) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(a), b0 = reinterpret_cast<uintptr_t>(b);
  return a0 < b0 + (uintptr_t)bbytes && b0 < a0 + (uintptr_t)abytes;
}

static ss_status_t validate_1d(const void* x, const void* y, int64_t N, int64_t batch, int64_t w,
                               int64_t stride, const char* wname, int64_t* L) {
  if (!x || !y) return fail(SS_ERR_NULL, "x and y must be non-NULL device pointers");
  if (N < 1 || batch < 1 || w < 1 || stride < 1)
    return fail(SS_ERR_BAD_SIZE, "N=%lld batch=%lld %s=%lld stride=%lld must all be >= 1",
                (long long)N, (long long)batch, wname, (long long)w, (long long)stride);
  if (N > INT64_MAX / 8 / batch) return fail(SS_ERR_BAD_SIZE, "batch*N*4 overflows int64");
  if (w > N)
    return fail(SS_ERR_WINDOW_EXCEEDS_INPUT, "window exceeds input: %s=%lld > N=%lld", wname,
                (long long)w, (long long)N);
  *L = (N - w) / stride + 1;
  if (overlaps(x, batch * N * 4, y, batch * *L * 4)) return fail(SS_ERR_OVERLAP, "x and y overlap");
  return SS_OK;
}

static int pool_pivot(int64_t w) {
  if (w >= 32) return 32;
  if (w >= 16) return 16;
  if (w >= 8) return 8;
  if (w >= 4) return 4;
  if (w >= 2) return 2;
  return 1;
}

static int conv_bucket(int64_t k) {
  static const int ks[] = {1, 2, 3, 4, 5, 7, 8, 15, 16, 24, 31, 32, 48, 63, 64};
  for (int v : ks)
    if (k <= v) return v;
  return 0;
}

static ss_status_t pool_impl(int op, const void* x, void* y, int64_t N, int64_t batch, int64_t w,
                             int64_t stride, ss_dtype_t dtype, void* stream) {
  int64_t L = 0;
  ss_status_t st = validate_1d(x, y, N, batch, w, stride, "w", &L);
  if (st != SS_OK) return st;
  if (dtype != SS_F32 && dtype != SS_I32) return fail(SS_ERR_UNSUPPORTED, "dtype %d", (int)dtype);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int grid = current_sms();
  if (stride == 1 && w <= kPoolTmaMaxW) {
    Slide1DParams p;
    if (make_slide_params(p, x, y, N, batch, L)) {
      p.w = w;
      cudaError_t e = launch_pool_tma(p, op, dtype == SS_I32 ? 1 : 0, pool_pivot(w), s, grid);
      if (e == cudaSuccess) return SS_OK;
      if (e != cudaErrorInvalidConfiguration) return cuda_fail(e, "pool tma launch");
    }
  }
  GenericParams g;
  memset(&g, 0, sizeof g);
  g.x = x; g.y = y; g.N = N; g.L = L; g.batch = batch; g.w = w; g.stride = stride;
  cudaError_t e = launch_pool_generic(g, op, dtype == SS_I32 ? 1 : 0, s, grid * 8);
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "pool generic launch");
}

}  // namespace ss

using namespace ss;

extern "C" {

int ss_abi_version(void) { return SS_ABI_VERSION; }

int64_t ss_out_len(int64_t N, int64_t w, int64_t stride) {
  if (N < 1 || w < 1 || stride < 1 || w > N) return -1;
  return (N - w) / stride + 1;
}

ss_status_t ss_pool_sum(const void* x, void* y, int64_t N, int64_t batch, int64_t w,
                        int64_t stride, ss_dtype_t dtype, void* stream) {
  return pool_impl(kOpSum, x, y, N, batch, w, stride, dtype, stream);
}

ss_status_t ss_pool_max(const void* x, void* y, int64_t N, int64_t batch, int64_t w,
                        int64_t stride, ss_dtype_t dtype, void* stream) {
  return pool_impl(kOpMax, x, y, N, batch, w, stride, dtype, stream);
}

ss_status_t ss_conv1d(const void* x, void* y, int64_t N, int64_t batch, const float* filter_host,
                      int64_t k, int64_t stride, ss_dtype_t dtype, void* stream) {
  int64_t L = 0;
  if (!filter_host) return fail(SS_ERR_NULL, "filter_host must be non-NULL");
  ss_status_t st = validate_1d(x, y, N, batch, k, stride, "k", &L);
  if (st != SS_OK) return st;
  if (dtype != SS_F32) return fail(SS_ERR_UNSUPPORTED, "conv1d supports SS_F32 only");
  if (k > SS_K_MAX) return fail(SS_ERR_UNSUPPORTED, "k=%lld > SS_K_MAX=%d", (long long)k, SS_K_MAX);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int grid = current_sms();
  const int KT = conv_bucket(k);
  if (stride == 1 && KT > 0) {
    Slide1DParams p;
    if (make_slide_params(p, x, y, N, batch, L)) {
      for (int j = 0; j < KT; ++j) p.taps[j] = j < k ? filter_host[j] : 0.0f;
      p.w = k;
      cudaError_t e = launch_conv_tma(p, KT, s, grid);
      if (e == cudaSuccess) return SS_OK;
      if (e != cudaErrorInvalidConfiguration) return cuda_fail(e, "conv tma launch");
    }
  }
  GenericParams g;
  memset(&g, 0, sizeof g);
  g.x = x; g.y = y; g.N = N; g.L = L; g.batch = batch; g.w = k; g.stride = stride;
  for (int64_t j = 0; j < k; ++j) g.taps[j] = filter_host[j];
  cudaError_t e = launch_conv_generic(g, s, grid * 8);
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "conv generic launch");
}

ss_status_t ss_pool2d(const void* x, void* y, int64_t planes, int64_t H, int64_t W, int64_t kh,
                      int64_t kw, int64_t sh, int64_t sw, ss_pool_mode_t mode, ss_dtype_t dtype,
                      void* stream) {
  if (!x || !y) return fail(SS_ERR_NULL, "x and y must be non-NULL device pointers");
  if (planes < 1 || H < 1 || W < 1 || kh < 1 || kw < 1 || sh < 1 || sw < 1)
    return fail(SS_ERR_BAD_SIZE, "planes, H, W, kh, kw, sh, sw must all be >= 1");
  if (H > INT64_MAX / 8 / W || H * W > INT64_MAX / 8 / planes)
    return fail(SS_ERR_BAD_SIZE, "planes*H*W*4 overflows int64");
  if (kh > H || kw > W)
    return fail(SS_ERR_WINDOW_EXCEEDS_INPUT, "window %lldx%lld exceeds input %lldx%lld",
                (long long)kh, (long long)kw, (long long)H, (long long)W);
  if (mode != SS_POOL_MAX && mode != SS_POOL_AVG) return fail(SS_ERR_UNSUPPORTED, "mode %d", (int)mode);
  if (dtype != SS_F32) return fail(SS_ERR_UNSUPPORTED, "pool2d supports SS_F32 only");
  if ((reinterpret_cast<uintptr_t>(x) & 3) || (reinterpret_cast<uintptr_t>(y) & 3))
    return fail(SS_ERR_BAD_SIZE, "x and y must be 4-byte aligned");
  Pool2DParams p;
  memset(&p, 0, sizeof p);
  p.x = static_cast<const float*>(x);
  p.y = static_cast<float*>(y);
  p.planes = planes; p.H = H; p.W = W; p.kh = kh; p.kw = kw; p.sh = sh; p.sw = sw;
  p.OH = (H - kh) / sh + 1;
  p.OW = (W - kw) / sw + 1;
  if (overlaps(x, planes * H * W * 4, y, planes * p.OH * p.OW * 4))
    return fail(SS_ERR_OVERLAP, "x and y overlap");
  p.mode = mode == SS_POOL_AVG ? 1 : 0;
  p.inv_area = (float)(1.0 / (double)(kh * kw));
  p.bulk = ((reinterpret_cast<uintptr_t>(x) & 15) == 0) && (W % 4 == 0);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = launch_pool2d(p, s, current_sms());
  if (e == cudaErrorInvalidConfiguration) e = launch_pool2d_direct(p, s, current_sms() * 8);
  if (e == cudaSuccess) return SS_OK;
  return cuda_fail(e, "pool2d launch");
}

const char* ss_status_string(ss_status_t s) {
  switch (s) {
    case SS_OK: return "SS_OK";
    case SS_ERR_NULL: return "SS_ERR_NULL: a required pointer is NULL";
    case SS_ERR_BAD_SIZE: return "SS_ERR_BAD_SIZE: invalid size or stride";
    case SS_ERR_WINDOW_EXCEEDS_INPUT: return "SS_ERR_WINDOW_EXCEEDS_INPUT: window exceeds input";
    case SS_ERR_UNSUPPORTED: return "SS_ERR_UNSUPPORTED: unsupported dtype/mode/size";
    case SS_ERR_CUDA: return "SS_ERR_CUDA: CUDA error";
    case SS_ERR_OVERLAP: return "SS_ERR_OVERLAP: x and y overlap";
  }
  return "unknown ss_status_t";
}

const char* ss_last_error(void) { return g_last_error.c_str(); }

uint64_t ss_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
