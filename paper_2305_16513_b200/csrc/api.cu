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

static int env_int(const char* name, int dflt);

// SS_FGRAD_TC=0: the FFMA filter-gradient kernels instead of the tensor-core one (A/B measurement)
bool tc_filter_grad_enabled() {
  static const bool on = [] {
    const char* e = getenv("SS_FGRAD_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

int dynamic_tiles() {
  static int on = env_int("SS_DYNAMIC_TILES", 1);
  return on != 0;
}

// SS_TILE_2D (read once, default 1): 0 routes stride-1 3x3 / 5x5 / 7x7 conv2d and its
// input gradient to the previous kernels (A/B only).
static int tile_2d_enabled() {
  static int on = env_int("SS_TILE_2D", 1);
  return on != 0;
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

// Chunk view for the tensor-core conv (conv_tc.cu): element (e, m, a) =
// base[128 m + 32 a + e], i.e. chunk m's K-atom a is the 128-B row 4m + a;
// box {32, nc + 8, 4} at {0, m0, 0} lands in smem as four (nc + 8) x 128-B
// K-major SWIZZLE_128B blocks, K-atoms 0..3 (atoms 4, 5 = blocks 0, 1 one row down).
bool encode_chunk_map(CUtensorMap* m, const void* base, int64_t m_ext, int atoms, int nc) {
  auto enc = encode_fn();
  if (!enc || m_ext < 1 || m_ext > (int64_t(1) << 31) - 1024) return false;
  cuuint64_t dims[3] = {32, (cuuint64_t)m_ext, (cuuint64_t)atoms};
  cuuint64_t strides[2] = {512, 128};
  cuuint32_t box[3] = {32, (cuuint32_t)(nc + 8), (cuuint32_t)atoms};  // one tile: nc + 8 chunks x 4 K-atoms
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Planes [planes][H][W] of fp32 for the 2-D tile kernel (conv2d_tile.cu): box
// {box_w, box_h, 1} lands as box_h dense rows of box_w floats (SWIZZLE_NONE),
// elements outside the plane (negative coordinates, columns >= W, rows >= H)
// zero-filled -- the tile's padding and pitch in one copy.  W*4 must be a
// multiple of 16 (TMA stride rule).
bool encode_plane_map(CUtensorMap* m, const float* base, int64_t W, int64_t H, int64_t planes, int box_w,
                      int box_h) {
  auto enc = encode_fn();
  if (!enc || (W * 4) % 16 || box_w > 256 || box_h > 256 || (box_w * 4) % 16) return false;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)(W * 4), (cuuint64_t)(H * W * 4)};
  cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Channels-last bf16 activations for the multi-channel conv (conv_mc.cu):
// element (e, p, a) = x[p * cin + 64 a + e]; box {64, box_rows, 1} lands one
// K-atom of box_rows positions as a SWIZZLE_128B K-major block, one position
// per 128-B row (positions past the array zero-filled).
bool encode_mc_map(CUtensorMap* m, const void* x, int64_t positions, int64_t cin, int box_rows) {
  auto enc = encode_fn();
  if (!enc || positions < 1 || positions > (int64_t(1) << 32) || cin % 64 || box_rows > 256 || box_rows < 8)
    return false;
  const int64_t at = cin / 64;
  cuuint64_t dims[3] = {64, (cuuint64_t)positions, (cuuint64_t)at};
  cuuint64_t strides[2] = {(cuuint64_t)(cin * 2), at > 1 ? 128 : (cuuint64_t)(positions * cin * 2)};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(x), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// fp32 rows of 128 (x viewed as [rows][128], 16-B aligned base), boxes of 33 rows, OOB zero fill.
bool encode_rows128_map(CUtensorMap* m, const void* base, int64_t rows) {
  auto enc = encode_fn();
  if (!enc || rows < 1 || rows >= (int64_t(1) << 31) || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
  cuuint64_t dims[2] = {128, (cuuint64_t)rows};
  cuuint64_t strides[1] = {512};
  cuuint32_t box[2] = {128, 33};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 1-D fp32 view of n elements (16-B aligned base), boxes of 256, OOB zero fill.
bool encode_flat_f32_map(CUtensorMap* m, const void* base, int64_t n) {
  auto enc = encode_fn();
  if (!enc || n < 1 || n >= (int64_t(1) << 31) || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
  cuuint64_t dims[1] = {(cuuint64_t)n};
  cuuint64_t strides[1] = {4};
  cuuint32_t box[1] = {256};
  cuuint32_t estr[1] = {1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Batched variant: 4-D {64, positions, cin/64, batch} (strides: position cin*2 B, atom 128 B, row
// positions*cin*2 B); a box starting before a row or running past it is zero-filled (row padding).
bool encode_mc_map_batched(CUtensorMap* m, const void* x, int64_t batch, int64_t positions, int64_t cin,
                           int box_rows) {
  auto enc = encode_fn();
  if (!enc || positions < 1 || positions > (int64_t(1) << 31) || batch < 1 || cin % 64 || box_rows > 256 ||
      box_rows < 8 || (positions * cin * 2) % 16)
    return false;
  const int64_t at = cin / 64;
  cuuint64_t dims[4] = {64, (cuuint64_t)positions, (cuuint64_t)at, (cuuint64_t)batch};
  cuuint64_t strides[3] = {(cuuint64_t)(cin * 2), 128, (cuuint64_t)(positions * cin * 2)};
  cuuint32_t box[4] = {64, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 5-D view of an NHWC bf16 image batch: {64 channels, OW, OH, c/64 atoms, batch}, box {64, box_w, box_h, 1, 1}
// (pad2d staging: boxes start up to kh-1 rows / kw-1 columns outside the image, zero-filled).
bool encode_mc_map_2d(CUtensorMap* m, const void* x, int64_t batch, int64_t OH, int64_t OW, int64_t c, int box_w,
                      int box_h) {
  auto enc = encode_fn();
  if (!enc || batch < 1 || OH < 1 || OW < 1 || c % 64 || box_w < 1 || box_w > 256 || box_h < 1 || box_h > 256 ||
      OH > (int64_t(1) << 31) || OW > (int64_t(1) << 31) || batch > (int64_t(1) << 31))
    return false;
  const int64_t at = c / 64;
  cuuint64_t dims[5] = {64, (cuuint64_t)OW, (cuuint64_t)OH, (cuuint64_t)at, (cuuint64_t)batch};
  cuuint64_t strides[4] = {(cuuint64_t)(c * 2), (cuuint64_t)(OW * c * 2), 128, (cuuint64_t)(OH * OW * c * 2)};
  cuuint32_t box[5] = {64, (cuuint32_t)box_w, (cuuint32_t)box_h, 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(x), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Tensor-core conv selection: k in [tc_min_k, kConvTcMaxK] at stride 1 without
// dilation (default 33: measured faster than the FFMA2 tile kernel for every
// k >= 33 on config 3).  SS_CONV_TC_MIN_K (read once) overrides the threshold, 0 disables
// the path; SS_CONV_TC_NC picks the chunk count per tile (32 / 48 / 64).
static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  if (!v || !*v) return dflt;
  return atoi(v);
}
static int tc_min_k() {
  static int v = env_int("SS_CONV_TC_MIN_K", 33);
  return v;
}
// Debug trace of the tensor-core conv: a CALLER-OWNED device buffer of 1024
// uint64 (64 x 8 CTA-0 role timestamps), set through ss_debug_conv_tc_set_trace
// (not in ss.h); null (the default) disables it.  The library allocates nothing.
static std::atomic<unsigned long long*> g_tc_trace{nullptr};
static std::atomic<uint64_t> g_tc_launches{0};

// Try the tensor-core conv for the interior outputs of every row (y_int =
// first interior output of row 0, rows y_pitch apart).  false: not applicable.
static bool try_conv_tc(const void* x, float* y_int, int64_t N, int64_t batch, int64_t k, int64_t y_pitch,
                        const float* taps, cudaStream_t s, int grid, cudaError_t* err, bool any_k = false) {
  *err = cudaSuccess;
  const int mk = tc_min_k();
  if (mk <= 0 || (!any_k && k < mk) || k > kConvTcMaxK) return false;
  const uintptr_t xa = reinterpret_cast<uintptr_t>(x);
  if (xa & 3) return false;
  ConvTCParams p;
  memset(&p, 0, sizeof p);
  p.x_view = reinterpret_cast<const float*>(xa & ~uintptr_t(15));
  p.shift_x = (int64_t)((xa & 15) >> 2);
  p.y = y_int;
  p.N = N;
  p.L_int = N - k + 1;
  p.batch = batch;
  p.y_pitch = y_pitch;
  p.y_off = 0;
  p.total_view = p.shift_x + batch * N;
  p.k = (int)k;
  p.K = 192;  // conv_tc.cu: fixed MMA depth, Toeplitz zero beyond k (k <= 65)
  p.atoms = 4;  // staged K-atoms per chunk; atoms 4, 5 are the next chunk's 0, 1
  if (p.total_view < 128 * 8) return false;
  // chunk m's 4 staged atoms are view rows 4m..4m+3: the map holds m_map chunks; chunk m's
  // outputs need chunk m + 1's atoms 0 and 1, so chunks [0, m_map - 1) run on the tensor cores
  const int64_t m_map = (p.total_view - 128) / 128 + 1;
  p.m_ext = m_map - 1;
  constexpr int nc = 64;  // chunks of 128 outputs per tile
  if (!encode_chunk_map(&p.tm_b, p.x_view, m_map, p.atoms, nc)) return false;
  for (int j = 0; j < (int)k; ++j) p.taps[j] = taps[j];
  p.trace = g_tc_trace.load(std::memory_order_relaxed);
  p.lo_bufs = 2;
  static int mixed = env_int("SS_CONV_TC_MIXED", 1);
  p.mixed = mixed;
  p.clc = dynamic_tiles();
  *err = launch_conv_tc(p, nc, s, grid);
  if (*err == cudaErrorInvalidConfiguration) { *err = cudaSuccess; return false; }
  g_tc_launches.fetch_add(1, std::memory_order_relaxed);
  return true;
}

// Fill the TMA-kernel geometry; false if this problem cannot take that path.
static bool make_slide_params(Slide1DParams& p, const void* x, void* y, int64_t N, int64_t batch,
                              int64_t L, int64_t y_pitch = -1, int64_t y_off = 0) {
  if (y_pitch < 0) y_pitch = L;
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
  p.y_pitch = y_pitch;
  p.y_off = y_off;
  const int64_t y_rows = (p.shift_y + batch * y_pitch) / 32;
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

// Window spec (ss.h): stride s, dilation d, zero padding pl/pr.  Computes the
// output length; validates everything before anything is enqueued.
static ss_status_t validate_1d(const void* x, const void* y, int64_t N, int64_t batch, int64_t w,
                               int64_t stride, int64_t d, int64_t pl, int64_t pr, const char* wname,
                               int64_t* L) {
  if (!x || !y) return fail(SS_ERR_NULL, "x and y must be non-NULL device pointers");
  if (N < 1 || batch < 1 || w < 1 || stride < 1 || d < 1)
    return fail(SS_ERR_BAD_SIZE, "N=%lld batch=%lld %s=%lld stride=%lld dilation=%lld must all be >= 1",
                (long long)N, (long long)batch, wname, (long long)w, (long long)stride, (long long)d);
  if (pl < 0 || pr < 0) return fail(SS_ERR_BAD_SIZE, "padding must be >= 0");
  if (N > INT64_MAX / 8 / batch || pl > INT64_MAX / 8 - N || pr > INT64_MAX / 8 - N - pl ||
      w > INT64_MAX / 8 / d)
    return fail(SS_ERR_BAD_SIZE, "sizes overflow int64");
  const int64_t E = (w - 1) * d + 1, Np = N + pl + pr;
  if (E > Np)
    return fail(SS_ERR_WINDOW_EXCEEDS_INPUT, "window exceeds input: extent %lld > padded N=%lld",
                (long long)E, (long long)Np);
  *L = (Np - E) / stride + 1;
  if (*L > INT64_MAX / 8 / batch) return fail(SS_ERR_BAD_SIZE, "batch*out_len*4 overflows int64");
  if (overlaps(x, batch * N * 4, y, batch * *L * 4)) return fail(SS_ERR_OVERLAP, "x and y overlap");
  return SS_OK;
}

static GenericParams generic_params(const void* x, void* y, int64_t N, int64_t L, int64_t batch,
                                    int64_t w, int64_t stride, int64_t d, int64_t pl) {
  GenericParams g;
  memset(&g, 0, sizeof g);
  g.x = x; g.y = y; g.N = N; g.L = L; g.batch = batch; g.w = w; g.stride = stride;
  g.dilation = d; g.pad_left = pl;
  return g;
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

// One 1-D window op.  Stride 1 without dilation takes the TMA tile kernel
// for every output whose window lies inside the row (with zero padding the
// tile kernel writes the interior of each padded output row, and a small
// generic launch fills the pl + pr edge outputs); everything else runs the
// direct-window generic kernels.
static ss_status_t window_impl(int op, const void* x, void* y, int64_t N, int64_t batch, int64_t w,
                               int64_t stride, int64_t d, int64_t pl, int64_t pr, int pad_mode,
                               ss_dtype_t dtype, const float* taps, void* stream) {
  int64_t L = 0;
  ss_status_t st = validate_1d(x, y, N, batch, w, stride, d, pl, pr, op == kOpConv ? "k" : "w", &L);
  if (st != SS_OK) return st;
  if (pad_mode < kPadZeros || pad_mode > kPadReplicate) return fail(SS_ERR_UNSUPPORTED, "pad_mode %d", pad_mode);
  if (pad_mode == kPadReflect && (pl > N - 1 || pr > N - 1))
    return fail(SS_ERR_BAD_SIZE, "reflect padding needs pad_left, pad_right <= N-1 (one reflection)");
  if (pad_mode == kPadCircular && (pl > N || pr > N))
    return fail(SS_ERR_BAD_SIZE, "circular padding needs pad_left, pad_right <= N (one period)");
  if (op == kOpConv) {
    if (dtype != SS_F32) return fail(SS_ERR_UNSUPPORTED, "conv1d supports SS_F32 only");
    if (w > SS_K_MAX) return fail(SS_ERR_UNSUPPORTED, "k=%lld > SS_K_MAX=%d", (long long)w, SS_K_MAX);
  } else if (dtype != SS_F32 && dtype != SS_I32) {
    return fail(SS_ERR_UNSUPPORTED, "dtype %d", (int)dtype);
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int grid = current_sms();
  const int dt = dtype == SS_I32 ? 1 : 0;
  const int64_t E = (w - 1) * d + 1;  // window extent
  const int64_t L_int = N - E + 1;     // outputs whose window is inside the row (stride 1)
  bool interior_done = false;
  if (stride == 1 && L_int >= 1 && op == kOpConv && E <= kConvTcMaxK) {
    // tensor cores: k >= the threshold, or any dilated filter whose extent fits (the
    // Toeplitz of the zero-expanded filter f_e[j d] = f_j)
    float expanded[kConvTcMaxK];
    const float* tt = taps;
    if (d > 1) {
      for (int64_t t = 0; t < E; ++t) expanded[t] = 0.0f;
      for (int64_t j = 0; j < w; ++j) expanded[j * d] = taps[j];
      tt = expanded;
    }
    cudaError_t e;
    if (try_conv_tc(x, static_cast<float*>(y) + pl, N, batch, E, L, tt, s, grid, &e, d > 1)) {
      if (e != cudaSuccess) return cuda_fail(e, "tensor-core conv launch");
      interior_done = true;
    }
  }
  if (!interior_done && stride == 1 && d > 1 && L_int >= 1 && w <= 32 && dtype == SS_F32) {
    // dilated windows: phase-decomposed tile kernel on the interior (dilated.cu)
    DilatedParams dp;
    memset(&dp, 0, sizeof dp);
    dp.x = x; dp.y = static_cast<float*>(y) + pl;
    dp.N = N; dp.L_int = L_int; dp.batch = batch; dp.w = w; dp.d = d; dp.y_pitch = L; dp.y_off = 0;
    if (op == kOpConv)
      for (int64_t j = 0; j < w; ++j) dp.taps[j] = taps[j];
    cudaError_t e = launch_dilated(dp, op, s, grid);
    if (e == cudaSuccess) interior_done = true;
    else if (e != cudaErrorInvalidConfiguration) return cuda_fail(e, "dilated launch");
  }
  if (!interior_done && stride == 1 && d == 1 && L_int >= 1) {
    const int KT = op == kOpConv ? conv_bucket(w) : 0;
    if (op == kOpConv ? KT > 0 : w <= kPoolTmaMaxW) {
      Slide1DParams p;
      // interior outputs land at y[b*L + pl + i], i < L_int
      char* y_int = static_cast<char*>(y) + 4 * pl;
      if (make_slide_params(p, x, y_int, N, batch, L_int, L, 0)) {
        p.w = w;
        p.clc = dynamic_tiles();
        cudaError_t e;
        if (op == kOpConv) {
          for (int j = 0; j < KT; ++j) p.taps[j] = j < w ? taps[j] : 0.0f;
          e = launch_conv_tma(p, KT, s, grid);
        } else {
          e = launch_pool_tma(p, op, dt, pool_pivot(w), s, grid);
        }
        if (e == cudaSuccess) interior_done = true;
        else if (e != cudaErrorInvalidConfiguration) return cuda_fail(e, "tma launch");
      }
    }
  }
  if (interior_done && pl == 0 && pr == 0) return SS_OK;
  GenericParams g = generic_params(x, y, N, L, batch, w, stride, d, pl);
  g.pad_mode = pad_mode;
  if (interior_done) {
    g.skip_lo = pl;
    g.skip_hi = pl + L_int;
  }
  if (op == kOpConv)
    for (int64_t j = 0; j < w; ++j) g.taps[j] = taps[j];
  cudaError_t e = op == kOpConv ? launch_conv_generic(g, s, grid * 8)
                                : launch_pool_generic(g, op, dt, s, grid * 8);
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "generic launch");
}

}  // namespace ss

using namespace ss;

extern "C" {

int ss_abi_version(void) { return SS_ABI_VERSION; }

/* Debug hook (not in ss.h): number of conv1d calls served by the tensor-core
 * kernel (tests use it to check which path ran). */
uint64_t ss_debug_conv_tc_launches(void) { return g_tc_launches.load(std::memory_order_relaxed); }

/* Debug hook (not in ss.h): later tensor-core conv launches write CTA 0's role
 * timestamps (64 x 8 clock64 values) into the caller's device buffer of 1024
 * uint64; null disables. */
void ss_debug_conv_tc_set_trace(void* device_buf) {
  g_tc_trace.store(static_cast<unsigned long long*>(device_buf), std::memory_order_relaxed);
}

int64_t ss_out_len(int64_t N, int64_t w, int64_t stride) {
  if (N < 1 || w < 1 || stride < 1 || w > N) return -1;
  return (N - w) / stride + 1;
}

ss_status_t ss_pool_sum(const void* x, void* y, int64_t N, int64_t batch, int64_t w,
                        int64_t stride, ss_dtype_t dtype, void* stream) {
  return window_impl(kOpSum, x, y, N, batch, w, stride, 1, 0, 0, kPadZeros, dtype, nullptr, stream);
}

ss_status_t ss_pool_max(const void* x, void* y, int64_t N, int64_t batch, int64_t w,
                        int64_t stride, ss_dtype_t dtype, void* stream) {
  return window_impl(kOpMax, x, y, N, batch, w, stride, 1, 0, 0, kPadZeros, dtype, nullptr, stream);
}

ss_status_t ss_pool_min(const void* x, void* y, int64_t N, int64_t batch, int64_t w,
                        int64_t stride, ss_dtype_t dtype, void* stream) {
  return window_impl(kOpMin, x, y, N, batch, w, stride, 1, 0, 0, kPadZeros, dtype, nullptr, stream);
}

ss_status_t ss_conv1d(const void* x, void* y, int64_t N, int64_t batch, const float* filter_host,
                      int64_t k, int64_t stride, ss_dtype_t dtype, void* stream) {
  if (!filter_host) return fail(SS_ERR_NULL, "filter_host must be non-NULL");
  return window_impl(kOpConv, x, y, N, batch, k, stride, 1, 0, 0, kPadZeros, dtype, filter_host, stream);
}

ss_status_t ss_pool_sum_ex(const void* x, void* y, int64_t N, int64_t batch, int64_t w,
                           int64_t stride, int64_t dilation, int64_t pad_left, int64_t pad_right,
                           ss_pad_mode_t pad_mode, ss_dtype_t dtype, void* stream) {
  return window_impl(kOpSum, x, y, N, batch, w, stride, dilation, pad_left, pad_right, (int)pad_mode, dtype,
                     nullptr, stream);
}

ss_status_t ss_pool_max_ex(const void* x, void* y, int64_t N, int64_t batch, int64_t w,
                           int64_t stride, int64_t dilation, int64_t pad_left, int64_t pad_right,
                           ss_pad_mode_t pad_mode, ss_dtype_t dtype, void* stream) {
  return window_impl(kOpMax, x, y, N, batch, w, stride, dilation, pad_left, pad_right, (int)pad_mode, dtype,
                     nullptr, stream);
}

ss_status_t ss_pool_min_ex(const void* x, void* y, int64_t N, int64_t batch, int64_t w,
                           int64_t stride, int64_t dilation, int64_t pad_left, int64_t pad_right,
                           ss_pad_mode_t pad_mode, ss_dtype_t dtype, void* stream) {
  return window_impl(kOpMin, x, y, N, batch, w, stride, dilation, pad_left, pad_right, (int)pad_mode, dtype,
                     nullptr, stream);
}

ss_status_t ss_conv1d_ex(const void* x, void* y, int64_t N, int64_t batch, const float* filter_host,
                         int64_t k, int64_t stride, int64_t dilation, int64_t pad_left,
                         int64_t pad_right, ss_pad_mode_t pad_mode, ss_dtype_t dtype, void* stream) {
  if (!filter_host) return fail(SS_ERR_NULL, "filter_host must be non-NULL");
  return window_impl(kOpConv, x, y, N, batch, k, stride, dilation, pad_left, pad_right, (int)pad_mode, dtype,
                     filter_host, stream);
}

// ---- backward passes (backward.cu) -----------------------
static ss_status_t validate_bwd(const void* a, const void* b, const void* dx, int64_t N, int64_t batch,
                                int64_t w, int64_t stride, const char* wname, int64_t* L) {
  if (!a || !b || !dx) return fail(SS_ERR_NULL, "pointers must be non-NULL device pointers");
  if (N < 1 || batch < 1 || w < 1 || stride < 1)
    return fail(SS_ERR_BAD_SIZE, "N=%lld batch=%lld %s=%lld stride=%lld must all be >= 1", (long long)N,
                (long long)batch, wname, (long long)w, (long long)stride);
  if (N > INT64_MAX / 8 / batch) return fail(SS_ERR_BAD_SIZE, "sizes overflow int64");
  if (w > N) return fail(SS_ERR_WINDOW_EXCEEDS_INPUT, "window exceeds input: %s=%lld > N=%lld", wname,
                         (long long)w, (long long)N);
  *L = (N - w) / stride + 1;
  return SS_OK;
}

static ss_status_t pool_sum_backward_impl(const void* dy, void* dx, int64_t N, int64_t batch, int64_t w, int64_t stride,
                                   ss_dtype_t dtype, void* stream) {
  int64_t L = 0;
  ss_status_t st = validate_bwd(dy, dy, dx, N, batch, w, stride, "w", &L);
  if (st != SS_OK) return st;
  if (dtype != SS_F32 && dtype != SS_I32) return fail(SS_ERR_UNSUPPORTED, "dtype %d", (int)dtype);
  if (overlaps(dy, batch * L * 4, dx, batch * N * 4)) return fail(SS_ERR_OVERLAP, "dy and dx overlap");
  if (stride == 1)  // dx = sliding sum of dy zero-padded by w-1 on both sides (length L + w - 1 = N)
    return window_impl(kOpSum, dy, dx, L, batch, w, 1, 1, w - 1, w - 1, kPadZeros, dtype, nullptr, stream);
  BackwardParams p;
  memset(&p, 0, sizeof p);
  p.dy = dy; p.dx = dx; p.N = N; p.L = L; p.batch = batch; p.w = w; p.stride = stride;
  cudaError_t e = launch_transpose_window(p, kOpSum, dtype == SS_I32 ? 1 : 0, static_cast<cudaStream_t>(stream),
                                          current_sms());
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "pool_sum_backward launch");
}

static ss_status_t conv1d_backward_input_impl(const void* dy, void* dx, int64_t N, int64_t batch, const float* f,
                                       int64_t k, int64_t stride, ss_dtype_t dtype, void* stream) {
  if (!f) return fail(SS_ERR_NULL, "filter_host must be non-NULL");
  int64_t L = 0;
  ss_status_t st = validate_bwd(dy, dy, dx, N, batch, k, stride, "k", &L);
  if (st != SS_OK) return st;
  if (dtype != SS_F32) return fail(SS_ERR_UNSUPPORTED, "conv1d backward supports SS_F32 only");
  if (k > SS_K_MAX) return fail(SS_ERR_UNSUPPORTED, "k=%lld > SS_K_MAX=%d", (long long)k, SS_K_MAX);
  if (overlaps(dy, batch * L * 4, dx, batch * N * 4)) return fail(SS_ERR_OVERLAP, "dy and dx overlap");
  if (stride == 1) {  // dx = dy zero-padded by k-1 on both sides, correlated with the flipped filter
    float flipped[SS_K_MAX];
    for (int64_t j = 0; j < k; ++j) flipped[j] = f[k - 1 - j];
    return window_impl(kOpConv, dy, dx, L, batch, k, 1, 1, k - 1, k - 1, kPadZeros, SS_F32, flipped, stream);
  }
  BackwardParams p;
  memset(&p, 0, sizeof p);
  p.dy = dy; p.dx = dx; p.N = N; p.L = L; p.batch = batch; p.w = k; p.stride = stride;
  for (int64_t j = 0; j < k; ++j) p.taps[j] = f[j];
  cudaError_t e = launch_transpose_window(p, kOpConv, 0, static_cast<cudaStream_t>(stream), current_sms());
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "conv1d_backward_input launch");
}

static ss_status_t pool_max_backward_impl(const void* x, const void* dy, void* dx, int64_t N, int64_t batch, int64_t w,
                                   int64_t stride, ss_dtype_t dtype, void* stream) {
  int64_t L = 0;
  ss_status_t st = validate_bwd(x, dy, dx, N, batch, w, stride, "w", &L);
  if (st != SS_OK) return st;
  if (dtype != SS_F32) return fail(SS_ERR_UNSUPPORTED, "pool_max backward supports SS_F32 only");
  if (overlaps(dy, batch * L * 4, dx, batch * N * 4) || overlaps(x, batch * N * 4, dx, batch * N * 4))
    return fail(SS_ERR_OVERLAP, "dx overlaps an input");
  BackwardParams p;
  memset(&p, 0, sizeof p);
  p.x = x; p.dy = dy; p.dx = dx; p.N = N; p.L = L; p.batch = batch; p.w = w; p.stride = stride;
  if (stride == 1 && pool_max_backward_s1_supported(w) && batch * N + 8192 < (int64_t(1) << 31)) {
    MaxBwdS1Params q;
    memset(&q, 0, sizeof q);
    q.dx = static_cast<float*>(dx); q.N = N; q.L = L; q.batch = batch; q.w = w;
    if (encode_flat_f32_map(&q.tm_x, x, batch * N) && encode_flat_f32_map(&q.tm_dy, dy, batch * L)) {
      cudaError_t e = launch_pool_max_backward_s1(q, static_cast<cudaStream_t>(stream), current_sms());
      return e == cudaSuccess ? SS_OK : cuda_fail(e, "pool_max_backward launch");
    }
  }
  cudaError_t e = launch_pool_max_backward(p, static_cast<cudaStream_t>(stream), current_sms());
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "pool_max_backward launch");
}

static ss_status_t conv1d_backward_filter_impl(const void* x, const void* dy, float* df, int64_t N, int64_t batch, int64_t k,
                                        int64_t stride, void* workspace, size_t ws_bytes, void* stream) {
  int64_t L = 0;
  ss_status_t st = validate_bwd(x, dy, df, N, batch, k, stride, "k", &L);
  if (st != SS_OK) return st;
  if (k > SS_K_MAX) return fail(SS_ERR_UNSUPPORTED, "k=%lld > SS_K_MAX=%d", (long long)k, SS_K_MAX);
  const int ctas = conv_filter_grad_ctas(current_sms());
  const size_t need = conv_filter_grad_workspace(k, ctas);
  if (!workspace || ws_bytes < need)
    return fail(SS_ERR_BAD_SIZE, "workspace of %zu bytes needed (ss_conv1d_backward_filter_workspace)", need);
  if (overlaps(workspace, (int64_t)need, x, batch * N * 4) || overlaps(workspace, (int64_t)need, dy, batch * L * 4) ||
      overlaps(workspace, (int64_t)need, df, k * 4) || overlaps(df, k * 4, x, batch * N * 4) ||
      overlaps(df, k * 4, dy, batch * L * 4))
    return fail(SS_ERR_OVERLAP, "df / workspace overlap an input");
  BackwardParams p;
  memset(&p, 0, sizeof p);
  p.x = x; p.dy = dy; p.N = N; p.L = L; p.batch = batch; p.w = k; p.stride = stride;
  FgradTcParams q;
  memset(&q, 0, sizeof q);
  if (conv_filter_grad_tc_supported(N, k, stride, x) && encode_rows128_map(&q.tm_x, x, batch * N / 128)) {
    q.x = static_cast<const float*>(x); q.dy = static_cast<const float*>(dy); q.part = static_cast<double*>(workspace);
    q.N = N; q.L = L; q.batch = batch; q.k = k;
    cudaError_t e = launch_conv_filter_grad_tc(q, df, ctas, current_sms(), static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? SS_OK : cuda_fail(e, "conv1d_backward_filter launch");
  }
  cudaError_t e = launch_conv_filter_grad(p, df, workspace, ctas, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "conv1d_backward_filter launch");
}

static size_t conv1d_backward_filter_workspace_impl(int64_t k) {
  if (k < 1 || k > SS_K_MAX) return 0;
  return conv_filter_grad_workspace(k, conv_filter_grad_ctas(current_sms()));
}

static ss_status_t pool2d_backward_impl(const void* x, const void* dy, void* dx, int64_t planes, int64_t H, int64_t W,
                                 int64_t kh, int64_t kw, int64_t sh, int64_t sw, ss_pool_mode_t mode,
                                 ss_dtype_t dtype, void* stream) {
  if (!dy || !dx || (mode == SS_POOL_MAX && !x)) return fail(SS_ERR_NULL, "pointers must be non-NULL");
  if (planes < 1 || H < 1 || W < 1 || kh < 1 || kw < 1 || sh < 1 || sw < 1)
    return fail(SS_ERR_BAD_SIZE, "planes/H/W/kh/kw/sh/sw must be >= 1");
  if (kh > H || kw > W) return fail(SS_ERR_WINDOW_EXCEEDS_INPUT, "window exceeds input");
  if (mode != SS_POOL_MAX && mode != SS_POOL_AVG) return fail(SS_ERR_UNSUPPORTED, "mode %d", (int)mode);
  if (dtype != SS_F32) return fail(SS_ERR_UNSUPPORTED, "pool2d backward supports SS_F32 only");
  if (H > INT64_MAX / 8 / W || H * W > INT64_MAX / 8 / planes) return fail(SS_ERR_BAD_SIZE, "sizes overflow int64");
  Pool2DBackwardParams p;
  memset(&p, 0, sizeof p);
  p.x = static_cast<const float*>(x); p.dy = static_cast<const float*>(dy); p.dx = static_cast<float*>(dx);
  p.planes = planes; p.H = H; p.W = W; p.kh = kh; p.kw = kw; p.sh = sh; p.sw = sw;
  p.OH = (H - kh) / sh + 1; p.OW = (W - kw) / sw + 1;
  p.mode = mode == SS_POOL_AVG ? 1 : 0;
  p.inv_area = 1.0f / (float)(kh * kw);
  const int64_t nx = planes * H * W * 4, ny = planes * p.OH * p.OW * 4;
  if (overlaps(dy, ny, dx, nx) || (x && overlaps(x, nx, dx, nx))) return fail(SS_ERR_OVERLAP, "dx overlaps an input");
  if (p.mode == 1 && sh == 1 && sw == 1 && tile_2d_enabled() && conv2d_tile_supported((int)kh, (int)kw, H, W)) {
    // average pooling at stride 1: dx = the full correlation of dy with the box 1/(kh kw) -- the
    // 2-D tile kernel's padded mode, as for the conv2d input gradient
    Conv2DTileParams t;
    memset(&t, 0, sizeof t);
    t.x = p.dy; t.y = p.dx; t.planes = planes;
    t.IH = (int)p.OH; t.IW = (int)p.OW; t.OH = (int)H; t.OW = (int)W; t.KH = (int)kh; t.KW = (int)kw;
    t.pad_t = (int)kh - 1; t.pad_l = (int)kw - 1;
    for (int64_t i = 0; i < kh * kw; ++i) t.taps[i] = p.inv_area;
    t.clc = dynamic_tiles();
    cudaError_t e = launch_conv2d_tile(t, static_cast<cudaStream_t>(stream), current_sms());
    if (e == cudaSuccess) return SS_OK;
    if (e != cudaErrorInvalidConfiguration) return cuda_fail(e, "pool2d_backward tile launch");
  }
  cudaError_t e = launch_pool2d_backward(p, static_cast<cudaStream_t>(stream), current_sms());
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "pool2d_backward launch");
}

static ss_status_t conv2d_bwd_check(int64_t planes, int64_t H, int64_t W, int64_t kh, int64_t kw, int64_t sh,
                                     int64_t sw) {
  if (planes < 1 || H < 1 || W < 1 || kh < 1 || kw < 1 || sh < 1 || sw < 1)
    return fail(SS_ERR_BAD_SIZE, "planes/H/W/kh/kw/sh/sw must be >= 1");
  if (H > INT64_MAX / 8 / W || H * W > INT64_MAX / 8 / planes) return fail(SS_ERR_BAD_SIZE, "sizes overflow int64");
  if (kh > H || kw > W) return fail(SS_ERR_WINDOW_EXCEEDS_INPUT, "window exceeds input: %lldx%lld > %lldx%lld",
                                    (long long)kh, (long long)kw, (long long)H, (long long)W);
  if (kh * kw > SS_K_MAX) return fail(SS_ERR_UNSUPPORTED, "kh*kw=%lld > SS_K_MAX=%d", (long long)(kh * kw), SS_K_MAX);
  return SS_OK;
}

ss_status_t ss_conv2d_backward_input(const void* dy, void* dx, int64_t planes, int64_t H, int64_t W,
                                     const float* filter_host, int64_t kh, int64_t kw, int64_t sh, int64_t sw,
                                     ss_dtype_t dtype, void* stream) {
  if (!dy || !dx || !filter_host) return fail(SS_ERR_NULL, "dy, dx and filter_host must be non-NULL");
  ss_status_t st = conv2d_bwd_check(planes, H, W, kh, kw, sh, sw);
  if (st != SS_OK) return st;
  if (dtype != SS_F32) return fail(SS_ERR_UNSUPPORTED, "conv2d backward supports SS_F32 only");
  if ((reinterpret_cast<uintptr_t>(dy) & 3) || (reinterpret_cast<uintptr_t>(dx) & 3))
    return fail(SS_ERR_BAD_SIZE, "dy and dx must be 4-byte aligned");
  Conv2DBwdParams p;
  memset(&p, 0, sizeof p);
  p.dy = static_cast<const float*>(dy); p.dx = static_cast<float*>(dx);
  p.planes = planes; p.H = H; p.W = W; p.kh = kh; p.kw = kw; p.sh = sh; p.sw = sw;
  p.OH = (H - kh) / sh + 1; p.OW = (W - kw) / sw + 1;
  if (overlaps(dy, planes * p.OH * p.OW * 4, dx, planes * H * W * 4)) return fail(SS_ERR_OVERLAP, "dx overlaps dy");
  if (sh == 1 && sw == 1 && tile_2d_enabled() && conv2d_tile_supported((int)kh, (int)kw, H, W)) {
    // stride 1: dx = the full correlation of dy with the flipped filter = the tile kernel's
    // valid correlation of dy bordered by kh-1 / kw-1 zeros (reading R21)
    Conv2DTileParams t;
    memset(&t, 0, sizeof t);
    t.x = p.dy; t.y = p.dx; t.planes = planes;
    t.IH = (int)p.OH; t.IW = (int)p.OW; t.OH = (int)H; t.OW = (int)W; t.KH = (int)kh; t.KW = (int)kw;
    t.pad_t = (int)kh - 1; t.pad_l = (int)kw - 1;
    for (int64_t i = 0; i < kh * kw; ++i) t.taps[i] = filter_host[kh * kw - 1 - i];
    t.clc = dynamic_tiles();
    cudaError_t e = launch_conv2d_tile(t, static_cast<cudaStream_t>(stream), current_sms());
    if (e == cudaSuccess) return SS_OK;
    if (e != cudaErrorInvalidConfiguration) return cuda_fail(e, "conv2d_backward_input tile launch");
  }
  for (int64_t t = 0; t < kh * kw; ++t) p.taps[t] = filter_host[t];
  cudaError_t e = launch_conv2d_backward_input(p, static_cast<cudaStream_t>(stream), current_sms());
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "conv2d_backward_input launch");
}

size_t ss_conv2d_backward_filter_workspace(int64_t kh, int64_t kw) {
  if (kh < 1 || kw < 1 || kh * kw > SS_K_MAX) return 0;
  return conv2d_backward_filter_workspace(kh * kw, conv2d_backward_filter_ctas(current_sms()));
}

ss_status_t ss_conv2d_backward_filter(const void* x, const void* dy, float* df, int64_t planes, int64_t H, int64_t W,
                                      int64_t kh, int64_t kw, int64_t sh, int64_t sw, void* workspace,
                                      size_t workspace_bytes, void* stream) {
  if (!x || !dy || !df || !workspace) return fail(SS_ERR_NULL, "x, dy, df and workspace must be non-NULL");
  ss_status_t st = conv2d_bwd_check(planes, H, W, kh, kw, sh, sw);
  if (st != SS_OK) return st;
  if ((reinterpret_cast<uintptr_t>(x) & 3) || (reinterpret_cast<uintptr_t>(dy) & 3) ||
      (reinterpret_cast<uintptr_t>(df) & 3) || (reinterpret_cast<uintptr_t>(workspace) & 7))
    return fail(SS_ERR_BAD_SIZE, "x, dy, df must be 4-byte and workspace 8-byte aligned");
  const int ctas = conv2d_backward_filter_ctas(current_sms());
  const size_t need = conv2d_backward_filter_workspace(kh * kw, ctas);
  if (workspace_bytes < need)
    return fail(SS_ERR_BAD_SIZE, "workspace of %zu bytes needed (ss_conv2d_backward_filter_workspace)", need);
  Conv2DBwdParams p;
  memset(&p, 0, sizeof p);
  p.x = static_cast<const float*>(x); p.dy = static_cast<const float*>(dy);
  p.planes = planes; p.H = H; p.W = W; p.kh = kh; p.kw = kw; p.sh = sh; p.sw = sw;
  p.OH = (H - kh) / sh + 1; p.OW = (W - kw) / sw + 1;
  const int64_t nx = planes * H * W * 4, ny = planes * p.OH * p.OW * 4, nw = (int64_t)need, nf = kh * kw * 4;
  if (overlaps(workspace, nw, x, nx) || overlaps(workspace, nw, dy, ny) || overlaps(workspace, nw, df, nf) ||
      overlaps(df, nf, x, nx) || overlaps(df, nf, dy, ny))
    return fail(SS_ERR_OVERLAP, "df / workspace overlap an input");
  cudaError_t e = launch_conv2d_backward_filter(p, df, workspace, ctas, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "conv2d_backward_filter launch");
}

// TMA boxes per staged atom: nbox boxes of box_rows (<= 256, a multiple of 8) cover p.rows.
static bool mc_boxes(ConvMcParams& p) {
  p.rows = mc_round_rows(p.rows, &p.nbox, &p.box_rows);
  return p.rows <= 2048;
}

ss_status_t ss_conv1d_mc(const void* x, const void* w, float* y, int64_t batch, int64_t N, int64_t cin,
                         int64_t cout, int64_t k, void* stream) {
  if (!x || !w || !y) return fail(SS_ERR_NULL, "x, w and y must be non-NULL device pointers");
  if (batch < 1 || N < 1 || cin < 1 || cout < 1 || k < 1)
    return fail(SS_ERR_BAD_SIZE, "batch/N/cin/cout/k must all be >= 1");
  if (N > INT64_MAX / 8 / batch / cin || cout > INT64_MAX / 8 / batch / N || k > INT64_MAX / 8 / cin / cout)
    return fail(SS_ERR_BAD_SIZE, "sizes overflow int64");
  if (k > N) return fail(SS_ERR_WINDOW_EXCEEDS_INPUT, "window exceeds input: k=%lld > N=%lld", (long long)k,
                         (long long)N);
  if ((reinterpret_cast<uintptr_t>(x) & 1) || (reinterpret_cast<uintptr_t>(w) & 1) ||
      (reinterpret_cast<uintptr_t>(y) & 3))
    return fail(SS_ERR_BAD_SIZE, "x / w must be 2-byte and y 4-byte aligned");
  const int64_t L = N - k + 1;
  if (overlaps(x, batch * N * cin * 2, y, batch * L * cout * 4) || overlaps(w, cout * cin * k * 2, y, batch * L * cout * 4))
    return fail(SS_ERR_OVERLAP, "y overlaps an input");
  ConvMcParams p;
  memset(&p, 0, sizeof p);
  p.x = x; p.w = w; p.y = y; p.batch = batch; p.N = N; p.L = L; p.cin = cin; p.cout = cout; p.k = k;
  for (int64_t j = 0; j < k && j < kMcMaxTaps; ++j) p.tap_off[j] = (int)j;
  p.mblk = conv_mc_choose_mblk(cin, cout, k, 136, k <= 4);
  p.rows = 128 * p.mblk + 8;  // 128 mblk outputs + k - 1 <= 8 halo positions
  const bool tc = (cin == 64 || cin == 128) && (cout == 64 || cout == 128) && k <= 9 &&
                  (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0 &&
                  mc_boxes(p) && encode_mc_map(&p.tm_x, x, batch * N, cin, p.box_rows);
  p.clc = dynamic_tiles();
  cudaError_t e = launch_conv_mc(p, tc, static_cast<cudaStream_t>(stream), current_sms());
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "conv1d_mc launch");
}

ss_status_t ss_conv1d_mc_backward_input(const void* dy, const void* w, float* dx, int64_t batch, int64_t N,
                                        int64_t cin, int64_t cout, int64_t k, void* stream) {
  if (!dy || !w || !dx) return fail(SS_ERR_NULL, "dy, w and dx must be non-NULL device pointers");
  if (batch < 1 || N < 1 || cin < 1 || cout < 1 || k < 1)
    return fail(SS_ERR_BAD_SIZE, "batch/N/cin/cout/k must all be >= 1");
  if (N > INT64_MAX / 8 / batch / cin || N > INT64_MAX / 8 / batch / cout || k > INT64_MAX / 8 / cin / cout)
    return fail(SS_ERR_BAD_SIZE, "sizes overflow int64");
  if (k > N) return fail(SS_ERR_WINDOW_EXCEEDS_INPUT, "window exceeds input: k=%lld > N=%lld", (long long)k,
                         (long long)N);
  if ((reinterpret_cast<uintptr_t>(dy) & 1) || (reinterpret_cast<uintptr_t>(w) & 1) ||
      (reinterpret_cast<uintptr_t>(dx) & 3))
    return fail(SS_ERR_BAD_SIZE, "dy / w must be 2-byte and dx 4-byte aligned");
  const int64_t L = N - k + 1;
  if (overlaps(dy, batch * L * cout * 2, dx, batch * N * cin * 4) || overlaps(w, cout * cin * k * 2, dx, batch * N * cin * 4))
    return fail(SS_ERR_OVERLAP, "dx overlaps an input");
  // dx[b][t][ci] = sum_j sum_co w[co][ci][k-1-j] dy[b][t - (k-1) + j][co]: the forward implicit GEMM on dy
  // (channels cout -> cin) with the weights transposed and flipped, over rows padded by k-1 zeros
  ConvMcParams p;
  memset(&p, 0, sizeof p);
  p.x = dy; p.w = w; p.y = dx; p.batch = batch; p.N = L; p.L = N; p.cin = cout; p.cout = cin; p.k = k;
  p.bwd_in = 1; p.batched = 1; p.pad = (int)(k - 1); p.n_out = N;
  for (int64_t j = 0; j < k && j < kMcMaxTaps; ++j) p.tap_off[j] = (int)j;
  p.mblk = conv_mc_choose_mblk(cout, cin, k, 136);
  p.rows = 128 * p.mblk + 8;
  const bool tc = (cin == 64 || cin == 128) && (cout == 64 || cout == 128) && k <= 9 &&
                  (reinterpret_cast<uintptr_t>(dy) & 15) == 0 && (reinterpret_cast<uintptr_t>(dx) & 15) == 0 &&
                  mc_boxes(p) && encode_mc_map_batched(&p.tm_x, dy, batch, L, cout, p.box_rows);
  p.clc = dynamic_tiles();
  cudaError_t e = launch_conv_mc(p, tc, static_cast<cudaStream_t>(stream), current_sms());
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "conv1d_mc_backward_input launch");
}

size_t ss_conv1d_mc_backward_filter_workspace(int64_t cin, int64_t cout, int64_t k) {
  return mc_filter_grad_workspace(cin, cout, k, current_sms());
}

ss_status_t ss_conv1d_mc_backward_filter(const void* dy, const void* x, float* dw, int64_t batch, int64_t N,
                                         int64_t cin, int64_t cout, int64_t k, void* workspace,
                                         size_t workspace_bytes, void* stream) {
  if (!dy || !x || !dw) return fail(SS_ERR_NULL, "dy, x and dw must be non-NULL device pointers");
  if (batch < 1 || N < 1 || cin < 1 || cout < 1 || k < 1)
    return fail(SS_ERR_BAD_SIZE, "batch/N/cin/cout/k must all be >= 1");
  if (N > INT64_MAX / 8 / batch / cin || N > INT64_MAX / 8 / batch / cout || k > INT64_MAX / 8 / cin / cout)
    return fail(SS_ERR_BAD_SIZE, "sizes overflow int64");
  if (k > N) return fail(SS_ERR_WINDOW_EXCEEDS_INPUT, "window exceeds input: k=%lld > N=%lld", (long long)k,
                         (long long)N);
  if ((reinterpret_cast<uintptr_t>(dy) & 1) || (reinterpret_cast<uintptr_t>(x) & 1) ||
      (reinterpret_cast<uintptr_t>(dw) & 3))
    return fail(SS_ERR_BAD_SIZE, "dy / x must be 2-byte and dw 4-byte aligned");
  const int64_t L = N - k + 1;
  const int sms = current_sms();
  const size_t need = mc_filter_grad_workspace(cin, cout, k, sms);
  if (need && (!workspace || workspace_bytes < need))
    return fail(SS_ERR_BAD_SIZE, "workspace of %zu bytes needed (ss_conv1d_mc_backward_filter_workspace)", need);
  const int64_t nw = cout * cin * k * 4;
  if (overlaps(dw, nw, dy, batch * L * cout * 2) || overlaps(dw, nw, x, batch * N * cin * 2) ||
      (need && (overlaps(workspace, (int64_t)need, dy, batch * L * cout * 2) ||
                overlaps(workspace, (int64_t)need, x, batch * N * cin * 2) || overlaps(workspace, (int64_t)need, dw, nw))))
    return fail(SS_ERR_OVERLAP, "dw / workspace overlap an input");
  McFgradParams p;
  memset(&p, 0, sizeof p);
  p.dy = static_cast<const uint16_t*>(dy); p.x = static_cast<const uint16_t*>(x); p.dw = dw;
  p.ws = static_cast<double*>(workspace);
  p.batch = batch; p.N = N; p.L = L; p.cin = cin; p.cout = cout; p.k = k;
  const bool tc = need && (reinterpret_cast<uintptr_t>(dy) & 15) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(workspace) & 7) == 0 &&
                  encode_mc_map_batched(&p.tm_dy, dy, batch, L, cout, 128) &&
                  encode_mc_map_batched(&p.tm_x, x, batch, N, cin, 136);
  cudaError_t e = launch_mc_filter_grad(p, tc, static_cast<cudaStream_t>(stream), sms);
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "conv1d_mc_backward_filter launch");
}

ss_status_t ss_conv2d_mc(const void* x, const void* w, float* y, int64_t batch, int64_t H, int64_t W, int64_t cin,
                         int64_t cout, int64_t kh, int64_t kw, void* stream) {
  if (!x || !w || !y) return fail(SS_ERR_NULL, "x, w and y must be non-NULL device pointers");
  if (batch < 1 || H < 1 || W < 1 || cin < 1 || cout < 1 || kh < 1 || kw < 1)
    return fail(SS_ERR_BAD_SIZE, "batch/H/W/cin/cout/kh/kw must all be >= 1");
  if (H > INT64_MAX / 8 / W || H * W > INT64_MAX / 8 / batch || batch * H * W > INT64_MAX / 8 / cin ||
      batch * H * W > INT64_MAX / 8 / cout || kh * kw > INT64_MAX / 8 / cin / cout)
    return fail(SS_ERR_BAD_SIZE, "sizes overflow int64");
  if (kh > H || kw > W)
    return fail(SS_ERR_WINDOW_EXCEEDS_INPUT, "window %lldx%lld exceeds input %lldx%lld", (long long)kh, (long long)kw,
                (long long)H, (long long)W);
  if ((reinterpret_cast<uintptr_t>(x) & 1) || (reinterpret_cast<uintptr_t>(w) & 1) ||
      (reinterpret_cast<uintptr_t>(y) & 3))
    return fail(SS_ERR_BAD_SIZE, "x / w must be 2-byte and y 4-byte aligned");
  const int64_t OH = H - kh + 1, OW = W - kw + 1;
  const int64_t ybytes = batch * OH * OW * cout * 4;
  if (overlaps(x, batch * H * W * cin * 2, y, ybytes) || overlaps(w, cout * cin * kh * kw * 2, y, ybytes))
    return fail(SS_ERR_OVERLAP, "y overlaps an input");
  ConvMcParams p;
  memset(&p, 0, sizeof p);
  p.x = x; p.w = w; p.y = y; p.batch = batch; p.N = H * W; p.cin = cin; p.cout = cout; p.k = kh * kw;
  p.two_d = 1; p.H = H; p.W = W; p.OH = OH; p.OW = OW;
  // flat positions over the image rows: tap (a, e) reads the staged tile shifted by a W + e
  // positions; a tile of 128 flat output positions stages 128 + (kh-1) W + kw - 1 positions
  bool tc = (cin == 64 || cin == 128) && (cout == 64 || cout == 128) && kh * kw <= kMcMaxTaps &&
            (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0 &&
            (kh - 1) * W + kw - 1 <= 1024;
  if (tc) {
    for (int64_t a = 0; a < kh; ++a)
      for (int64_t e = 0; e < kw; ++e) p.tap_off[a * kw + e] = (int)(a * W + e);
    p.mblk = conv_mc_choose_mblk(cin, cout, kh * kw, (int)(128 + (kh - 1) * W + kw - 1), true);
    p.rows = (int)(128 * p.mblk + (kh - 1) * W + kw - 1);
    tc = mc_boxes(p) && encode_mc_map(&p.tm_x, x, batch * H * W, cin, p.box_rows);
  }
  p.clc = dynamic_tiles();
  cudaError_t e = launch_conv_mc(p, tc, static_cast<cudaStream_t>(stream), current_sms());
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "conv2d_mc launch");
}

ss_status_t ss_conv2d_mc_backward_input(const void* dy, const void* w, float* dx, int64_t batch, int64_t H,
                                        int64_t W, int64_t cin, int64_t cout, int64_t kh, int64_t kw, void* stream) {
  if (!dy || !w || !dx) return fail(SS_ERR_NULL, "dy, w and dx must be non-NULL device pointers");
  if (batch < 1 || H < 1 || W < 1 || cin < 1 || cout < 1 || kh < 1 || kw < 1)
    return fail(SS_ERR_BAD_SIZE, "batch/H/W/cin/cout/kh/kw must all be >= 1");
  if (H > INT64_MAX / 8 / W || H * W > INT64_MAX / 8 / batch || batch * H * W > INT64_MAX / 8 / cin ||
      batch * H * W > INT64_MAX / 8 / cout || kh * kw > INT64_MAX / 8 / cin / cout)
    return fail(SS_ERR_BAD_SIZE, "sizes overflow int64");
  if (kh > H || kw > W)
    return fail(SS_ERR_WINDOW_EXCEEDS_INPUT, "window %lldx%lld exceeds input %lldx%lld", (long long)kh, (long long)kw,
                (long long)H, (long long)W);
  if ((reinterpret_cast<uintptr_t>(dy) & 1) || (reinterpret_cast<uintptr_t>(w) & 1) ||
      (reinterpret_cast<uintptr_t>(dx) & 3))
    return fail(SS_ERR_BAD_SIZE, "dy / w must be 2-byte and dx 4-byte aligned");
  const int64_t OH = H - kh + 1, OW = W - kw + 1;
  const int64_t dxbytes = batch * H * W * cin * 4;
  if (overlaps(dy, batch * OH * OW * cout * 2, dx, dxbytes) || overlaps(w, cout * cin * kh * kw * 2, dx, dxbytes))
    return fail(SS_ERR_OVERLAP, "dx overlaps an input");
  // dx = the forward on dy zero-padded by (kh-1, kw-1) with the weights transposed and flipped (reading R26):
  // tiles of R dx rows x Cw columns, each staged as one TMA box per atom that starts outside dy
  ConvMcParams p;
  memset(&p, 0, sizeof p);
  p.x = dy; p.w = w; p.y = dx; p.batch = batch; p.cin = cout; p.cout = cin; p.k = kh * kw;
  p.H = H; p.W = W; p.OH = OH; p.OW = OW; p.N = OH * OW; p.L = H * W;
  p.pad2d = 1; p.bwd_in = 1; p.pd_kh = (int)(kh < 1024 ? kh : 1024); p.pd_kw = (int)(kw < 1024 ? kw : 1024);  // tc: kh kw <= 64
  const bool tc = (cin == 64 || cin == 128) && (cout == 64 || cout == 128) && kh * kw <= kMcMaxTaps &&
                  (reinterpret_cast<uintptr_t>(dy) & 15) == 0 && (reinterpret_cast<uintptr_t>(dx) & 15) == 0 &&
                  H < (int64_t(1) << 31) && W < (int64_t(1) << 31) && conv_mc_plan_pad2d(p) &&
                  encode_mc_map_2d(&p.tm_x, dy, batch, OH, OW, cout, p.pd_P, p.pd_R + (int)kh - 1);
  p.clc = dynamic_tiles();
  cudaError_t e = launch_conv_mc(p, tc, static_cast<cudaStream_t>(stream), current_sms());
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "conv2d_mc_backward_input launch");
}

size_t ss_conv2d_mc_backward_filter_workspace(int64_t cin, int64_t cout, int64_t kh, int64_t kw) {
  if (kh < 1 || kh > 64) return 0;
  return mc_filter_grad_workspace(cin, cout, kw, current_sms(), true);
}

ss_status_t ss_conv2d_mc_backward_filter(const void* dy, const void* x, float* dw, int64_t batch, int64_t H,
                                         int64_t W, int64_t cin, int64_t cout, int64_t kh, int64_t kw,
                                         void* workspace, size_t workspace_bytes, void* stream) {
  if (!dy || !x || !dw) return fail(SS_ERR_NULL, "dy, x and dw must be non-NULL device pointers");
  if (batch < 1 || H < 1 || W < 1 || cin < 1 || cout < 1 || kh < 1 || kw < 1)
    return fail(SS_ERR_BAD_SIZE, "batch/H/W/cin/cout/kh/kw must all be >= 1");
  if (H > INT64_MAX / 8 / W || H * W > INT64_MAX / 8 / batch || batch * H * W > INT64_MAX / 8 / cin ||
      batch * H * W > INT64_MAX / 8 / cout || kh * kw > INT64_MAX / 8 / cin / cout)
    return fail(SS_ERR_BAD_SIZE, "sizes overflow int64");
  if (kh > H || kw > W)
    return fail(SS_ERR_WINDOW_EXCEEDS_INPUT, "window %lldx%lld exceeds input %lldx%lld", (long long)kh, (long long)kw,
                (long long)H, (long long)W);
  if ((reinterpret_cast<uintptr_t>(dy) & 1) || (reinterpret_cast<uintptr_t>(x) & 1) ||
      (reinterpret_cast<uintptr_t>(dw) & 3))
    return fail(SS_ERR_BAD_SIZE, "dy / x must be 2-byte and dw 4-byte aligned");
  const int64_t OH = H - kh + 1, OW = W - kw + 1;
  const int sms = current_sms();
  const size_t need = ss_conv2d_mc_backward_filter_workspace(cin, cout, kh, kw);
  if (need && (!workspace || workspace_bytes < need))
    return fail(SS_ERR_BAD_SIZE, "workspace of %zu bytes needed (ss_conv2d_mc_backward_filter_workspace)", need);
  const int64_t nw = cout * cin * kh * kw * 4, ndy = batch * OH * OW * cout * 2, nx = batch * H * W * cin * 2;
  if (overlaps(dw, nw, dy, ndy) || overlaps(dw, nw, x, nx) ||
      (need && (overlaps(workspace, (int64_t)need, dy, ndy) || overlaps(workspace, (int64_t)need, x, nx) ||
                overlaps(workspace, (int64_t)need, dw, nw))))
    return fail(SS_ERR_OVERLAP, "dw / workspace overlap an input");
  McFgradParams p;
  memset(&p, 0, sizeof p);
  p.dy = static_cast<const uint16_t*>(dy); p.x = static_cast<const uint16_t*>(x); p.dw = dw;
  p.ws = static_cast<double*>(workspace);
  p.batch = batch; p.N = H * W; p.L = OH * OW; p.cin = cin; p.cout = cout; p.k = kw;
  p.two_d = 1; p.kh = (int)(kh < 1024 ? kh : 1024); p.H = H; p.W = W; p.OH = OH; p.OW = OW;
  // dy rows staged with pitch W (the box runs past OW: zero fill) against x rows shifted by the tap row
  const bool tc = need && (reinterpret_cast<uintptr_t>(dy) & 15) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(workspace) & 7) == 0 && mc_filter_grad_2d_plan(p) &&
                  encode_mc_map_2d(&p.tm_dy, dy, batch, OH, OW, cout, (int)W, p.dy_fill / (int)W) &&
                  encode_mc_map_2d(&p.tm_x, x, batch, H, W, cin, (int)W, p.R + 1);
  cudaError_t e = launch_mc_filter_grad(p, tc, static_cast<cudaStream_t>(stream), sms);
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "conv2d_mc_backward_filter launch");
}

ss_status_t ss_conv2d(const void* x, void* y, int64_t planes, int64_t H, int64_t W, const float* filter_host,
                      int64_t kh, int64_t kw, int64_t sh, int64_t sw, ss_dtype_t dtype, void* stream) {
  if (!x || !y || !filter_host) return fail(SS_ERR_NULL, "x, y and filter_host must be non-NULL");
  if (planes < 1 || H < 1 || W < 1 || kh < 1 || kw < 1 || sh < 1 || sw < 1)
    return fail(SS_ERR_BAD_SIZE, "planes/H/W/kh/kw/sh/sw must be >= 1");
  if (H > INT64_MAX / 8 / W || H * W > INT64_MAX / 8 / planes) return fail(SS_ERR_BAD_SIZE, "sizes overflow int64");
  if (kh > H || kw > W) return fail(SS_ERR_WINDOW_EXCEEDS_INPUT, "window exceeds input: %lldx%lld > %lldx%lld",
                                    (long long)kh, (long long)kw, (long long)H, (long long)W);
  if (dtype != SS_F32) return fail(SS_ERR_UNSUPPORTED, "conv2d supports SS_F32 only");
  if (kh * kw > SS_K_MAX) return fail(SS_ERR_UNSUPPORTED, "kh*kw=%lld > SS_K_MAX=%d", (long long)(kh * kw), SS_K_MAX);
  if ((reinterpret_cast<uintptr_t>(x) & 3) || (reinterpret_cast<uintptr_t>(y) & 3))
    return fail(SS_ERR_BAD_SIZE, "x and y must be 4-byte aligned");
  Conv2DParams p;
  memset(&p, 0, sizeof p);
  p.x = static_cast<const float*>(x); p.y = static_cast<float*>(y);
  p.planes = planes; p.H = H; p.W = W; p.kh = kh; p.kw = kw; p.sh = sh; p.sw = sw;
  p.OH = (H - kh) / sh + 1; p.OW = (W - kw) / sw + 1;
  if (overlaps(x, planes * H * W * 4, y, planes * p.OH * p.OW * 4)) return fail(SS_ERR_OVERLAP, "x and y overlap");
  // stride-1 5x5 / 7x7: the FFMA2 tile kernel (FP32-pipe bound); 3x3 stays on the
  // memory-bound vector kernel, measured faster there
  if (sh == 1 && sw == 1 && kh * kw >= 25 && tile_2d_enabled() && conv2d_tile_supported((int)kh, (int)kw, p.OH, p.OW)) {
    Conv2DTileParams t;
    memset(&t, 0, sizeof t);
    t.x = p.x; t.y = p.y; t.planes = planes;
    t.IH = (int)H; t.IW = (int)W; t.OH = (int)p.OH; t.OW = (int)p.OW; t.KH = (int)kh; t.KW = (int)kw;
    for (int64_t i = 0; i < kh * kw; ++i) t.taps[i] = filter_host[i];
    t.clc = dynamic_tiles();
    cudaError_t e = launch_conv2d_tile(t, static_cast<cudaStream_t>(stream), current_sms());
    if (e == cudaSuccess) return SS_OK;
    if (e != cudaErrorInvalidConfiguration) return cuda_fail(e, "conv2d tile launch");
  }
  for (int64_t t = 0; t < kh * kw; ++t) p.taps[t] = filter_host[t];
  p.clc = dynamic_tiles();
  cudaError_t e = launch_conv2d(p, static_cast<cudaStream_t>(stream), current_sms());
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "conv2d launch");
}

ss_status_t ss_pool_sum_backward(const void* dy, void* dx, int64_t N, int64_t batch, int64_t w, int64_t stride,
                                 ss_dtype_t dtype, void* stream) {
  return pool_sum_backward_impl(dy, dx, N, batch, w, stride, dtype, stream);
}

ss_status_t ss_pool_max_backward(const void* x, const void* dy, void* dx, int64_t N, int64_t batch, int64_t w,
                                 int64_t stride, ss_dtype_t dtype, void* stream) {
  return pool_max_backward_impl(x, dy, dx, N, batch, w, stride, dtype, stream);
}

ss_status_t ss_conv1d_backward_input(const void* dy, void* dx, int64_t N, int64_t batch, const float* filter_host,
                                     int64_t k, int64_t stride, ss_dtype_t dtype, void* stream) {
  return conv1d_backward_input_impl(dy, dx, N, batch, filter_host, k, stride, dtype, stream);
}

size_t ss_conv1d_backward_filter_workspace(int64_t k) { return conv1d_backward_filter_workspace_impl(k); }

ss_status_t ss_conv1d_backward_filter(const void* x, const void* dy, float* df, int64_t N, int64_t batch, int64_t k,
                                      int64_t stride, void* workspace, size_t workspace_bytes, void* stream) {
  return conv1d_backward_filter_impl(x, dy, df, N, batch, k, stride, workspace, workspace_bytes, stream);
}

ss_status_t ss_pool2d_backward(const void* x, const void* dy, void* dx, int64_t planes, int64_t H, int64_t W,
                               int64_t kh, int64_t kw, int64_t sh, int64_t sw, ss_pool_mode_t mode, ss_dtype_t dtype,
                               void* stream) {
  return pool2d_backward_impl(x, dy, dx, planes, H, W, kh, kw, sh, sw, mode, dtype, stream);
}

int64_t ss_out_len_ex(int64_t N, int64_t w, int64_t stride, int64_t dilation, int64_t pad_left,
                      int64_t pad_right) {
  if (N < 1 || w < 1 || stride < 1 || dilation < 1 || pad_left < 0 || pad_right < 0) return -1;
  if (w > INT64_MAX / 8 / dilation || pad_left > INT64_MAX / 8 - N || pad_right > INT64_MAX / 8 - N - pad_left)
    return -1;
  const int64_t E = (w - 1) * dilation + 1, Np = N + pad_left + pad_right;
  if (E > Np) return -1;
  return (Np - E) / stride + 1;
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
  p.clc = dynamic_tiles();
  cudaError_t e = launch_pool2d(p, s, current_sms());
  if (e == cudaErrorInvalidConfiguration) e = launch_pool2d_direct(p, s, current_sms() * 8);
  if (e == cudaSuccess) return SS_OK;
  return cuda_fail(e, "pool2d launch");
}

ss_status_t ss_affine_window(const float* u, const float* v, float* U, float* V, int64_t N,
                             int64_t batch, int64_t w, int64_t stride, void* stream) {
  if (!u || !v || !V) return fail(SS_ERR_NULL, "u, v and V must be non-NULL device pointers");
  if (N < 1 || batch < 1 || w < 1 || stride < 1)
    return fail(SS_ERR_BAD_SIZE, "N, batch, w, stride must all be >= 1");
  if (N > INT64_MAX / 8 / batch) return fail(SS_ERR_BAD_SIZE, "batch*N*4 overflows int64");
  if (w > N)
    return fail(SS_ERR_WINDOW_EXCEEDS_INPUT, "window exceeds input: w=%lld > N=%lld", (long long)w,
                (long long)N);
  if (w > SS_AFFINE_W_MAX) return fail(SS_ERR_UNSUPPORTED, "w > SS_AFFINE_W_MAX");
  if ((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(v) |
       reinterpret_cast<uintptr_t>(U) | reinterpret_cast<uintptr_t>(V)) & 3)
    return fail(SS_ERR_BAD_SIZE, "u, v, U, V must be 4-byte aligned");
  const int64_t L = (N - w) / stride + 1;
  const int64_t in_b = batch * N * 4, out_b = batch * L * 4;
  if (overlaps(u, in_b, V, out_b) || overlaps(v, in_b, V, out_b) ||
      (U && (overlaps(u, in_b, U, out_b) || overlaps(v, in_b, U, out_b) || overlaps(U, out_b, V, out_b))))
    return fail(SS_ERR_OVERLAP, "outputs overlap an input or each other");
  AffineParams p;
  memset(&p, 0, sizeof p);
  p.u = u; p.v = v; p.U = U; p.V = V;
  p.N = N; p.L = L; p.batch = batch; p.w = w; p.stride = stride;
  const cudaError_t e = launch_affine(p, static_cast<cudaStream_t>(stream), current_sms());
  if (e == cudaSuccess) return SS_OK;
  return cuda_fail(e, "affine_window launch");
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
