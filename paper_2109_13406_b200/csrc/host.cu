// host.cu -- host-side plumbing shared by the C ABI translation units
// (capi.cu: the BLAS entry points; capi_lapack.cu: Rtrsm / Rgetrf / Rgetrs /
// Rpotrf): error state, launch accounting, the stream-ordered workspace pool,
// the GEMM driver `run`, host staging helpers and the auxiliary streams.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/ddblas.h"
#include "host.h"

namespace ddb {
namespace host {

thread_local std::string g_last_error;
thread_local int g_last_route = -1;
std::atomic<long long> g_launches{0};

int fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? DDB_ENOMEM : DDB_ECUDA;
}

int upflag(char c) { return (c >= 'a' && c <= 'z') ? c - 32 : c; }
bool is_zero(double h, double l) { return h == 0.0 && l == 0.0; }
bool is_one(double h, double l) { return h == 1.0 && l == 0.0; }

static int bexp(double x) {
  long long b;
  std::memcpy(&b, &x, sizeof b);
  return (int)((b >> 52) & 0x7ff);
}
// scalar safe-window test (same window as dd_prescan.cu)
bool in_window(double h, double l) {
  const int eh = bexp(h), el = bexp(l);
  return !((h != 0.0 && eh < WIN_LO) || eh > WIN_HI || el > WIN_HI);
}

bool debug_sync() {
  static const bool on = [] {
    const char* v = std::getenv("DDB_DEBUG_SYNC");
    return v != nullptr && v[0] != '\0' && v[0] != '0';
  }();
  return on;
}

// The per-call workspace and host staging buffers come from the device's
// stream-ordered pool; keep freed blocks cached instead of returning them to
// the driver at every synchronisation (release threshold = unlimited).
void retain_pool_memory() {
  static thread_local int done_mask = 0;   // bit per device id < 32
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 32 || (done_mask >> dev) & 1) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    unsigned long long thr = ~0ULL;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done_mask |= 1 << dev;
}

// Rpotrf's panel stream (highest priority), one per host thread and device.
cudaError_t panel_stream(cudaStream_t* out) {
  static thread_local cudaStream_t streams[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 64) return cudaErrorInvalidDevice;
  if (streams[dev] == nullptr) {
    int least = 0, greatest = 0;
    e = cudaDeviceGetStreamPriorityRange(&least, &greatest);
    if (e == cudaSuccess)
      e = cudaStreamCreateWithPriority(&streams[dev], cudaStreamNonBlocking, greatest);
    if (e != cudaSuccess) return e;
  }
  *out = streams[dev];
  return cudaSuccess;
}

// Runs one validated, non-trivial call: prescan (+ route summary) -> [fast:
// bound] -> the mode's tiled kernel (EC_FAST elements) -> [fast: TwoSum
// fallback for EC_WIDE elements] -> [split-K reduce] -> reference-semantics
// kernel for the EC_REF elements (exits at once when there are none).
int run(const GemmArgs& g0, int mode, cudaStream_t s) {
  int nl = 0;
  cudaError_t e;
  GemmArgs g = g0;
  {
    static const int gm_env = [] {
      const char* v = std::getenv("DDB_GROUP_M");
      return v ? std::atoi(v) : 0;
    }();
    g.group_m = gm_env;
  }
  if (g.f64) {   // binary64: bit-exact tiled kernel for every input (no window)
    if (g.alpha.h == 0.0 || g.k == 0 || mode == MODE_REFERENCE) {
      e = launch_reference(g, nullptr, GATE_ALWAYS, s, &nl);
      g_launches += nl;
      if (e != cudaSuccess) return fail(e, "reference kernel launch");
      g_last_route = 2;
      return DDB_OK;
    }
    g.kchunk = g.k;
    e = launch_tiled(g, ALG_F64, nullptr, nullptr, nullptr, s, &nl);
    g_launches += nl;
    if (e != cudaSuccess) return fail(e, "f64 kernel launch");
    g_last_route = debug_sync() ? 4 : -1;
    return DDB_OK;
  }
  const bool trivial_ref = mode == MODE_REFERENCE || is_zero(g.alpha.h, g.alpha.l) || g.k == 0;
  bool scalars_ok = true;
  if (mode == MODE_EXACT)
    scalars_ok = in_window(g.alpha.h, g.alpha.l) && in_window(g.beta.h, g.beta.l);
  if (trivial_ref || !scalars_ok) {
    e = launch_reference(g, nullptr, GATE_ALWAYS, s, &nl);
    g_launches += nl;
    if (e != cudaSuccess) return fail(e, "reference kernel launch");
    g_last_route = 2;
    return DDB_OK;
  }
  retain_pool_memory();
  int alg = alg_for_mode(mode);
  // The certified bound's accumulation factor (1 + k 2^-21, below) keeps
  // S' <= 1.064 sum |ab| up to k = 2^16; deeper calls take the TwoSum MAC,
  // whose error bound holds at any depth.
  if (alg == ALG_CERT && g.k > kCertMaxK) alg = ALG_TWOSUM;
  const int64_t nrow = g.m, ncol = g.n;
  const size_t head = route_ws_bytes(nrow, ncol, g.syrk);
  int64_t kchunk = g.k;
  const int splits = choose_ksplit(g, alg, &kchunk);
  g.kchunk = kchunk;
  const size_t part_bytes = splits > 1 ? (size_t)splits * 2 * g.m * g.n * sizeof(double) : 0;
  const size_t bnd_bytes = alg == ALG_CERT ? ((bound_workspace_bytes(g) + 255) / 256) * 256 : 0;
  const size_t ws_bytes = head + bnd_bytes + part_bytes;
  void* ws = nullptr;
  e = cudaMallocAsync(&ws, ws_bytes, s);
  if (e != cudaSuccess) return fail(e, "workspace allocation");
  const RouteWs r = route_ws_carve(ws, nrow, ncol, g.syrk);
  const char* what = "dd kernel launch";
  e = cudaMemsetAsync(ws, 0, head, s);
  if (e == cudaSuccess) e = launch_prescan(g, alg, r, s, &nl);
  g.rsp = r.rsp; g.csp = r.csp; g.rsb = r.rsb; g.csb = r.csb; g.flag = r.flag;
  g.bad_rows = r.bad_rows; g.bad_cols = r.bad_cols;
  g.wide_lim = alg == ALG_CERT ? wide_limit(g.k) : 0;
  if (e == cudaSuccess && alg == ALG_CERT) {
    char* bw = static_cast<char*>(ws) + head;
    float* bound = bound_carve(g, bw);
    g.bound = bound;
    g.bnd_fac = 1.0 + (double)g.k * 0x1p-21;
    g.bnd_floor = (double)g.k * 0x1p-120;
    e = launch_bound(g, r.rmax, r.cmax, bw, bound, s, &nl, &what);
  }
  if (splits > 1) g.part = reinterpret_cast<double*>(static_cast<char*>(ws) + head + bnd_bytes);
  if (e == cudaSuccess) e = launch_tiled(g, alg, r.rmax, r.cmax, r.flag, s, &nl);
  if (e == cudaSuccess && alg == ALG_CERT) e = launch_wide_fallback(g, s, &nl);
  if (e == cudaSuccess && splits > 1) e = launch_splitk_reduce(g, splits, r.flag, s, &nl);
  if (e == cudaSuccess) e = launch_reference(g, r.flag, GATE_IF_UNSAFE, s, &nl);
  g_launches += nl;
  int route = -1;
  if (e == cudaSuccess && debug_sync()) {
    // 0 exact, 1 fast, 3 twosum; 2 = some elements took the reference
    // kernel, 5 = some took the TwoSum fallback (fast mode)
    int f[3] = {0, 0, 0};
    e = cudaMemcpyAsync(f, r.flag, sizeof f, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    route = f[0] != ROUTE_SAFE ? 2
            : (g.wide_lim > 0 && f[1] + f[2] > g.wide_lim) ? 5
            : (mode == MODE_EXACT ? 0 : (alg == ALG_CERT ? 1 : 3));
  }
  cudaError_t e2 = cudaFreeAsync(ws, s);
  if (e != cudaSuccess) return fail(e, what);
  if (e2 != cudaSuccess) return fail(e2, "workspace free");
  g_last_route = route;
  return DDB_OK;
}


int64_t span(int64_t nrow, int64_t ncol, int64_t ld) {
  return (nrow <= 0 || ncol <= 0) ? 0 : (ncol - 1) * ld + nrow;
}


int stage_in(DevBuf& b, const double* hi, const double* lo, int64_t n, cudaStream_t s) {
  b.s = s;
  retain_pool_memory();
  if (n == 0) return DDB_OK;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&b.p), sizeof(double) * 2 * n, s);
  if (e != cudaSuccess) return fail(e, "host staging allocation");
  e = cudaMemcpyAsync(b.p, hi, sizeof(double) * n, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(b.p + n, lo, sizeof(double) * n, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return fail(e, "host to device copy");
  return DDB_OK;
}

int stage_in1(DevBuf& b, const double* x, int64_t n, cudaStream_t s) {
  b.s = s;
  retain_pool_memory();
  if (n == 0) return DDB_OK;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&b.p), sizeof(double) * n, s);
  if (e != cudaSuccess) return fail(e, "host staging allocation");
  e = cudaMemcpyAsync(b.p, x, sizeof(double) * n, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return fail(e, "host to device copy");
  return DDB_OK;
}
int stage_out1(double* x, const DevBuf& b, int64_t n, cudaStream_t s) {
  cudaError_t e = cudaMemcpyAsync(x, b.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(e, "device to host copy");
  return DDB_OK;
}

}  // namespace host
}  // namespace ddb
