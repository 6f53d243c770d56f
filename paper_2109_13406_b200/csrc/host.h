// host.h -- host-side plumbing shared by the C ABI translation units (host.cu).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "internal.h"

namespace ddb {
namespace host {

extern thread_local std::string g_last_error;
extern thread_local int g_last_route;
extern std::atomic<long long> g_launches;

int fail(cudaError_t e, const char* what);         // records the error, returns DDB_E*
int upflag(char c);
bool is_zero(double h, double l);
bool is_one(double h, double l);
bool in_window(double h, double l);                // the prescan's safe window, scalar form
bool debug_sync();
void retain_pool_memory();                         // keep the stream-ordered pool warm
cudaError_t panel_stream(cudaStream_t* out);       // high-priority stream per thread, device
int run(const GemmArgs& g, int mode, cudaStream_t s);   // one validated GEMM / SYRK call

int64_t span(int64_t nrow, int64_t ncol, int64_t ld);   // elements a column-major view covers

struct DevBuf {                                    // device staging buffer, freed on its stream
  double* p = nullptr;
  cudaStream_t s = nullptr;
  ~DevBuf() { if (p) cudaFreeAsync(p, s); }
};

int stage_in(DevBuf& b, const double* hi, const double* lo, int64_t n, cudaStream_t s);
int stage_in1(DevBuf& b, const double* x, int64_t n, cudaStream_t s);
int stage_out1(double* x, const DevBuf& b, int64_t n, cudaStream_t s);

}  // namespace host
}  // namespace ddb
