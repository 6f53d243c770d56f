// dd_getrf.cu -- blocked dd LU with partial pivoting (Rgetrf, mplapack/lu.py:74-114).
//
// The reference is unblocked right-looking: per column j, pivot search
// (DDBackend.argmax_abs, elem.py:246-259: max |hi|, ties by max lo*sign(hi),
// first index), interchange of the whole rows, scaling of the column by the
// pivot's reciprocal (or a division when |pivot| < safmin), then the rank-1
// update a(i, c) += mul2(a(i, j), -a(j, c)) of everything right of / below.
// Per element the updates arrive in j order, so the LAPACK blocking keeps
// the result bit-identical in exact mode:
//   1. getrf_panel_kernel  factors the nb-column panel over all rows below j0
//      -- one cooperative launch, rows split over the CTAs, two grid barriers
//      per column (after the partial pivot searches; after the interchange);
//   2. getrf_laswp_kernel  applies the panel's interchanges to the columns
//      left and right of it (in order, per column);
//   3. getrf_trsm_kernel   U12 = L11^-1 A12, one thread per column, the
//      reference's per-element order;
//   4. the trailing update A22 += L21 (-U12) as Rgemm (alpha = -1, beta = 1)
//      in the caller's mode: per element c = c + mul2(L, mul2(-1, U)), which
//      equals the reference's mul2(L, -U) bit for bit (mul2(-1, u) differs
//      from -u at most in the sign of a zero low word, which mul2 absorbs).
// A zero pivot sets info (first one) and skips the interchange and scaling
// but not the update, as the reference does; the pivot index is recorded
// either way (lu.py:93-106).
#include <cooperative_groups.h>

#include <cstdlib>

#include "lapack_num.cuh"

namespace ddb {

namespace {

// pivot-search key: larger |hi| wins, then larger lo*sign(hi), then the
// smaller row index; a NaN |hi| anywhere makes the search return its first
// row (np.max propagates NaN and no entry compares equal to it)
struct PivKey {
  double ah, al;     // |hi|, lo * sign(hi)
  double h, l;       // the entry itself (the pivot value, read before any interchange)
  long long idx;
  int nan;
};
__device__ __forceinline__ bool better(const PivKey& x, const PivKey& y) {
  if (x.idx < 0) return false;
  if (y.idx < 0) return true;
  if (x.ah != y.ah) return x.ah > y.ah;
  if (x.al != y.al) return x.al > y.al;
  return x.idx < y.idx;
}
__device__ __forceinline__ PivKey merge(PivKey x, const PivKey& y) {
  PivKey r = better(y, x) ? y : x;
  r.nan = x.nan | y.nan;
  return r;
}

__device__ __forceinline__ PivKey shfl_down(const PivKey& k, int o) {
  PivKey y;
  y.ah = __shfl_down_sync(0xffffffffu, k.ah, o);
  y.al = __shfl_down_sync(0xffffffffu, k.al, o);
  y.h = __shfl_down_sync(0xffffffffu, k.h, o);
  y.l = __shfl_down_sync(0xffffffffu, k.l, o);
  y.idx = __shfl_down_sync(0xffffffffu, k.idx, o);
  y.nan = __shfl_down_sync(0xffffffffu, k.nan, o);
  return y;
}

__device__ __forceinline__ double ldg_cg(const double* p) { return __ldcg(p); }

// grid-wide barrier for a cooperative launch: arrival counter in global
// memory, target = gridDim.x * (number of barriers so far)
__device__ void grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (true) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if (v >= target) break;
      __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

constexpr int kPanelThreads = 256;

// block-wide best key (all threads get it)
__device__ PivKey block_best(PivKey k) {
  __shared__ PivKey red[kPanelThreads / 32];
  for (int o = 16; o > 0; o >>= 1) k = merge(k, shfl_down(k, o));
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = k;
  __syncthreads();
  PivKey r = red[0];
  for (int i = 1; i < kPanelThreads / 32; ++i) r = merge(r, red[i]);
  return r;
}

}  // namespace

// Panel [j0, j0 + nb) over rows [j0, m).  CTA c owns rows [r0c, r1c).
template <class N>
__global__ void __launch_bounds__(kPanelThreads)
getrf_panel_kernel(GetrfArgs g, int64_t j0, int nb) {
  using T = typename N::T;
  __shared__ PivKey best_s;
  __shared__ T piv_s, rec_s;
  __shared__ int use_rec_s, nonzero_s;
  const int64_t rows = g.m - j0;
  const int64_t chunk = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = j0 + (int64_t)blockIdx.x * chunk;
  const int64_t r1 = r0 + chunk < g.m ? r0 + chunk : g.m;
  const int64_t lda = g.lda;
  double* ah = g.a_hi;
  double* al = g.a_lo;
  unsigned nbar = 0;
  auto local_search = [&](int64_t j) {
    PivKey k{0.0, 0.0, 0.0, 0.0, -1, 0};
    for (int64_t i = (r0 > j ? r0 : j) + threadIdx.x; i < r1; i += blockDim.x) {
      const T v = N::ldcg(ah, al, i + j * lda);
      PivKey y{N::key_hi(v), N::key_lo(v), N::hi(v), N::lo(v), (long long)i, N::key_nan(v) ? 1 : 0};
      k = merge(k, y);
    }
    k = block_best(k);
    if (threadIdx.x == 0) {
      g.part_ah[blockIdx.x] = k.ah;
      g.part_al[blockIdx.x] = k.al;
      g.part_h[blockIdx.x] = k.h;
      g.part_l[blockIdx.x] = k.l;
      g.part_idx[blockIdx.x] = k.idx;
      g.part_nan[blockIdx.x] = k.nan;
    }
  };
  local_search(j0);
  const int64_t jend = j0 + nb;
  for (int64_t j = j0; j < jend; ++j) {
    grid_barrier(g.bar, gridDim.x * ++nbar);
    if (threadIdx.x < 32) {   // merge the partial searches (warp 0)
      PivKey k{0.0, 0.0, 0.0, 0.0, -1, 0};
      for (int c = threadIdx.x; c < (int)gridDim.x; c += 32) {
        PivKey y{__ldcg(g.part_ah + c), __ldcg(g.part_al + c), __ldcg(g.part_h + c),
                 __ldcg(g.part_l + c), __ldcg(g.part_idx + c), __ldcg(g.part_nan + c)};
        k = merge(k, y);
      }
      for (int o = 16; o > 0; o >>= 1) k = merge(k, shfl_down(k, o));
      if (threadIdx.x == 0) {
        T piv = N::make(k.h, k.l);
        if (k.nan || k.idx < 0) {   // argmax_abs returns 0 -> the diagonal entry
          k.idx = j;
          piv = N::ldcg(ah, al, j + j * lda);
        }
        best_s = k;
        const int64_t jp = k.idx;
        piv_s = piv;
        nonzero_s = N::nonzero(piv);
        use_rec_s = N::ge_safmin(piv);                     // |pivot| >= safmin (lu.py:98)
        if (nonzero_s && use_rec_s) rec_s = N::sdiv(N::one(), piv);
        if (blockIdx.x == 0) {
          g.ipiv[j] = jp + 1;
          g.swap[j] = nonzero_s ? jp : j;
          if (!nonzero_s && *g.info == 0) *g.info = (int)(j + 1);
        }
      }
    }
    __syncthreads();
    const int64_t jp = best_s.idx;
    const bool nonzero = nonzero_s;
    if (blockIdx.x == 0 && nonzero && jp != j) {   // interchange within the panel
      for (int64_t c = j0 + threadIdx.x; c < jend; c += blockDim.x) {
        const T tj = N::ldcg(ah, al, j + c * lda);
        N::st(ah, al, j + c * lda, N::ldcg(ah, al, jp + c * lda));
        N::st(ah, al, jp + c * lda, tj);
      }
    }
    grid_barrier(g.bar, gridDim.x * ++nbar);
    // scale the column below the pivot (own rows), then the rank-1 update of
    // the panel's later columns
    const int64_t lo_row = r0 > j + 1 ? r0 : j + 1;
    if (nonzero) {
      const bool use_rec = use_rec_s;
      const T rec = rec_s, piv = piv_s;
      for (int64_t i = lo_row + threadIdx.x; i < r1; i += blockDim.x) {
        const T x = N::ldcg(ah, al, i + j * lda);
        N::st(ah, al, i + j * lda, use_rec ? N::mul(rec, x) : N::vdiv(x, piv));
      }
    }
    __syncthreads();
    const int64_t ncol = jend - j - 1;
    const int64_t nrow = r1 - lo_row;
    if (ncol > 0 && nrow > 0 && j < g.mn - 1) {
      for (int64_t t = threadIdx.x; t < ncol * nrow; t += blockDim.x) {
        const int64_t i = lo_row + t % nrow, c = j + 1 + t / nrow;
        const T x = N::ldcg(ah, al, i + j * lda), u = N::ldcg(ah, al, j + c * lda);
        N::st(ah, al, i + c * lda, N::add(N::ldcg(ah, al, i + c * lda), N::mul(x, N::neg(u))));
      }
    }
    __syncthreads();
    if (j + 1 < jend) local_search(j + 1);
  }
}

// Shared-memory panel, one grid barrier per column: CTA c stages its rows
// [r0, r1) of the panel in shared memory for the whole factorization.  With
// its partial pivot search each CTA publishes its candidate's whole panel row
// (double-buffered by column parity), and the owner of row j publishes row j,
// so after the single barrier every CTA has both rows of the interchange:
// the winner's candidate row becomes row j, the old row j goes to row jp.
// Falls back to the global-memory kernel when a CTA's share would not fit
// (kSmemRowsMax rows).
constexpr int kSmemRowsMax = 192;

// The shared-memory kernel's search key: argmax_abs's order (elem.py:246-259)
// as integers -- |hi| by its bits (non-negative doubles order like their bit
// patterns; a NaN |hi| sorts above +inf, so a NaN anywhere wins and is
// recognised on the winner), then lo * sign(hi) through the order-preserving
// map of signed doubles (after -0 -> +0: the reference compares with ==), then
// the smaller row.  The pivot value itself is read from the winner's
// published row, so the key is three words and a merge is integer compares.
struct SKey {
  unsigned long long ah, al;
  long long idx;                         // kNoRow: empty
};
constexpr long long kNoRow = 0x7fffffffffffffffLL;
__device__ __forceinline__ SKey skey_merge(const SKey& x, const SKey& y) {
  const bool yb = y.ah != x.ah ? y.ah > x.ah : (y.al != x.al ? y.al > x.al : y.idx < x.idx);
  return yb ? y : x;
}
__device__ __forceinline__ SKey skey_shfl_down(const SKey& k, int o) {
  return SKey{__shfl_down_sync(0xffffffffu, k.ah, o), __shfl_down_sync(0xffffffffu, k.al, o),
              __shfl_down_sync(0xffffffffu, k.idx, o)};
}
template <class N>
__device__ __forceinline__ SKey skey_of(typename N::T v, long long idx) {
  unsigned long long b = (unsigned long long)__double_as_longlong(dadd(N::key_lo(v), 0.0));
  b ^= (b >> 63) ? ~0ull : (1ull << 63);
  return SKey{(unsigned long long)__double_as_longlong(N::key_hi(v)), b, idx};
}

__device__ __forceinline__ void named_sync(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kPanelThreads) : "memory");
}
__device__ __forceinline__ void named_arrive(int id) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(kPanelThreads) : "memory");
}
constexpr int kPanelMaxNb = 64;          // panel width (the driver's inner block)

#ifdef DDB_DIAG_TIMING
// diagnostics build only: per-step clock64 stamps of CTA 0 in the last panel
__device__ long long g_panel_t[64][8];
#define PANEL_T(jj, k) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_panel_t[jj][k] = clock64(); } while (0)
extern "C" int ddb_debug_panel_timing(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_panel_t, sizeof(g_panel_t));
}
#else
#define PANEL_T(jj, k) ((void)0)
#endif

template <class N>
__global__ void __launch_bounds__(kPanelThreads)
getrf_panel_smem_kernel(GetrfArgs g, int64_t j0, int nb, int64_t chunk) {
  using T = typename N::T;
  extern __shared__ double sm[];
  __shared__ T rec_s;
  __shared__ int flags_s;                // bit 0 nonzero pivot, bit 1 |pivot| >= safmin
  const int G = gridDim.x;
  const int64_t r0 = j0 + (int64_t)blockIdx.x * chunk;
  const int64_t r1 = r0 + chunk < g.m ? r0 + chunk : g.m;
  const int nr = r1 > r0 ? (int)(r1 - r0) : 0;
  const int ch = (int)chunk | 1;         // odd row stride: a row read across lanes is conflict-free
  double* xh = sm;                       // rows x nb, ld = ch
  double* xl = sm + (size_t)ch * nb;
  // the pivot rows of two consecutive steps (step jj's at parity jj & 1)
  auto prow_h = [&](int par) { return xl + (size_t)ch * nb + (size_t)par * 2 * nb; };
  auto prow_l = [&](int par) { return prow_h(par) + nb; };
  const int64_t lda = g.lda;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = threadIdx.x; t < nr * nb; t += blockDim.x) {
    const int r = t % nr, c = t / nr;
    N::st(xh, xl, r + c * ch, N::ld(g.a_hi, g.a_lo, (r0 + r) + (j0 + c) * lda));
  }
  __syncthreads();
  auto owner = [&](int64_t row) { return (int)((row - j0) / chunk); };
  auto mine = [&](int64_t row) { return row >= r0 && row < r1; };
  auto first_row = [&](int64_t j) { return r0 > j ? 0 : (int)(j - r0); };   // local rows >= j
  // global scratch, two parities: keys [2][G], candidate rows [2][G][2 nb +
  // 2], row j [2][2 nb + 2]: hi row | lo row | the reciprocal of the row's
  // entry in the column searched (formed speculatively by the publisher)
  const size_t RS = 2 * (size_t)nb + 2;
  auto cand = [&](int par, int c) { return g.rowbuf + ((size_t)par * G + c) * RS; };
  auto jrow = [&](int par) { return g.rowbuf + (size_t)2 * G * RS + (size_t)par * RS; };
  // step jj's rank-1 update of x(r, c) (check-free inside the safe window)
  auto upd = [&](int r, int c, int jj) {
    const T x = N::ld(xh, xl, r + jj * ch), a = N::ld(xh, xl, r + c * ch);
    const T pc = N::ld(prow_h(jj & 1), prow_l(jj & 1), c);
    const T out = N::win(x) && N::win(a) && N::win(pc) ? N::fadd2(a, N::fmul(x, N::neg(pc)))
                                                       : N::add(a, N::mul(x, N::neg(pc)));
    N::st(xh, xl, r + c * ch, out);
  };
  // warps 1 / 2: the reciprocal of the candidate's / row j's pivot-column
  // entry (the reference's scalar _div2, needed only when the entry is a
  // non-zero >= safmin), in the shadow of warp 0's row output
  auto spec_rec = [&](double* out, int rr, int jj) {
    if (lane != 0) return;
    const T v = N::ld(xh, xl, rr + jj * ch);
    T rec = N::zero();
    if (N::nonzero(v) && N::ge_safmin(v)) rec = N::sdiv(N::one(), v);
    N::st(out + 2 * nb, out + 2 * nb + 1, 0, rec);
  };
  // search column jj (warps 0 and 1 alike), publish the candidate (+ row j0
  // + jj).  Columns > u of the published rows carry step jj - 1's rank-1
  // update (the same operations the bulk update performs on them later), so
  // the CTA can arrive at the barrier before its bulk update.
  auto publish = [&](int jj, int u) {
    const int par = jj & 1;
    const int64_t j = j0 + jj;
    auto row_out = [&](double* out, int rr) {
      for (int c = lane; c < nb; c += 32) {
        T v = N::ld(xh, xl, rr + c * ch);
        if (c > u) {
          const T pc = N::ld(prow_h((jj - 1) & 1), prow_l((jj - 1) & 1), c);
          const T x = N::ld(xh, xl, rr + (jj - 1) * ch);
          // check-free inside the window: bit-identical to the checked forms
          v = N::win(v) && N::win(x) && N::win(pc) ? N::fadd2(v, N::fmul(x, N::neg(pc)))
                                                   : N::add(v, N::mul(x, N::neg(pc)));
        }
        N::st(out, out + nb, c, v);
      }
    };
    if (warp == 2) {
      if (mine(j)) spec_rec(jrow(par), (int)(j - r0), jj);
      return;
    }
    if (warp == 3) {                           // row j (no search needed)
      if (mine(j)) row_out(jrow(par), (int)(j - r0));
      return;
    }
    SKey k{0ull, 0ull, kNoRow};
    for (int r = first_row(j) + lane; r < nr; r += 32)
      k = skey_merge(k, skey_of<N>(N::ld(xh, xl, r + jj * ch), (long long)(r0 + r)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      k = skey_merge(k, SKey{__shfl_xor_sync(0xffffffffu, k.ah, o), __shfl_xor_sync(0xffffffffu, k.al, o),
                             __shfl_xor_sync(0xffffffffu, k.idx, o)});
    if (warp == 1) {
      if (k.idx != kNoRow) spec_rec(cand(par, blockIdx.x), (int)(k.idx - r0), jj);
      return;
    }
    const int slot = par * G + blockIdx.x;
    if (lane == 0) {
      reinterpret_cast<unsigned long long*>(g.part_ah)[slot] = k.ah;
      reinterpret_cast<unsigned long long*>(g.part_al)[slot] = k.al;
      g.part_idx[slot] = k.idx;
    }
    if (k.idx != kNoRow) row_out(cand(par, blockIdx.x), (int)(k.idx - r0));
  };
  // split grid barrier: release-add after the CTA's writes, acquire-poll
  auto arrive = [&]() {
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(g.bar) : "memory");
  };
  auto wait = [&](unsigned target) {
    if (threadIdx.x == 0) {
      while (true) {
        unsigned v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(g.bar) : "memory");
        if (v >= target) break;
        __nanosleep(20);
      }
    }
    __syncthreads();
  };
  if (warp < 4) publish(0, nb);
  arrive();
  unsigned nbar = 0;
  for (int jj = 0; jj < nb; ++jj) {
    const int par = jj & 1;
    const int64_t j = j0 + jj;
    PANEL_T(jj, 0);
    wait(G * ++nbar);
    PANEL_T(jj, 1);
    if (warp == 0) {
      // merge the G partial keys, fetch the pivot row (and row j) and the
      // publisher's reciprocal; the rows go into x only once the other warps
      // have finished step jj - 1's deferred bulk update (named barrier 1)
      SKey k{0ull, 0ull, kNoRow};
      for (int c = lane; c < G; c += 32) {
        const int slot = par * G + c;
        k = skey_merge(k, SKey{__ldcg(reinterpret_cast<const unsigned long long*>(g.part_ah) + slot),
                               __ldcg(reinterpret_cast<const unsigned long long*>(g.part_al) + slot),
                               __ldcg(g.part_idx + slot)});
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
        k = skey_merge(k, SKey{__shfl_xor_sync(0xffffffffu, k.ah, o), __shfl_xor_sync(0xffffffffu, k.al, o),
                               __shfl_xor_sync(0xffffffffu, k.idx, o)});
      // NaN |hi| (np.max propagates it: argmax_abs returns 0 -> the diagonal
      // entry) or no candidate: row j stays
      const bool nan = k.idx == kNoRow || isnan(__longlong_as_double((long long)k.ah));
      const int64_t jp = nan ? j : k.idx;
      // nonzero(pivot) from the key: |hi| != 0 or lo != 0 (+0 is the map's 1 << 63)
      const bool swapped = !nan && (k.ah != 0ull || k.al != (1ull << 63)) && jp != j;
      const double* src = swapped ? cand(par, owner(jp)) : jrow(par);
      const double* jr = jrow(par);
      const bool own_j = mine(j), own_jp = swapped && mine(jp);
      constexpr int kMaxPer = (kPanelMaxNb + 31) / 32;
      T v[kMaxPer], o[kMaxPer];
#pragma unroll
      for (int i = 0; i < kMaxPer; ++i) {
        const int c = lane + 32 * i;
        v[i] = o[i] = N::zero();
        if (c < nb) {
          v[i] = N::ldcg(src, src + nb, c);
          if (own_jp) o[i] = N::ldcg(jr, jr + nb, c);
        }
      }
      T piv = N::zero(), rec = N::zero();
      if (lane == 0) {
        piv = N::ldcg(src, src + nb, jj);
        rec = N::ldcg(src + 2 * nb, src + 2 * nb + 1, 0);
      }
      PANEL_T(jj, 7);
      named_sync(1);
#pragma unroll
      for (int i = 0; i < kMaxPer; ++i) {
        const int c = lane + 32 * i;
        if (c < nb) {
          N::st(prow_h(par), prow_l(par), c, v[i]);
          if (own_j) N::st(xh, xl, (j - r0) + c * ch, v[i]);
          if (own_jp) N::st(xh, xl, (jp - r0) + c * ch, o[i]);
        }
      }
      if (lane == 0) {
        const bool nz = N::nonzero(piv), ur = N::ge_safmin(piv);     // lu.py:98
        flags_s = (nz ? 1 : 0) | (ur ? 2 : 0);
        if (nz && ur) rec_s = rec;             // = _div2(1, piv), formed by the publisher
        if (blockIdx.x == 0) {
          g.ipiv[j] = jp + 1;
          g.swap[j] = swapped ? jp : j;
          if (!nz && *g.info == 0) *g.info = (int)(j + 1);
        }
      }
      PANEL_T(jj, 2);
    } else {
      // step jj - 1's bulk update of columns >= jj + 2 (column jj + 1 was
      // done before the barrier), 64 rows x 7 column phases
      if (jj > 0) {
        const int t = threadIdx.x - 32, rr = t % 32, cc = t / 32;
        const int rs = first_row(j), pj = (jj - 1) & 1;
        for (int r = rs + rr; r < nr; r += 32) {
          const T x = N::ld(xh, xl, r + (jj - 1) * ch);
          const bool wx = N::win(x);
          for (int c = jj + 2 + cc; c < nb; c += (kPanelThreads - 32) / 32) {
            const T a = N::ld(xh, xl, r + c * ch), pc = N::ld(prow_h(pj), prow_l(pj), c);
            // mul2(x, -p): the sign moves between the factors exactly
            const T out = wx && N::win(a) && N::win(pc) ? N::fadd2(a, N::fmul(x, N::neg(pc)))
                                                        : N::add(a, N::mul(x, N::neg(pc)));
            N::st(xh, xl, r + c * ch, out);
          }
        }
      }
      named_arrive(1);
    }
    __syncthreads();
    PANEL_T(jj, 3);
    const int flags = flags_s;
    const int rs = first_row(j + 1);
    // this thread's row (chunk <= kSmemRowsMax < kPanelThreads): scale
    // column jj, then step jj's update of column jj + 1 (the next search)
    {
      const int r = rs + threadIdx.x;
      if (r < nr) {
        T x = N::ld(xh, xl, r + jj * ch);
        if (flags & 1) {
          x = (flags & 2) ? N::mul(rec_s, x) : N::vdiv(x, N::ld(prow_h(par), prow_l(par), jj));
          N::st(xh, xl, r + jj * ch, x);
        }
        if (jj + 1 < nb) upd(r, jj + 1, jj);
      }
    }
    if (jj + 1 == nb) break;              // (j < mn - 1 holds below: the panel lies inside mn)
    __syncthreads();
    PANEL_T(jj, 4);
    if (warp < 4) publish(jj + 1, jj + 1);
    PANEL_T(jj, 5);
    arrive();
    PANEL_T(jj, 6);
    // column jj + 2 of step jj's update now (the next step's first update
    // needs it); the other columns go to the other warps in the shadow of
    // the next step's key merge (the deferral keeps every element's update
    // order: step jj before step jj + 1)
    if (jj + 2 < nb)
      for (int r = rs + threadIdx.x; r < nr; r += blockDim.x) upd(r, jj + 2, jj);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nr * nb; t += blockDim.x) {
    const int r = t % nr, c = t / nr;
    N::st(g.a_hi, g.a_lo, (r0 + r) + (j0 + c) * lda, N::ld(xh, xl, r + c * ch));
  }
}

// Row interchanges (laswp, lu.py:61-65) of steps [j0, j1), in order (or in
// reverse), on columns [c0, c1).  getrf_perm_kernel (one warp) composes them
// into a permutation of the touched rows -- the step rows [j0, j1) at fixed
// slots, the other targets appended -- and getrf_apply_perm_kernel moves the
// touched entries of a group of columns through shared memory: every load is
// independent, then every store.
constexpr int kPermSteps = 256;                 // steps per composition
constexpr int kPermMax = 2 * kPermSteps;        // touched rows

__global__ void __launch_bounds__(32)
getrf_perm_kernel(GetrfArgs g, int64_t j0, int64_t j1, int reverse, PermBuf pb) {
  // one thread composes (the steps are inherently sequential); the step rows
  // [j0, j1) sit at fixed slots, other targets are found through a small
  // open-addressing table in shared memory
  constexpr int kHash = 1024;
  __shared__ long long rows_s[kPermMax];
  __shared__ int src_s[kPermMax];
  __shared__ long long key_s[kHash];
  __shared__ int slot_s[kHash];
  __shared__ int nt_s;
  __shared__ long long swap_s[kPermSteps];
  const int nb = (int)(j1 - j0);
  for (int t = threadIdx.x; t < kHash; t += blockDim.x) key_s[t] = -1;
  for (int t = threadIdx.x; t < nb; t += blockDim.x) {
    rows_s[t] = j0 + t;
    src_s[t] = t;
    swap_s[t] = g.swap[j0 + t];        // all steps' targets in one coalesced read
  }
  __syncwarp();
  if (threadIdx.x == 0) {
    int nt = nb;
    auto find = [&](long long r) {
      if (r >= j0 && r < j1) return (int)(r - j0);
      unsigned h = (unsigned)(((unsigned long long)r * 0x9E3779B97F4A7C15ull) >> 54);   // 10 bits
      while (true) {
        const long long k = key_s[h];
        if (k == r) return slot_s[h];
        if (k < 0) {
          key_s[h] = r;
          slot_s[h] = nt;
          rows_s[nt] = r;
          src_s[nt] = nt;
          return nt++;
        }
        h = (h + 1) & (kHash - 1);
      }
    };
    for (int64_t s = j0; s < j1; ++s) {
      const int64_t j = reverse ? j0 + j1 - 1 - s : s;
      const long long p = swap_s[j - j0];
      if (p == j) continue;
      const int a = find(j), b = find(p);
      const int t = src_s[a];
      src_s[a] = src_s[b];
      src_s[b] = t;
    }
    nt_s = nt;
  }
  __syncwarp();
  const int nt = nt_s;
  for (int t = threadIdx.x; t < nt; t += blockDim.x) {
    pb.rows[t] = rows_s[t];
    pb.src[t] = src_s[t];
  }
  if (threadIdx.x == 0) *pb.n = nt;
}

constexpr int kPermCols = 8;                    // columns per CTA

__global__ void __launch_bounds__(256)
getrf_apply_perm_kernel(GetrfArgs g, PermBuf pb, int64_t c0, int64_t c1) {
  extern __shared__ double sm[];
  const int nt = *pb.n;
  double* vh = sm;                              // [kPermCols][nt]
  double* vl = sm + (size_t)kPermCols * nt;
  for (int64_t cb = c0 + (int64_t)blockIdx.x * kPermCols; cb < c1;
       cb += (int64_t)gridDim.x * kPermCols) {
    const int ncol = (int)(c1 - cb < kPermCols ? c1 - cb : kPermCols);
    for (int e = threadIdx.x; e < nt * ncol; e += blockDim.x) {
      const int t = e % nt, c = e / nt;
      const int64_t x = pb.rows[pb.src[t]] + (cb + c) * g.lda;
      vh[c * nt + t] = g.a_hi[x];
      if (!g.f64) vl[c * nt + t] = g.a_lo[x];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nt * ncol; e += blockDim.x) {
      const int t = e % nt, c = e / nt;
      const int64_t x = pb.rows[t] + (cb + c) * g.lda;
      g.a_hi[x] = vh[c * nt + t];
      if (!g.f64) g.a_lo[x] = vl[c * nt + t];
    }
    __syncthreads();
  }
}

// U12 = L11^-1 A12 for columns [c0, c1): one warp per column, lane t holding
// rows t and t + 32 of the block.  Step l: the owner finalises U(l, c) and
// broadcasts it; every later row r gets a(r, c) += mul2(L(r, l), -U(l, c)) --
// per element the reference's order (l ascending).
template <class N>
__global__ void __launch_bounds__(256)
getrf_trsm_kernel(GetrfArgs g, int64_t j0, int nb, int64_t c0, int64_t c1) {
  using T = typename N::T;
  extern __shared__ double sm[];
  double* lh = sm;
  double* ll = sm + nb * nb;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int r = e % nb, l = e / nb;
    if (l < r) N::st(lh, ll, e, N::ld(g.a_hi, g.a_lo, (j0 + r) + (j0 + l) * g.lda));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t c = c0 + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (c >= c1) return;                       // whole warps
  double* uh = g.a_hi + j0 + c * g.lda;
  double* ul = g.f64 ? nullptr : g.a_lo + j0 + c * g.lda;
  const int ra = lane, rb = lane + 32;
  T acc_a = N::zero(), acc_b = N::zero();
  if (ra < nb) acc_a = N::ld(uh, ul, ra);
  if (rb < nb) acc_b = N::ld(uh, ul, rb);
  for (int l = 0; l < nb - 1; ++l) {
    // U(l, c) is final once its turn comes
    const T nu = N::neg(N::shfl(l < 32 ? acc_a : acc_b, l & 31));
    if (ra > l && ra < nb) acc_a = N::add(acc_a, N::mul(N::ld(lh, ll, ra + l * nb), nu));
    if (rb > l && rb < nb) acc_b = N::add(acc_b, N::mul(N::ld(lh, ll, rb + l * nb), nu));
  }
  if (ra < nb) N::st(uh, ul, ra, acc_a);
  if (rb < nb) N::st(uh, ul, rb, acc_b);
}

// U12 of a block row in one launch: columns c in [c0, c1) of rows [j0, j0 +
// w) (w <= 256) after the block's interchanges, U(l, c) = A(l, c) - sum_{t <
// l} L(l, t) U(t, c) with the products in t order -- the same operation
// sequence as getrf_trsm_kernel per inner block plus the alpha = -1 Rgemm
// between inner blocks (add2(acc, mul2(L, -U)) per element, t ascending), so
// exact mode stays bitwise.  One warp per column, lane t holding rows t + 32
// i (chains); step l finalises entry l (unit diagonal: no scaling),
// broadcasts it, and every lane extends its later rows -- lanes whose row is
// already final update dead accumulators, so there are no per-lane
// predicates.  L is read through L1 one step ahead; the check-free forms run
// while the step is inside the safe window (mask: L block rows, from
// launch_window_mask; the starting column; each broadcast value).
// TwoSum accumulation (fast / twosum modes, as potrf_rows_kernel's
// RK_TWOSUM): unnormalised (H, L), 13 FP64 operations per product
__device__ __forceinline__ dd ts_mac(dd acc, dd x, dd y) {
  const double p = dmul(x.h, y.h);
  const double e = dfma(x.h, y.h, -p);
  const double c = dfma(x.h, y.l, dmul(x.l, y.h));
  double s, err;
  two_sum(acc.h, p, s, err);
  return dd{s, dadd(acc.l, dadd(err, dadd(e, c)))};
}
__device__ __forceinline__ dd ts_norm(dd a) {
  double s, e;
  quick_two_sum(a.h, a.l, s, e);
  return dd{s, e};
}
__device__ __forceinline__ double ts_mac(double acc, double x, double y) { return dadd(acc, dmul(x, y)); }
__device__ __forceinline__ double ts_norm(double a) { return a; }

template <class N, int NPER, bool TS>
__global__ void __launch_bounds__(256)
getrf_u12_kernel(GetrfArgs g, int64_t j0, int w, int64_t c0, int64_t c1,
                 const unsigned* __restrict__ lmask) {
  using T = typename N::T;
  const int lane = threadIdx.x & 31;
  const int64_t c = c0 + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (c >= c1) return;                       // whole warps
  const int64_t lda = g.lda;
  double* uh = g.a_hi + j0 + c * lda;
  double* ul = g.f64 ? nullptr : g.a_lo + j0 + c * lda;
  const double* lh = g.a_hi + j0 + j0 * lda;  // L(j0 + r, j0 + t) at r + t * lda
  const double* ll = g.f64 ? nullptr : g.a_lo + j0 + j0 * lda;
  T acc[NPER];
  bool ok = !N::kF64 && lmask != nullptr;
#pragma unroll
  for (int i = 0; i < NPER; ++i) {
    const int r = lane + 32 * i;
    acc[i] = N::zero();
    if (r < w) {
      acc[i] = N::ld(uh, ul, r);
      ok &= N::win(acc[i]) && (lmask[i] >> lane & 1u) != 0;
    }
  }
  const bool fast_ok = __all_sync(0xffffffffu, ok);
  const bool ts = TS && fast_ok;             // TwoSum only on an all-in-window column
  T tn[NPER];
#pragma unroll
  for (int i = 0; i < NPER; ++i) tn[i] = N::zero();
  auto fetch = [&](int t, int s) {           // L(r, t) for chains >= s
#pragma unroll
    for (int i = 0; i < NPER; ++i)
      if (i >= s && lane + 32 * i < w) tn[i] = N::ldg(lh, ll, (int64_t)(lane + 32 * i) + (int64_t)t * lda);
  };
  if (w > 1) fetch(0, 0);
#pragma unroll
  for (int s = 0; s < NPER; ++s) {
    if (32 * s >= w) break;
    const int tend = min(32, w - 32 * s);
    for (int tt = 0; tt < tend; ++tt) {
      const int t = 32 * s + tt;
      T lv[NPER];
#pragma unroll
      for (int i = s; i < NPER; ++i) lv[i] = tn[i];
      if (t + 1 < w) fetch(t + 1, tt + 1 < 32 ? s : s + 1);
      T as = acc[s];
      if (ts) as = ts_norm(as);
      const T u = N::shfl(as, tt);           // U(j0 + t, c): final
      if (lane == tt) N::st(uh, ul, t, u);
      const T nu = N::neg(u);
      if (ts && N::win(u)) {                 // fast modes: TwoSum accumulation
#pragma unroll
        for (int i = s; i < NPER; ++i) acc[i] = ts_mac(acc[i], lv[i], nu);
      } else if (ts) {
#pragma unroll
        for (int i = s; i < NPER; ++i) acc[i] = N::add(ts_norm(acc[i]), N::mul(lv[i], nu));
      } else if (fast_ok && N::win(u)) {     // warp-uniform
#pragma unroll
        for (int i = s; i < NPER; ++i) acc[i] = N::fadd2(acc[i], N::fmul(lv[i], nu));
      } else {
#pragma unroll
        for (int i = s; i < NPER; ++i) acc[i] = N::add(acc[i], N::mul(lv[i], nu));
      }
    }
  }
}

// The inner panels' trailing update inside an outer block row, A(r, c) +=
// L(r, l) (-U(l, c)) for rows [r0, r1), columns [c0, c1) (<= 256), l < kb
// (<= 64), as one lean launch instead of an Rgemm call (~10 launches of
// routing / bound / split machinery around a k = 64 tile that the TMA kernel
// runs in ~66 us).  CTA: 128 rows (one per thread) x 8 columns, the 8 x kb
// slice of U staged in shared memory with a window flag.  Per element the
// products arrive in l order: exact mode the check-free add2(mul2(L, -U))
// inside the safe window (bit-identical to the checked forms and to the
// alpha = -1 Rgemm it replaces), the checked forms otherwise; fast / twosum
// modes the TwoSum accumulation (ts_mac) inside the window.
template <class N, bool TS>
__global__ void __launch_bounds__(128)
getrf_inner_upd_kernel(GetrfArgs g, int64_t l0, int kb, int64_t r0, int64_t r1, int64_t c0,
                       int64_t c1) {
  using T = typename N::T;
  constexpr int CW = 8;
  __shared__ T us[kPanelMaxNb][CW];
  __shared__ int uok;
  const int64_t lda = g.lda;
  const int64_t cb = c0 + (int64_t)blockIdx.y * CW;
  if (threadIdx.x == 0) uok = 1;
  __syncthreads();
  for (int e = threadIdx.x; e < kb * CW; e += blockDim.x) {
    const int l = e % kb, cc = e / kb;
    T u = N::zero();
    if (cb + cc < c1) u = N::ld(g.a_hi, g.a_lo, (l0 + l) + (cb + cc) * lda);
    us[l][cc] = N::neg(u);
    if (!N::win(u)) uok = 0;
  }
  __syncthreads();
  const int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= r1) return;
  T acc[CW];
  bool ok = uok != 0 && !N::kF64;
#pragma unroll
  for (int cc = 0; cc < CW; ++cc) {
    acc[cc] = N::zero();
    if (cb + cc < c1) {
      acc[cc] = N::ld(g.a_hi, g.a_lo, r + (cb + cc) * lda);
      ok &= N::win(acc[cc]);
    }
  }
  T ln = N::ld(g.a_hi, g.a_lo, r + l0 * lda);
  for (int l = 0; l < kb; ++l) {
    const T lv = ln;
    if (l + 1 < kb) ln = N::ld(g.a_hi, g.a_lo, r + (l0 + l + 1) * lda);
    if (ok && N::win(lv)) {
#pragma unroll
      for (int cc = 0; cc < CW; ++cc)
        acc[cc] = TS ? ts_mac(acc[cc], lv, us[l][cc]) : N::fadd2(acc[cc], N::fmul(lv, us[l][cc]));
    } else {
#pragma unroll
      for (int cc = 0; cc < CW; ++cc) {
        const T a = TS ? ts_norm(acc[cc]) : acc[cc];
        acc[cc] = N::add(a, N::mul(lv, us[l][cc]));
      }
    }
  }
#pragma unroll
  for (int cc = 0; cc < CW; ++cc)
    if (cb + cc < c1) N::st(g.a_hi, g.a_lo, r + (cb + cc) * lda, TS ? ts_norm(acc[cc]) : acc[cc]);
}

cudaError_t launch_getrf_inner_upd(const GetrfArgs& g, int64_t l0, int kb, int64_t r0, int64_t r1,
                                   int64_t c0, int64_t c1, cudaStream_t s) {
  if (r1 <= r0 || c1 <= c0 || kb <= 0) return cudaSuccess;
  if (kb > kPanelMaxNb) return cudaErrorInvalidValue;
  dim3 grid((unsigned)((r1 - r0 + 127) / 128), (unsigned)((c1 - c0 + 7) / 8));
  if (g.f64) getrf_inner_upd_kernel<NumF64, false><<<grid, 128, 0, s>>>(g, l0, kb, r0, r1, c0, c1);
  else if (g.fastacc) getrf_inner_upd_kernel<NumDD, true><<<grid, 128, 0, s>>>(g, l0, kb, r0, r1, c0, c1);
  else getrf_inner_upd_kernel<NumDD, false><<<grid, 128, 0, s>>>(g, l0, kb, r0, r1, c0, c1);
  return cudaGetLastError();
}

template <class N, int NPER>
static cudaError_t u12_launch(const GetrfArgs& g, int64_t j0, int w, int64_t c0, int64_t c1,
                              const unsigned* lmask, cudaStream_t s) {
  const int64_t threads = (c1 - c0) * 32;
  const unsigned grid = (unsigned)((threads + 255) / 256);
  if (g.fastacc) getrf_u12_kernel<N, NPER, true><<<grid, 256, 0, s>>>(g, j0, w, c0, c1, lmask);
  else getrf_u12_kernel<N, NPER, false><<<grid, 256, 0, s>>>(g, j0, w, c0, c1, lmask);
  return cudaGetLastError();
}

template <class N>
static cudaError_t u12_dispatch(const GetrfArgs& g, int64_t j0, int w, int64_t c0, int64_t c1,
                                const unsigned* lmask, cudaStream_t s) {
  if (w <= 64) return u12_launch<N, 2>(g, j0, w, c0, c1, lmask, s);
  if (w <= 128) return u12_launch<N, 4>(g, j0, w, c0, c1, lmask, s);
  return u12_launch<N, 8>(g, j0, w, c0, c1, lmask, s);
}

cudaError_t launch_getrf_u12(const GetrfArgs& g, int64_t j0, int w, int64_t c0, int64_t c1,
                             unsigned* lmask, cudaStream_t s) {
  if (c1 <= c0 || w <= 0) return cudaSuccess;
  if (w > 256) return cudaErrorInvalidValue;
  if (!g.f64) {
    const cudaError_t e = launch_window_mask(g.a_hi + j0 + j0 * g.lda, g.a_lo + j0 + j0 * g.lda, w, 1,
                                             g.lda, lmask, s);
    if (e != cudaSuccess) return e;
  }
  return g.f64 ? u12_dispatch<NumF64>(g, j0, w, c0, c1, nullptr, s)
               : u12_dispatch<NumDD>(g, j0, w, c0, c1, lmask, s);
}

static int panel_grid(int64_t rows) {
  static thread_local int cached_dev = -1, cached_max = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cached_dev) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, getrf_panel_kernel<NumDD>, kPanelThreads,
                                                  0);
    // the shared-memory variants at their largest share: also >= 1 CTA / SM
    cudaFuncSetAttribute(getrf_panel_smem_kernel<NumDD>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(getrf_panel_smem_kernel<NumF64>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cached_max = per > 0 ? sms : 1;                            // one CTA per SM
    cached_dev = dev;
  }
  // rows per CTA (env DDB_GETRF_ROWS): each step's rank-1 update of a CTA's
  // rows sits on the panel's critical path, so thinner slices (more CTAs,
  // capped at one per SM) shorten it
  static const int64_t per_cta = [] {
    const char* v = std::getenv("DDB_GETRF_ROWS");
    const int64_t r = v ? (int64_t)std::atoll(v) : 0;
    return r > 0 ? r : (int64_t)32;   // 32: 141.0 vs 141.5 ms at n = 8192 (64)
  }();
  int64_t want = (rows + per_cta - 1) / per_cta;
  if (want < 1) want = 1;
  return (int)(want < cached_max ? want : cached_max);
}

int getrf_max_panel_ctas() { return panel_grid(1LL << 40); }

cudaError_t launch_getrf_panel(const GetrfArgs& g, int64_t j0, int nb, cudaStream_t s) {
  const int64_t rows = g.m - j0;
  int grid = panel_grid(rows);
  cudaError_t e = cudaMemsetAsync(g.bar, 0, sizeof(unsigned), s);
  if (e != cudaSuccess) return e;
  GetrfArgs ga = g;
  int nbv = nb;
  int64_t chunk = (rows + grid - 1) / grid;
  if (chunk < 32) {                       // >= 32 rows per CTA: fewer barrier arrivals
    chunk = rows < 32 ? rows : 32;
    grid = (int)((rows + chunk - 1) / chunk);
  }
  if (chunk <= kSmemRowsMax && nb <= kPanelMaxNb) {
    const size_t smem = sizeof(double) * (2 * (size_t)(chunk | 1) * nb + 4 * (size_t)nb);
    // A cooperative launch guarantees co-residency but may wait for an idle
    // device; with grid <= one CTA per SM an ordinary launch also completes
    // (the other stream's CTAs always retire), and can overlap the trailing
    // update (measured: no difference).  DDB_GETRF_COOP=0 selects it.
    static const bool coop = [] {
      const char* v = std::getenv("DDB_GETRF_COOP");
      return v == nullptr || v[0] != '0';
    }();
    void* kern = g.f64 ? reinterpret_cast<void*>(getrf_panel_smem_kernel<NumF64>)
                       : reinterpret_cast<void*>(getrf_panel_smem_kernel<NumDD>);
    if (!coop) {
      if (g.f64) getrf_panel_smem_kernel<NumF64><<<grid, kPanelThreads, smem, s>>>(ga, j0, nbv, chunk);
      else getrf_panel_smem_kernel<NumDD><<<grid, kPanelThreads, smem, s>>>(ga, j0, nbv, chunk);
      return cudaGetLastError();
    }
    void* args[] = {&ga, &j0, &nbv, &chunk};
    return cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kPanelThreads), args, smem, s);
  }
  grid = panel_grid(rows);
  void* args[] = {&ga, &j0, &nbv};
  void* kern = g.f64 ? reinterpret_cast<void*>(getrf_panel_kernel<NumF64>)
                     : reinterpret_cast<void*>(getrf_panel_kernel<NumDD>);
  return cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kPanelThreads), args, 0, s);
}

cudaError_t launch_getrf_compose(const GetrfArgs& g, int64_t j0, int64_t j1, int reverse,
                                 const PermBuf& pb, cudaStream_t s) {
  getrf_perm_kernel<<<1, 32, 0, s>>>(g, j0, j1, reverse, pb);
  return cudaGetLastError();
}

cudaError_t launch_getrf_apply(const GetrfArgs& g, const PermBuf& pb, int64_t nsteps, int64_t c0,
                               int64_t c1, cudaStream_t s) {
  if (c1 <= c0 || nsteps <= 0) return cudaSuccess;
  static thread_local int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaFuncSetAttribute(getrf_apply_perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(2 * sizeof(double) * kPermCols * kPermMax));
    attr_dev = dev;
  }
  int64_t grid = (c1 - c0 + kPermCols - 1) / kPermCols;
  if (grid > 148 * 8) grid = 148 * 8;
  const size_t smem = 2 * sizeof(double) * kPermCols * (size_t)(2 * nsteps);
  getrf_apply_perm_kernel<<<(unsigned)grid, 256, smem, s>>>(g, pb, c0, c1);
  return cudaGetLastError();
}

cudaError_t launch_getrf_laswp(const GetrfArgs& g, int64_t j0, int64_t j1, int64_t c0, int64_t c1,
                               cudaStream_t s, int reverse, const PermBuf& pb) {
  if (c1 <= c0 || j1 <= j0) return cudaSuccess;
  for (int64_t t = j0; t < j1; t += kPermSteps) {        // compositions in order
    int64_t a = t, b = t + kPermSteps < j1 ? t + kPermSteps : j1;
    if (reverse) {                                       // chunks from the end
      b = j1 - (t - j0);
      a = b - kPermSteps > j0 ? b - kPermSteps : j0;
    }
    cudaError_t e = launch_getrf_compose(g, a, b, reverse, pb, s);
    if (e == cudaSuccess) e = launch_getrf_apply(g, pb, b - a, c0, c1, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_getrf_trsm(const GetrfArgs& g, int64_t j0, int nb, int64_t c0, int64_t c1,
                              cudaStream_t s) {
  if (c1 <= c0 || nb <= 1) return cudaSuccess;
  const size_t smem = 2 * sizeof(double) * (size_t)nb * nb;
  static thread_local int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaFuncSetAttribute(getrf_trsm_kernel<NumDD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    cudaFuncSetAttribute(getrf_trsm_kernel<NumF64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr_dev = dev;
  }
  if (g.f64) getrf_trsm_kernel<NumF64><<<(unsigned)((c1 - c0 + 7) / 8), 256, smem, s>>>(g, j0, nb, c0, c1);
  else getrf_trsm_kernel<NumDD><<<(unsigned)((c1 - c0 + 7) / 8), 256, smem, s>>>(g, j0, nb, c0, c1);
  return cudaGetLastError();
}

}  // namespace ddb
