// LSH hash kernels: SimHash (reference hashing.py:121-178) and
// DWTA / WTA (hashing.py:196-287).  One kernel serves both the per-sample
// queries (x = hidden activations, B rows) and the table rebuild (x = W2,
// N rows): rows are staged in shared memory, the projection / permutation
// tables stay resident in shared memory for the whole (grid-stride) launch.
#include "internal.cuh"
#include <algorithm>

namespace slide {

// ---------------------------------------------------------------- SimHash
// bit = [sum_j sign_j * x[idx_j] > 0] (sign(0) -> 0, hashing.py:169).  The
// sum is taken in fp64 over fp32 inputs: exact whenever the c terms span
// < 2^23 in magnitude, so the sign equals the reference's f64 sign.
template <int ROWS>
__global__ void __launch_bounds__(256) simhash_kernel(SimHashDev f, const float* __restrict__ x,
                                                      int64_t n, int ld, uint32_t* __restrict__ keys) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int KL = f.k * f.l;
  // rows transposed: xs[idx * ROWS + r], so one entry fetches all ROWS rows
  float* xs = reinterpret_cast<float*>(sm);
  uint16_t* proj = reinterpret_cast<uint16_t*>(xs + ROWS * f.dim);  // (c, KL)
  uint8_t* bits = reinterpret_cast<uint8_t*>(proj + ((KL * f.c + 1) & ~1));
  for (int q = threadIdx.x; q < KL * f.c; q += blockDim.x) {
    int p = q / f.c, j = q - p * f.c;
    proj[j * KL + p] = f.packed[q];
  }
  for (int64_t row0 = (int64_t)blockIdx.x * ROWS; row0 < n; row0 += (int64_t)gridDim.x * ROWS) {
    const int nr = (int)(n - row0 < ROWS ? n - row0 : ROWS);
    __syncthreads();
    for (int q = threadIdx.x; q < ROWS * f.dim; q += blockDim.x) {
      int r = q / f.dim, c = q - r * f.dim;
      xs[c * ROWS + r] = r < nr ? x[(row0 + r) * ld + c] : 0.f;
    }
    __syncthreads();
    for (int p = threadIdx.x; p < KL; p += blockDim.x) {
      double acc[ROWS];
#pragma unroll
      for (int r = 0; r < ROWS; ++r) acc[r] = 0.0;
      for (int j = 0; j < f.c; ++j) {
        uint16_t e = proj[j * KL + p];
        int idx = e & 0x7fff;
        bool neg = e >> 15;
        float vals[ROWS];
        if constexpr (ROWS % 4 == 0) {
#pragma unroll
          for (int r4 = 0; r4 < ROWS / 4; ++r4)
            *reinterpret_cast<float4*>(vals + 4 * r4) = *reinterpret_cast<const float4*>(xs + idx * ROWS + 4 * r4);
        } else {
#pragma unroll
          for (int r = 0; r < ROWS; ++r) vals[r] = xs[idx * ROWS + r];
        }
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
          double v = (double)vals[r];
          acc[r] += neg ? -v : v;
        }
      }
#pragma unroll
      for (int r = 0; r < ROWS; ++r) bits[r * KL + p] = acc[r] > 0.0;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nr * f.l; q += blockDim.x) {
      int r = q / f.l, t = q - r * f.l;
      const uint8_t* b = bits + r * KL + t * f.k;
      uint32_t key = 0;
      for (int kk = 0; kk < f.k; ++kk) key |= (uint32_t)b[kk] << kk;
      keys[(row0 + r) * f.l + t] = key;
    }
  }
}

template <int ROWS>
static void launch_simhash_t(const SimHashDev& f, const float* x, int64_t n, int ld, uint32_t* keys, cudaStream_t s) {
  const int KL = f.k * f.l;
  size_t smem = (size_t)ROWS * f.dim * 4 + (size_t)((KL * f.c + 1) & ~1) * 2 + (size_t)ROWS * KL;
  SLIDE_CHECK(smem <= 227 * 1024, kNotSupported, "simhash tables too large for shared memory");
  SLIDE_CUDA(cudaFuncSetAttribute(simhash_kernel<ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  int64_t blocks = ceil_div(n, ROWS);
  int grid = (int)std::min<int64_t>(blocks, (int64_t)kSms * 4);
  simhash_kernel<ROWS><<<grid, 256, smem, s>>>(f, x, n, ld, keys);
  SLIDE_LAUNCH_CHECK();
}

// Per-sample queries: one row per CTA, the row in shared memory, the
// transposed projection table read straight from L1/L2 (coalesced across
// the projections) instead of being staged by every CTA.
__global__ void __launch_bounds__(512) simhash_query_kernel(SimHashDev f, const float* __restrict__ x, int ld,
                                                            uint32_t* __restrict__ keys) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int KL = f.k * f.l;
  float* xs = reinterpret_cast<float*>(sm);
  uint8_t* bits = reinterpret_cast<uint8_t*>(xs + f.dim);
  const int64_t row = blockIdx.x;
  for (int c = threadIdx.x; c < f.dim; c += blockDim.x) xs[c] = x[row * ld + c];
  __syncthreads();
  for (int p = threadIdx.x; p < KL; p += blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < f.c; ++j) {
      const uint16_t e = __ldg(f.packed_t + j * KL + p);
      const double v = (double)xs[e & 0x7fff];
      acc += (e >> 15) ? -v : v;
    }
    bits[p] = acc > 0.0;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < f.l; t += blockDim.x) {
    uint32_t key = 0;
    for (int kk = 0; kk < f.k; ++kk) key |= (uint32_t)bits[t * f.k + kk] << kk;
    keys[row * f.l + t] = key;
  }
}

void launch_simhash_keys(const SimHashDev& f, const float* x, int64_t n, int ld, uint32_t* keys,
                         cudaStream_t s, DBuf* tc_scratch) {
  if (n <= 0) return;
  if (tc_scratch && n >= (int64_t)kSms * 128 && launch_simhash_keys_tc(f, x, n, ld, keys, *tc_scratch, s)) return;
  const int KL = f.k * f.l;
  if (f.packed_t && n <= (int64_t)kSms * 8) {
    const size_t smem = (size_t)f.dim * 4 + KL;
    SLIDE_CHECK(smem <= 200 * 1024, kNotSupported, "simhash dim too large for shared memory");
    if (smem > 48 * 1024)
      SLIDE_CUDA(cudaFuncSetAttribute(simhash_query_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    simhash_query_kernel<<<(int)n, 512, smem, s>>>(f, x, ld, keys);
    SLIDE_LAUNCH_CHECK();
    return;
  }
  // few rows (per-sample queries): one row per CTA fills the SMs
  if (n <= (int64_t)kSms * 8) launch_simhash_t<1>(f, x, n, ld, keys, s);
  else launch_simhash_t<8>(f, x, n, ld, keys, s);
}

// ------------------------------------------------------------------- DWTA
// Global bin g: permutation g / bins_per_perm, bin g % bins_per_perm, the m
// dims perms[q][b*m .. b*m+m) (ragged last bin).  Winner = largest value,
// ties to the smallest in-bin offset; only nonzeros take part unless
// dense_mode (WTA, hashing.py:262-274).  Empty bins copy the code of the
// first occupied donor mix(salt, g, a) % KL, a = 1..100, else 0
// (hashing.py:219-231).  key_t = sum_k code[t*K+k] << (bits*k).
template <int ROWS>
__global__ void __launch_bounds__(256) dwta_kernel(DwtaDev f, const float* __restrict__ x, int64_t n,
                                                   int ld, uint32_t* __restrict__ keys) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int KL = f.k * f.l;
  float* xs = reinterpret_cast<float*>(sm);
  int16_t* perm = reinterpret_cast<int16_t*>(xs + ROWS * f.dim);
  uint8_t* codes = reinterpret_cast<uint8_t*>(perm + ((f.n_perms * f.dim + 1) & ~1));
  uint8_t* occ = codes + ROWS * KL;
  // a row without any occupied bin (an all-zero activation row: every hidden
  // unit dead for that sample) has nothing to borrow: all its codes are 0 --
  // without the 100-step donor walk of every one of its bins (40 us a row)
  __shared__ int row_any[ROWS];
  for (int q = threadIdx.x; q < f.n_perms * f.dim; q += blockDim.x) perm[q] = f.perms[q];
  for (int64_t row0 = (int64_t)blockIdx.x * ROWS; row0 < n; row0 += (int64_t)gridDim.x * ROWS) {
    const int nr = (int)(n - row0 < ROWS ? n - row0 : ROWS);
    __syncthreads();
    if (threadIdx.x < ROWS) row_any[threadIdx.x] = 0;
    for (int q = threadIdx.x; q < ROWS * f.dim; q += blockDim.x) {
      int r = q / f.dim, c = q - r * f.dim;
      xs[q] = r < nr ? x[(row0 + r) * ld + c] : 0.f;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < ROWS * KL; q += blockDim.x) {
      int r = q / KL, g = q - r * KL;
      int pq = g / f.bins_per_perm, b = g - pq * f.bins_per_perm;
      int lo = b * f.m, hi = min(lo + f.m, f.dim);
      const int16_t* pp = perm + pq * f.dim;
      const float* xr = xs + r * f.dim;
      float best = 0.f;
      int code = 0, oc = 0;
      for (int o = 0; o < hi - lo; ++o) {
        float v = xr[pp[lo + o]];
        if ((f.dense_mode || v != 0.f) && (!oc || v > best)) {
          best = v;
          code = o;
          oc = 1;
        }
      }
      codes[q] = (uint8_t)code;
      occ[q] = (uint8_t)oc;
      if (oc) row_any[r] = 1;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < ROWS * KL; q += blockDim.x) {
      if (occ[q]) continue;
      int r = q / KL, g = q - r * KL;
      int code = 0;
      for (int a = 0; a < 100 && row_any[r]; ++a) {
        int d = f.donors[g * 100 + a];
        if (occ[r * KL + d]) {
          code = codes[r * KL + d];
          break;
        }
      }
      codes[q] = (uint8_t)code;  // only empty bins are written; donors are occupied
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nr * f.l; q += blockDim.x) {
      int r = q / f.l, t = q - r * f.l;
      const uint8_t* cc = codes + r * KL + t * f.k;
      uint32_t key = 0;
      for (int kk = 0; kk < f.k; ++kk) key |= (uint32_t)cc[kk] << (f.bits * kk);
      keys[(row0 + r) * f.l + t] = key;
    }
  }
}

// Rebuild path: 16 rows at a time, transposed in shared memory so one
// 16-byte load fetches a dimension for 4 rows; one thread per bin keeps the
// bin's m permutation positions in registers for all 16 rows.  Same winner /
// tie / nonzero rules and the same donor densification as dwta_kernel.
constexpr int kDwRows = 16;
constexpr int kDwMaxM = 16;
// the transposed tile's row stride: 20 floats (16-byte aligned quads, and the
// transposing stores of consecutive columns hit 8 banks instead of 2)
constexpr int kDwLd = kDwRows + 4;

__global__ void __launch_bounds__(256) dwta_rows_kernel(DwtaDev f, const float* __restrict__ x, int64_t n, int ld,
                                                        uint32_t* __restrict__ keys) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int KL = f.k * f.l;
  float* xs = reinterpret_cast<float*>(sm);  // [dim][kDwLd]
  int16_t* perm = reinterpret_cast<int16_t*>(xs + kDwLd * f.dim);
  uint8_t* codes = reinterpret_cast<uint8_t*>(perm + ((f.n_perms * f.dim + 7) & ~7));
  uint8_t* occ = codes + kDwRows * KL;
  for (int q = threadIdx.x; q < f.n_perms * f.dim; q += blockDim.x) perm[q] = f.perms[q];
  for (int64_t row0 = (int64_t)blockIdx.x * kDwRows; row0 < n; row0 += (int64_t)gridDim.x * kDwRows) {
    const int nr = (int)(n - row0 < kDwRows ? n - row0 : kDwRows);
    __syncthreads();
    for (int q = threadIdx.x; q < kDwRows * f.dim; q += blockDim.x) {
      const int r = q / f.dim, c = q - r * f.dim;
      xs[c * kDwLd + r] = r < nr ? x[(row0 + r) * ld + c] : 0.f;
    }
    __syncthreads();
    for (int g = threadIdx.x; g < KL; g += blockDim.x) {
      const int pq = g / f.bins_per_perm, b = g - pq * f.bins_per_perm;
      const int lo = b * f.m, cnt = min(f.m, f.dim - lo);
      int idx[kDwMaxM];
#pragma unroll
      for (int o = 0; o < kDwMaxM; ++o) idx[o] = o < cnt ? perm[pq * f.dim + lo + o] : 0;
#pragma unroll
      for (int r4 = 0; r4 < kDwRows / 4; ++r4) {
        float best[4] = {0.f, 0.f, 0.f, 0.f};
        int code[4] = {0, 0, 0, 0}, oc[4] = {0, 0, 0, 0};
#pragma unroll
        for (int o = 0; o < kDwMaxM; ++o) {
          if (o >= cnt) break;
          const float4 v4 = *reinterpret_cast<const float4*>(xs + idx[o] * kDwLd + r4 * 4);
          const float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const bool take = (f.dense_mode || v[e] != 0.f) && (!oc[e] || v[e] > best[e]);
            best[e] = take ? v[e] : best[e];
            code[e] = take ? o : code[e];
            oc[e] = take ? 1 : oc[e];
          }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          codes[(r4 * 4 + e) * KL + g] = (uint8_t)code[e];
          occ[(r4 * 4 + e) * KL + g] = (uint8_t)oc[e];
        }
      }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nr * KL; q += blockDim.x) {
      if (occ[q]) continue;
      const int r = q / KL, g = q - r * KL;
      int code = 0;
      for (int a = 0; a < 100; ++a) {
        const int d = f.donors[g * 100 + a];
        if (occ[r * KL + d]) {
          code = codes[r * KL + d];
          break;
        }
      }
      codes[q] = (uint8_t)code;  // only empty bins are written; donors are occupied
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nr * f.l; q += blockDim.x) {
      const int r = q / f.l, t = q - r * f.l;
      const uint8_t* cc = codes + r * KL + t * f.k;
      uint32_t key = 0;
      for (int kk = 0; kk < f.k; ++kk) key |= (uint32_t)cc[kk] << (f.bits * kk);
      keys[(row0 + r) * f.l + t] = key;
    }
  }
}

// Rebuild path, lanes = rows.  A tile of 64 rows sits transposed in shared
// memory ([dim + 1][66], zeros stored as -inf so "only nonzeros take part,
// the first of equal values wins" is one strict compare per element; the
// extra row is all -inf and pads ragged / short bins).  Lane l holds rows 2l
// and 2l + 1: a bin position is ONE conflict-free 8-byte load per lane whose
// address is uniform across the warp up to the lane offset, so the shared-
// memory pipe moves exactly the 2 x 4 bytes per (row, position) the bin
// needs (the bin-per-thread form gathers 16-byte quads at random dims: ~2.4
// bank conflicts per load).  A warp walks whole tables: the K codes of a key
// are packed in registers and stored straight to the key array.  The codes
// (bit 7 = empty bin) are also kept per tile; only a tile that saw an empty
// bin runs the donor densification (hashing.py:219-231) and rewrites its
// keys from them -- dense weight rows never do.
constexpr int kDtRows = 64;            // rows per tile (2 per lane)
constexpr int kDtLd = kDtRows + 2;     // transposed row stride (8-byte aligned, 2-way store conflicts)

__host__ __device__ inline size_t dt_xs_bytes(int dim) { return ((size_t)(dim + 1) * kDtLd * 4 + 15) & ~(size_t)15; }

// Largest of MM values and its position, ties to the lowest position: a
// binary tournament (strict > keeps the left entry), MM - 1 compares instead
// of a chain of MM -- the compare / select work runs on the half-rate ALU
// pipe, which bounds this kernel.
template <int MM>
__device__ __forceinline__ void dt_winner(const float (&v)[MM], float& best, int& code) {
  float bv[MM / 2];
  int bc[MM / 2];
#pragma unroll
  for (int i = 0; i < MM / 2; ++i) {
    const bool t = v[2 * i + 1] > v[2 * i];
    bv[i] = t ? v[2 * i + 1] : v[2 * i];
    bc[i] = t ? 2 * i + 1 : 2 * i;
  }
#pragma unroll
  for (int n = MM / 2; n > 1; n >>= 1) {
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const bool t = bv[2 * i + 1] > bv[2 * i];
      bv[i] = t ? bv[2 * i + 1] : bv[2 * i];
      bc[i] = t ? bc[2 * i + 1] : bc[2 * i];
    }
  }
  best = bv[0];
  code = bc[0];
}

template <int MM, int kDtWarps>
__global__ void __launch_bounds__(kDtWarps * 32) dwta_tile_kernel(DwtaDev f, const float* __restrict__ x, int64_t n,
                                                                   int ld, uint32_t* __restrict__ keys) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int KL = f.k * f.l;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* xs = reinterpret_cast<float*>(sm);                                    // [dim + 1][kDtLd]
  uint32_t* offs = reinterpret_cast<uint32_t*>(sm + dt_xs_bytes(f.dim));       // [KL][MM] byte offsets into xs
  // [KL][kDtRows] codes, bit 7 = empty; bins of up to 8 positions pack two rows per byte
  constexpr bool kPacked = MM <= 8;
  uint8_t* codes = reinterpret_cast<uint8_t*>(offs + (size_t)KL * MM);
  const float ninf = __int_as_float(0xff800000);
  // every bin's positions as byte offsets of their transposed rows; positions
  // past the bin's end point at the -inf row
  for (int q = threadIdx.x; q < KL * MM; q += blockDim.x) {
    const int g = q / MM, o = q - g * MM;
    const int pq = g / f.bins_per_perm, b = g - pq * f.bins_per_perm;
    const int lo = b * f.m, cnt = min(f.m, f.dim - lo);
    const int dimi = o < cnt ? (int)f.perms[pq * f.dim + lo + o] : f.dim;
    offs[q] = (uint32_t)dimi * (kDtLd * 4);
  }
  for (int q = threadIdx.x; q < kDtLd; q += blockDim.x) xs[f.dim * kDtLd + q] = ninf;
  const int d4 = f.dim >> 2;  // float4s per row (dim % 4 == 0, checked by the launcher)
  const char* xl = reinterpret_cast<const char*>(xs) + lane * 8;
  const int64_t n_tiles = (n + kDtRows - 1) / kDtRows;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t row0 = tile * kDtRows;
    const int nr = (int)(n - row0 < kDtRows ? n - row0 : kDtRows);
    __syncthreads();  // the previous tile's readers are done
    // coalesced 16-byte loads (8 lanes along a row, 4 rows per warp access),
    // transposed 4-byte stores
    for (int u = threadIdx.x; u < kDtRows * d4; u += blockDim.x) {
      const int c_lo = u & 7, r_lo = (u >> 3) & 3, rest = u >> 5;
      const int c_hi = rest % (d4 >> 3), r_hi = rest / (d4 >> 3);
      const int c4 = c_hi * 8 + c_lo, r = r_hi * 4 + r_lo;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < nr) v = __ldcs(reinterpret_cast<const float4*>(x + (row0 + r) * ld) + c4);
      const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        xs[(c4 * 4 + j) * kDtLd + r] = (f.dense_mode || e[j] != 0.f) ? e[j] : ninf;
    }
    __syncthreads();
    int any_empty = 0;
    for (int t = warp; t < f.l; t += kDtWarps) {
      uint32_t key0 = 0, key1 = 0;
      for (int kk = 0; kk < f.k; ++kk) {
        const int g = t * f.k + kk;
        uint32_t po[MM];
#pragma unroll
        for (int o4 = 0; o4 < MM / 4; ++o4) {
          const uint4 p4 = *reinterpret_cast<const uint4*>(offs + (size_t)g * MM + o4 * 4);
          po[o4 * 4 + 0] = p4.x, po[o4 * 4 + 1] = p4.y, po[o4 * 4 + 2] = p4.z, po[o4 * 4 + 3] = p4.w;
        }
        float2 v[MM];
#pragma unroll
        for (int o = 0; o < MM; ++o) v[o] = *reinterpret_cast<const float2*>(xl + po[o]);
        float vx[MM], vy[MM];
#pragma unroll
        for (int o = 0; o < MM; ++o) vx[o] = v[o].x, vy[o] = v[o].y;
        float b0, b1;
        int c0, c1;
        dt_winner<MM>(vx, b0, c0);
        dt_winner<MM>(vy, b1, c1);
        const bool e0 = b0 == ninf, e1 = b1 == ninf;
        any_empty |= ((e0 && lane * 2 < nr) || (e1 && lane * 2 + 1 < nr)) ? 1 : 0;  // (rows past the end are all -inf)
        if (kPacked)  // two rows' codes per byte: 3 code bits + the empty flag each
          codes[(size_t)g * (kDtRows / 2) + lane] = (uint8_t)((e0 ? 8 : c0) | ((e1 ? 8 : c1) << 4));
        else
          *reinterpret_cast<uint16_t*>(codes + (size_t)g * kDtRows + lane * 2) =
              (uint16_t)((e0 ? 0x80 : c0) | ((e1 ? 0x80 : c1) << 8));
        key0 |= (uint32_t)c0 << (f.bits * kk);
        key1 |= (uint32_t)c1 << (f.bits * kk);
      }
      const int r = lane * 2;
      if (r < nr) keys[(row0 + r) * f.l + t] = key0;
      if (r + 1 < nr) keys[(row0 + r + 1) * f.l + t] = key1;
    }
    if (!__syncthreads_or(any_empty)) continue;
    // densification: empty bins copy their first occupied donor's code (flag kept
    // so that a filled bin is never taken for an occupied donor)
    auto code_of = [&](int g, int r) -> int {  // bit 7: empty
      if (!kPacked) return codes[(size_t)g * kDtRows + r];
      const int nib = (codes[(size_t)g * (kDtRows / 2) + (r >> 1)] >> (4 * (r & 1))) & 15;
      return (nib & 7) | ((nib & 8) << 4);
    };
    // (packed: a thread owns a byte = rows 2p, 2p + 1 of a bin; occupied nibbles never change)
    for (int q = threadIdx.x; q < KL * (kDtRows / 2); q += blockDim.x) {
      const int g = q / (kDtRows / 2), p = q - g * (kDtRows / 2);
      int filled[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = 2 * p + e;
        int cd = code_of(g, r);
        if (r < nr && (cd & 0x80)) {
          int code = 0;
          for (int a = 0; a < 100; ++a) {
            const int dcd = code_of(f.donors[g * 100 + a], r);
            if (!(dcd & 0x80)) {
              code = dcd;
              break;
            }
          }
          cd = 0x80 | code;
        }
        filled[e] = cd;
      }
      if (kPacked)
        codes[(size_t)g * (kDtRows / 2) + p] =
            (uint8_t)((filled[0] & 7) | ((filled[0] & 0x80) >> 4) | ((filled[1] & 7) << 4) | (filled[1] & 0x80));
      else
        *reinterpret_cast<uint16_t*>(codes + (size_t)g * kDtRows + 2 * p) = (uint16_t)(filled[0] | (filled[1] << 8));
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nr * f.l; q += blockDim.x) {
      const int r = q / f.l, t = q - r * f.l;
      uint32_t key = 0;
      for (int kk = 0; kk < f.k; ++kk) key |= (uint32_t)(code_of(t * f.k + kk, r) & 0x7f) << (f.bits * kk);
      keys[(row0 + r) * f.l + t] = key;
    }
  }
}

template <int MM, int NW>
static int dwta_tile_per_sm(size_t smem) {
  SLIDE_CUDA(cudaFuncSetAttribute(dwta_tile_kernel<MM, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SLIDE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dwta_tile_kernel<MM, NW>, NW * 32, smem));
  return per_sm;
}

template <int MM>
static bool launch_dwta_tile_t(const DwtaDev& f, const float* x, int64_t n, int ld, uint32_t* keys, cudaStream_t s) {
  const int KL = f.k * f.l;
  const size_t smem = dt_xs_bytes(f.dim) + (size_t)KL * MM * 4 + (size_t)KL * (MM <= 8 ? kDtRows / 2 : kDtRows);
  if (smem > 227 * 1024) return false;
  // wide rows leave room for one tile per SM: 16 warps share it instead of 8
  const int per8 = dwta_tile_per_sm<MM, 8>(smem);
  if (per8 >= 2) {
    const int grid = (int)std::min<int64_t>(ceil_div(n, kDtRows), (int64_t)kSms * per8);
    dwta_tile_kernel<MM, 8><<<grid, 8 * 32, smem, s>>>(f, x, n, ld, keys);
  } else {
    const int per16 = std::max(1, dwta_tile_per_sm<MM, 16>(smem));
    const int grid = (int)std::min<int64_t>(ceil_div(n, kDtRows), (int64_t)kSms * per16);
    dwta_tile_kernel<MM, 16><<<grid, 16 * 32, smem, s>>>(f, x, n, ld, keys);
  }
  SLIDE_LAUNCH_CHECK();
  return true;
}

// false when the shape does not fit (the callers fall back)
static bool launch_dwta_tile(const DwtaDev& f, const float* x, int64_t n, int ld, uint32_t* keys, cudaStream_t s) {
  if (f.dim % 32 || ld % 4 || (reinterpret_cast<uintptr_t>(x) & 15) || f.m > 16 || f.m < 1) return false;
  if (f.m <= 4) return launch_dwta_tile_t<4>(f, x, n, ld, keys, s);
  if (f.m <= 8) return launch_dwta_tile_t<8>(f, x, n, ld, keys, s);
  return launch_dwta_tile_t<16>(f, x, n, ld, keys, s);
}

template <int ROWS>
static void launch_dwta_t(const DwtaDev& f, const float* x, int64_t n, int ld, uint32_t* keys, cudaStream_t s) {
  const int KL = f.k * f.l;
  size_t smem = (size_t)ROWS * f.dim * 4 + (size_t)((f.n_perms * f.dim + 1) & ~1) * 2 + (size_t)2 * ROWS * KL;
  SLIDE_CHECK(smem <= 227 * 1024, kNotSupported, "dwta tables too large for shared memory");
  SLIDE_CUDA(cudaFuncSetAttribute(dwta_kernel<ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int64_t blocks = ceil_div(n, ROWS);
  // (per-sample queries, ROWS = 1: a CTA per row up to 8 resident per SM --
  // the phases of a row are latency-bound, a second row per CTA doubles them)
  int grid = (int)std::min<int64_t>(blocks, (int64_t)kSms * (ROWS == 1 ? 8 : 4));
  dwta_kernel<ROWS><<<grid, 256, smem, s>>>(f, x, n, ld, keys);
  SLIDE_LAUNCH_CHECK();
}

void launch_dwta_keys(const DwtaDev& f, const float* x, int64_t n, int ld, uint32_t* keys, cudaStream_t s) {
  if (n <= 0) return;
  if (n <= (int64_t)kSms * 8) {
    launch_dwta_t<1>(f, x, n, ld, keys, s);
    return;
  }
  static const bool old_rows = getenv("SLIDE_DWTA_OLD") != nullptr;  // A/B timing only
  if (!old_rows && launch_dwta_tile(f, x, n, ld, keys, s)) return;
  const int KL = f.k * f.l;
  const size_t smem = (size_t)kDwLd * f.dim * 4 + (size_t)((f.n_perms * f.dim + 7) & ~7) * 2 + (size_t)2 * kDwRows * KL;
  if (f.m > kDwMaxM || smem > 227 * 1024) {
    launch_dwta_t<8>(f, x, n, ld, keys, s);
    return;
  }
  SLIDE_CUDA(cudaFuncSetAttribute(dwta_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = (int)std::min<int64_t>(ceil_div(n, kDwRows), (int64_t)kSms * 4);
  dwta_rows_kernel<<<grid, 256, smem, s>>>(f, x, n, ld, keys);
  SLIDE_LAUNCH_CHECK();
}

}  // namespace slide
