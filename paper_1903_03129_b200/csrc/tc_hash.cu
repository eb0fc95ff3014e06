// SimHash table rebuild on the 5th-generation tensor cores (tcgen05).
//
// The rebuild hashes every W2 row: bit p of row r is [sum_j s_pj W[r, i_pj] > 0]
// over the c-sparse +-1 projection p (reference hashing.py:121-178).  Dense,
// that is D = W P with P (hidden x K*L) in {-1, 0, +1}: a GEMM.
//
//  * W is split exactly into three bf16 parts, W = hi + mid + lo (a float
//    has 24 significant bits, a bf16 8), so every product part x P is exact
//    and D = hi P + mid P + lo P is accumulated in fp32 in TMEM by 3 x
//    (hidden / 16) tcgen05.mma (M = 128 rows, N <= 256 per instruction, K = 16).
//  * The sign is certified: with S_r = sum |W[r, :]| the accumulated value
//    is within 384 * 2^-20 * S_r of the exact dot product (a loose bound on
//    fp32 accumulation), so whenever |D| exceeds it, sign(D) is the exact
//    sign -- which is the reference's f64 sign.  The remaining (row, bit)
//    cases go to a list and are recomputed in fp64 in the reference's term
//    order by simhash_fix_kernel, then patched into the keys.
//
// One CTA (4 warps) per SM, persistent over 128-row tiles: P stays in shared
// memory for the whole launch, the W tile is loaded, split and written in the
// canonical K-major no-swizzle layout, thread 0 issues the MMAs and commits to
// an mbarrier, then every thread reads its row's accumulators with
// tcgen05.ld and packs the keys.
#include "internal.cuh"
#include "tc_common.cuh"
#include <cuda_bf16.h>
#include <algorithm>

namespace slide {

using namespace tc;

namespace {

constexpr int kTcRows = 128;              // M per tile = TMEM lanes
constexpr int kTcThreads = 256;           // 8 warps: warp w reads TMEM lanes 32(w%4).., columns half w/4
constexpr int kTcMaxCols = 512;           // TMEM columns (fp32 accumulators)
constexpr double kTcBoundRel = 384.0 / 1048576.0;  // 384 * 2^-20
constexpr int kBitsLd = kTcMaxCols / 32 + 1;       // sign-bit words per row (+1: banks)
constexpr int kTcK = 128;                          // hidden width of the tensor-core path
constexpr int kTcChunks = kTcK / 16;               // 8-column chunks per thread (two threads per row)

struct TcFix {
  int32_t row, bit;
};

}  // namespace

// smem: P [np_pad x kdim] bf16 | W parts 3 x [128 x kdim] bf16 | mbarrier | tmem base | S_r | sign bits
__global__ void __launch_bounds__(kTcThreads, 1) simhash_tc_kernel(SimHashDev f, const float* __restrict__ x,
                                                                   int64_t n, int ld, int kdim, int np_pad,
                                                                   uint32_t* __restrict__ keys,
                                                                   TcFix* __restrict__ fix, int32_t* __restrict__ n_fix,
                                                                   int fix_cap) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int KL = f.k * f.l;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint8_t* p_s = sm;
  const uint32_t p_bytes = (uint32_t)np_pad * kdim * 2;
  uint8_t* a_s = sm + p_bytes;
  const uint32_t part_bytes = (uint32_t)kTcRows * kdim * 2;
  uint64_t* bar = reinterpret_cast<uint64_t*>(a_s + 3 * part_bytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);
  float* srow = reinterpret_cast<float*>(bar + 2);                  // [2][kTcRows] S_r halves
  uint32_t* bits_s = reinterpret_cast<uint32_t*>(srow + 2 * kTcRows);  // [kTcRows][kBitsLd]
  const int row = tid & (kTcRows - 1), half = tid >> 7;  // two threads per tile row
  const int pgroups = np_pad / 8, agroups = kTcRows / 8;

  // P in the canonical layout: zero, then one projection per thread
  for (uint32_t q = tid; q < p_bytes / 16; q += kTcThreads) reinterpret_cast<uint4*>(p_s)[q] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  for (int p = tid; p < KL; p += kTcThreads)
    for (int j = 0; j < f.c; ++j) {
      const uint16_t e = f.packed[p * f.c + j];
      __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p_s + kmajor_off(p, e & 0x7fff, pgroups));
      *dst = __float2bfloat16_rn(__bfloat162float(*dst) + ((e >> 15) ? -1.f : 1.f));
    }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTcMaxCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  const uint32_t p_addr = smem_u32(p_s), a_addr = smem_u32(a_s);
  const uint32_t n1 = np_pad < 256 ? np_pad : 256, n2 = np_pad - n1;
  const uint32_t id1 = idesc_bf16(kTcRows, n1), id2 = n2 ? idesc_bf16(kTcRows, n2) : 0u;
  const uint32_t a_lbo = agroups * 128, p_lbo = pgroups * 128;
  uint32_t phase = 0;
  const int64_t tiles = (n + kTcRows - 1) / kTcRows;
  // W rows of a tile: thread (row, half) loads k chunks [8 half, 8 half + 8)
  // of 8 floats (kdim = 128), kept in registers so the next tile's loads are
  // in flight during this tile's MMAs and epilogue
  float4 wbuf[kTcChunks * 2];
  auto load_w = [&](int64_t row0) {
    const int64_t gr = row0 + row;
    const float* xr = x + gr * ld + half * kTcChunks * 8;
#pragma unroll
    for (int q = 0; q < kTcChunks * 2; ++q)
      wbuf[q] = gr < n ? *reinterpret_cast<const float4*>(xr + q * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  if ((int64_t)blockIdx.x < tiles) load_w((int64_t)blockIdx.x * kTcRows);
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t row0 = tile * kTcRows;
    // split into hi / mid / lo: per 8-column chunk one 16-byte store per part
    // (a core-matrix row; a warp's stores are contiguous); S_r = sum |w|
    {
      float s = 0.f;
#pragma unroll
      for (int c = 0; c < kTcChunks; ++c) {
        const int kc = half * kTcChunks + c;
        const float4 v0 = wbuf[2 * c], v1 = wbuf[2 * c + 1];
        const float e[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
        uint32_t hw[4], mw[4], lw[4];
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
          __nv_bfloat16 h[2], m[2], l[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const float w = kc * 8 + q + u < f.dim ? e[q + u] : 0.f;
            h[u] = __float2bfloat16_rn(w);
            const float r1 = w - __bfloat162float(h[u]);
            m[u] = __float2bfloat16_rn(r1);
            l[u] = __float2bfloat16_rn(r1 - __bfloat162float(m[u]));
            s += fabsf(w);
          }
          hw[q / 2] = (uint32_t)__bfloat16_as_ushort(h[0]) | ((uint32_t)__bfloat16_as_ushort(h[1]) << 16);
          mw[q / 2] = (uint32_t)__bfloat16_as_ushort(m[0]) | ((uint32_t)__bfloat16_as_ushort(m[1]) << 16);
          lw[q / 2] = (uint32_t)__bfloat16_as_ushort(l[0]) | ((uint32_t)__bfloat16_as_ushort(l[1]) << 16);
        }
        const uint32_t off = kmajor_off(row, kc * 8, agroups);
        *reinterpret_cast<uint4*>(a_s + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(a_s + part_bytes + off) = make_uint4(mw[0], mw[1], mw[2], mw[3]);
        *reinterpret_cast<uint4*>(a_s + 2 * part_bytes + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
      }
      srow[half * kTcRows + row] = s;
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (tid == 0) {
      uint32_t acc = 0;
      for (int part = 0; part < 3; ++part)
        for (int k = 0; k < kdim; k += 16) {
          // a K step of 16 = two core-matrix columns (LBO apart)
          const uint64_t ad = smem_desc(a_addr + part * part_bytes + (k >> 3) * a_lbo, a_lbo, 128);
          const uint64_t b1 = smem_desc(p_addr + (k >> 3) * p_lbo, p_lbo, 128);
          mma_bf16(tmem, ad, b1, id1, acc);
          if (n2) {
            const uint64_t b2 = smem_desc(p_addr + (k >> 3) * p_lbo + (n1 / 8) * 128, p_lbo, 128);
            mma_bf16(tmem + n1, ad, b2, id2, acc);
          }
          acc = 1;
        }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       smem_u32(bar))
                   : "memory");
    }
    if (tile + gridDim.x < tiles) load_w((tile + gridDim.x) * kTcRows);  // next tile, in flight
    mbar_wait(smem_u32(bar), phase);
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    // epilogue: thread (row, half) reads TMEM lane `row`, columns
    // [256 half, 256 half + 256): sign bits to shared memory, uncertain
    // masks kept in registers; one atomic per warp reserves fix-up space.
    const int64_t gr = row0 + row;
    const float bound = (float)(kTcBoundRel * (double)(srow[row] + srow[kTcRows + row]));
    const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t um[8];
    int cnt = 0;
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const int c0 = half * 256 + cc * 32;
      um[cc] = 0u;
      if (c0 < KL) {  // warp-uniform
        uint32_t v[32];
        tmem_ld32(lane_base + c0, v);
        uint32_t word = 0, umask = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float d = __uint_as_float(v[j]);
          word |= (d > 0.f ? 1u : 0u) << j;
          umask |= (fabsf(d) > bound ? 0u : 1u) << j;  // NaN-safe
        }
        const uint32_t valid = KL - c0 >= 32 ? 0xffffffffu : ((1u << (KL - c0)) - 1u);
        um[cc] = gr < n ? umask & valid : 0u;
        bits_s[row * kBitsLd + (c0 >> 5)] = gr < n ? word : 0u;
        cnt += __popc(um[cc]);
      }
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (total) {  // warp-uniform
      int base = 0;
      if (lane == 31) base = atomicAdd(n_fix, total);
      int pos = __shfl_sync(0xffffffffu, base, 31) + incl - cnt;
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        uint32_t m = um[cc];
        while (m) {
          const int j = __ffs(m) - 1;
          m &= m - 1;
          if (pos < fix_cap) fix[pos] = TcFix{(int32_t)gr, half * 256 + cc * 32 + j};
          ++pos;
        }
      }
    }
    __syncthreads();  // both halves of every row's bits are in shared memory
    // keys of the tile into shared memory (the A parts are free once the
    // MMAs completed), then one coalesced copy: rows are consecutive
    uint32_t* keys_s = reinterpret_cast<uint32_t*>(a_s);
    const int nrow = (int)min((int64_t)kTcRows, n - row0);
    if (row < nrow) {  // tables split between the row's two threads
      const uint32_t kmask = (uint32_t)((1ull << f.k) - 1);
      const uint32_t* bw = bits_s + row * kBitsLd;
      const int t0 = half ? f.l / 2 : 0, t1 = half ? f.l : f.l / 2;
      for (int t = t0, b0 = t0 * f.k; t < t1; ++t, b0 += f.k) {
        const int w0 = b0 >> 5, sh = b0 & 31;
        uint64_t two = bw[w0];
        if (sh + f.k > 32) two |= (uint64_t)bw[w0 + 1] << 32;
        keys_s[row * f.l + t] = (uint32_t)(two >> sh) & kmask;
      }
    }
    __syncthreads();
    {
      uint32_t* dst = keys + row0 * f.l;
      const int nk = nrow * f.l;
      for (int q = tid; q < nk; q += kTcThreads) dst[q] = keys_s[q];
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();  // accumulators read before the next tile's MMAs; A reusable
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTcMaxCols));
}

// exact fp64 recompute of the uncertain (row, bit) cases, in the reference's
// term order, patched into the keys
__global__ void simhash_fix_kernel(SimHashDev f, const float* __restrict__ x, int ld, const TcFix* __restrict__ fix,
                                   const int32_t* __restrict__ n_fix, int fix_cap, uint32_t* __restrict__ keys) {
  const int nf = min(*n_fix, fix_cap);
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nf; q += gridDim.x * blockDim.x) {
    const TcFix e = fix[q];
    const float* xr = x + (int64_t)e.row * ld;
    const uint16_t* pp = f.packed + (int64_t)e.bit * f.c;
    double acc = 0.0;
    for (int j0 = 0; j0 < f.c; j0 += 8) {  // 8 gathers in flight, terms added in order
      uint16_t pe[8];
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) pe[u] = j0 + u < f.c ? pp[j0 + u] : (uint16_t)0;
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = j0 + u < f.c ? xr[pe[u] & 0x7fff] : 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j0 + u < f.c) acc += (pe[u] >> 15) ? -(double)v[u] : (double)v[u];
    }
    const int t = e.bit / f.k, kk = e.bit - t * f.k;
    uint32_t* kw = keys + (int64_t)e.row * f.l + t;
    if (acc > 0.0) atomicOr(kw, 1u << kk);
    else atomicAnd(kw, ~(1u << kk));
  }
}

// false when the shape does not fit (caller uses the CUDA-core kernel)
bool launch_simhash_keys_tc(const SimHashDev& f, const float* x, int64_t n, int ld, uint32_t* keys, DBuf& scratch,
                            cudaStream_t s) {
  const int KL = f.k * f.l;
  const int kdim = kTcK;  // W rows padded to 128 columns (hp = 128)
  if (KL > kTcMaxCols || f.dim > kTcK || kdim > ld || ld % 4 != 0 || n < kTcRows) return false;
  const int np_pad = (KL + 15) / 16 * 16;
  const size_t smem =
      (size_t)np_pad * kdim * 2 + 3 * (size_t)kTcRows * kdim * 2 + 16 + 2 * kTcRows * 4 + kTcRows * kBitsLd * 4;
  if (smem > 227 * 1024) return false;
  const int fix_cap = (int)std::min<int64_t>(std::max<int64_t>(1 << 16, n * KL / 16), 1 << 26);
  uint8_t* buf = scratch.ensure<uint8_t>(16 + (size_t)fix_cap * sizeof(TcFix));
  int32_t* n_fix = reinterpret_cast<int32_t*>(buf);
  TcFix* fix = reinterpret_cast<TcFix*>(buf + 16);
  SLIDE_CUDA(cudaMemsetAsync(n_fix, 0, 4, s));
  SLIDE_CUDA(cudaFuncSetAttribute(simhash_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = (int)std::min<int64_t>(ceil_div(n, kTcRows), (int64_t)kSms);
  simhash_tc_kernel<<<grid, kTcThreads, smem, s>>>(f, x, n, ld, kdim, np_pad, keys, fix, n_fix, fix_cap);
  SLIDE_LAUNCH_CHECK();
  simhash_fix_kernel<<<kSms * 4, 256, 0, s>>>(f, x, ld, fix, n_fix, fix_cap, keys);
  SLIDE_LAUNCH_CHECK();
  int32_t cnt = 0;
  SLIDE_CUDA(cudaMemcpyAsync(&cnt, n_fix, 4, cudaMemcpyDeviceToHost, s));
  SLIDE_CUDA(cudaStreamSynchronize(s));
  if (cnt > fix_cap) return false;  // list overflowed: redo on the CUDA cores
  return true;
}

}  // namespace slide
