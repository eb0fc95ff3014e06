// Bit-exact restatement of the random streams the reference consumes on the
// hot path, usable on host and device.
//
// * numpy Generator(PCG64) seeded from SeedSequence(entropy):
//   reference network.py:353 `default_rng((seed, iteration, slot))`.
//   - permutation(n): Fisher-Yates with `random_interval` (samplers.py:69).
//   - choice(pop, size, replace=False): Floyd with a hash set + tail
//     shuffle of the result, or the partial "tail shuffle" of arange(pop)
//     when pop > 10000 and size > pop // 50 (network.py:231).
//   numpy's RNG source is not vendored in the container; this
//   restates its published algorithms (numpy 2.3, PCG64 XSL-RR 128/64,
//   SeedSequence hashmix, Lemire bounded ints) and is pinned by golden
//   streams produced by numpy itself (tests/golden/rng_streams.npz).
// * CPython random.Random (MT19937, 53-bit random()): tables.py:101,149-161,
//   pinned by tests/golden/mt19937.npz.  Host only.
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define SL_HD __host__ __device__ __forceinline__
#else
#define SL_HD inline
#endif

namespace slide {

typedef unsigned __int128 u128;

// ---------------------------------------------------------------- SeedSequence
struct SeedSeq {
  static constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u;
  static constexpr uint32_t INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
  static constexpr uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
  uint32_t pool[4];

  SL_HD static uint32_t hashmix(uint32_t v, uint32_t& hc) {
    v ^= hc;
    hc *= MULT_A;
    v *= hc;
    v ^= v >> 16;
    return v;
  }
  SL_HD static uint32_t mix(uint32_t x, uint32_t y) {
    uint32_t r = MIX_L * x - MIX_R * y;
    r ^= r >> 16;
    return r;
  }
  // entropy: a sequence of non-negative integers, each split into 32-bit
  // little-endian words (0 -> one zero word).
  SL_HD void init(const uint64_t* ent, int n_ent) {
    uint32_t words[16];
    int nw = 0;
    for (int i = 0; i < n_ent && nw < 15; ++i) {
      uint64_t x = ent[i];
      if (x == 0) {
        words[nw++] = 0;
      } else {
        while (x && nw < 16) {
          words[nw++] = (uint32_t)(x & 0xffffffffu);
          x >>= 32;
        }
      }
    }
    uint32_t hc = INIT_A;
    for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < nw ? words[i] : 0u, hc);
    for (int s = 0; s < 4; ++s)
      for (int d = 0; d < 4; ++d)
        if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], hc));
    for (int s = 4; s < nw; ++s)
      for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(words[s], hc));
  }
  // generate_state(n64, uint64)
  SL_HD void generate(uint64_t* out, int n64) const {
    uint32_t hc = INIT_B;
    for (int i = 0; i < 2 * n64; ++i) {
      uint32_t v = pool[i & 3];
      v ^= hc;
      hc *= MULT_B;
      v *= hc;
      v ^= v >> 16;
      if (i & 1)
        out[i >> 1] |= (uint64_t)v << 32;
      else
        out[i >> 1] = v;
    }
  }
};

// ---------------------------------------------------------------------- PCG64
struct Pcg64 {
  u128 state, inc;
  uint32_t has32, u32;

  SL_HD static u128 mult() {
    return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
  }
  SL_HD void step() { state = state * mult() + inc; }
  SL_HD void seed_from(const uint64_t* ent, int n_ent) {
    SeedSeq ss;
    ss.init(ent, n_ent);
    uint64_t v[4];
    ss.generate(v, 4);
    u128 s = ((u128)v[0] << 64) | v[1];
    u128 i = ((u128)v[2] << 64) | v[3];
    inc = (i << 1) | 1u;
    state = 0;
    step();
    state += s;
    step();
    has32 = 0;
    u32 = 0;
  }
  SL_HD uint64_t next64() {
    step();
    uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    unsigned rot = (unsigned)(state >> 122);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  SL_HD uint32_t next32() {
    if (has32) {
      has32 = 0;
      return u32;
    }
    uint64_t n = next64();
    has32 = 1;
    u32 = (uint32_t)(n >> 32);
    return (uint32_t)n;
  }
  // random_interval(max) / random_bounded_uint64: rng_interval / rng_bounded below
  SL_HD uint64_t interval(uint64_t mx);
  SL_HD uint64_t bounded(uint64_t rng);
  SL_HD static uint64_t xsl_rr(u128 st) {
    uint64_t hi = (uint64_t)(st >> 64), lo = (uint64_t)st;
    unsigned rot = (unsigned)(st >> 122);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }

  // serialised as 6 uint64: state hi/lo, inc hi/lo, has_uint32, uinteger
  SL_HD void store(uint64_t* s) const {
    s[0] = (uint64_t)(state >> 64);
    s[1] = (uint64_t)state;
    s[2] = (uint64_t)(inc >> 64);
    s[3] = (uint64_t)inc;
    s[4] = has32;
    s[5] = u32;
  }
  SL_HD void load(const uint64_t* s) {
    state = ((u128)s[0] << 64) | s[1];
    inc = ((u128)s[2] << 64) | s[3];
    has32 = (uint32_t)s[4];
    u32 = (uint32_t)s[5];
  }
};

// random_interval(max): masked rejection (used by Generator.shuffle); G is
// any source with next32 / next64 (Pcg64, PcgBuf)
template <class G>
SL_HD uint64_t rng_interval(G& g, uint64_t mx) {
  if (mx == 0) return 0;
  uint64_t mask = mx;
  mask |= mask >> 1;
  mask |= mask >> 2;
  mask |= mask >> 4;
  mask |= mask >> 8;
  mask |= mask >> 16;
  mask |= mask >> 32;
  uint64_t v;
  if (mx <= 0xffffffffull) {
    while ((v = (g.next32() & mask)) > mx) {
    }
  } else {
    while ((v = (g.next64() & mask)) > mx) {
    }
  }
  return v;
}

// random_bounded_uint64(off=0, rng, use_masked=false): Lemire
template <class G>
SL_HD uint64_t rng_bounded(G& g, uint64_t rng) {
  if (rng == 0) return 0;
  if (rng <= 0xffffffffull) {
    if (rng == 0xffffffffull) return g.next32();
    uint32_t rx = (uint32_t)rng + 1u;
    uint64_t m = (uint64_t)g.next32() * rx;
    uint32_t left = (uint32_t)m;
    if (left < rx) {
      uint32_t th = (uint32_t)((0xffffffffu - (uint32_t)rng) % rx);
      while (left < th) {
        m = (uint64_t)g.next32() * rx;
        left = (uint32_t)m;
      }
    }
    return m >> 32;
  }
  if (rng == 0xffffffffffffffffull) return g.next64();
  uint64_t rx = rng + 1;
  u128 m = (u128)g.next64() * rx;
  uint64_t left = (uint64_t)m;
  if (left < rx) {
    uint64_t th = (0xffffffffffffffffull - rng) % rx;
    while (left < th) {
      m = (u128)g.next64() * rx;
      left = (uint64_t)m;
    }
  }
  return (uint64_t)(m >> 64);
}

SL_HD uint64_t Pcg64::interval(uint64_t mx) { return rng_interval(*this, mx); }
SL_HD uint64_t Pcg64::bounded(uint64_t rng) { return rng_bounded(*this, rng); }

// Jump-ahead: after k steps the state is A_k s + S_k inc (A_k = a^k, S_k =
// 1 + a + ... + a^(k-1) mod 2^128), so k outputs of one stream can be made
// in parallel and the state after any prefix of them restored exactly.
constexpr int kPcgJump = 65536;
SL_HD void pcg_jump_coeffs(int k, u128& A, u128& S) {
  A = 1;
  S = 0;
  for (int i = 0; i < k; ++i) {
    S = S * Pcg64::mult() + 1;
    A = A * Pcg64::mult();
  }
}

#ifdef __CUDACC__
// the device jump table: jump[2k], jump[2k + 1] = (A_k, S_k), k = 0..kPcgJump
// (built once on the host, select.cu)
const u128* pcg_jump_table();

// A stream consumer reading a precomputed run of outputs: buf[k] = output
// k + 1 of the generator `base`; past the run it steps serially.  The
// interval / bounded / has32 logic is the generator's own, so the values
// and the final state equal Pcg64's.
struct PcgBuf {
  const uint64_t* buf;
  int n, pos;
  Pcg64 g;  // the base state; after the run, the serial continuation
  uint32_t has32, u32;
  const u128* jump;
  __device__ PcgBuf(const Pcg64& base, const uint64_t* b, int nb, const u128* jt)
      : buf(b), n(nb), pos(0), g(base), has32(base.has32), u32(base.u32), jump(jt) {}
  __device__ uint64_t next64() {
    if (pos < n) return buf[pos++];
    if (pos == n) {  // leave the run: the state after n steps
      const u128 A = jump[2 * n], S = jump[2 * n + 1];
      g.state = A * g.state + S * g.inc;
    }
    ++pos;
    g.step();
    return Pcg64::xsl_rr(g.state);
  }
  __device__ uint32_t next32() {
    if (has32) {
      has32 = 0;
      return u32;
    }
    uint64_t v = next64();
    has32 = 1;
    u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  // the generator after everything consumed so far
  __device__ void finish(Pcg64& out) {
    out = g;
    if (pos <= n) {
      const u128 A = jump[2 * pos], S = jump[2 * pos + 1];
      out.state = A * g.state + S * g.inc;
    }
    out.has32 = has32;
    out.u32 = u32;
  }
};

// the first n (<= kPcgJump) outputs of `g`, threads t of nt in parallel
__device__ __forceinline__ void pcg_fill(const Pcg64& g, uint64_t* buf, int n, int t, int nt, const u128* jump) {
  for (int k = t; k < n; k += nt) {
    const u128 A = jump[2 * (k + 1)], S = jump[2 * (k + 1) + 1];
    buf[k] = Pcg64::xsl_rr(A * g.state + S * g.inc);
  }
}
#endif

// Generator.permutation(n) on an int array (n small: L tables)
template <typename T, class G>
SL_HD void pcg_permutation(G& g, T* a, int n) {
  for (int i = 0; i < n; ++i) a[i] = (T)i;
  for (int i = n - 1; i >= 1; --i) {
    int j = (int)rng_interval(g, (uint64_t)i);
    T t = a[i];
    a[i] = a[j];
    a[j] = t;
  }
}

SL_HD uint64_t gen_mask(uint64_t x) {
  x |= x >> 1;
  x |= x >> 2;
  x |= x >> 4;
  x |= x >> 8;
  x |= x >> 16;
  x |= x >> 32;
  return x;
}

// Sizes of the scratch choice() needs (int64 entries).
SL_HD bool choice_uses_tail(int64_t pop, int64_t size) { return pop > 10000 && size > pop / 50; }
SL_HD int64_t choice_scratch_entries(int64_t pop, int64_t size) {
  if (choice_uses_tail(pop, size)) return 2 * (int64_t)(gen_mask((uint64_t)(2 * size)) + 1);
  return (int64_t)(gen_mask((uint64_t)(1.2 * (double)size)) + 1);
}

// Generator.choice(pop, size, replace=False) -> out[size] (numpy order).
// scratch: choice_scratch_entries(pop,size) int64 slots; any contents.
// keep_order = false: the final shuffle's draws are consumed (the generator
// ends in numpy's state) but not applied -- for callers that only need the
// set (the training fallback unions it with the labels and sorts).
template <class G>
SL_HD void pcg_choice(G& g, int64_t pop, int64_t size, int64_t* out, int64_t* scratch, bool keep_order = true) {
  if (size <= 0) return;
  if (choice_uses_tail(pop, size)) {
    // partial Fisher-Yates of arange(pop) over positions [first, pop);
    // sparse position->value map (open addressing, key -1 = empty)
    const uint64_t cap = gen_mask((uint64_t)(2 * size)) + 1;
    const uint64_t mask = cap - 1;
    int64_t* keys = scratch;
    int64_t* vals = scratch + cap;
    for (uint64_t q = 0; q < cap; ++q) keys[q] = -1;
    auto find = [&](int64_t pos) -> uint64_t {
      uint64_t h = ((uint64_t)pos * 0x9E3779B97F4A7C15ull) >> 17;
      uint64_t loc = h & mask;
      while (keys[loc] != -1 && keys[loc] != pos) loc = (loc + 1) & mask;
      return loc;
    };
    const int64_t lo = pop - size;
    const int64_t first = lo > 1 ? lo : 1;
    for (int64_t i = pop - 1; i >= first; --i) {
      int64_t j = (int64_t)rng_bounded(g, (uint64_t)i);
      uint64_t li = find(i);
      int64_t vi = keys[li] == i ? vals[li] : i;
      uint64_t lj = find(j);
      int64_t vj = keys[lj] == j ? vals[lj] : j;
      out[i - lo] = vj;
      if (j != i) {
        keys[lj] = j;
        vals[lj] = vi;
      }
    }
    for (int64_t i = lo; i < first; ++i) {  // only when size == pop
      uint64_t l = find(i);
      out[i - lo] = keys[l] == i ? vals[l] : i;
    }
    return;
  }
  // Floyd's algorithm with numpy's open-addressing hash set
  const uint64_t mask = gen_mask((uint64_t)(1.2 * (double)size));
  int64_t* hs = scratch;
  for (uint64_t q = 0; q <= mask; ++q) hs[q] = -1;
  for (int64_t j = pop - size; j < pop; ++j) {
    int64_t val = (int64_t)rng_bounded(g, (uint64_t)j);
    uint64_t loc = (uint64_t)val & mask;
    while (hs[loc] != -1 && hs[loc] != val) loc = (loc + 1) & mask;
    if (hs[loc] == -1) {
      hs[loc] = val;
      out[j - pop + size] = val;
    } else {
      loc = (uint64_t)j & mask;
      while (hs[loc] != -1) loc = (loc + 1) & mask;
      hs[loc] = j;
      out[j - pop + size] = j;
    }
  }
  // shuffle=True: _shuffle_int(size, 1, out)
  for (int64_t i = size - 1; i >= 1; --i) {
    int64_t j = (int64_t)rng_bounded(g, (uint64_t)i);
    if (!keep_order) continue;
    int64_t t = out[i];
    out[i] = out[j];
    out[j] = t;
  }
}

// ------------------------------------------------------------------- MT19937
// CPython random.Random: state = 624 words + index (getstate()[1]).
struct Mt19937 {
  uint32_t mt[624];
  int idx;
  void load(const uint64_t* s) {
    for (int i = 0; i < 624; ++i) mt[i] = (uint32_t)s[i];
    idx = (int)s[624];
  }
  void store(uint64_t* s) const {
    for (int i = 0; i < 624; ++i) s[i] = mt[i];
    s[624] = (uint64_t)idx;
  }
  uint32_t next() {
    if (idx >= 624) {
      for (int k = 0; k < 624; ++k) {
        uint32_t y = (mt[k] & 0x80000000u) | (mt[(k + 1) % 624] & 0x7fffffffu);
        mt[k] = mt[(k + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
      }
      idx = 0;
    }
    uint32_t y = mt[idx++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
  }
  double random() {  // genrand_res53
    uint32_t a = next() >> 5, b = next() >> 6;
    return ((double)a * 67108864.0 + (double)b) * (1.0 / 9007199254740992.0);
  }
};

}  // namespace slide
