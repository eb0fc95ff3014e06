// Internal declarations shared by the SLIDE B200 translation units.
#pragma once
#include "common.cuh"
#include "rng.cuh"
#include <vector>

namespace slide {

// Bumped whenever any DBuf changes its address: a captured step graph holds
// raw pointers, so a step graph captured before the bump must be re-captured.
extern unsigned long long g_slide_realloc_gen;

// Growable device buffer (cudaMalloc'd; contents undefined after grow).
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  // grows geometrically (x1.5) so steady-state steps never reallocate
  template <typename T>
  T* ensure(size_t n) {
    size_t need = n * sizeof(T);
    if (need == 0) need = 16;
    if (need > bytes) {
      if (p) SLIDE_CUDA(cudaFree(p));
      p = nullptr;
      ++g_slide_realloc_gen;
      size_t grow = bytes ? bytes + bytes / 2 : 0;
      size_t alloc = need > grow ? need : grow;
      alloc = (alloc + 255) & ~(size_t)255;
      SLIDE_CUDA(cudaMalloc(&p, alloc));
      bytes = alloc;
    }
    return reinterpret_cast<T*>(p);
  }
  template <typename T>
  T* as() const { return reinterpret_cast<T*>(p); }
  void release() {
    if (p) {
      cudaFree(p);
      ++g_slide_realloc_gen;
    }
    p = nullptr;
    bytes = 0;
  }
};

// ---------------------------------------------------------------- hashing
struct SimHashDev {
  int dim, k, l, c;
  const uint16_t* packed;  // (K*L, c): idx | (sign<0) << 15
  const uint16_t* packed_t = nullptr;  // optional (c, K*L) copy: queries read it from L1/L2
};
struct DwtaDev {
  int dim, k, l, m, bins_per_perm, n_perms, bits;
  int dense_mode;          // 1 = WTA (zeros take part), 0 = DWTA
  const int16_t* perms;    // (n_perms, dim)
  const int16_t* donors;   // (K*L, 100)
};

// Tensor-core rebuild path (tc_hash.cu); false when the shape does not fit.
bool launch_simhash_keys_tc(const SimHashDev& f, const float* x, int64_t n, int ld, uint32_t* keys, DBuf& scratch,
                            cudaStream_t s);
// tc_scratch: when given, large row counts (table rebuilds) go to the
// tensor-core path
void launch_simhash_keys(const SimHashDev& f, const float* x, int64_t n, int ld, uint32_t* keys,
                         cudaStream_t s, DBuf* tc_scratch = nullptr);
void launch_dwta_keys(const DwtaDev& f, const float* x, int64_t n, int ld, uint32_t* keys,
                      cudaStream_t s);

// ----------------------------------------------------------------- tables
// Built structure of the L tables of one layer.  Runs = distinct (table,
// key) pairs after a stable (table,key) sort of the N*L inserts.
struct TablesDev {
  int l = 0, key_bits = 0, cap = 0;
  int dense_dir = 0;          // 1: dir is (L << key_bits) int32 run ids
  int validated = 0;          // dense dir never cleared: an entry counts only if run_keys[r] == key
  const uint32_t* run_keys = nullptr;  // per run: its (table << key_bits | key)
  int empty = 1;              // no buckets (unbuilt or cleared)
  uint64_t disabled = 0;      // bit t: table t reads as empty
  uint64_t hash_mask = 0;     // hash directory size - 1
  const int32_t* dir = nullptr;
  const uint64_t* hdir = nullptr;
  const int32_t* bstart = nullptr;  // per run: first bucket slot in ids
  const int32_t* blen = nullptr;    // per run: occupancy (<= cap)
  const int32_t* bcount = nullptr;  // per run: insert count
  const int32_t* ids = nullptr;     // bucket contents
  int64_t n_runs = 0;
  // two-level directory for long keys (DWTA): per (table, top key bits)
  // prefix p the first run whose prefix is >= p, stored reversed
  // (coarse[coarse_n - 1 - p]); a lookup binary-searches the prefix's runs
  const int32_t* coarse = nullptr;
  int coarse_shift = 0;
  int64_t coarse_n = 0;
};

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x85ebca6bu;
  x ^= x >> 13;
  x *= 0xc2b2ae35u;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ int tables_lookup(const TablesDev& t, uint32_t skey) {
  if (t.empty || ((t.disabled >> (skey >> t.key_bits)) & 1ull)) return -1;
  if (t.coarse) {
    const int64_t p = skey >> t.coarse_shift;
    int lo = t.coarse[t.coarse_n - 1 - p];
    int hi = p + 1 < t.coarse_n ? t.coarse[t.coarse_n - 2 - p] : (int)t.n_runs;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (t.run_keys[mid] < skey) lo = mid + 1;
      else hi = mid;
    }
    return lo < t.n_runs && t.run_keys[lo] == skey ? lo : -1;
  }
  if (t.dense_dir) {
    const int r = t.dir[skey];
    if (t.validated && ((uint64_t)(uint32_t)r >= (uint64_t)t.n_runs || t.run_keys[r] != skey)) return -1;
    return r;
  }
  uint64_t loc = hash32(skey) & t.hash_mask;
  while (true) {
    uint64_t e = t.hdir[loc];
    if (e == ~0ull) return -1;
    if ((uint32_t)(e >> 32) == skey) return (int)(uint32_t)e;
    loc = (loc + 1) & t.hash_mask;
  }
}

struct TablesHost {
  TablesDev dev;
  DBuf skeys_a, skeys_b, vals_a, vals_b, uniq, counts, offsets, nruns, dir, hdir, bstart, blen, temp,
      ovf_cnt, ovf_off, ovf_ev, patch, coarse, ctemp;
  int64_t n_items = 0, n_slots = 0;
  int policy = 0;  // 0 fifo, 1 reservoir
  bool built = false;
  void release();
};

// Build all L tables from row keys (n, L).  mt_state (625 words, host) is the
// reservoir stream, consumed and updated when a bucket overflows.
// id_mul / id_add: stored id of row r is r * id_mul + id_add (a column shard
// of the output layer stores its rows' global ids; reservoir overflows are
// then not replayed -- the sharded caller proves there are none)
void tables_build(TablesHost& tb, const uint32_t* keys, int64_t n, int l, int key_bits, int cap,
                  int policy, uint64_t* mt_state, cudaStream_t s, int id_mul = 1, int id_add = 0);
// sharded FIFO reconciliation (see tables.cu)
int64_t tables_pack_size(const TablesHost& tb);
void tables_pack(const TablesHost& tb, int32_t* out, cudaStream_t s);
void tables_reconcile(TablesHost& tb, const int32_t* packs, int64_t stride, int G, int g, int cap, cudaStream_t s);
// Install host-made buckets (device copies of the arrays), directory rebuilt.
void tables_load(TablesHost& tb, const uint32_t* skeys, const int32_t* counts, const int32_t* starts,
                 const int32_t* lens, int64_t n_runs, const int32_t* ids, int64_t n_slots, int64_t n_items, int l,
                 int key_bits, int cap, cudaStream_t s);

// ------------------------------------------------------------------ misc
void launch_iota_slots(const int32_t* ptr, int b, int32_t* slot_of, cudaStream_t s);

}  // namespace slide
