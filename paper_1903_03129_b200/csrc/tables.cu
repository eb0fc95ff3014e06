// (K, L) bucket index build (reference tables.py:105-161).
//
// Ids 0..N-1 enter every table in ascending order.  On the device that is
// one stable radix sort of the N*L (table, key) inserts with the id as value:
// each run of equal (table, key) is a bucket's insert history in insertion
// order.  FIFO keeps the last min(count, cap) entries of the run
// (tables.py:130-145); reservoir keeps the first cap and replays the
// overflowing inserts through the MT19937 stream on the host, in (table, id)
// order (tables.py:146-161).  A directory maps (table, key) to its run:
// dense (L << key_bits entries) for short keys, open addressing otherwise.
#include "internal.cuh"
#include <cub/cub.cuh>
#include <algorithm>

namespace slide {

void TablesHost::release() {
  for (DBuf* b : {&skeys_a, &skeys_b, &vals_a, &vals_b, &uniq, &counts, &offsets, &nruns, &dir, &hdir,
                  &bstart, &blen, &temp, &ovf_cnt, &ovf_off, &ovf_ev, &patch, &coarse, &ctemp})
    b->release();
  built = false;
}

__global__ void runs_kernel(const uint32_t* __restrict__ uniq, const int32_t* __restrict__ counts,
                            const int32_t* __restrict__ offsets, int64_t n_runs, int cap, int fifo,
                            int dense, int32_t* dir, uint64_t* hdir, uint64_t hmask,
                            int32_t* __restrict__ bstart, int32_t* __restrict__ blen,
                            int32_t* __restrict__ ovf) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_runs;
       r += (int64_t)gridDim.x * blockDim.x) {
    int cnt = counts[r];
    int len = cnt < cap ? cnt : cap;
    bstart[r] = fifo ? offsets[r] + cnt - len : offsets[r];
    blen[r] = len;
    if (ovf) ovf[r] = cnt > cap ? cnt - cap : 0;
    uint32_t sk = uniq[r];
    if (dense) {
      dir[sk] = (int32_t)r;
    } else if (hdir) {
      uint64_t ent = ((uint64_t)sk << 32) | (uint32_t)r;
      uint64_t loc = hash32(sk) & hmask;
      while (true) {
        unsigned long long prev = atomicCAS((unsigned long long*)&hdir[loc], ~0ull, (unsigned long long)ent);
        if (prev == ~0ull) break;
        loc = (loc + 1) & hmask;
      }
    }
  }
}

__global__ void dir_kernel(const uint32_t* __restrict__ uniq, int64_t n_runs, int dense, int32_t* dir,
                           uint64_t* hdir, uint64_t hmask) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_runs;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint32_t sk = uniq[r];
    if (dense) {
      dir[sk] = (int32_t)r;
      continue;
    }
    if (!hdir) return;  // two-level directory: built from the runs afterwards
    uint64_t ent = ((uint64_t)sk << 32) | (uint32_t)r;
    uint64_t loc = hash32(sk) & hmask;
    while (atomicCAS((unsigned long long*)&hdir[loc], ~0ull, (unsigned long long)ent) != ~0ull)
      loc = (loc + 1) & hmask;
  }
}

struct OvfEvent {
  int32_t id, table, off, count;
};

__global__ void overflow_events_kernel(const uint32_t* __restrict__ uniq, const int32_t* __restrict__ counts,
                                       const int32_t* __restrict__ offsets, const int32_t* __restrict__ ovf,
                                       const int32_t* __restrict__ ovf_off, const int32_t* __restrict__ ids,
                                       int64_t n_runs, int cap, int kb, OvfEvent* ev) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_runs;
       r += (int64_t)gridDim.x * blockDim.x) {
    int o = ovf[r];
    if (!o) continue;
    int base = ovf_off[r], off = offsets[r];
    int t = (int)(uniq[r] >> kb);
    for (int p = 0; p < o; ++p) {
      OvfEvent e;
      e.id = ids[off + cap + p];
      e.table = t;
      e.off = off;
      e.count = cap + p + 1;
      ev[base + p] = e;
    }
  }
}

__global__ void patch_kernel(const int2* __restrict__ patches, int64_t n, int32_t* ids) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    ids[patches[q].x] = patches[q].y;
}


// Directory choice.  Short keys (<= 16 bits): a dense (table, key) -> run
// table, reset per build.  Longer keys with a key space at most 64x the
// inserts and <= 2^30 entries (DWTA 24-bit keys at wide-out / scaled): the
// same dense table but never cleared -- a lookup validates the entry against
// the run's own key (stale entries of earlier builds fail the check), so a
// build only scatters its runs.  Otherwise an open-addressing hash.
__global__ void fill_kernel(int32_t* __restrict__ a, int64_t n, int32_t v) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) a[q] = v;
}

// the two-level directory's prefix marks: run r starts its prefix when the
// previous run's prefix differs (runs are sorted by (table, key))
__global__ void coarse_mark_kernel(const uint32_t* __restrict__ uniq, int64_t n_runs, int shift, int64_t n_p,
                                   int32_t* __restrict__ crev) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_runs; r += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = uniq[r] >> shift;
    if (r == 0 || (uniq[r - 1] >> shift) != p) crev[n_p - 1 - p] = (int32_t)r;
  }
}

static int grid_for(int64_t n, int bs = 256);

// Long keys: the two-level directory (built after the runs, see
// build_coarse).  A dense (L << key_bits) table of run ids would be one
// random 4-byte write per run into up to 4 GB (DWTA 24-bit keys at 4M rows:
// 2.5 ms per build); the coarse table holds ~8 runs per prefix.
static void build_coarse(TablesHost& tb, TablesDev& d, int l, int kb, int64_t n_runs, const uint32_t* uniq,
                         cudaStream_t s) {
  int cb = 1;
  while (cb < kb && ((int64_t)l << (cb + 3)) < n_runs) ++cb;  // ~8 runs per prefix
  const int64_t n_p = (int64_t)l << cb;
  int32_t* crev = tb.coarse.ensure<int32_t>(n_p);
  fill_kernel<<<grid_for(n_p, 256), 256, 0, s>>>(crev, n_p, (int32_t)n_runs);
  SLIDE_LAUNCH_CHECK();
  if (n_runs > 0) {
    coarse_mark_kernel<<<grid_for(n_runs, 256), 256, 0, s>>>(uniq, n_runs, kb - cb, n_p, crev);
    SLIDE_LAUNCH_CHECK();
  }
  size_t bytes = 0;
  SLIDE_CUDA(cub::DeviceScan::InclusiveScan(nullptr, bytes, crev, crev, cub::Min(), (int)n_p, s));
  void* tmp = tb.ctemp.ensure<uint8_t>(bytes);
  SLIDE_CUDA(cub::DeviceScan::InclusiveScan(tmp, bytes, crev, crev, cub::Min(), (int)n_p, s));  // suffix minimum
  d.coarse = crev;
  d.coarse_shift = kb - cb;
  d.coarse_n = n_p;
}

static void choose_dir(TablesHost& tb, TablesDev& d, int l, int kb, int64_t n_items, int64_t n_runs, cudaStream_t s) {
  (void)n_items;
  const uint64_t nd = (uint64_t)l << kb;
  d.dense_dir = kb <= 16;
  d.validated = 0;
  d.dir = nullptr;
  d.hdir = nullptr;
  d.hash_mask = 0;
  d.coarse = nullptr;
  if (kb > 16) return;  // two-level directory, built from the runs (build_coarse)
  if (d.dense_dir) {
    int32_t* dir = tb.dir.ensure<int32_t>(nd);
    if (!d.validated) SLIDE_CUDA(cudaMemsetAsync(dir, 0xff, nd * 4, s));
    d.dir = dir;
  } else {
    uint64_t hc = gen_mask((uint64_t)std::max<int64_t>(2 * n_runs, 16)) + 1;
    uint64_t* hdir = tb.hdir.ensure<uint64_t>(hc);
    SLIDE_CUDA(cudaMemsetAsync(hdir, 0xff, hc * 8, s));
    d.hdir = hdir;
    d.hash_mask = hc - 1;
  }
}

// (n, L) row-major keys -> the inserts (t << kb | key, id) in the same
// row-major order: a stable sort by (table, key) then yields every bucket's
// ids ascending, the order they were inserted in (tables.py:127-161) -- no
// transpose needed.  Four inserts per thread, 16-byte loads.
template <typename K>
__global__ void __launch_bounds__(256) composite_keys_kernel(const uint32_t* __restrict__ keys, int64_t total, int l,
                                                             int kb, K* __restrict__ skeys,
                                                             int32_t* __restrict__ vals, int id_mul, int id_add) {
  for (int64_t q0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; q0 < total;
       q0 += (int64_t)gridDim.x * blockDim.x * 4) {
    uint32_t k[4];
    if (q0 + 4 <= total && (q0 & 3) == 0) {
      const uint4 v = __ldcs(reinterpret_cast<const uint4*>(keys + q0));
      k[0] = v.x, k[1] = v.y, k[2] = v.z, k[3] = v.w;
    } else {
      for (int j = 0; j < 4; ++j) k[j] = q0 + j < total ? keys[q0 + j] : 0u;
    }
    const int64_t r0 = q0 / l;
    int t = (int)(q0 - r0 * l);
    int64_t r = r0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (q0 + j < total) {
        skeys[q0 + j] = (K)(((uint32_t)t << kb) | k[j]);
        vals[q0 + j] = (int32_t)(r * id_mul + id_add);
      }
      if (++t == l) {
        t = 0;
        ++r;
      }
    }
  }
}

__global__ void widen_keys_kernel(const uint16_t* __restrict__ in, const int32_t* __restrict__ n_dev,
                                  uint32_t* __restrict__ out) {
  const int n = *n_dev;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) out[q] = in[q];
}

static int grid_for(int64_t n, int bs) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, bs), kSms * 16)); }

void tables_build(TablesHost& tb, const uint32_t* keys, int64_t n, int l, int kb, int cap, int policy,
                  uint64_t* mt_state, cudaStream_t s, int id_mul, int id_add) {
  int tbits = 0;
  while ((1 << tbits) < l) ++tbits;
  SLIDE_CHECK(kb + tbits <= 32, kNotSupported, "table index + key bits must fit in 32 bits");
  SLIDE_CHECK(n * l < (int64_t)INT32_MAX, kNotSupported, "N*L inserts exceed int32 range");
  const int64_t total = n * l;
  uint32_t* ska = tb.skeys_a.ensure<uint32_t>(total);
  uint32_t* skb = tb.skeys_b.ensure<uint32_t>(total);
  int32_t* va = tb.vals_a.ensure<int32_t>(total);
  int32_t* vb = tb.vals_b.ensure<int32_t>(total);
  uint32_t* uniq = tb.uniq.ensure<uint32_t>(total);
  int32_t* counts = tb.counts.ensure<int32_t>(total);
  int32_t* offsets = tb.offsets.ensure<int32_t>(total);
  int32_t* nr_d = tb.nruns.ensure<int32_t>(1);
  const int end_bit = kb + tbits;
  const int cgrid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 1024), (int64_t)kSms * 16));
  size_t tbytes = 0;
  void* temp = nullptr;
  if (end_bit <= 16) {
    // short keys (SimHash): 16-bit (table, key) keys -- a quarter less
    // traffic in each radix pass and in the run-length encode
    uint16_t* ska16 = reinterpret_cast<uint16_t*>(ska);
    uint16_t* skb16 = reinterpret_cast<uint16_t*>(skb);
    uint16_t* uniq16 = reinterpret_cast<uint16_t*>(offsets);  // scratch until the runs are counted
    if (total > 0) {
      composite_keys_kernel<uint16_t><<<cgrid, 256, 0, s>>>(keys, total, l, kb, ska16, va, id_mul, id_add);
      SLIDE_LAUNCH_CHECK();
    }
    size_t b1 = 0, b2 = 0, b3 = 0;
    SLIDE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b1, ska16, skb16, va, vb, (int)total, 0, end_bit, s));
    SLIDE_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, b2, skb16, uniq16, counts, nr_d, (int)total, s));
    SLIDE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b3, counts, offsets, (int)total, s));
    tbytes = std::max(b1, std::max(b2, b3));
    temp = tb.temp.ensure<uint8_t>(tbytes);
    SLIDE_CUDA(cub::DeviceRadixSort::SortPairs(temp, tbytes, ska16, skb16, va, vb, (int)total, 0, end_bit, s));
    SLIDE_CUDA(cub::DeviceRunLengthEncode::Encode(temp, tbytes, skb16, uniq16, counts, nr_d, (int)total, s));
    widen_keys_kernel<<<grid_for(std::min<int64_t>(total, (int64_t)1 << end_bit)), 256, 0, s>>>(uniq16, nr_d, uniq);
    SLIDE_LAUNCH_CHECK();
  } else {
    if (total > 0) {
      composite_keys_kernel<uint32_t><<<cgrid, 256, 0, s>>>(keys, total, l, kb, ska, va, id_mul, id_add);
      SLIDE_LAUNCH_CHECK();
    }
    size_t b1 = 0, b2 = 0, b3 = 0;
    SLIDE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b1, ska, skb, va, vb, (int)total, 0, end_bit, s));
    SLIDE_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, b2, skb, uniq, counts, nr_d, (int)total, s));
    SLIDE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b3, counts, offsets, (int)total, s));
    tbytes = std::max(b1, std::max(b2, b3));
    temp = tb.temp.ensure<uint8_t>(tbytes);
    SLIDE_CUDA(cub::DeviceRadixSort::SortPairs(temp, tbytes, ska, skb, va, vb, (int)total, 0, end_bit, s));
    SLIDE_CUDA(cub::DeviceRunLengthEncode::Encode(temp, tbytes, skb, uniq, counts, nr_d, (int)total, s));
  }
  int32_t n_runs = 0;
  SLIDE_CUDA(cudaMemcpyAsync(&n_runs, nr_d, 4, cudaMemcpyDeviceToHost, s));
  SLIDE_CUDA(cudaStreamSynchronize(s));
  if (n_runs > 0) SLIDE_CUDA(cub::DeviceScan::ExclusiveSum(temp, tbytes, counts, offsets, n_runs, s));

  TablesDev& d = tb.dev;
  d.l = l;
  d.key_bits = kb;
  d.cap = cap;
  d.n_runs = n_runs;
  choose_dir(tb, d, l, kb, total, n_runs, s);
  d.run_keys = uniq;
  int32_t* dir = const_cast<int32_t*>(d.dir);
  uint64_t* hdir = const_cast<uint64_t*>(d.hdir);
  const uint64_t hmask = d.hash_mask;
  // per-run arrays sized by the bound (runs <= inserts), like uniq / counts /
  // offsets above: a rebuild whose run count passed the previous one must not
  // free and re-allocate GB-sized buffers between two training steps (seen as
  // 50-700 ms rebuild barriers at the scaled shape) nor move what a captured
  // step graph points at
  const int64_t run_cap = std::max<int64_t>(total, 1);
  int32_t* bstart = tb.bstart.ensure<int32_t>(run_cap);
  int32_t* blen = tb.blen.ensure<int32_t>(run_cap);
  int32_t* ovf = policy == 1 ? tb.ovf_cnt.ensure<int32_t>(run_cap) : nullptr;
  if (n_runs > 0) {
    runs_kernel<<<grid_for(n_runs), 256, 0, s>>>(uniq, counts, offsets, n_runs, cap, policy == 0, d.dense_dir,
                                                 dir, hdir, hmask, bstart, blen, ovf);
    SLIDE_LAUNCH_CHECK();
  }
  if (kb > 16) build_coarse(tb, d, l, kb, n_runs, uniq, s);
  if (policy == 1 && n_runs > 0 && id_mul == 1) {
    // reservoir: host replay of the overflowing inserts (tables.py:156-161)
    int32_t* ovf_off = tb.ovf_off.ensure<int32_t>(run_cap);
    size_t b4 = 0;
    SLIDE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b4, ovf, ovf_off, (int)n_runs, s));
    if (b4 > tbytes) {
      // temp grows; contents are not needed any more
      temp = tb.temp.ensure<uint8_t>(b4);
      tbytes = b4;
    }
    SLIDE_CUDA(cub::DeviceScan::ExclusiveSum(temp, tbytes, ovf, ovf_off, (int)n_runs, s));
    int32_t last[2] = {0, 0};
    SLIDE_CUDA(cudaMemcpyAsync(&last[0], ovf_off + n_runs - 1, 4, cudaMemcpyDeviceToHost, s));
    SLIDE_CUDA(cudaMemcpyAsync(&last[1], ovf + n_runs - 1, 4, cudaMemcpyDeviceToHost, s));
    SLIDE_CUDA(cudaStreamSynchronize(s));
    int64_t n_ev = (int64_t)last[0] + last[1];
    if (n_ev > 0) {
      SLIDE_CHECK(mt_state != nullptr, kValueError, "reservoir build needs the random.Random state");
      OvfEvent* ev = tb.ovf_ev.ensure<OvfEvent>(n_ev);
      overflow_events_kernel<<<grid_for(n_runs), 256, 0, s>>>(uniq, counts, offsets, ovf, ovf_off, vb, n_runs,
                                                               cap, kb, ev);
      SLIDE_LAUNCH_CHECK();
      std::vector<OvfEvent> h(n_ev);
      SLIDE_CUDA(cudaMemcpyAsync(h.data(), ev, n_ev * sizeof(OvfEvent), cudaMemcpyDeviceToHost, s));
      SLIDE_CUDA(cudaStreamSynchronize(s));
      std::sort(h.begin(), h.end(), [](const OvfEvent& a, const OvfEvent& b) {
        return a.table != b.table ? a.table < b.table : a.id < b.id;
      });
      Mt19937 mt;
      mt.load(mt_state);
      std::vector<int2> patches;
      patches.reserve(n_ev / 4 + 16);
      for (const OvfEvent& e : h) {
        if (mt.random() * (double)e.count < (double)cap) {
          int slot = (int)(mt.random() * (double)cap);
          patches.push_back(make_int2(e.off + slot, e.id));
        }
      }
      mt.store(mt_state);
      if (!patches.empty()) {
        // later patches to the same slot win: apply in order on one thread
        // block per unique position is unnecessary -- dedupe on the host
        std::vector<int2> last_w;
        last_w.reserve(patches.size());
        std::stable_sort(patches.begin(), patches.end(), [](const int2& a, const int2& b) { return a.x < b.x; });
        for (size_t q = 0; q < patches.size(); ++q)
          if (q + 1 == patches.size() || patches[q + 1].x != patches[q].x) last_w.push_back(patches[q]);
        int2* dp = tb.patch.ensure<int2>(last_w.size());
        SLIDE_CUDA(cudaMemcpyAsync(dp, last_w.data(), last_w.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
        patch_kernel<<<grid_for((int64_t)last_w.size()), 256, 0, s>>>(dp, (int64_t)last_w.size(), vb);
        SLIDE_LAUNCH_CHECK();
        SLIDE_CUDA(cudaStreamSynchronize(s));  // host vector lifetime
      }
    }
  }
  d.dir = dir;
  d.hdir = hdir;
  d.hash_mask = hmask;
  d.bstart = bstart;
  d.blen = blen;
  d.bcount = counts;
  d.ids = vb;
  d.empty = n_runs == 0;
  d.disabled = 0;
  tb.n_items = n;
  tb.n_slots = total;
  tb.policy = policy;
  tb.built = true;
}

void tables_load(TablesHost& tb, const uint32_t* skeys, const int32_t* counts, const int32_t* starts,
                 const int32_t* lens, int64_t n_runs, const int32_t* ids, int64_t n_slots, int64_t n_items, int l,
                 int kb, int cap, cudaStream_t s) {
  uint32_t* uniq = tb.uniq.ensure<uint32_t>(std::max<int64_t>(n_runs, 1));
  int32_t* cnt = tb.counts.ensure<int32_t>(std::max<int64_t>(n_runs, 1));
  int32_t* bstart = tb.bstart.ensure<int32_t>(std::max<int64_t>(n_runs, 1));
  int32_t* blen = tb.blen.ensure<int32_t>(std::max<int64_t>(n_runs, 1));
  int32_t* vb = tb.vals_b.ensure<int32_t>(std::max<int64_t>(n_slots, 1));
  if (n_runs) {
    SLIDE_CUDA(cudaMemcpyAsync(uniq, skeys, n_runs * 4, cudaMemcpyHostToDevice, s));
    SLIDE_CUDA(cudaMemcpyAsync(cnt, counts, n_runs * 4, cudaMemcpyHostToDevice, s));
    SLIDE_CUDA(cudaMemcpyAsync(bstart, starts, n_runs * 4, cudaMemcpyHostToDevice, s));
    SLIDE_CUDA(cudaMemcpyAsync(blen, lens, n_runs * 4, cudaMemcpyHostToDevice, s));
  }
  if (n_slots) SLIDE_CUDA(cudaMemcpyAsync(vb, ids, n_slots * 4, cudaMemcpyHostToDevice, s));
  TablesDev& d = tb.dev;
  d.l = l;
  d.key_bits = kb;
  d.cap = cap;
  d.n_runs = n_runs;
  choose_dir(tb, d, l, kb, n_items, n_runs, s);
  d.run_keys = uniq;
  if (n_runs) {
    dir_kernel<<<grid_for(n_runs), 256, 0, s>>>(uniq, n_runs, d.dense_dir, const_cast<int32_t*>(d.dir),
                                                const_cast<uint64_t*>(d.hdir), d.hash_mask);
    SLIDE_LAUNCH_CHECK();
  }
  if (kb > 16) build_coarse(tb, d, l, kb, n_runs, uniq, s);
  SLIDE_CUDA(cudaStreamSynchronize(s));  // host arrays may go away
  d.bstart = bstart;
  d.blen = blen;
  d.bcount = cnt;
  d.ids = vb;
  d.empty = n_runs == 0;
  d.disabled = 0;
  tb.n_items = n_items;
  tb.built = true;
}

// ------------------------------------------------ column-sharded tables
// rank g builds its tables from its own rows (global ids
// r G + g, ascending within a bucket, like the unsharded insert order).  A
// global FIFO bucket keeps its cap highest ids (tables.py:130-145); when a
// bucket may overflow globally the ranks exchange their runs (packed below)
// and each keeps the ids at or above the bucket's cap-th highest id over all
// ranks.  Pack layout (int32): [R, S, skeys R, counts R, starts R, lens R,
// ids S] -- the runs' keys ascending, insert counts, kept tails (start, len)
// into the rank's sorted id array, which follows whole (S = its inserts).
int64_t tables_pack_size(const TablesHost& tb) { return 2 + 4 * tb.dev.n_runs + tb.n_slots; }

__global__ void pack_header_kernel(int32_t* out, int32_t r, int32_t sl) {
  out[0] = r;
  out[1] = sl;
}

void tables_pack(const TablesHost& tb, int32_t* out, cudaStream_t s) {
  const int64_t r = tb.dev.n_runs, ns = tb.n_slots;
  pack_header_kernel<<<1, 1, 0, s>>>(out, (int32_t)r, (int32_t)ns);
  SLIDE_LAUNCH_CHECK();
  if (r) {
    SLIDE_CUDA(cudaMemcpyAsync(out + 2, tb.dev.run_keys, r * 4, cudaMemcpyDeviceToDevice, s));
    SLIDE_CUDA(cudaMemcpyAsync(out + 2 + r, tb.dev.bcount, r * 4, cudaMemcpyDeviceToDevice, s));
    SLIDE_CUDA(cudaMemcpyAsync(out + 2 + 2 * r, tb.dev.bstart, r * 4, cudaMemcpyDeviceToDevice, s));
    SLIDE_CUDA(cudaMemcpyAsync(out + 2 + 3 * r, tb.dev.blen, r * 4, cudaMemcpyDeviceToDevice, s));
  }
  if (ns) SLIDE_CUDA(cudaMemcpyAsync(out + 2 + 4 * r, tb.dev.ids, ns * 4, cudaMemcpyDeviceToDevice, s));
}

constexpr int kRecWarps = 8;

// one warp per local run: the bucket's lists on every rank (<= cap ids each,
// ascending) are staged in shared memory; the threshold T = the cap-th
// highest id overall is found by bisection on the id value with warp-wide
// counts; the local run keeps its ids >= T.
__global__ void __launch_bounds__(kRecWarps * 32) reconcile_kernel(const int32_t* __restrict__ packs, int64_t stride,
                                                                   int G, int g, int cap, int64_t n_runs,
                                                                   const uint32_t* __restrict__ run_keys,
                                                                   int32_t* __restrict__ bstart,
                                                                   int32_t* __restrict__ blen,
                                                                   int32_t* __restrict__ bcount,
                                                                   const int32_t* __restrict__ ids) {
  extern __shared__ int32_t lists[];  // [kRecWarps][G * cap]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* buf = lists + (size_t)warp * G * cap;
  for (int64_t r = (int64_t)blockIdx.x * kRecWarps + warp; r < n_runs; r += (int64_t)gridDim.x * kRecWarps) {
    const uint32_t sk = run_keys[r];
    int total = 0, n = 0;
    for (int q = 0; q < G; ++q) {
      const int32_t* pk = packs + q * stride;
      const int R = pk[0];
      const uint32_t* keys = reinterpret_cast<const uint32_t*>(pk + 2);
      int start = 0, len = 0, cnt = 0;
      if (q == g) {
        start = -1;
        len = blen[r];
        cnt = bcount[r];
      } else if (lane == 0) {
        int lo = 0, hi = R;  // first key >= sk
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (keys[mid] < sk) lo = mid + 1;
          else hi = mid;
        }
        if (lo < R && keys[lo] == sk) {
          cnt = pk[2 + R + lo];
          start = pk[2 + 2 * R + lo];
          len = pk[2 + 3 * R + lo];
        }
      }
      start = __shfl_sync(0xffffffffu, start, 0);
      len = __shfl_sync(0xffffffffu, len, 0);
      cnt = __shfl_sync(0xffffffffu, cnt, 0);
      total += cnt;
      const int32_t* src = q == g ? ids + bstart[r] : pk + 2 + 4 * R + start;
      for (int j = lane; j < len; j += 32) buf[n + j] = src[j];
      n += len;
    }
    __syncwarp();
    if (total > cap) {
      // largest T with #(ids >= T) >= cap; ids are distinct and < 2^31
      int64_t lo = 0, hi = 0x7fffffff;
      while (lo < hi) {  // <= 31 rounds
        const int64_t mid = lo + ((hi - lo + 1) >> 1);
        int c = 0;
        for (int j = lane; j < n; j += 32) c += buf[j] >= mid;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (c >= cap) lo = mid;
        else hi = mid - 1;
      }
      const int32_t* own = ids + bstart[r];
      const int len = blen[r];
      int below = 0;
      for (int j = lane; j < len; j += 32) below += (int64_t)own[j] < lo;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) below += __shfl_xor_sync(0xffffffffu, below, o);
      if (lane == 0) {
        bstart[r] += below;
        blen[r] = len - below;
      }
    }
    if (lane == 0) bcount[r] = total;
    __syncwarp();
  }
}

void tables_reconcile(TablesHost& tb, const int32_t* packs, int64_t stride, int G, int g, int cap, cudaStream_t s) {
  const int64_t r = tb.dev.n_runs;
  if (r <= 0) return;
  SLIDE_CHECK((int64_t)G * cap <= 4096, kNotSupported, "sharded table reconciliation needs shard_count * cap <= 4096");
  const size_t smem = (size_t)kRecWarps * G * cap * 4;
  if (smem > 48 * 1024)
    SLIDE_CUDA(cudaFuncSetAttribute(reconcile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = (int)std::min<int64_t>(ceil_div(r, kRecWarps), (int64_t)kSms * 8);
  reconcile_kernel<<<grid, kRecWarps * 32, smem, s>>>(packs, stride, G, g, cap, r, tb.dev.run_keys,
                                                      const_cast<int32_t*>(tb.dev.bstart),
                                                      const_cast<int32_t*>(tb.dev.blen),
                                                      const_cast<int32_t*>(tb.dev.bcount), tb.dev.ids);
  SLIDE_LAUNCH_CHECK();
}

}  // namespace slide
