// Host-side native code: synthetic power-law graph generator, k-hop sampler,
// label generator. Plain C++17 with std::thread; deterministic regardless of
// the thread count (all randomness is counter-based, rng.h).
#include <stdint.h>

#include <emmintrin.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/splitgnn_b200.h"
#include "rng.h"

namespace sg {
void set_error(const std::string& msg);
}

namespace {

int pick_threads(int t) {
  if (t > 0) return t;
  unsigned h = std::thread::hardware_concurrency();
  return h ? (int)h : 1;
}

template <typename F>
void parallel_for(int64_t n, int threads, F fn) {
  threads = pick_threads(threads);
  if (n <= 0) return;
  if (threads <= 1 || n < 4096) {
    fn(0, n);
    return;
  }
  std::vector<std::thread> ts;
  const int64_t chunk = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const int64_t b = t * chunk, e = std::min<int64_t>(n, b + chunk);
    if (b >= e) break;
    ts.emplace_back([=]() { fn(b, e); });
  }
  for (auto& th : ts) th.join();
}

// ---------------------------------------------------------------- generator
struct PowerLaw {
  int64_t n;
  int32_t blocks;
  double p_local;
  uint64_t seed;
  std::vector<double> C;  // prefix sums of vertex weights, size n+1

  int64_t block_lo(int64_t b) const { return (b * n + blocks - 1) / blocks; }

  void build(double gamma, int threads) {
    C.assign(n + 1, 0.0);
    const double ex = -1.0 / (gamma - 1.0);
    // relabel: rank r_v = perm(v)+1, perm(v) = (A v + B) mod n, gcd(A, n) = 1
    uint64_t A = (sg_mix64(seed ^ 0xA5A5ull) % (uint64_t)std::max<int64_t>(n, 1)) | 1ull;
    while (std::gcd<uint64_t, uint64_t>(A, (uint64_t)n) != 1) A += 2;
    const uint64_t B = sg_mix64(seed ^ 0x5A5Aull) % (uint64_t)std::max<int64_t>(n, 1);
    std::vector<double> w(n);
    parallel_for(n, threads, [&](int64_t b, int64_t e) {
      for (int64_t v = b; v < e; ++v) {
        const uint64_t r = (uint64_t)(((unsigned __int128)A * (uint64_t)v + B) % (uint64_t)n) + 1;
        w[v] = std::pow((double)r, ex);
      }
    });
    double acc = 0.0;
    for (int64_t v = 0; v < n; ++v) {
      C[v] = acc;
      acc += w[v];
    }
    C[n] = acc;
  }

  int64_t draw(double u, int64_t lo, int64_t hi) const {
    const double t = C[lo] + u * (C[hi] - C[lo]);
    int64_t x = (int64_t)(std::upper_bound(C.begin() + lo, C.begin() + hi + 1, t) - C.begin()) - 1;
    return std::min(std::max(x, lo), hi - 1);
  }

  void edge(int64_t e, int64_t* src, int64_t* dst) const {
    const int64_t d = draw(sg_uniform53(sg_hash3(seed, (uint64_t)e, 0)), 0, n);
    const bool local = sg_uniform53(sg_hash3(seed, (uint64_t)e, 1)) < p_local;
    const double u = sg_uniform53(sg_hash3(seed, (uint64_t)e, 2));
    int64_t s;
    if (local) {
      const int64_t b = d * blocks / n;
      s = draw(u, block_lo(b), block_lo(b + 1));
    } else {
      s = draw(u, 0, n);
    }
    *src = s;
    *dst = d;
  }
};

// ---------------------------------------------------------------- sampler
struct Sampler {
  int64_t n;
  const int64_t* ro;
  const int32_t* ci;
  std::vector<int32_t> pos_of, stamp;
  int32_t gen = 0;
  std::vector<std::vector<int32_t>> layers;
  std::vector<std::vector<int32_t>> es, ed;
};

}  // namespace

extern "C" int sg_gen_powerlaw(int64_t n, int64_t m, int32_t blocks, double p_local,
                               double gamma, uint64_t seed, int32_t threads, int64_t* row_offsets,
                               int32_t* col_indices) {
  if (n <= 0 || n >= (int64_t(1) << 31) || m < 0 || blocks < 1 || gamma <= 1.0) {
    sg::set_error("gen_powerlaw: bad arguments");
    return SG_ERR_ARG;
  }
  PowerLaw g{n, blocks, p_local, seed, {}};
  g.build(gamma, threads);
  std::vector<int64_t> cnt(n, 0);
  parallel_for(m, threads, [&](int64_t b, int64_t e) {
    for (int64_t i = b; i < e; ++i) {
      int64_t s, d;
      g.edge(i, &s, &d);
      __atomic_fetch_add(&cnt[d], 1, __ATOMIC_RELAXED);
    }
  });
  row_offsets[0] = 0;
  for (int64_t v = 0; v < n; ++v) row_offsets[v + 1] = row_offsets[v] + cnt[v];
  std::vector<int64_t> cur(row_offsets, row_offsets + n);
  parallel_for(m, threads, [&](int64_t b, int64_t e) {
    for (int64_t i = b; i < e; ++i) {
      int64_t s, d;
      g.edge(i, &s, &d);
      const int64_t pos = __atomic_fetch_add(&cur[d], 1, __ATOMIC_RELAXED);
      col_indices[pos] = (int32_t)s;
    }
  });
  parallel_for(n, threads, [&](int64_t b, int64_t e) {
    for (int64_t v = b; v < e; ++v) std::sort(col_indices + row_offsets[v], col_indices + row_offsets[v + 1]);
  });
  return SG_OK;
}

extern "C" int sg_gen_labels(int64_t n, int32_t num_classes, uint64_t seed, int32_t* out) {
  if (n < 0 || num_classes < 1) {
    sg::set_error("gen_labels: bad arguments");
    return SG_ERR_ARG;
  }
  for (int64_t v = 0; v < n; ++v)
    out[v] = (int32_t)sg_bounded(sg_hash3(seed, (uint64_t)v, 7), (uint64_t)num_classes);
  return SG_OK;
}

extern "C" int sg_fill_uniform_host(float* out, int64_t rows, int32_t width, uint64_t seed,
                                    int64_t row0, const int64_t* row_ids) {
  for (int64_t r = 0; r < rows; ++r) {
    const uint64_t rid = row_ids ? (uint64_t)row_ids[r] : (uint64_t)(row0 + r);
    for (int32_t c = 0; c < width; ++c) out[r * width + c] = sg_uniform24(seed, rid, (uint64_t)c);
  }
  return SG_OK;
}

extern "C" void* sg_sampler_create(int64_t n, const int64_t* row_offsets,
                                   const int32_t* col_indices) {
  Sampler* s = new Sampler();
  s->n = n;
  s->ro = row_offsets;
  s->ci = col_indices;
  return s;
}

extern "C" void sg_sampler_destroy(void* h) { delete (Sampler*)h; }

// sample_minibatch (sampling.py:118-177) with a counter-based RNG.
extern "C" int sg_sampler_run(void* h, const int64_t* targets, int64_t n_targets,
                              const int32_t* fanouts, int32_t L, uint64_t seed, int32_t threads,
                              int64_t* nV_out, int64_t* nE_out) {
  Sampler& S = *(Sampler*)h;
  if (n_targets <= 0) {
    sg::set_error("targets must be non-empty");
    return SG_ERR_ARG;
  }
  if (L < 1 || L > SG_MAXL) {
    sg::set_error("fanouts must be non-empty");
    return SG_ERR_ARG;
  }
  if (S.pos_of.empty()) {
    S.pos_of.assign(S.n, 0);
    S.stamp.assign(S.n, 0);
  }
  S.layers.assign(L + 1, {});
  S.es.assign(L, {});
  S.ed.assign(L, {});
  auto& top = S.layers[L];
  top.resize(n_targets);
  ++S.gen;
  for (int64_t i = 0; i < n_targets; ++i) {
    const int64_t t = targets[i];
    if (t < 0 || t >= S.n) {
      sg::set_error("target id out of range");
      return SG_ERR_ARG;
    }
    if (S.stamp[t] == S.gen) {
      sg::set_error("targets must be distinct");
      return SG_ERR_ARG;
    }
    S.stamp[t] = S.gen;
    top[i] = (int32_t)t;
  }
  for (int l = L; l >= 1; --l) {
    const auto& cur = S.layers[l];
    const int64_t nc = (int64_t)cur.size();
    const int f = std::max(0, (int)fanouts[l - 1]);
    std::vector<int32_t> picks((size_t)nc * std::max(f, 1));
    std::vector<int32_t> npk(nc, 0);
    parallel_for(nc, threads, [&](int64_t b, int64_t e) {
      std::vector<int64_t> mk, mv;  // sparse swap map of the partial Fisher-Yates
      for (int64_t i = b; i < e; ++i) {
        const int32_t v = cur[i];
        const int64_t s0 = S.ro[v], m = S.ro[v + 1] - s0;
        const int64_t k = std::min<int64_t>(f, m);
        if (k <= 0) continue;
        int32_t* out = &picks[(size_t)i * f];
        int cnt = 0;
        auto accept = [&](int32_t u) {
          if (u == v) return;  // the input's own self-loop
          for (int t = 0; t < cnt; ++t)
            if (out[t] == u) return;  // parallel edge
          out[cnt++] = u;
        };
        if (k >= m) {
          for (int64_t j = 0; j < m; ++j) accept(S.ci[s0 + j]);
        } else {
          mk.clear();
          mv.clear();
          auto get = [&](int64_t x) -> int64_t {
            for (size_t t = 0; t < mk.size(); ++t)
              if (mk[t] == x) return mv[t];
            return S.ci[s0 + x];
          };
          auto set = [&](int64_t x, int64_t val) {
            for (size_t t = 0; t < mk.size(); ++t)
              if (mk[t] == x) {
                mv[t] = val;
                return;
              }
            mk.push_back(x);
            mv.push_back(val);
          };
          for (int64_t j = 0; j < k; ++j) {
            const uint64_t hsh = sg_hash3(seed, ((uint64_t)l << 40) ^ (uint64_t)i, (uint64_t)j);
            const int64_t r = j + (int64_t)sg_bounded(hsh, (uint64_t)(m - j));
            const int64_t vj = get(j), vr = get(r);
            set(r, vj);
            set(j, vr);
            accept((int32_t)vr);
          }
        }
        npk[i] = cnt;
      }
    });
    // first-seen ordering (sequential, as the reference's dict insertion order)
    ++S.gen;
    std::vector<int32_t> order(cur.begin(), cur.end());
    for (int64_t i = 0; i < nc; ++i) {
      S.stamp[cur[i]] = S.gen;
      S.pos_of[cur[i]] = (int32_t)i;
    }
    auto& src = S.es[l - 1];
    auto& dst = S.ed[l - 1];
    int64_t tot = nc;
    for (int64_t i = 0; i < nc; ++i) tot += npk[i];
    src.reserve(tot);
    dst.reserve(tot);
    for (int64_t i = 0; i < nc; ++i) {
      src.push_back((int32_t)i);
      dst.push_back((int32_t)i);
      const int32_t* pk = &picks[(size_t)i * f];
      for (int t = 0; t < npk[i]; ++t) {
        const int32_t u = pk[t];
        int32_t j;
        if (S.stamp[u] == S.gen) {
          j = S.pos_of[u];
        } else {
          j = (int32_t)order.size();
          S.stamp[u] = S.gen;
          S.pos_of[u] = j;
          order.push_back(u);
        }
        src.push_back(j);
        dst.push_back((int32_t)i);
      }
    }
    S.layers[l - 1] = std::move(order);
  }
  for (int l = 0; l <= L; ++l) nV_out[l] = (int64_t)S.layers[l].size();
  for (int l = 0; l < L; ++l) nE_out[l] = (int64_t)S.es[l].size();
  return SG_OK;
}

// sg_sampler_fetch plus the per-destination run starts of every layer
// (starts: layer 1..L back to back, |V^l| ints each; starts[i] = first edge of
// destination i in E^l -- the sampler emits each destination's edges as one
// run, destinations ascending, the self edge first, so every run is non-empty).
extern "C" int sg_sampler_fetch_starts(void* h, int32_t* V, int32_t* esrc, int32_t* edst, int32_t* starts) {
  Sampler& S = *(Sampler*)h;
  int64_t o = 0;
  for (auto& lv : S.layers) {
    std::memcpy(V + o, lv.data(), lv.size() * 4);
    o += (int64_t)lv.size();
  }
  o = 0;
  int64_t so = 0;
  for (size_t l = 0; l < S.es.size(); ++l) {
    const int64_t m = (int64_t)S.es[l].size();
    std::memcpy(esrc + o, S.es[l].data(), m * 4);
    const int32_t* d = S.ed[l].data();
    int32_t* out = edst + o;
    int32_t* st = starts + so;
    int32_t prev = -1;
    for (int64_t j = 0; j < m; ++j) {
      const int32_t v = d[j];
      out[j] = v;
      if (v != prev) {
        st[v] = (int32_t)j;
        prev = v;
      }
    }
    o += m;
    so += (int64_t)S.layers[l + 1].size();
  }
  return SG_OK;
}

extern "C" int sg_sampler_fetch(void* h, int32_t* V, int32_t* esrc, int32_t* edst) {
  Sampler& S = *(Sampler*)h;
  int64_t o = 0;
  for (auto& lv : S.layers) {
    std::memcpy(V + o, lv.data(), lv.size() * 4);
    o += (int64_t)lv.size();
  }
  o = 0;
  for (size_t l = 0; l < S.es.size(); ++l) {
    std::memcpy(esrc + o, S.es[l].data(), S.es[l].size() * 4);
    std::memcpy(edst + o, S.ed[l].data(), S.ed[l].size() * 4);
    o += (int64_t)S.es[l].size();
  }
  return SG_OK;
}

// ---------------------------------------------------------------- coarsest-level partition
// Initial partition of the coarsest level of the multilevel partitioner
// (partition.py drives the GPU levels; the contract is reference
// partition.py:186-233 + 236-270: greedy region growing, best of a few
// restarts after sequential boundary refinement, every part within cap).
// Symmetric weighted CSR (off, nbr, wt), vertex weights vw.
namespace {

struct CoarseGraph {
  int64_t n;
  const int64_t* off;
  const int32_t* nbr;
  const int32_t* wt;
  const int32_t* vw;
};

int64_t coarse_cut(const CoarseGraph& G, const std::vector<int32_t>& part) {
  int64_t c = 0;
  for (int64_t v = 0; v < G.n; ++v)
    for (int64_t j = G.off[v]; j < G.off[v + 1]; ++j)
      if (part[G.nbr[j]] != part[v]) c += G.wt[j];
  return c / 2;
}

// Grow parts 0..g-2 one at a time from a seeded start vertex, always taking the
// unassigned vertex most connected to the growing part (ties by a seeded hash);
// the last part takes the rest.
void grow(const CoarseGraph& G, int g, int64_t cap, uint64_t seed, std::vector<int32_t>& part) {
  const int64_t n = G.n;
  part.assign(n, -1);
  int64_t total = 0;
  for (int64_t v = 0; v < n; ++v) total += G.vw[v];
  std::vector<int64_t> conn(n, 0);
  std::vector<int64_t> unassigned(n);
  std::iota(unassigned.begin(), unassigned.end(), 0);
  int64_t left = total, n_left = n;
  typedef std::pair<std::pair<int64_t, uint64_t>, int64_t> Item;
  for (int p = 0; p < g - 1 && n_left > 0; ++p) {
    const int64_t target = left / (g - p);
    std::vector<Item> heap;
    std::vector<int64_t> touched;
    auto push = [&](int64_t v) {
      heap.push_back({{conn[v], sg_hash3(seed, (uint64_t)v, (uint64_t)p)}, v});
      std::push_heap(heap.begin(), heap.end());
    };
    int64_t wp = 0;
    // a seeded unassigned vertex that still fits the part (scanning on from a
    // random position); false when none does
    auto random_start = [&]() {
      int64_t k = 0;
      for (int64_t v : unassigned)
        if (part[v] < 0) unassigned[k++] = v;
      unassigned.resize(k);
      if (k == 0) return false;
      const int64_t r = (int64_t)sg_bounded(sg_hash3(seed, 0x5eedull + p, (uint64_t)k), (uint64_t)k);
      for (int64_t i = 0; i < k; ++i) {
        const int64_t v = unassigned[(r + i) % k];
        if (wp + G.vw[v] <= cap) {
          push(v);
          return true;
        }
      }
      return false;
    };
    if (!random_start()) continue;
    while (wp < target && n_left > 0) {
      if (heap.empty() && !random_start()) break;
      std::pop_heap(heap.begin(), heap.end());
      const Item it = heap.back();
      heap.pop_back();
      const int64_t v = it.second;
      if (part[v] >= 0 || it.first.first != conn[v]) continue;  // taken or stale
      if (wp + G.vw[v] > cap) continue;
      part[v] = p;
      wp += G.vw[v];
      left -= G.vw[v];
      --n_left;
      for (int64_t j = G.off[v]; j < G.off[v + 1]; ++j) {
        const int64_t x = G.nbr[j];
        if (part[x] >= 0) continue;
        if (conn[x] == 0) touched.push_back(x);
        conn[x] += G.wt[j];
        push(x);
      }
    }
    for (int64_t x : touched) conn[x] = 0;
  }
  for (int64_t v = 0; v < n; ++v)
    if (part[v] < 0) part[v] = g - 1;
}

// Sequential boundary refinement: first repair overfull parts (move the vertex
// whose move loses the least into a part with room), then passes of strictly
// positive gain moves within the cap (lowest part on ties) until none applies.
void refine_seq(const CoarseGraph& G, int g, int64_t cap, std::vector<int32_t>& part, int max_passes) {
  const int64_t n = G.n;
  std::vector<int64_t> size(g, 0);
  for (int64_t v = 0; v < n; ++v) size[part[v]] += G.vw[v];
  std::vector<int64_t> conn(g);
  auto connect = [&](int64_t v) {
    std::fill(conn.begin(), conn.end(), 0);
    for (int64_t j = G.off[v]; j < G.off[v + 1]; ++j)
      if (G.nbr[j] != v) conn[part[G.nbr[j]]] += G.wt[j];
  };
  for (int guard = 0; guard < 4 * n + 8; ++guard) {
    int a = -1;
    for (int p = 0; p < g; ++p)
      if (size[p] > cap && (a < 0 || size[p] > size[a])) a = p;
    if (a < 0) break;
    int64_t bv = -1, bgain = 0;
    int bq = -1;
    for (int64_t v = 0; v < n; ++v) {
      if (part[v] != a) continue;
      connect(v);
      for (int q = 0; q < g; ++q) {
        if (q == a || size[q] + G.vw[v] > cap) continue;
        const int64_t gain = conn[q] - conn[a];
        if (bv < 0 || gain > bgain) {
          bv = v;
          bgain = gain;
          bq = q;
        }
      }
    }
    if (bv < 0) break;  // nothing fits anywhere: leave it to the caller's check
    part[bv] = bq;
    size[a] -= G.vw[bv];
    size[bq] += G.vw[bv];
  }
  for (int pass = 0; pass < max_passes; ++pass) {
    int64_t moved = 0;
    for (int64_t v = 0; v < n; ++v) {
      connect(v);
      const int a = part[v];
      int best = -1;
      int64_t bgain = 0;
      for (int q = 0; q < g; ++q) {
        if (q == a || size[q] + G.vw[v] > cap) continue;
        const int64_t gain = conn[q] - conn[a];
        if (gain > bgain) {
          bgain = gain;
          best = q;
        }
      }
      if (best >= 0) {
        part[v] = best;
        size[a] -= G.vw[v];
        size[best] += G.vw[v];
        ++moved;
      }
    }
    if (!moved) break;
  }
}

}  // namespace

extern "C" int sg_partition_coarse_host(int64_t n, const int64_t* off, const int32_t* nbr, const int32_t* wt,
                                        const int32_t* vw, int32_t g, int64_t cap, uint64_t seed,
                                        int32_t restarts, int32_t* part_out, int64_t* cut_out) {
  if (n < 0 || g < 1 || (n > 0 && (!off || !nbr || !wt || !vw)) || !part_out || !cut_out) {
    sg::set_error("partition_coarse_host: bad argument");
    return SG_ERR_ARG;
  }
  const CoarseGraph G{n, off, nbr, wt, vw};
  std::vector<int32_t> part, best;
  int64_t best_cut = -1;
  bool best_ok = false;
  for (int r = 0; r < std::max(1, (int)restarts); ++r) {
    grow(G, g, cap, sg_hash3(seed, 0xC0A55ull, (uint64_t)r), part);
    refine_seq(G, g, cap, part, 10);
    std::vector<int64_t> size(g, 0);
    for (int64_t v = 0; v < n; ++v) size[part[v]] += vw[v];
    const bool ok = *std::max_element(size.begin(), size.end()) <= cap;
    const int64_t cut = coarse_cut(G, part);
    if (best_cut < 0 || (ok && !best_ok) || (ok == best_ok && cut < best_cut)) {
      best = part;
      best_cut = cut;
      best_ok = ok;
    }
  }
  std::memcpy(part_out, best.data(), sizeof(int32_t) * n);
  *cut_out = best_cut;
  return SG_OK;
}

// Sequential boundary refinement of one level (partition.py:236-270 semantics:
// overfull parts repaired first, then passes of strictly positive gain moves
// within the cap, ascending vertex id, lowest part on ties). The multilevel
// driver runs it on the levels small enough for one core; larger levels are
// refined by the parallel GPU rounds (sg_partition_round).
extern "C" int sg_partition_refine_host(int64_t n, const int64_t* off, const int32_t* nbr, const int32_t* wt,
                                        const int32_t* vw, int32_t g, int64_t cap, int32_t max_passes,
                                        int32_t* part, int64_t* cut_out) {
  if (n < 0 || g < 1 || (n > 0 && (!off || !nbr || !wt || !vw || !part)) || !cut_out) {
    sg::set_error("partition_refine_host: bad argument");
    return SG_ERR_ARG;
  }
  const CoarseGraph G{n, off, nbr, wt, vw};
  std::vector<int32_t> p(part, part + n);
  refine_seq(G, g, cap, p, max_passes);
  std::memcpy(part, p.data(), sizeof(int32_t) * n);
  *cut_out = coarse_cut(G, p);
  return SG_OK;
}

// ---------------------------------------------------------------- sample packing
// split_minibatch's host side (scheduler.py:164 entry): the sample's arrays
// (V^0..V^L, then E^l sources, then E^l destinations; int32 or int64 each)
// copied as int32 into one pinned buffer at the given word offsets, after a
// header of the sizes as int64 [nV_0..nV_L, nE_1..nE_L]. The copy is split
// evenly over `threads` host threads (it is a few MB per C2 sample).
extern "C" int sg_pack_sample(int32_t* out, int32_t L, const int64_t* sizes, const int64_t* dst_off,
                              const void* const* src, const int32_t* elem_bytes, int32_t threads,
                              int64_t* vrange) {
  if (!out || L < 1 || !sizes || !dst_off || !src || !elem_bytes) {
    sg::set_error("pack_sample: bad argument");
    return SG_ERR_ARG;
  }
  const int narr = 3 * L + 1;
  std::memcpy(out, sizes, sizeof(int64_t) * (2 * L + 1));
  std::vector<int64_t> len(narr), start(narr + 1, 0);
  for (int i = 0; i < narr; ++i) {
    len[i] = i <= L ? sizes[i] : sizes[L + 1 + (i - L - 1) % L];
    if (elem_bytes[i] != 4 && elem_bytes[i] != 8 && len[i] > 0) {
      sg::set_error("pack_sample: element size must be 4 or 8");
      return SG_ERR_ARG;
    }
    start[i + 1] = start[i] + len[i];
  }
  const int64_t total = start[narr];
  // non-temporal stores unless SG_PACK_NT=0: right after a cached multi-core
  // write the pinned buffer's H2D copy measured ~7 GB/s against ~48 GB/s
  static const bool nt = [] {
    const char* e = std::getenv("SG_PACK_NT");
    return !(e && e[0] == '0');
  }();
  std::vector<int64_t> vmin(64, INT64_MAX), vmax(64, INT64_MIN);  // per thread, over V^0..V^L
  auto copy_range = [&](int64_t a, int64_t b, int tix) {  // global element range [a, b)
    int i = (int)(std::upper_bound(start.begin(), start.end(), a) - start.begin()) - 1;
    while (a < b && i < narr) {
      const int64_t e = std::min(b, start[i + 1]);
      if (e > a) {
        const int64_t o = a - start[i], k = e - a;
        int32_t* dst = out + dst_off[i] + o;
        if (i <= L) {  // vertex ids: also their range (split_minibatch's validation)
          int64_t lo = vmin[tix], hi = vmax[tix];
          for (int64_t j = 0; j < k; ++j) {
            const int64_t v = elem_bytes[i] == 4 ? (int64_t)((const int32_t*)src[i])[o + j]
                                                 : ((const int64_t*)src[i])[o + j];
            lo = std::min(lo, v);
            hi = std::max(hi, v);
            if (nt) _mm_stream_si32(dst + j, (int32_t)v);
            else dst[j] = (int32_t)v;
          }
          vmin[tix] = lo;
          vmax[tix] = hi;
        } else if (elem_bytes[i] == 4) {
          const int32_t* s = (const int32_t*)src[i] + o;
          if (nt) {  // streaming stores: the DMA engine reads the buffer next, not a CPU
            int64_t j = 0;
            for (; j < k && ((uintptr_t)(dst + j) & 15); ++j) _mm_stream_si32(dst + j, s[j]);
            for (; j + 4 <= k; j += 4)
              _mm_stream_si128((__m128i*)(dst + j), _mm_loadu_si128((const __m128i*)(s + j)));
            for (; j < k; ++j) _mm_stream_si32(dst + j, s[j]);
          } else {
            std::memcpy(dst, s, 4 * k);
          }
        } else {
          const int64_t* s = (const int64_t*)src[i] + o;
          if (nt) {
            for (int64_t j = 0; j < k; ++j) _mm_stream_si32(dst + j, (int32_t)s[j]);
          } else {
            for (int64_t j = 0; j < k; ++j) dst[j] = (int32_t)s[j];
          }
        }
      }
      a = e;
      ++i;
    }
    if (nt) _mm_sfence();
  };
  static const int env_threads = [] {
    const char* e = std::getenv("SG_PACK_THREADS");
    return e ? std::atoi(e) : 0;
  }();
  if (env_threads > 0) threads = env_threads;
  const int T = std::max(1, std::min<int>(pick_threads(threads), (int)(total / (1 << 16)) + 1));
  const int TT = std::min(T, 64);
  if (TT == 1) {
    copy_range(0, total, 0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < TT; ++t) pool.emplace_back(copy_range, total * t / TT, total * (t + 1) / TT, t);
    for (auto& th : pool) th.join();
  }
  if (vrange) {
    vrange[0] = *std::min_element(vmin.begin(), vmin.end());
    vrange[1] = *std::max_element(vmax.begin(), vmax.end());
  }
  return SG_OK;
}

// SplitExecutor.run / allreduce_and_step on host ModelParams (engine.py:95-117,
// 633-647): the k parameter arrays (contiguous, fp64 or fp32: elem_bytes 8 / 4)
// flattened to fp32 in order -- the upload snapshot.
extern "C" int sg_host_params_gather(int32_t k, const void* const* ptrs, const int64_t* sizes,
                                     const int32_t* elem_bytes, float* out) {
  if (k < 0 || (k > 0 && (!ptrs || !sizes || !elem_bytes || !out))) {
    sg::set_error("host_params_gather: bad argument");
    return SG_ERR_ARG;
  }
  for (int32_t i = 0; i < k; ++i) {
    const int64_t m = sizes[i];
    if (elem_bytes[i] == 8) {
      const double* s = (const double*)ptrs[i];
      for (int64_t j = 0; j < m; ++j) out[j] = (float)s[j];
    } else if (elem_bytes[i] == 4) {
      std::memcpy(out, ptrs[i], 4 * m);
    } else {
      sg::set_error("host_params_gather: element size must be 4 or 8");
      return SG_ERR_ARG;
    }
    out += m;
  }
  return SG_OK;
}

// allreduce_and_step's host side for gradients already on the host: when the
// parameters still equal `snapshot` (the values the step ran with),
// total = the g flat gradients summed in device order (fp32), and every
// parameter p <- fp32(p - scale * total) with the product formed exactly (in
// fp64) and rounded once, as the device kernel's fused multiply-add; written
// back into the arrays in their own element type. *applied = 0 (nothing
// written) when the parameters changed since the snapshot.
extern "C" int sg_host_sum_sgd(int32_t k, void* const* ptrs, const int64_t* sizes, const int32_t* elem_bytes,
                               const float* snapshot, const float* const* grads, int32_t g, int64_t n,
                               float scale, float* total_out, int32_t* applied) {
  if (k < 0 || g < 1 || n < 0 || !grads || !total_out || !applied || (k > 0 && (!ptrs || !sizes || !elem_bytes))) {
    sg::set_error("host_sum_sgd: bad argument");
    return SG_ERR_ARG;
  }
  int64_t tot = 0;
  for (int32_t i = 0; i < k; ++i) tot += sizes[i];
  if (tot != n) {
    sg::set_error("host_sum_sgd: parameter sizes do not add up to n");
    return SG_ERR_ARG;
  }
  *applied = 0;
  if (snapshot) {  // unchanged since the run? (bit compare, branch-free: vectorised)
    auto bits = [](float x) {
      uint32_t u;
      std::memcpy(&u, &x, 4);
      return u;
    };
    int64_t o = 0;
    for (int32_t i = 0; i < k; ++i) {
      const int64_t m = sizes[i];
      uint32_t diff = 0;
      if (elem_bytes[i] == 8) {
        const double* s = (const double*)ptrs[i];
        for (int64_t j = 0; j < m; ++j) diff |= bits((float)s[j]) ^ bits(snapshot[o + j]);
      } else {
        const float* s = (const float*)ptrs[i];
        for (int64_t j = 0; j < m; ++j) diff |= bits(s[j]) ^ bits(snapshot[o + j]);
      }
      if (diff) return SG_OK;
      o += m;
    }
  }
  for (int64_t j = 0; j < n; ++j) {
    float t = grads[0][j];
    for (int32_t d = 1; d < g; ++d) t += grads[d][j];
    total_out[j] = t;
  }
  const double sc = (double)scale;
  int64_t o = 0;
  for (int32_t i = 0; i < k; ++i) {
    const int64_t m = sizes[i];
    if (elem_bytes[i] == 8) {
      double* s = (double*)ptrs[i];
      for (int64_t j = 0; j < m; ++j) s[j] = (double)(float)((double)(float)s[j] - sc * (double)total_out[o + j]);
    } else {
      float* s = (float*)ptrs[i];
      for (int64_t j = 0; j < m; ++j) s[j] = (float)((double)s[j] - sc * (double)total_out[o + j]);
    }
    o += m;
  }
  *applied = 1;
  return SG_OK;
}
