// Host-side native code: synthetic power-law graph generator, k-hop sampler,
// label generator. Plain C++17 with std::thread; deterministic regardless of
// the thread count (all randomness is counter-based, rng.h).
#include <stdint.h>

#include <algorithm>
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
