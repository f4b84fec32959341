// hanf_host.cpp -- host side of libhanf.so: CSR construction, synthetic graph
// generators, HBG1 cache I/O and the N(t) statistics.
//
// None of this is on the per-iteration hot path; it feeds the engine
// (graph.hpp:23-229 surface) and post-processes its output (stats.hpp:33-77).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <functional>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/hanf.h"
#include "hanf_graph_internal.h"
#include "hanf_rng.h"

namespace {

hanf_status fail(hanf_status st, const std::string& msg) {
  hanf_host_detail::set_error(msg);
  return st;
}

unsigned worker_count() {
  const unsigned h = std::thread::hardware_concurrency();
  return h == 0 ? 1 : (h > 64 ? 64 : h);
}

// Runs fn(begin, end) over [0, total) split into contiguous ranges.
void parallel_for(uint64_t total, const std::function<void(uint64_t, uint64_t)>& fn,
                  uint64_t min_grain = 1 << 16) {
  unsigned t = worker_count();
  if (total < min_grain * 2 || t == 1) {
    fn(0, total);
    return;
  }
  const uint64_t parts = std::min<uint64_t>(t, (total + min_grain - 1) / min_grain);
  std::vector<std::thread> pool;
  for (uint64_t p = 0; p < parts; ++p) {
    const uint64_t b = total * p / parts, e = total * (p + 1) / parts;
    pool.emplace_back([&fn, b, e] { fn(b, e); });
  }
  for (auto& th : pool) th.join();
}

// hash.hpp:8-15 / 27-55 (the reference's own mixers, used so that the
// reference fixtures gen_uniform_random / gen_clique_path are reproduced
// bit for bit).
using hanf_rng::mix64;
struct SplitMix64 {
  uint64_t state;
  uint64_t next() {
    state += 0x9e3779b97f4a7c15ULL;
    uint64_t z = state;
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return z;
  }
  uint64_t next_below(uint64_t bound) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(next()) * bound) >> 64);
  }
  double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

using hanf_rng::Feistel;
using hanf_rng::hash3;
using hanf_rng::u01;

// Graph::from_edges (graph.hpp:29-44): ids < n checked; rows sorted and
// deduplicated.  Parallel counting sort by source, then per-row sort.
hanf_status build_csr(uint64_t n, const uint32_t* src, const uint32_t* dst, uint64_t count,
                      bool drop_self_loops, hanf_graph** out) {
  std::atomic<bool> bad{false};
  parallel_for(count, [&](uint64_t b, uint64_t e) {
    for (uint64_t i = b; i < e; ++i)
      if (src[i] >= n || dst[i] >= n) bad = true;
  });
  if (bad) return fail(HANF_INVALID_ARGUMENT, "arc endpoint out of range");
  hanf_graph* g = new (std::nothrow) hanf_graph();
  if (!g) return fail(HANF_OUT_OF_MEMORY, "graph allocation failed");
  try {
    g->n = n;
    // counting sort by source, parallel: atomic row counts, prefix sum,
    // atomic row cursors (the order inside a row does not matter, rows are
    // sorted next)
    std::vector<uint64_t> deg(n + 1, 0);
    parallel_for(count, [&](uint64_t b, uint64_t e) {
      for (uint64_t i = b; i < e; ++i)
        if (!(drop_self_loops && src[i] == dst[i]))
          std::atomic_ref<uint64_t>(deg[src[i] + 1]).fetch_add(1, std::memory_order_relaxed);
    });
    for (uint64_t v = 0; v < n; ++v) deg[v + 1] += deg[v];
    std::vector<uint32_t> tmp(deg[n]);
    {
      std::vector<uint64_t> cursor(deg.begin(), deg.end() - 1);
      parallel_for(count, [&](uint64_t b, uint64_t e) {
        for (uint64_t i = b; i < e; ++i)
          if (!(drop_self_loops && src[i] == dst[i])) {
            const uint64_t pos =
                std::atomic_ref<uint64_t>(cursor[src[i]]).fetch_add(1, std::memory_order_relaxed);
            tmp[pos] = dst[i];
          }
      });
    }
    // sort + unique each row, compute new degrees
    std::vector<uint64_t> newdeg(n + 1, 0);
    parallel_for(n, [&](uint64_t b, uint64_t e) {
      for (uint64_t v = b; v < e; ++v) {
        uint32_t* first = tmp.data() + deg[v];
        uint32_t* last = tmp.data() + deg[v + 1];
        std::sort(first, last);
        newdeg[v + 1] = static_cast<uint64_t>(std::unique(first, last) - first);
      }
    }, 1 << 12);
    g->offsets.assign(n + 1, 0);
    for (uint64_t v = 0; v < n; ++v) g->offsets[v + 1] = g->offsets[v] + newdeg[v + 1];
    g->succ.resize(g->offsets[n]);
    parallel_for(n, [&](uint64_t b, uint64_t e) {
      for (uint64_t v = b; v < e; ++v)
        std::memcpy(g->succ.data() + g->offsets[v], tmp.data() + deg[v],
                    sizeof(uint32_t) * newdeg[v + 1]);
    }, 1 << 12);
  } catch (const std::bad_alloc&) {
    delete g;
    return fail(HANF_OUT_OF_MEMORY, "graph allocation failed");
  }
  *out = g;
  return HANF_OK;
}

}  // namespace

extern "C" {

hanf_status hanf_graph_from_edges(uint64_t n, const uint32_t* src, const uint32_t* dst,
                                  uint64_t count, hanf_graph** out) {
  if (!out || (count && (!src || !dst))) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (n > (1ull << 32)) return fail(HANF_INVALID_ARGUMENT, "graph too large for 32-bit node ids");
  return build_csr(n, src, dst, count, false, out);
}

// graph.hpp:262-285, same RNG stream as the reference.
hanf_status hanf_gen_uniform_random(uint64_t n, double d, uint64_t seed, hanf_graph** out) {
  if (!out) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (n < 1) return fail(HANF_INVALID_ARGUMENT, "random graph needs n >= 1");
  if (n > 0xffffffffull) return fail(HANF_INVALID_ARGUMENT, "graph too large for 32-bit node ids");
  const uint64_t deg = static_cast<uint64_t>(std::llround(d));
  if (d < 0 || deg >= n) return fail(HANF_INVALID_ARGUMENT, "average degree must satisfy 0 <= d < n");
  SplitMix64 rng{mix64(seed ^ 0x5eedULL)};
  std::vector<uint32_t> src, dst, picks;
  src.reserve(n * deg);
  dst.reserve(n * deg);
  for (uint64_t v = 0; v < n; ++v) {
    picks.clear();
    while (picks.size() < deg) {
      const auto w = static_cast<uint32_t>(rng.next_below(n));
      if (std::find(picks.begin(), picks.end(), w) == picks.end()) picks.push_back(w);
    }
    for (uint32_t w : picks) {
      src.push_back(static_cast<uint32_t>(v));
      dst.push_back(w);
    }
  }
  return build_csr(n, src.data(), dst.data(), src.size(), false, out);
}

// graph.hpp:238-258
hanf_status hanf_gen_clique_path(uint64_t k, uint64_t l, hanf_graph** out) {
  if (!out) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (k < 1 || l < 1) return fail(HANF_INVALID_ARGUMENT, "clique-path needs k,l >= 1");
  const uint64_t n = 2 * k + l;
  if (n > 0xffffffffull) return fail(HANF_INVALID_ARGUMENT, "graph too large for 32-bit node ids");
  std::vector<uint32_t> src, dst;
  auto arc = [&](uint64_t a, uint64_t b) {
    src.push_back(static_cast<uint32_t>(a));
    dst.push_back(static_cast<uint32_t>(b));
  };
  for (uint64_t a = 0; a < k; ++a)
    for (uint64_t b = 0; b < k; ++b)
      if (a != b) arc(a, b);
  for (uint64_t a = 0; a < k; ++a) arc(a, k);
  for (uint64_t i = 0; i + 1 < l; ++i) arc(k + i, k + i + 1);
  for (uint64_t b = 0; b < k; ++b) arc(k + l - 1, k + l + b);
  for (uint64_t a = 0; a < k; ++a)
    for (uint64_t b = 0; b < k; ++b)
      if (a != b) arc(k + l + a, k + l + b);
  return build_csr(n, src.data(), dst.data(), src.size(), false, out);
}

// Config 1: directed G(n, p), p = mean_degree / (n - 1), no self-loops.
// Row v is drawn independently by geometric skipping over the n - 1
// candidate targets with the counter-based stream (seed, v).
hanf_status hanf_gen_erdos_renyi(uint64_t n, double mean_degree, uint64_t seed, hanf_graph** out) {
  if (!out) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (n < 2 || n > 0xffffffffull) return fail(HANF_INVALID_ARGUMENT, "G(n,p) needs 2 <= n < 2^32");
  const double p = mean_degree / static_cast<double>(n - 1);
  if (!(p > 0.0 && p < 1.0)) return fail(HANF_INVALID_ARGUMENT, "G(n,p) needs 0 < p < 1");
  hanf_graph* g = new (std::nothrow) hanf_graph();
  if (!g) return fail(HANF_OUT_OF_MEMORY, "graph allocation failed");
  g->n = n;
  const double lq = std::log1p(-p);
  std::vector<std::vector<uint32_t>> rows(n);
  parallel_for(n, [&](uint64_t b, uint64_t e) {
    for (uint64_t v = b; v < e; ++v) {
      uint64_t k = 0;
      int64_t x = -1;  // position in the n-1 candidates (self excluded)
      for (;;) {
        const double u = u01(hash3(seed, v, k++));
        const double skip = std::floor(std::log1p(-u) / lq);
        x += 1 + static_cast<int64_t>(skip);
        if (skip >= static_cast<double>(n) || x >= static_cast<int64_t>(n - 1)) break;
        const uint64_t w = static_cast<uint64_t>(x) < v ? static_cast<uint64_t>(x) : static_cast<uint64_t>(x) + 1;
        rows[v].push_back(static_cast<uint32_t>(w));
      }
    }
  }, 1 << 10);
  g->offsets.assign(n + 1, 0);
  for (uint64_t v = 0; v < n; ++v) g->offsets[v + 1] = g->offsets[v] + rows[v].size();
  g->succ.resize(g->offsets[n]);
  for (uint64_t v = 0; v < n; ++v)
    std::copy(rows[v].begin(), rows[v].end(), g->succ.begin() + g->offsets[v]);
  *out = g;
  return HANF_OK;
}

// Configs 2 and 5: R-MAT(a, b, c, d = 1-a-b-c), 2^scale nodes,
// edge_factor * 2^scale draws; self-loops and duplicates removed; node ids
// permuted by a seeded Feistel bijection.  Draw i descends `scale` levels;
// each level consumes 16 bits of the stream (seed, i).
hanf_status hanf_gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                          uint64_t seed, uint64_t permute_seed, hanf_graph** out) {
  if (!out) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (scale < 2 || scale > 32) return fail(HANF_INVALID_ARGUMENT, "R-MAT scale must be in [2, 32]");
  if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0))
    return fail(HANF_INVALID_ARGUMENT, "R-MAT probabilities must be non-negative, a+b+c <= 1");
  const uint64_t n = 1ull << scale;
  const uint64_t draws = n * edge_factor;
  const uint32_t ta = static_cast<uint32_t>(a * 65536.0);
  const uint32_t tb = static_cast<uint32_t>((a + b) * 65536.0);
  const uint32_t tc = static_cast<uint32_t>((a + b + c) * 65536.0);
  const Feistel perm(scale, permute_seed);
  std::vector<uint32_t> src, dst;
  try {
    src.resize(draws);
    dst.resize(draws);
  } catch (const std::bad_alloc&) {
    return fail(HANF_OUT_OF_MEMORY, "edge buffer allocation failed");
  }
  parallel_for(draws, [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) {
      uint64_t u = 0, v = 0;
      hanf_rng::rmat_draw(seed, i, scale, ta, tb, tc, &u, &v);
      src[i] = static_cast<uint32_t>(perm(u));
      dst[i] = static_cast<uint32_t>(perm(v));
    }
  });
  return build_csr(n, src.data(), dst.data(), draws, true, out);
}

// Config 3: web-like copying model.  Node v draws an out-degree from a
// power law P(d) ~ d^-exponent on [1, max_degree] (continuous Pareto,
// x_min solved for the requested mean, rounded), and a prototype p_v
// uniform within +-window of v.  Arc j copies the prototype's j-th base
// successor with probability copy_prob, else it is a uniform target within
// +-window of v; the base successor of x is uniform within +-window of x.
// Self-loops and duplicates are removed.
hanf_status hanf_gen_copying(uint64_t n, double exponent, double mean_degree, uint64_t max_degree,
                             double copy_prob, uint64_t window, uint64_t seed, hanf_graph** out) {
  if (!out) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (n < 2 || n > 0xffffffffull) return fail(HANF_INVALID_ARGUMENT, "copying model needs 2 <= n < 2^32");
  if (!(exponent > 2.0) || !(mean_degree >= 1.0) || max_degree < 1)
    return fail(HANF_INVALID_ARGUMENT, "copying model needs exponent > 2, mean >= 1, max >= 1");
  const double al = exponent - 1.0;  // Pareto tail index
  const double xmax = static_cast<double>(max_degree);
  auto mean_of = [&](double xmin) {
    // mean of the truncated Pareto(xmin, al) on [xmin, xmax]
    const double r = xmin / xmax;
    return xmin * al / (al - 1.0) * (1.0 - std::pow(r, al - 1.0)) / (1.0 - std::pow(r, al));
  };
  double lo = 1e-6, hi = xmax;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    (mean_of(mid) < mean_degree ? lo : hi) = mid;
  }
  const double xmin = 0.5 * (lo + hi);
  const double r = xmin / xmax;
  const double tail = 1.0 - std::pow(r, al);
  const int64_t w = static_cast<int64_t>(window);
  auto clampi = [&](int64_t x) {
    return static_cast<uint32_t>(x < 0 ? 0 : (x >= static_cast<int64_t>(n) ? static_cast<int64_t>(n) - 1 : x));
  };
  auto window_pick = [&](uint64_t x, uint64_t key, uint64_t k) {
    const uint64_t h = hash3(seed ^ 0xc0ffee, key, k);
    const int64_t off = static_cast<int64_t>(h % static_cast<uint64_t>(2 * w + 1)) - w;
    return clampi(static_cast<int64_t>(x) + off);
  };
  std::vector<uint64_t> deg(n + 1, 0);
  parallel_for(n, [&](uint64_t b, uint64_t e) {
    for (uint64_t v = b; v < e; ++v) {
      const double u = u01(hash3(seed, v, 0));
      const double x = xmin * std::pow(1.0 - u * tail, -1.0 / al);  // inverse CDF
      uint64_t d = static_cast<uint64_t>(std::llround(x));
      deg[v + 1] = std::min<uint64_t>(std::max<uint64_t>(d, 1), max_degree);
    }
  });
  for (uint64_t v = 0; v < n; ++v) deg[v + 1] += deg[v];
  std::vector<uint32_t> src, dst;
  try {
    src.resize(deg[n]);
    dst.resize(deg[n]);
  } catch (const std::bad_alloc&) {
    return fail(HANF_OUT_OF_MEMORY, "edge buffer allocation failed");
  }
  parallel_for(n, [&](uint64_t b, uint64_t e) {
    for (uint64_t v = b; v < e; ++v) {
      const uint32_t proto = window_pick(v, v, 1ull << 40);
      for (uint64_t i = deg[v], j = 0; i < deg[v + 1]; ++i, ++j) {
        src[i] = static_cast<uint32_t>(v);
        const double u = u01(hash3(seed, v, 1 + j));
        dst[i] = u < copy_prob ? window_pick(proto, proto, j) : window_pick(v, v, (1ull << 41) + j);
      }
    }
  }, 1 << 12);
  return build_csr(n, src.data(), dst.data(), deg[n], true, out);
}

// Config 4: Barabasi-Albert preferential attachment (m edges per new node,
// seeded with an (m+1)-clique), generated in parallel with the
// Sanders-Schulz recurrence: edge i (source node i/m + m + 1) picks position
// r uniform in [0, 2i'); even r -> source of edge r/2, odd r -> target of
// edge (r-1)/2, resolved by following strictly decreasing edge indices.
// Arcs are stored in both directions; self-loops and duplicates removed;
// node ids permuted by a seeded Feistel bijection when n is a power of two.
hanf_status hanf_gen_barabasi_albert(uint64_t n, uint32_t m, uint64_t seed, uint64_t permute_seed,
                                     hanf_graph** out) {
  if (!out) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (m < 1 || n <= m + 1 || n > 0xffffffffull)
    return fail(HANF_INVALID_ARGUMENT, "Barabasi-Albert needs 1 <= m < n - 1, n < 2^32");
  const uint64_t m0 = m + 1;
  const uint64_t clique = m0 * (m0 - 1) / 2;        // undirected seed edges
  const uint64_t grown = (n - m0) * m;
  const uint64_t edges = clique + grown;
  std::vector<uint32_t> es, et;
  try {
    es.resize(edges);
    et.resize(edges);
  } catch (const std::bad_alloc&) {
    return fail(HANF_OUT_OF_MEMORY, "edge buffer allocation failed");
  }
  {
    uint64_t k = 0;
    for (uint64_t a = 0; a < m0; ++a)
      for (uint64_t b = a + 1; b < m0; ++b, ++k) {
        es[k] = static_cast<uint32_t>(b);
        et[k] = static_cast<uint32_t>(a);
      }
  }
  // target of edge i (i >= clique): uniform endpoint among edges [0, i)
  auto resolve = [&](uint64_t i) -> uint32_t {
    uint64_t cur = i, k = 0;
    for (;;) {
      const uint64_t r = hash3(seed, cur, k++) % (2 * cur);
      const uint64_t e = r >> 1;
      if ((r & 1) == 0) {
        return e < clique ? es[e] : static_cast<uint32_t>((e - clique) / m + m0);
      }
      if (e < clique) return et[e];
      cur = e;  // target of an earlier grown edge: recurse
      k = 0;
    }
  };
  parallel_for(grown, [&](uint64_t b, uint64_t e) {
    for (uint64_t j = b; j < e; ++j) {
      const uint64_t i = clique + j;
      es[i] = static_cast<uint32_t>(j / m + m0);
      et[i] = resolve(i);
    }
  });
  const bool pow2 = (n & (n - 1)) == 0 && n >= 4;
  uint32_t bits = 0;
  while ((1ull << bits) < n) ++bits;
  const Feistel perm(bits, permute_seed);
  std::vector<uint32_t> src(2 * edges), dst(2 * edges);
  parallel_for(edges, [&](uint64_t b, uint64_t e) {
    for (uint64_t i = b; i < e; ++i) {
      const uint32_t u = pow2 ? static_cast<uint32_t>(perm(es[i])) : es[i];
      const uint32_t v = pow2 ? static_cast<uint32_t>(perm(et[i])) : et[i];
      src[2 * i] = u;
      dst[2 * i] = v;
      src[2 * i + 1] = v;
      dst[2 * i + 1] = u;
    }
  });
  es.clear();
  es.shrink_to_fit();
  et.clear();
  et.shrink_to_fit();
  return build_csr(n, src.data(), dst.data(), src.size(), true, out);
}

// graph.hpp:72-84
hanf_status hanf_graph_transpose(const hanf_graph* g, hanf_graph** out) {
  if (!g || !out) return fail(HANF_INVALID_ARGUMENT, "null argument");
  hanf_graph* t = new (std::nothrow) hanf_graph();
  if (!t) return fail(HANF_OUT_OF_MEMORY, "graph allocation failed");
  t->n = g->n;
  t->offsets.assign(g->n + 1, 0);
  t->succ.resize(g->succ.size());
  for (uint32_t w : g->succ) ++t->offsets[w + 1];
  for (uint64_t v = 0; v < g->n; ++v) t->offsets[v + 1] += t->offsets[v];
  std::vector<uint64_t> cursor(t->offsets.begin(), t->offsets.end() - 1);
  for (uint64_t v = 0; v < g->n; ++v)
    for (uint64_t i = g->offsets[v]; i < g->offsets[v + 1]; ++i)
      t->succ[cursor[g->succ[i]]++] = static_cast<uint32_t>(v);
  *out = t;
  return HANF_OK;
}

// HBG1: "HBG1", u64 n, u64 a, (n+1) u64 offsets, a u32 successors, LE
// (graph.hpp:145-218, FORMATS.md:13-23).  Hosts here are little-endian.
hanf_status hanf_graph_save_csr(const hanf_graph* g, const char* path) {
  if (!g || !path) return fail(HANF_INVALID_ARGUMENT, "null argument");
  std::ofstream out(path, std::ios::binary);
  if (!out) return fail(HANF_IO_ERROR, std::string("cannot open for writing: ") + path);
  const uint64_t a = g->succ.size();
  out.write("HBG1", 4);
  out.write(reinterpret_cast<const char*>(&g->n), 8);
  out.write(reinterpret_cast<const char*>(&a), 8);
  out.write(reinterpret_cast<const char*>(g->offsets.data()), 8 * g->offsets.size());
  out.write(reinterpret_cast<const char*>(g->succ.data()), 4 * a);
  if (!out) return fail(HANF_IO_ERROR, std::string("write failed: ") + path);
  return HANF_OK;
}

hanf_status hanf_graph_load_csr(const char* path, hanf_graph** out) {
  if (!path || !out) return fail(HANF_INVALID_ARGUMENT, "null argument");
  std::ifstream in(path, std::ios::binary);
  if (!in) return fail(HANF_IO_ERROR, std::string("cannot open: ") + path);
  char magic[4] = {};
  in.read(magic, 4);
  if (!in || std::memcmp(magic, "HBG1", 4) != 0)
    return fail(HANF_PARSE_ERROR, std::string(path) + ": bad graph cache magic");
  uint64_t n = 0, a = 0;
  in.read(reinterpret_cast<char*>(&n), 8);
  in.read(reinterpret_cast<char*>(&a), 8);
  if (!in || n > (1ull << 32))
    return fail(HANF_PARSE_ERROR, std::string(path) + ": truncated or inconsistent cache");
  hanf_graph* g = new (std::nothrow) hanf_graph();
  if (!g) return fail(HANF_OUT_OF_MEMORY, "graph allocation failed");
  try {
    g->n = n;
    g->offsets.resize(n + 1);
    in.read(reinterpret_cast<char*>(g->offsets.data()), 8 * (n + 1));
    g->succ.resize(a);
    in.read(reinterpret_cast<char*>(g->succ.data()), 4 * a);
  } catch (const std::bad_alloc&) {
    delete g;
    return fail(HANF_OUT_OF_MEMORY, "graph allocation failed");
  }
  bool ok = static_cast<bool>(in) && g->offsets[0] == 0 && g->offsets[n] == a;
  for (uint64_t v = 0; ok && v < n; ++v) ok = g->offsets[v] <= g->offsets[v + 1];
  for (uint64_t i = 0; ok && i < a; ++i) ok = g->succ[i] < n;
  if (!ok) {
    delete g;
    return fail(HANF_PARSE_ERROR, std::string(path) + ": truncated or inconsistent cache");
  }
  // load_csr rebuilds through from_edges (graph.hpp:207-217): rows sorted,
  // duplicates collapsed
  for (uint64_t v = 0; v < n; ++v) {
    auto first = g->succ.begin() + g->offsets[v], last = g->succ.begin() + g->offsets[v + 1];
    if (!std::is_sorted(first, last) || std::adjacent_find(first, last) != last) {
      std::vector<uint32_t> src(a), dst(g->succ.begin(), g->succ.end());
      for (uint64_t u = 0; u < n; ++u)
        for (uint64_t i = g->offsets[u]; i < g->offsets[u + 1]; ++i) src[i] = static_cast<uint32_t>(u);
      delete g;
      return build_csr(n, src.data(), dst.data(), a, false, out);
    }
  }
  *out = g;
  return HANF_OK;
}

hanf_status hanf_graph_view_of(const hanf_graph* g, hanf_graph_view* view) {
  if (!g || !view) return fail(HANF_INVALID_ARGUMENT, "null argument");
  view->n = g->n;
  view->num_arcs = g->succ.size();
  view->offsets = g->offsets.data();
  view->arcs = g->succ.data();
  return HANF_OK;
}

void hanf_graph_free(hanf_graph* g) { delete g; }

// stats.hpp:33-60 (cdf_from_nf + distribution_from_cdf)
hanf_status hanf_distance_distribution(const double* nf, uint64_t len, double* mean,
                                       double* variance, double* spid) {
  if (!nf || !mean || !variance || !spid) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (len == 0) return fail(HANF_INVALID_ARGUMENT, "cdf: empty neighbourhood function");
  const double last = nf[len - 1];
  if (!(last > 0.0)) return fail(HANF_INVALID_ARGUMENT, "cdf: neighbourhood function is all zero");
  double prev = 0.0, mu = 0.0, second = 0.0;
  for (uint64_t t = 0; t < len; ++t) {
    const double cdf = nf[t] / last;
    const double h = cdf - prev;
    prev = cdf;
    mu += static_cast<double>(t) * h;
    second += static_cast<double>(t) * static_cast<double>(t) * h;
  }
  *mean = mu;
  *variance = std::max(0.0, second - mu * mu);
  *spid = mu > 0.0 ? *variance / mu : 0.0;
  return HANF_OK;
}

// stats.hpp:65-77
hanf_status hanf_effective_diameter(const double* nf, uint64_t len, double alpha,
                                    int32_t interpolated, double* out) {
  if (!nf || !out) return fail(HANF_INVALID_ARGUMENT, "null argument");
  if (!(alpha > 0.0 && alpha <= 1.0))
    return fail(HANF_INVALID_ARGUMENT, "effective diameter: alpha must be in (0, 1]");
  if (len == 0) return fail(HANF_INVALID_ARGUMENT, "effective diameter: empty input");
  const double target = alpha * nf[len - 1];
  uint64_t t = 0;
  while (t + 1 < len && nf[t] < target) ++t;
  if (!interpolated || t == 0) {
    *out = static_cast<double>(t);
    return HANF_OK;
  }
  const double rise = nf[t] - nf[t - 1];
  if (rise <= 0.0) {
    *out = static_cast<double>(t - 1);
    return HANF_OK;
  }
  *out = static_cast<double>(t - 1) + (target - nf[t - 1]) / rise;
  return HANF_OK;
}

}  // extern "C"
