// ab2_synth.cpp -- seeded benchmark inputs.  Host C++, std::thread.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "aires_b200_synth.h"

namespace {

thread_local std::string tl_synth_error;

struct SynthError {
  int code;
  std::string msg;
};

inline uint64_t splitmix(uint64_t x) {
  uint64_t z = x + 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline double u01(uint64_t h) { return static_cast<double>(h >> 11) * 0x1.0p-53; }

int nthreads(int want) {
  int hw = static_cast<int>(std::thread::hardware_concurrency());
  if (hw < 1) hw = 1;
  return want > 0 ? std::min(want, hw * 2) : hw;
}

template <class F>
void parallel_for(int64_t n, int threads, F&& f) {
  if (threads <= 1 || n < 4096) {
    f(int64_t(0), n, 0);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < threads; t++) {
    int64_t a = n * t / threads, b = n * (t + 1) / threads;
    th.emplace_back([&, a, b, t] { f(a, b, t); });
  }
  for (auto& x : th) x.join();
}

// Continuous power law on [0, n): density proportional to (x + i0)^-alpha.
struct PowerLaw {
  double alpha, i0, a1, lo, hi;
  uint64_t n;
  PowerLaw(uint64_t n_, double alpha_, double i0_) : alpha(alpha_), i0(i0_), n(n_) {
    a1 = 1.0 - alpha;
    lo = std::pow(i0, a1);
    hi = std::pow(static_cast<double>(n) + i0, a1);
  }
  uint64_t sample(double u) const {
    double t = lo + u * (hi - lo);
    double x = std::pow(t, 1.0 / a1) - i0;
    if (!(x >= 0)) x = 0;
    uint64_t i = static_cast<uint64_t>(x);
    return i >= n ? n - 1 : i;
  }
  double mass(double a, double b) const { return (std::pow(b + i0, a1) - std::pow(a + i0, a1)) / (hi - lo); }
};

double solve_i0(uint64_t n, double alpha, double pairs, double cap) {
  auto top = [&](double i0) { return 2.0 * pairs * PowerLaw(n, alpha, i0).mass(0.0, 1.0); };
  if (top(1e-9) <= cap) return 1e-9;
  double lo = 1e-9, hi = static_cast<double>(n);
  for (int it = 0; it < 200; it++) {
    double mid = std::sqrt(lo * hi);
    if (top(mid) > cap)
      lo = mid;
    else
      hi = mid;
  }
  return hi;
}

struct Csr {
  std::vector<uint64_t> ptr;
  std::vector<uint32_t> col;
};

// One sampling round: M pairs -> symmetric, loop-free, duplicate-free CSR.
Csr build(uint64_t n, uint64_t M, const PowerLaw& pl, const std::vector<uint32_t>& perm, uint64_t seed,
          int threads) {
  std::vector<std::atomic<uint32_t>> deg(n);
  for (auto& d : deg) d.store(0, std::memory_order_relaxed);
  auto pair_of = [&](uint64_t p, uint32_t& u, uint32_t& v) {
    uint64_t h1 = splitmix(seed * 0x100000001b3ULL + 2 * p), h2 = splitmix(seed * 0x100000001b3ULL + 2 * p + 1);
    uint64_t a = pl.sample(u01(h1)), b = pl.sample(u01(h2));
    u = perm.empty() ? static_cast<uint32_t>(a) : perm[a];
    v = perm.empty() ? static_cast<uint32_t>(b) : perm[b];
  };
  parallel_for(static_cast<int64_t>(M), threads, [&](int64_t a, int64_t b, int) {
    for (int64_t p = a; p < b; p++) {
      uint32_t u, v;
      pair_of(static_cast<uint64_t>(p), u, v);
      if (u == v) continue;
      deg[u].fetch_add(1, std::memory_order_relaxed);
      deg[v].fetch_add(1, std::memory_order_relaxed);
    }
  });
  std::vector<uint64_t> off(n + 1, 0);
  for (uint64_t i = 0; i < n; i++) off[i + 1] = off[i] + deg[i].load(std::memory_order_relaxed);
  std::vector<uint32_t> raw(off[n]);
  std::vector<std::atomic<uint64_t>> cur(n);
  for (uint64_t i = 0; i < n; i++) cur[i].store(off[i], std::memory_order_relaxed);
  parallel_for(static_cast<int64_t>(M), threads, [&](int64_t a, int64_t b, int) {
    for (int64_t p = a; p < b; p++) {
      uint32_t u, v;
      pair_of(static_cast<uint64_t>(p), u, v);
      if (u == v) continue;
      raw[cur[u].fetch_add(1, std::memory_order_relaxed)] = v;
      raw[cur[v].fetch_add(1, std::memory_order_relaxed)] = u;
    }
  });
  // sort + unique per row
  std::vector<uint64_t> cnt(n + 1, 0);
  parallel_for(static_cast<int64_t>(n), threads, [&](int64_t a, int64_t b, int) {
    for (int64_t r = a; r < b; r++) {
      auto s = raw.begin() + off[r], e = raw.begin() + off[r + 1];
      std::sort(s, e);
      cnt[r + 1] = static_cast<uint64_t>(std::unique(s, e) - s);
    }
  });
  Csr g;
  g.ptr.assign(n + 1, 0);
  for (uint64_t i = 0; i < n; i++) g.ptr[i + 1] = g.ptr[i] + cnt[i + 1];
  g.col.resize(g.ptr[n]);
  parallel_for(static_cast<int64_t>(n), threads, [&](int64_t a, int64_t b, int) {
    for (int64_t r = a; r < b; r++)
      std::copy(raw.begin() + off[r], raw.begin() + off[r] + (g.ptr[r + 1] - g.ptr[r]), g.col.begin() + g.ptr[r]);
  });
  return g;
}

int alloc_out(aires_b200_output* out, uint64_t rows, uint64_t nnz, void** p, void** i, void** v) {
  if (!out || !out->alloc) throw SynthError{AIRES_B200_INVALID_ARGUMENT, "output allocator is null"};
  if (out->location != AIRES_B200_HOST) throw SynthError{AIRES_B200_INVALID_ARGUMENT, "synth output must be HOST"};
  if ((out->idx_bytes != 4 && out->idx_bytes != 8) || (out->val_bytes != 4 && out->val_bytes != 8))
    throw SynthError{AIRES_B200_INVALID_ARGUMENT, "idx/val widths must be 4 or 8"};
  int rc = out->alloc(out->user, rows, nnz, p, i, v);
  if (rc) throw SynthError{rc, "allocator failed"};
  out->n_rows = rows;
  out->nnz = nnz;
  return 0;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const SynthError& e) {
    tl_synth_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    tl_synth_error = "host out of memory";
    return AIRES_B200_CAPACITY_EXCEEDED;
  } catch (const std::exception& e) {
    tl_synth_error = e.what();
    return AIRES_B200_INVALID_ARGUMENT;
  }
}

}  // namespace

extern "C" {

int aires_b200_synth_graph(const aires_b200_graph_spec* s, aires_b200_output* out, double* stats) {
  return guarded([&] {
    if (!s) throw SynthError{AIRES_B200_INVALID_ARGUMENT, "null spec"};
    if (s->n == 0 || s->n >= (1ull << 32)) throw SynthError{AIRES_B200_INVALID_ARGUMENT, "n must be in [1, 2^32)"};
    if (!(s->alpha > 0.0 && s->alpha < 1.0)) throw SynthError{AIRES_B200_INVALID_ARGUMENT, "alpha must be in (0,1)"};
    auto t0 = std::chrono::steady_clock::now();
    const int th = nthreads(s->threads);
    const uint64_t n = s->n;
    std::vector<uint32_t> perm;
    if (s->relabel) {
      perm.resize(n);
      std::iota(perm.begin(), perm.end(), 0u);
      std::mt19937_64 rng(s->relabel_seed);
      for (uint64_t i = n - 1; i > 0; i--) {
        uint64_t j = rng() % (i + 1);
        std::swap(perm[i], perm[j]);
      }
    }
    double pairs = std::max(1.0, static_cast<double>(s->target_nnz) / 2.0);
    double cap = s->degree_cap ? static_cast<double>(s->degree_cap) : static_cast<double>(n);
    Csr g;
    int rounds = 0;
    double i0 = 0;
    for (; rounds < 4; rounds++) {
      i0 = solve_i0(n, s->alpha, pairs, cap);
      PowerLaw pl(n, s->alpha, i0);
      g = build(n, static_cast<uint64_t>(pairs), pl, perm, s->seed, th);
      double got = static_cast<double>(g.ptr[n]);
      if (s->target_nnz == 0 || got <= 0) break;
      double ratio = static_cast<double>(s->target_nnz) / got;
      if (std::fabs(ratio - 1.0) < 0.005) break;
      pairs *= ratio * (ratio > 1 ? 1.02 : 1.0);
    }
    const uint64_t nnz_a = g.ptr[n];
    uint64_t maxdeg = 0;
    for (uint64_t r = 0; r < n; r++) maxdeg = std::max(maxdeg, g.ptr[r + 1] - g.ptr[r]);
    const uint64_t nnz = s->normalize ? nnz_a + n : nnz_a;
    void *pp, *ip, *vp;
    alloc_out(out, n, nnz, &pp, &ip, &vp);
    out->n_cols = n;
    auto* optr = static_cast<uint64_t*>(pp);
    optr[0] = 0;
    for (uint64_t r = 0; r < n; r++) optr[r + 1] = optr[r] + (g.ptr[r + 1] - g.ptr[r]) + (s->normalize ? 1 : 0);
    // gcn.hpp:29-72: A-hat = A + I (diagonal placed in column order), d_i = sum of row,
    // value / sqrt(d_r * d_c).  A has unit weights and no loops, so d_i = deg_i + 1.
    parallel_for(static_cast<int64_t>(n), th, [&](int64_t a, int64_t b, int) {
      for (int64_t r = a; r < b; r++) {
        uint64_t w = optr[r];
        const double dr = static_cast<double>(g.ptr[r + 1] - g.ptr[r] + 1);
        bool placed = !s->normalize;
        auto emit = [&](uint64_t c, double v) {
          if (out->idx_bytes == 4)
            static_cast<uint32_t*>(ip)[w] = static_cast<uint32_t>(c);
          else
            static_cast<uint64_t*>(ip)[w] = c;
          if (out->val_bytes == 4)
            static_cast<float*>(vp)[w] = static_cast<float>(v);
          else
            static_cast<double*>(vp)[w] = v;
          w++;
        };
        auto value = [&](uint64_t c) {
          if (!s->normalize) return 1.0;
          const double dc = static_cast<double>(g.ptr[c + 1] - g.ptr[c] + 1);
          return 1.0 / std::sqrt(dr * dc);
        };
        for (uint64_t k = g.ptr[r]; k < g.ptr[r + 1]; k++) {
          uint64_t c = g.col[k];
          if (!placed && c > static_cast<uint64_t>(r)) {
            emit(static_cast<uint64_t>(r), value(static_cast<uint64_t>(r)));
            placed = true;
          }
          emit(c, value(c));
        }
        if (!placed) emit(static_cast<uint64_t>(r), value(static_cast<uint64_t>(r)));
      }
    });
    if (stats) {
      double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      double v[8] = {static_cast<double>(nnz_a), static_cast<double>(maxdeg),
                     static_cast<double>(nnz_a) / static_cast<double>(n), static_cast<double>(rounds + 1),
                     secs, i0, 0, 0};
      std::memcpy(stats, v, sizeof v);
    }
  });
}

// synth.hpp:14-16 (uniform01), 49-69 (gen_sparse), 73-78 (gen_features): same draws.
int aires_b200_synth_features(uint64_t n, uint64_t dim, double sparsity_pct, uint64_t seed,
                              aires_b200_output* out) {
  return guarded([&] {
    if (sparsity_pct < 0.0 || sparsity_pct >= 100.0)
      throw SynthError{13 /* 1 + errc::invalid_density */, "feature sparsity must be in [0, 100)"};
    const double density = (100.0 - sparsity_pct) / 100.0;
    const double lo = 0.1, hi = 1.0;
    std::mt19937_64 rng(seed);
    auto uniform01 = [&] { return static_cast<double>(rng() >> 11) * 0x1.0p-53; };
    std::vector<uint64_t> ptr(n + 1, 0);
    std::vector<uint32_t> col;
    std::vector<double> val;
    col.reserve(static_cast<size_t>(n * dim * density * 1.05) + 16);
    val.reserve(col.capacity());
    for (uint64_t i = 0; i < n; i++) {
      for (uint64_t j = 0; j < dim; j++) {
        if (uniform01() < density) {
          double v = lo + (hi - lo) * uniform01();
          if (v == 0.0) continue;
          col.push_back(static_cast<uint32_t>(j));
          val.push_back(v);
        }
      }
      ptr[i + 1] = col.size();
    }
    void *pp, *ip, *vp;
    alloc_out(out, n, col.size(), &pp, &ip, &vp);
    out->n_cols = dim;
    std::memcpy(pp, ptr.data(), (n + 1) * 8);
    for (size_t k = 0; k < col.size(); k++) {
      if (out->idx_bytes == 4)
        static_cast<uint32_t*>(ip)[k] = col[k];
      else
        static_cast<uint64_t*>(ip)[k] = col[k];
      if (out->val_bytes == 4)
        static_cast<float*>(vp)[k] = static_cast<float>(val[k]);
      else
        static_cast<double*>(vp)[k] = val[k];
    }
  });
}

const char* aires_b200_synth_last_error(void) { return tl_synth_error.c_str(); }

// synth.hpp:81-86 (gen_weights): dense in_dim x out_dim, uniform01 - 0.5, row-major, same draws.
int aires_b200_synth_weights(uint64_t in_dim, uint64_t out_dim, uint64_t seed, double* out) {
  if (!out && in_dim * out_dim) return AIRES_B200_INVALID_ARGUMENT;
  std::mt19937_64 rng(seed);
  for (uint64_t i = 0; i < in_dim * out_dim; i++) out[i] = static_cast<double>(rng() >> 11) * 0x1.0p-53 - 0.5;
  return AIRES_B200_OK;
}

}  // extern "C"
