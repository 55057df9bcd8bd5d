// oracle/pmmf_oracle.cpp — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// A single-threaded CPU restatement of the reference pMMF stage loop
// (/root/reference/proj/include/pmmf, cited file:line per function), written
// over flat arrays in "stage numbering" (stage id = cluster offset + position
// in cluster), the same data model the CUDA path uses.  It exports the flat
// C-ABI of include/pmmf_b200.h under the prefix pmmf_oracle_.
//
// Parity pin: tests/test_oracle.py checks this restatement bit-for-bit
// against oracle/_ref/libpmmf_ref.so (the reference compiled in place) and
// against the committed golden fixtures in tests/golden/.
//
// Value-neutral reformulations (verified there and
// re-verified by the tests): identity rotations are skipped in the stage
// apply and exact zeros are not stored.  Neither changes any value or
// decision of the reference.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
// load this library.

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../include/pmmf_b200.h"

namespace orc {

using i64 = int64_t;

struct Error {
  int code;
  std::string msg;
};
[[noreturn]] void fail(int code, const std::string& m) { throw Error{code, m}; }

// ---------------------------------------------------------------- rng.hpp
inline uint64_t splitmix(uint64_t& s) {  // rng.hpp:16-21
  uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
struct Rng {  // rng.hpp:24-90
  uint64_t s[4];
  explicit Rng(uint64_t seed) {
    uint64_t sm = seed;
    for (auto& w : s) w = splitmix(sm);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {  // rng.hpp:31-41
    const uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  uint64_t below(uint64_t bound) {  // rng.hpp:44-50
    const uint64_t limit = ~uint64_t{0} - ~uint64_t{0} % bound;
    uint64_t x = next();
    while (x >= limit) x = next();
    return x % bound;
  }
};
uint64_t derive(uint64_t root, std::initializer_list<uint64_t> path) {  // rng.hpp:74-82
  uint64_t st = root, out = splitmix(st);
  for (uint64_t tag : path) {
    st ^= tag + 0x9e3779b97f4a7c15ull + (st << 6) + (st >> 2);
    out = splitmix(st);
  }
  return out;
}

// ------------------------------------------------------------ small dense
// Row-major k x k helpers following DenseMatrix (dense.hpp:19-113).
struct Mat {
  i64 r = 0, c = 0;
  std::vector<double> d;
  Mat() = default;
  Mat(i64 rr, i64 cc) : r(rr), c(cc), d(static_cast<size_t>(rr * cc), 0.0) {}
  double& operator()(i64 i, i64 j) { return d[i * c + j]; }
  double operator()(i64 i, i64 j) const { return d[i * c + j]; }
};
Mat multiply(const Mat& a, const Mat& b) {  // dense.hpp:55-65 (zero left factor skipped)
  Mat o(a.r, b.c);
  for (i64 i = 0; i < a.r; ++i)
    for (i64 k = 0; k < a.c; ++k) {
      const double x = a(i, k);
      if (x == 0.0) continue;
      for (i64 j = 0; j < b.c; ++j) o(i, j) += x * b(k, j);
    }
  return o;
}
Mat transposed(const Mat& a) {  // dense.hpp:48-53
  Mat t(a.c, a.r);
  for (i64 i = 0; i < a.r; ++i)
    for (i64 j = 0; j < a.c; ++j) t(j, i) = a(i, j);
  return t;
}
std::pair<double, double> jacobi_angle(double gpp, double grr, double gpr) {  // dense.hpp:132-138
  if (gpr == 0.0) return {1.0, 0.0};
  const double tau = (grr - gpp) / (2.0 * gpr);
  const double t = (tau >= 0.0 ? 1.0 : -1.0) / (std::abs(tau) + std::sqrt(1.0 + tau * tau));
  const double c = 1.0 / std::sqrt(1.0 + t * t);
  return {c, t * c};
}
Mat jacobi_diagonalize(Mat& a, double rel_tol = 1e-15, int max_sweeps = 64) {  // dense.hpp:144-183
  const i64 n = a.r;
  Mat q(n, n);
  for (i64 i = 0; i < n; ++i) q(i, i) = 1.0;
  double fro = 0.0;
  for (double v : a.d) fro += v * v;
  const double scale = std::sqrt(fro);
  if (scale == 0.0 || n < 2) return q;
  const double stop = rel_tol * scale;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    double off = 0.0;
    for (i64 i = 0; i < n; ++i)
      for (i64 j = i + 1; j < n; ++j) off += 2.0 * a(i, j) * a(i, j);
    if (std::sqrt(off) <= stop) break;
    for (i64 p = 0; p < n; ++p)
      for (i64 r = p + 1; r < n; ++r) {
        if (a(p, r) == 0.0) continue;
        const auto [c, s] = jacobi_angle(a(p, p), a(r, r), a(p, r));
        for (i64 t = 0; t < n; ++t) {
          const double ap = a(p, t), ar = a(r, t);
          a(p, t) = c * ap - s * ar;
          a(r, t) = s * ap + c * ar;
        }
        for (i64 t = 0; t < n; ++t) {
          const double ap = a(t, p), ar = a(t, r);
          a(t, p) = c * ap - s * ar;
          a(t, r) = s * ap + c * ar;
        }
        a(p, r) = 0.0;
        a(r, p) = 0.0;
        for (i64 t = 0; t < n; ++t) {
          const double qp = q(p, t), qr = q(r, t);
          q(p, t) = c * qp - s * qr;
          q(r, t) = s * qp + c * qr;
        }
      }
  }
  return q;
}
Mat rotation_from_gram(const Mat& g) {  // factorizer.hpp:150-171
  const i64 k = g.r;
  if (k != g.c || k < 1) fail(PMMF_INVALID_ARGUMENT, "rotation_from_gram: not square");
  double asym = 0.0, mx = 0.0;
  for (i64 i = 0; i < k; ++i)
    for (i64 j = 0; j < k; ++j) {
      mx = std::max(mx, std::abs(g(i, j)));
      if (j > i) asym = std::max(asym, std::abs(g(i, j) - g(j, i)));
    }
  if (asym > 1e-9 * std::max(1.0, mx)) fail(PMMF_INVALID_ARGUMENT, "rotation_from_gram: input not symmetric");
  Mat w(k, k);
  for (i64 i = 0; i < k; ++i)
    for (i64 j = 0; j < k; ++j) w(i, j) = 0.5 * (g(i, j) + g(j, i));
  Mat q;
  if (k == 2) {
    const auto [c, s] = jacobi_angle(w(0, 0), w(1, 1), w(0, 1));
    q = Mat(2, 2);
    q(0, 0) = c;
    q(0, 1) = -s;
    q(1, 0) = s;
    q(1, 1) = c;
  } else {
    q = jacobi_diagonalize(w);
  }
  for (i64 i = 0; i < q.r; ++i) {  // fix_row_signs, factorizer.hpp:130-144
    i64 arg = 0;
    double best = std::abs(q(i, 0));
    for (i64 j = 1; j < q.c; ++j)
      if (std::abs(q(i, j)) > best) {
        best = std::abs(q(i, j));
        arg = j;
      }
    if (q(i, arg) < 0.0)
      for (i64 j = 0; j < q.c; ++j) q(i, j) = -q(i, j);
  }
  return q;
}
bool is_exact_identity(const Mat& q) {
  for (i64 i = 0; i < q.r; ++i)
    for (i64 j = 0; j < q.c; ++j)
      if (q(i, j) != (i == j ? 1.0 : 0.0)) return false;
  return true;
}

// --------------------------------------------------------- sparse columns
struct Ent {
  i64 r;
  double v;
};
using Col = std::vector<Ent>;  // sorted by stage row id, no stored zeros

// A stage numbering: clusters of global ids laid end to end
// (Partition, partition.hpp:19-93).
struct Numbering {
  std::vector<i64> s2g, off, g2s, blk;  // blk: stage id -> cluster
  void build(const std::vector<std::vector<i64>>& clusters, i64 n) {
    s2g.clear();
    off.assign(1, 0);
    g2s.assign(static_cast<size_t>(n), -1);
    blk.clear();
    for (size_t u = 0; u < clusters.size(); ++u) {
      for (i64 g : clusters[u]) {
        if (g < 0) fail(PMMF_INVALID_ARGUMENT, "Partition: negative index");
        if (g >= n) fail(PMMF_OUT_OF_RANGE, "Partition: index beyond matrix dimension");
        if (g2s[g] >= 0) fail(PMMF_INVALID_ARGUMENT, "Partition: duplicate index across clusters");
        g2s[g] = static_cast<i64>(s2g.size());
        s2g.push_back(g);
        blk.push_back(static_cast<i64>(u));
      }
      off.push_back(static_cast<i64>(s2g.size()));
    }
  }
  i64 size() const { return static_cast<i64>(s2g.size()); }
  i64 clusters() const { return static_cast<i64>(off.size()) - 1; }
};

// ||A_:,j||^2 summed per block row, then over blocks
// (blocked_matrix.hpp:203-209 with sparse.hpp:99-103).
double norm_sq_two_level(const Col& col, const Numbering& nb) {
  double s = 0.0, inner = 0.0;
  i64 cur = -1;
  for (const Ent& e : col) {
    const i64 b = nb.blk[e.r];
    if (b != cur) {
      if (cur >= 0) s += inner;
      inner = 0.0;
      cur = b;
    }
    inner += e.v * e.v;
  }
  if (cur >= 0) s += inner;
  return s;
}
// <A_:,j1, A_:,j2> as a sum of per-block merges (blocked_matrix.hpp:193-201,
// sparse.hpp:81-97).  Blocks with no common row add +0.0 (a no-op).
double dot_two_level(const Col& a, const Col& b, const Numbering& nb) {
  double s = 0.0, inner = 0.0;
  i64 cur = -1;
  size_t i = 0, j = 0;
  while (i < a.size() && j < b.size()) {
    if (a[i].r < b[j].r) {
      ++i;
    } else if (b[j].r < a[i].r) {
      ++j;
    } else {
      const i64 blk = nb.blk[a[i].r];
      if (blk != cur) {
        if (cur >= 0) s += inner;
        inner = 0.0;
        cur = blk;
      }
      inner += a[i].v * b[j].v;
      ++i;
      ++j;
    }
  }
  if (cur >= 0) s += inner;
  return s;
}

// ------------------------------------------------------------- clustering
struct Params {
  int k, n_stages;
  double eta;
  i64 m_target, c_min, c_max;
  int d_max;
  bool bypass;
  i64 core_min, core_cap;
  uint64_t seed;
};

struct ClusterCtx {  // clustering.hpp:51-59
  const std::vector<Col>* cols;
  const Numbering* nb;
  const std::vector<double>* norm;  // by global id
  const Params* p;
  int max_depth = 0;
  double score(i64 j, i64 a) const {  // clustering.hpp:62-67
    const double nj = (*norm)[j], na = (*norm)[a];
    if (nj <= 0.0 || na <= 0.0) return 0.0;
    return std::abs(dot_two_level((*cols)[nb->g2s[j]], (*cols)[nb->g2s[a]], *nb)) / (nj * na);
  }
  std::pair<size_t, double> best(i64 j, const std::vector<i64>& anchors) const {  // clustering.hpp:71-83
    size_t b = 0;
    double bs = 0.0;
    for (size_t a = 0; a < anchors.size(); ++a) {
      const double s = score(j, anchors[a]);
      if (s > bs) {
        bs = s;
        b = a;
      }
    }
    return {b, bs};
  }
};

void cluster_recursive(ClusterCtx& ctx, std::vector<i64> pool, i64 m_request, int depth, Rng& rng,
                       std::vector<std::vector<i64>>& out) {  // clustering.hpp:85-177
  ctx.max_depth = std::max(ctx.max_depth, depth);
  if (pool.empty()) return;
  std::vector<i64> shuffled;
  for (i64 g : pool)
    if ((*ctx.norm)[g] > 0.0) shuffled.push_back(g);
  if (shuffled.empty()) {
    out.push_back(std::move(pool));
    return;
  }
  const size_t m = static_cast<size_t>(std::min<i64>(m_request, static_cast<i64>(shuffled.size())));
  for (size_t t = 0; t < m; ++t) std::swap(shuffled[t], shuffled[t + rng.below(shuffled.size() - t)]);
  std::vector<i64> anchors(shuffled.begin(), shuffled.begin() + static_cast<std::ptrdiff_t>(m));
  std::sort(anchors.begin(), anchors.end());
  const size_t kUn = static_cast<size_t>(-1);
  std::vector<std::vector<i64>> clusters(m);
  size_t rr = 0;
  for (i64 j : pool) {
    auto it = std::lower_bound(anchors.begin(), anchors.end(), j);
    size_t a;
    if (it != anchors.end() && *it == j) {
      a = static_cast<size_t>(it - anchors.begin());
    } else {
      auto [b, s] = ctx.best(j, anchors);
      a = s > 0.0 ? b : kUn;
    }
    if (a == kUn) a = (rr++) % m;
    clusters[a].push_back(j);
  }
  std::vector<size_t> alive(m);
  std::iota(alive.begin(), alive.end(), size_t{0});
  while (alive.size() > 1) {  // undersize repair, :138-163
    size_t worst = alive[0];
    for (size_t a : alive)
      if (clusters[a].size() < clusters[worst].size()) worst = a;
    if (static_cast<i64>(clusters[worst].size()) >= ctx.p->c_min) break;
    alive.erase(std::find(alive.begin(), alive.end(), worst));
    std::vector<i64> orphans = std::move(clusters[worst]);
    clusters[worst].clear();
    std::vector<i64> remaining;
    for (size_t a : alive) remaining.push_back(anchors[a]);
    size_t orr = 0;
    for (i64 o : orphans) {
      auto [b, s] = ctx.best(o, remaining);
      size_t a = s > 0.0 ? b : (orr++) % alive.size();
      clusters[alive[a]].push_back(o);
    }
    for (size_t a : alive) std::sort(clusters[a].begin(), clusters[a].end());
  }
  for (size_t a : alive) {  // oversize recursion, :165-176
    auto& mem = clusters[a];
    if (mem.empty()) continue;
    if (static_cast<i64>(mem.size()) > ctx.p->c_max && depth < ctx.p->d_max) {
      const i64 sub = (static_cast<i64>(mem.size()) + ctx.p->c_max - 1) / ctx.p->c_max;
      cluster_recursive(ctx, std::move(mem), sub, depth + 1, rng, out);
    } else {
      out.push_back(std::move(mem));
    }
  }
}

// ------------------------------------------------------- Gram / diag block
// Dense column-major c x c tiles: M[col * c + row].
struct Tile {
  i64 c;
  std::vector<double> m;
  explicit Tile(i64 cc) : c(cc), m(static_cast<size_t>(cc * cc), 0.0) {}
  double& at(i64 row, i64 col) { return m[col * c + row]; }
};

// G_u = A[:,B_u]^T A[:,B_u] summed row by row in stage order
// (blocked_matrix.hpp:238-254, sparse.hpp:177-187).
Tile gram(const std::vector<Col>& A, i64 off, i64 c, i64 N) {
  std::vector<std::vector<Ent>> rows(static_cast<size_t>(N));
  for (i64 a = 0; a < c; ++a)
    for (const Ent& e : A[off + a]) rows[e.r].push_back({a, e.v});
  Tile g(c);
  for (const auto& row : rows)
    for (size_t s = 0; s < row.size(); ++s)
      for (size_t t = s; t < row.size(); ++t) g.at(row[s].r, row[t].r) += row[s].v * row[t].v;
  for (i64 b = 0; b < c; ++b)
    for (i64 a = 0; a < b; ++a) g.at(b, a) = g.at(a, b);
  return g;
}
// D_u = A[B_u,B_u] from its upper triangle (blocked_matrix.hpp:257-266).
Tile diag_block(const std::vector<Col>& A, i64 off, i64 c) {
  Tile d(c);
  for (i64 a = 0; a < c; ++a)
    for (const Ent& e : A[off + a]) {
      const i64 r = e.r - off;
      if (r < 0 || r >= c || r > a) continue;
      d.at(r, a) = e.v;
      d.at(a, r) = e.v;
    }
  return d;
}
// M <- q M q^T on local indices idx (sparse.hpp:190-242), full storage.
void rotate_tile(Tile& M, const std::vector<i64>& idx, const Mat& q) {
  const i64 k = static_cast<i64>(idx.size()), c = M.c;
  Mat corner(k, k);
  for (i64 a = 0; a < k; ++a)
    for (i64 b = 0; b < k; ++b) corner(a, b) = M.at(idx[a], idx[b]);
  std::vector<double> v(k), mixed(k);
  for (i64 r = 0; r < c; ++r) {
    if (std::find(idx.begin(), idx.end(), r) != idx.end()) continue;
    for (i64 b = 0; b < k; ++b) v[b] = M.at(r, idx[b]);
    for (i64 a = 0; a < k; ++a) {
      double acc = 0.0;
      for (i64 b = 0; b < k; ++b) acc += q(a, b) * v[b];
      mixed[a] = acc;
    }
    for (i64 a = 0; a < k; ++a) {
      M.at(r, idx[a]) = mixed[a];
      M.at(idx[a], r) = mixed[a];
    }
  }
  const Mat nc = multiply(multiply(q, corner), transposed(q));
  for (i64 a = 0; a < k; ++a)
    for (i64 pos = 0; pos < k; ++pos) M.at(idx[pos], idx[a]) = nc(pos, a);
}
inline double off_diag_norm_sq(double ns, double d) { return std::max(0.0, ns - d * d); }  // factorizer.hpp:122-124

struct FoundRot {
  std::vector<i64> locals;
  Mat q;
};
struct Found {
  std::vector<FoundRot> rots;
  std::vector<i64> elim;  // local ids, elimination order
};
// Algorithm 2 (factorizer.hpp:198-319) on dense tiles.
Found search(i64 c, Tile& G, Tile& D, int k, double eta, i64 cap, uint64_t seed) {
  Found res;
  if (c < k) return res;
  i64 budget = static_cast<i64>(std::floor(eta * static_cast<double>(c)));
  if (cap >= 0) budget = std::min(budget, cap);
  if (budget <= 0) return res;
  Rng rng(seed);
  std::vector<i64> active(static_cast<size_t>(c));
  std::iota(active.begin(), active.end(), i64{0});
  std::vector<uint8_t> on(static_cast<size_t>(c), 1);
  auto eliminate = [&](i64 l) {
    res.elim.push_back(l);
    on[l] = 0;
    active.erase(std::lower_bound(active.begin(), active.end(), l));
  };
  for (i64 s = 0; s < budget; ++s) {
    if (static_cast<i64>(active.size()) <= k - 1) break;
    const i64 draw = active[rng.below(active.size())];
    if (G.at(draw, draw) <= 0.0) {
      eliminate(draw);
      continue;
    }
    std::vector<i64> partners;
    if (k == 2) {
      i64 best = -1;
      double bs = 0.0;
      for (i64 l = 0; l < c; ++l) {
        if (l == draw || !on[l]) continue;
        const double nl = G.at(l, l);
        if (nl <= 0.0) continue;
        const double g = G.at(l, draw);
        const double sc = g * g / nl;
        if (sc > bs) {
          bs = sc;
          best = l;
        }
      }
      if (best < 0) best = (active[0] == draw) ? active[1] : active[0];
      partners.push_back(best);
    } else {
      std::vector<std::pair<double, i64>> cand;
      for (i64 l = 0; l < c; ++l) {
        if (l == draw || !on[l]) continue;
        const double nl = G.at(l, l);
        if (nl <= 0.0) continue;
        const double g = G.at(l, draw);
        const double sc = g * g / nl;
        if (sc > 0.0) cand.push_back({sc, l});
      }
      std::sort(cand.begin(), cand.end(), [](const auto& x, const auto& y) {
        if (x.first != y.first) return x.first > y.first;
        return x.second < y.second;
      });
      for (const auto& cd : cand) {
        if (static_cast<i64>(partners.size()) == k - 1) break;
        partners.push_back(cd.second);
      }
      for (i64 l : active) {
        if (static_cast<i64>(partners.size()) == k - 1) break;
        if (l != draw && std::find(partners.begin(), partners.end(), l) == partners.end()) partners.push_back(l);
      }
    }
    std::vector<i64> locals{draw};
    locals.insert(locals.end(), partners.begin(), partners.end());
    Mat gs(k, k);
    for (i64 a = 0; a < k; ++a)
      for (i64 b = 0; b < k; ++b) gs(a, b) = G.at(locals[a], locals[b]);
    Mat q = rotation_from_gram(gs);
    rotate_tile(G, locals, q);
    rotate_tile(D, locals, q);
    i64 victim = -1;
    double vn = 0.0;
    for (size_t a = 1; a < locals.size(); ++a) {
      const double off = off_diag_norm_sq(G.at(locals[a], locals[a]), D.at(locals[a], locals[a]));
      if (victim < 0 || off < vn) {
        victim = locals[a];
        vn = off;
      }
    }
    if (off_diag_norm_sq(G.at(draw, draw), D.at(draw, draw)) < vn) victim = draw;
    res.rots.push_back({locals, q});
    eliminate(victim);
  }
  return res;
}

// Column mix over the union support (sparse.hpp:123-156); zeros dropped.
void mix_columns(std::vector<Col>& cols, const std::vector<i64>& ids, const Mat& q) {
  const size_t k = ids.size();
  std::vector<size_t> cur(k, 0);
  std::vector<Col> out(k);
  std::vector<double> v(k);
  for (;;) {
    i64 row = -1;
    for (size_t b = 0; b < k; ++b) {
      const Col& c = cols[ids[b]];
      if (cur[b] < c.size() && (row < 0 || c[cur[b]].r < row)) row = c[cur[b]].r;
    }
    if (row < 0) break;
    for (size_t b = 0; b < k; ++b) {
      const Col& c = cols[ids[b]];
      if (cur[b] < c.size() && c[cur[b]].r == row) {
        v[b] = c[cur[b]].v;
        ++cur[b];
      } else {
        v[b] = 0.0;
      }
    }
    for (size_t a = 0; a < k; ++a) {
      double acc = 0.0;
      for (size_t b = 0; b < k; ++b) acc += q(static_cast<i64>(a), static_cast<i64>(b)) * v[b];
      if (acc != 0.0) out[a].push_back({row, acc});
    }
  }
  for (size_t a = 0; a < k; ++a) cols[ids[a]] = std::move(out[a]);
}
std::vector<Col> transpose(const std::vector<Col>& A) {
  std::vector<Col> T(A.size());
  for (size_t j = 0; j < A.size(); ++j)
    for (const Ent& e : A[j]) T[e.r].push_back({static_cast<i64>(j), e.v});
  return T;
}

// ----------------------------------------------------------- result types
struct Rot {
  std::vector<i64> idx;
  Mat q;
};
struct Elim {
  i64 index;
  double diag, mass;
};
struct Stage {
  std::vector<i64> off, members, bypassed;
  std::vector<Rot> rots;
  std::vector<Elim> elim;
};
struct Result {
  i64 n = 0;
  int k = 2;
  std::vector<Stage> stages;
  std::vector<i64> core_idx, hist;
  Mat core;
  std::vector<std::pair<i64, double>> diag;
  double residual_sq = 0.0;
  bool trivial = false;
  double phases[6] = {0, 0, 0, 0, 0, 0};
  std::vector<std::array<i64, 7>> info;
};

using clk = std::chrono::steady_clock;
double ms_since(clk::time_point t) { return std::chrono::duration<double, std::milli>(clk::now() - t).count(); }

void validate(const Params& p) {  // factorizer.hpp:44-50, clustering.hpp:36-40
  if (p.k < 2 || p.k > 8) fail(PMMF_INVALID_ARGUMENT, "FactorizeParams: k must be in [2, 8]");
  if (p.n_stages < 1) fail(PMMF_INVALID_ARGUMENT, "FactorizeParams: n_stages < 1");
  if (!(p.eta > 0.0 && p.eta < 1.0)) fail(PMMF_INVALID_ARGUMENT, "FactorizeParams: eta not in (0,1)");
  if (p.core_min < 1) fail(PMMF_INVALID_ARGUMENT, "FactorizeParams: core_min < 1");
  if (p.m_target < 1) fail(PMMF_INVALID_ARGUMENT, "ClusterParams: m_target < 1");
  if (p.c_min > p.c_max) fail(PMMF_INVALID_ARGUMENT, "ClusterParams: c_min > c_max");
  if (p.d_max < 0) fail(PMMF_INVALID_ARGUMENT, "ClusterParams: d_max < 0");
}

// pmmf::factorize (factorizer.hpp:397-595) over the flat model.
Result factorize(const pmmf_b200_coo* in, const Params& p) {
  const i64 n = in->n;
  Numbering cur;
  {
    std::vector<std::vector<i64>> init;
    if (in->n_clusters == 0) {  // Partition::trivial, partition.hpp:57-61
      init.emplace_back(static_cast<size_t>(std::max<i64>(n, 0)));
      std::iota(init[0].begin(), init[0].end(), i64{0});
    } else {
      for (i64 u = 0; u < in->n_clusters; ++u)
        init.emplace_back(in->cluster_members + in->cluster_offsets[u], in->cluster_members + in->cluster_offsets[u + 1]);
    }
    cur.build(init, std::max<i64>(n, 0));
  }
  // from_triplets (blocked_matrix.hpp:138-156): per-column stable order,
  // duplicates summed in input order.
  std::vector<Col> A(static_cast<size_t>(cur.size()));
  for (i64 t = 0; t < in->nnz; ++t) {
    const i64 r = in->rows[t], c = in->cols[t];
    const double v = in->vals[t];
    if (r < 0 || r >= n || c < 0 || c >= n) fail(PMMF_OUT_OF_RANGE, "from_triplets: index out of range");
    if (!std::isfinite(v)) fail(PMMF_INVALID_ARGUMENT, "from_triplets: non-finite value");
    const i64 sr = cur.g2s[r], sc = cur.g2s[c];
    if (sr < 0 || sc < 0) fail(PMMF_OUT_OF_RANGE, "from_triplets: index not covered by partition");
    A[sc].push_back({sr, v});
  }
  for (Col& col : A) {
    std::stable_sort(col.begin(), col.end(), [](const Ent& x, const Ent& y) { return x.r < y.r; });
    size_t o = 0;
    for (size_t i = 0; i < col.size();) {
      double s = col[i].v;
      size_t j = i + 1;
      while (j < col.size() && col[j].r == col[i].r) s += col[j++].v;
      col[o++] = {col[i].r, s};
      i = j;
    }
    col.resize(o);
  }
  validate(p);
  if (n < 1) fail(PMMF_INVALID_ARGUMENT, "factorize: empty matrix");
  {  // symmetry check (factorizer.hpp:405-409, blocked_matrix.hpp:447-463)
    double fro = 0.0, worst = 0.0;
    for (const Col& col : A)
      for (const Ent& e : col) fro += e.v * e.v;
    for (i64 j = 0; j < cur.size(); ++j)
      for (const Ent& e : A[j]) {
        if (cur.blk[e.r] > cur.blk[j]) continue;
        const Col& mirror = A[e.r];
        auto it = std::lower_bound(mirror.begin(), mirror.end(), j, [](const Ent& x, i64 key) { return x.r < key; });
        const double m = (it != mirror.end() && it->r == j) ? it->v : 0.0;
        worst = std::max(worst, std::abs(e.v - m));
      }
    if (worst > 1e-9 * std::max(std::sqrt(fro), 1e-300))
      fail(PMMF_INVALID_ARGUMENT, "factorize: input matrix is not symmetric");
  }
  // Drop stored zeros (value-neutral, P12).
  for (Col& col : A) col.erase(std::remove_if(col.begin(), col.end(), [](const Ent& e) { return e.v == 0.0; }), col.end());

  const auto run_start = clk::now();
  Result R;
  R.n = n;
  R.k = p.k;
  std::vector<i64> active;
  for (i64 g = 0; g < n; ++g)
    if (cur.g2s[g] >= 0) active.push_back(g);
  R.hist.push_back(static_cast<i64>(active.size()));
  std::vector<uint8_t> is_active(static_cast<size_t>(n), 0);
  std::vector<i64> rank(static_cast<size_t>(n), -1);
  for (i64 g : active) is_active[g] = 1;
  if (static_cast<i64>(active.size()) <= p.core_min) R.trivial = true;

  for (int stage_no = 1; stage_no <= p.n_stages && !R.trivial; ++stage_no) {
    if (static_cast<i64>(active.size()) <= p.core_min) break;
    // ---- clustering on the pre-reblock matrix (clustering.hpp:183-225)
    auto t0 = clk::now();
    std::vector<double> norm(static_cast<size_t>(n), 0.0);
    for (i64 g : active) norm[g] = std::sqrt(norm_sq_two_level(A[cur.g2s[g]], cur));
    std::vector<i64> pool, bypassed;
    for (i64 g : active) (!p.bypass || norm[g] > 0.0 ? pool : bypassed).push_back(g);
    ClusterCtx ctx{&A, &cur, &norm, &p};
    std::vector<std::vector<i64>> clusters;
    if (!pool.empty()) {
      Rng rng(derive(p.seed, {0xC1u, static_cast<uint64_t>(stage_no)}));
      cluster_recursive(ctx, std::move(pool), p.m_target, 0, rng, clusters);
    }
    R.phases[0] += ms_since(t0);
    const i64 rc = static_cast<i64>(clusters.size());
    if (!bypassed.empty()) clusters.push_back(bypassed);
    // ---- reblock (blocked_matrix.hpp:318-367): relabel, drop retired, sort
    t0 = clk::now();
    Numbering nxt;
    nxt.build(clusters, n);
    std::vector<Col> B(static_cast<size_t>(nxt.size()));
    for (i64 J = 0; J < nxt.size(); ++J) {
      const Col& src = A[cur.g2s[nxt.s2g[J]]];
      Col& dst = B[J];
      for (const Ent& e : src) {
        const i64 nr = nxt.g2s[cur.s2g[e.r]];
        if (nr >= 0) dst.push_back({nr, e.v});
      }
      std::sort(dst.begin(), dst.end(), [](const Ent& x, const Ent& y) { return x.r < y.r; });
    }
    A = std::move(B);
    cur = std::move(nxt);
    R.phases[4] += ms_since(t0);
    Stage st;
    st.off = cur.off;
    st.members = cur.s2g;
    st.bypassed = bypassed;
    // ---- budgets (factorizer.hpp:463-479)
    std::vector<i64> budget(static_cast<size_t>(rc), 0);
    i64 planned = 0;
    for (i64 u = 0; u < rc; ++u) {
      const i64 c = cur.off[u + 1] - cur.off[u];
      i64 b = c < p.k ? 0 : static_cast<i64>(std::floor(p.eta * static_cast<double>(c)));
      b = std::min(b, std::max<i64>(0, c - (p.k - 1)));
      budget[u] = b;
      planned += b;
    }
    const i64 allowance = std::max<i64>(0, static_cast<i64>(active.size()) - p.core_min);
    while (planned > allowance) {
      i64 arg = 0;
      for (i64 u = 1; u < rc; ++u)
        if (budget[u] > budget[arg]) arg = u;
      --budget[arg];
      --planned;
    }
    // ---- Gram + search per cluster (factorizer.hpp:482-509)
    std::vector<Found> found(static_cast<size_t>(rc));
    double gram_ms = 0.0, search_ms = 0.0;
    for (i64 u = 0; u < rc; ++u) {
      const i64 off = cur.off[u], c = cur.off[u + 1] - off;
      t0 = clk::now();
      Tile G = gram(A, off, c, cur.size());
      Tile D = diag_block(A, off, c);
      gram_ms += ms_since(t0);
      t0 = clk::now();
      found[u] = search(c, G, D, p.k, p.eta, budget[u],
                        derive(p.seed, {0xF0u, static_cast<uint64_t>(stage_no), static_cast<uint64_t>(u)}));
      search_ms += ms_since(t0);
    }
    R.phases[1] += gram_ms;
    R.phases[2] += search_ms;
    for (i64 u = 0; u < rc; ++u)
      for (const auto& fr : found[u].rots) {
        Rot rot;
        for (i64 l : fr.locals) rot.idx.push_back(cur.s2g[cur.off[u] + l]);
        rot.q = fr.q;
        st.rots.push_back(std::move(rot));
      }
    // ---- stage apply (factorizer.hpp:336-394): column pass, transpose,
    // column pass, transpose; identity rotations skipped.
    t0 = clk::now();
    for (int side = 0; side < 2; ++side) {
      for (i64 u = 0; u < rc; ++u)
        for (const auto& fr : found[u].rots) {
          if (is_exact_identity(fr.q)) continue;
          std::vector<i64> ids;
          for (i64 l : fr.locals) ids.push_back(cur.off[u] + l);
          mix_columns(A, ids, fr.q);
        }
      A = transpose(A);
    }
    R.phases[3] += ms_since(t0);
    // ---- residual accounting (factorizer.hpp:521-547)
    std::vector<i64> order;
    for (i64 u = 0; u < rc; ++u)
      for (i64 l : found[u].elim) order.push_back(cur.s2g[cur.off[u] + l]);
    for (size_t r = 0; r < order.size(); ++r) {
      rank[order[r]] = static_cast<i64>(r);
      is_active[order[r]] = 0;
    }
    for (size_t r = 0; r < order.size(); ++r) {
      const i64 g = order[r];
      double mass = 0.0, d = 0.0;
      for (const Ent& e : A[cur.g2s[g]]) {
        const i64 l = cur.s2g[e.r];
        if (l == g) {
          d = e.v;
          continue;
        }
        if (is_active[l] || rank[l] > static_cast<i64>(r)) mass += e.v * e.v;
      }
      st.elim.push_back({g, d, mass});
    }
    for (const Elim& e : st.elim) {
      R.residual_sq += 2.0 * e.mass;
      R.diag.push_back({e.index, e.diag});
    }
    for (i64 g : order) rank[g] = -1;
    {
      std::vector<i64> next;
      for (i64 g : active)
        if (is_active[g]) next.push_back(g);
      active = std::move(next);
    }
    R.hist.push_back(static_cast<i64>(active.size()));
    R.info.push_back({stage_no, rc, static_cast<i64>(bypassed.size()), static_cast<i64>(st.rots.size()),
                      static_cast<i64>(st.elim.size()), static_cast<i64>(active.size()), ctx.max_depth});
    R.stages.push_back(std::move(st));
  }
  if (static_cast<i64>(active.size()) > p.core_cap)  // factorizer.hpp:573-576
    fail(PMMF_NUMERIC, "factorize: core of size " + std::to_string(active.size()) + " exceeds the cap of " +
                           std::to_string(p.core_cap) + "; raise core_cap or add stages");
  const i64 g = static_cast<i64>(active.size());
  R.core_idx = active;
  R.core = Mat(g, g);
  std::vector<i64> pos(static_cast<size_t>(n), -1);
  for (i64 a = 0; a < g; ++a) pos[active[a]] = a;
  for (i64 b = 0; b < g; ++b)
    for (const Ent& e : A[cur.g2s[active[b]]]) {
      const i64 a = pos[cur.s2g[e.r]];
      if (a >= 0) R.core(a, b) = e.v;
    }
  std::sort(R.diag.begin(), R.diag.end());
  R.phases[5] = ms_since(run_start);
  return R;
}

// ------------------------------------------------------------ MmfOperator
struct Operator {  // transform_ops.hpp:30-137
  std::shared_ptr<Result> f;
  double thr;
  std::vector<double> eval;
  Mat evec;  // eigenvectors as columns
  int64_t neg = 0;
  double factor(int mode, double d) const {  // :76-86
    if (mode == 0) return d;
    if (mode == 1) return std::abs(d) < thr ? 0.0 : 1.0 / d;
    return d < thr ? 0.0 : 1.0 / std::sqrt(d);
  }
  void apply(int mode, const double* in, double* out) const {  // :51-67
    const i64 n = f->n;
    std::vector<double> v(in, in + n);
    double vals[8];
    for (const Stage& st : f->stages)
      for (const Rot& r : st.rots) {
        const i64 k = static_cast<i64>(r.idx.size());
        for (i64 b = 0; b < k; ++b) vals[b] = v[r.idx[b]];
        for (i64 a = 0; a < k; ++a) {
          double acc = 0.0;
          for (i64 b = 0; b < k; ++b) acc += r.q(a, b) * vals[b];
          v[r.idx[a]] = acc;
        }
      }
    const i64 g = static_cast<i64>(f->core_idx.size());
    if (g > 0) {  // apply_core, :88-106
      std::vector<double> x(g), y(g, 0.0);
      for (i64 a = 0; a < g; ++a) x[a] = v[f->core_idx[a]];
      for (i64 e = 0; e < g; ++e) {
        double dot = 0.0;
        for (i64 a = 0; a < g; ++a) dot += evec(a, e) * x[a];
        dot *= factor(mode, eval[e]);
        for (i64 a = 0; a < g; ++a) y[a] += evec(a, e) * dot;
      }
      for (i64 a = 0; a < g; ++a) v[f->core_idx[a]] = y[a];
    }
    for (const auto& [i, d] : f->diag) v[i] *= factor(mode, d);
    for (auto sit = f->stages.rbegin(); sit != f->stages.rend(); ++sit)
      for (auto rit = sit->rots.rbegin(); rit != sit->rots.rend(); ++rit) {
        const i64 k = static_cast<i64>(rit->idx.size());
        for (i64 b = 0; b < k; ++b) vals[b] = v[rit->idx[b]];
        for (i64 a = 0; a < k; ++a) {
          double acc = 0.0;
          for (i64 b = 0; b < k; ++b) acc += rit->q(b, a) * vals[b];
          v[rit->idx[a]] = acc;
        }
      }
    std::copy(v.begin(), v.end(), out);
  }
};

// CSR-like row view for y = A x in multiply_flat order (blocked_matrix.hpp:390-407):
// each output row sums its columns in stage (input partition) order.
struct SpMat {
  i64 n;
  std::vector<std::vector<std::pair<i64, double>>> rows;  // (col, value) in stage-column order
};
SpMat make_spmat(const pmmf_b200_coo* in) {
  SpMat S;
  S.n = in->n;
  Numbering nb;
  std::vector<std::vector<i64>> init;
  if (in->n_clusters == 0) {
    init.emplace_back(static_cast<size_t>(in->n));
    std::iota(init[0].begin(), init[0].end(), i64{0});
  } else {
    for (i64 u = 0; u < in->n_clusters; ++u)
      init.emplace_back(in->cluster_members + in->cluster_offsets[u], in->cluster_members + in->cluster_offsets[u + 1]);
  }
  nb.build(init, in->n);
  std::vector<Col> cols(static_cast<size_t>(nb.size()));
  for (i64 t = 0; t < in->nnz; ++t) cols[nb.g2s[in->cols[t]]].push_back({nb.g2s[in->rows[t]], in->vals[t]});
  S.rows.resize(static_cast<size_t>(in->n));
  for (i64 j = 0; j < nb.size(); ++j) {
    Col& col = cols[j];
    std::stable_sort(col.begin(), col.end(), [](const Ent& x, const Ent& y) { return x.r < y.r; });
    for (size_t i = 0; i < col.size();) {
      double s = col[i].v;
      size_t k = i + 1;
      while (k < col.size() && col[k].r == col[i].r) s += col[k++].v;
      S.rows[nb.s2g[col[i].r]].push_back({nb.s2g[j], s});
      i = k;
    }
  }
  return S;
}
void spmv(const SpMat& S, const std::vector<double>& x, std::vector<double>& y) {
  for (i64 r = 0; r < S.n; ++r) {
    double acc = 0.0;
    for (const auto& [c, v] : S.rows[r]) {
      if (x[c] == 0.0) continue;
      acc += v * x[c];
    }
    y[r] = acc;
  }
}
double vdot(const std::vector<double>& a, const std::vector<double>& b) {  // solver.hpp:98-102
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

// ---- comparison preconditioners (solver.hpp:174-340), restated
// Entries of A after from_triplets in to_triplets order (blocked_matrix.hpp:
// 422-436): row clusters, then column clusters, then the block's columns,
// then rows; duplicates summed in input order, stored zeros KEPT.
struct Trip {
  i64 r, c;
  double v;
};
std::vector<Trip> to_triplets_kept(const pmmf_b200_coo* in) {
  Numbering nb;
  std::vector<std::vector<i64>> init;
  if (in->n_clusters == 0) {
    init.emplace_back(static_cast<size_t>(in->n));
    std::iota(init[0].begin(), init[0].end(), i64{0});
  } else {
    for (i64 u = 0; u < in->n_clusters; ++u)
      init.emplace_back(in->cluster_members + in->cluster_offsets[u], in->cluster_members + in->cluster_offsets[u + 1]);
  }
  nb.build(init, in->n);
  std::vector<Col> cols(static_cast<size_t>(nb.size()));
  for (i64 t = 0; t < in->nnz; ++t) {
    if (in->rows[t] < 0 || in->rows[t] >= in->n || in->cols[t] < 0 || in->cols[t] >= in->n)
      fail(PMMF_OUT_OF_RANGE, "from_triplets: index out of range");
    cols[nb.g2s[in->cols[t]]].push_back({nb.g2s[in->rows[t]], in->vals[t]});
  }
  // per stage column: stable sort by row, sum duplicates (sparse.hpp:66-79)
  std::vector<std::vector<std::pair<i64, double>>> summed(cols.size());
  for (size_t j = 0; j < cols.size(); ++j) {
    Col& col = cols[j];
    std::stable_sort(col.begin(), col.end(), [](const Ent& x, const Ent& y) { return x.r < y.r; });
    for (size_t i = 0; i < col.size();) {
      double s = col[i].v;
      size_t k = i + 1;
      while (k < col.size() && col[k].r == col[i].r) s += col[k++].v;
      summed[j].push_back({col[i].r, s});
      i = k;
    }
  }
  std::vector<Trip> out;
  const i64 m = nb.clusters();
  for (i64 u = 0; u < m; ++u)
    for (i64 v = 0; v < m; ++v)
      for (i64 j = nb.off[v]; j < nb.off[v + 1]; ++j)
        for (const auto& [r, val] : summed[j])
          if (r >= nb.off[u] && r < nb.off[u + 1]) out.push_back({nb.s2g[r], nb.s2g[j], val});
  return out;
}

struct LowerTri {  // detail::LowerTriangle (solver.hpp:174-202)
  std::vector<double> diag;
  std::vector<std::vector<std::pair<i64, double>>> cols;  // strictly lower, rows ascending
  i64 n() const { return static_cast<i64>(diag.size()); }
  void forward_solve(const double* b, double* x) const {  // solver.hpp:183-191
    std::copy(b, b + n(), x);
    for (i64 j = 0; j < n(); ++j) {
      x[j] /= diag[j];
      const double xj = x[j];
      for (const auto& [r, v] : cols[j]) x[r] -= v * xj;
    }
  }
  void backward_solve(const double* b, double* x) const {  // solver.hpp:193-201
    for (i64 j = n() - 1; j >= 0; --j) {
      double acc = b[j];
      for (const auto& [r, v] : cols[j]) acc -= v * x[r];
      x[j] = acc / diag[j];
    }
  }
};

LowerTri extract_lower(const std::vector<Trip>& t, i64 n) {  // solver.hpp:204-218
  LowerTri l;
  l.diag.assign(static_cast<size_t>(n), 0.0);
  l.cols.resize(static_cast<size_t>(n));
  for (const Trip& e : t) {
    if (e.r == e.c)
      l.diag[e.r] = e.v;
    else if (e.r > e.c)
      l.cols[e.c].push_back({e.r, e.v});
  }
  for (auto& c : l.cols) std::stable_sort(c.begin(), c.end(), [](auto& a, auto& b) { return a.first < b.first; });
  return l;
}

struct Pre {
  int kind = 0;
  i64 n = 0;
  std::vector<double> scale;  // jacobi
  LowerTri lower;             // ssor / ic
  std::vector<double> sqrt_d;  // ssor
  int compensated = 0;
  double alpha = 0.0;
  const Operator* op = nullptr;  // pmmf
  void apply(int side, const double* in, double* out) const {
    if (kind == PMMF_PRECOND_JACOBI) {
      for (i64 i = 0; i < n; ++i) out[i] = scale[i] * in[i];
    } else if (kind == PMMF_PRECOND_SSOR) {
      if (side == 0) {
        lower.forward_solve(in, out);
        for (i64 i = 0; i < n; ++i) out[i] *= sqrt_d[i];
      } else {
        std::vector<double> sc(static_cast<size_t>(n));
        for (i64 i = 0; i < n; ++i) sc[i] = in[i] * sqrt_d[i];
        lower.backward_solve(sc.data(), out);
      }
    } else if (kind == PMMF_PRECOND_IC) {
      if (side == 0)
        lower.forward_solve(in, out);
      else
        lower.backward_solve(in, out);
    } else if (kind == PMMF_PRECOND_PMMF) {
      op->apply(2, in, out);
    } else {
      std::copy(in, in + n, out);
    }
  }
};

bool ic_attempt(const LowerTri& pattern, double boost, LowerTri& l) {  // solver.hpp:284-313
  const i64 n = pattern.n();
  l = pattern;
  for (i64 j = 0; j < n; ++j) l.diag[j] *= (1.0 + boost);
  std::vector<std::vector<std::pair<i64, size_t>>> rows(static_cast<size_t>(n));
  std::vector<double> work;
  for (i64 j = 0; j < n; ++j) {
    auto& col = l.cols[j];
    double pivot = l.diag[j];
    work.assign(col.size(), 0.0);
    for (size_t t = 0; t < col.size(); ++t) work[t] = col[t].second;
    for (const auto& [k, pos] : rows[j]) {
      const auto& ck = l.cols[k];
      const double ljk = ck[pos].second;
      pivot -= ljk * ljk;
      size_t t = 0;
      for (size_t s = pos + 1; s < ck.size(); ++s) {
        const i64 r = ck[s].first;
        while (t < col.size() && col[t].first < r) ++t;
        if (t == col.size()) break;
        if (col[t].first == r) work[t] -= ck[s].second * ljk;
      }
    }
    if (!(pivot > 0.0)) return false;
    l.diag[j] = std::sqrt(pivot);
    for (size_t t = 0; t < col.size(); ++t) {
      col[t].second = work[t] / l.diag[j];
      rows[col[t].first].emplace_back(j, t);
    }
  }
  return true;
}

std::unique_ptr<Pre> make_pre(const pmmf_b200_coo* a, int kind, double omega) {
  auto p = std::make_unique<Pre>();
  p->kind = kind;
  p->n = a->n;
  const i64 n = a->n;
  if (kind == PMMF_PRECOND_SSOR && !(omega > 0.0 && omega < 2.0))
    fail(PMMF_INVALID_ARGUMENT, "ssor: omega must be in (0, 2)");
  const std::vector<Trip> t = to_triplets_kept(a);
  if (kind == PMMF_PRECOND_JACOBI) {  // solver.hpp:222-233
    p->scale.assign(static_cast<size_t>(n), 0.0);
    for (const Trip& e : t)
      if (e.r == e.c && e.v > 0.0) p->scale[e.r] = 1.0 / std::sqrt(e.v);
  } else if (kind == PMMF_PRECOND_SSOR) {  // solver.hpp:237-267
    p->lower = extract_lower(t, n);
    for (i64 i = 0; i < n; ++i)
      if (p->lower.diag[i] == 0.0) fail(PMMF_NUMERIC, "ssor: zero diagonal entry at row " + std::to_string(i));
    p->sqrt_d.resize(static_cast<size_t>(n));
    const double front = std::sqrt((2.0 - omega) / omega);
    for (i64 i = 0; i < n; ++i) {
      const double d = p->lower.diag[i];
      p->sqrt_d[i] = front * std::sqrt(std::abs(d));
      p->lower.diag[i] = d / omega;
    }
  } else if (kind == PMMF_PRECOND_IC) {  // solver.hpp:278-340
    const LowerTri pattern = extract_lower(t, n);
    if (!ic_attempt(pattern, 0.0, p->lower)) {
      std::vector<double> row_abs(static_cast<size_t>(n), 0.0), diag(static_cast<size_t>(n), 0.0);
      for (const Trip& e : t) {
        row_abs[e.r] += std::abs(e.v);
        if (e.r == e.c) diag[e.r] = e.v;
      }
      double alpha = 0.0;
      for (i64 i = 0; i < n; ++i) {
        if (!(diag[i] > 0.0))
          fail(PMMF_NUMERIC, "ic: non-positive diagonal, cannot compensate row " + std::to_string(i));
        alpha = std::max(alpha, row_abs[i] / diag[i]);
      }
      p->compensated = 1;
      p->alpha = alpha;
      if (!ic_attempt(pattern, alpha, p->lower))
        fail(PMMF_NUMERIC, "ic: breakdown persists after diagonal compensation");
    }
  } else {
    fail(PMMF_INVALID_ARGUMENT, "preconditioner: unknown kind");
  }
  return p;
}

}  // namespace orc

// =================================================================== C-ABI
using namespace orc;

namespace {
void set_err(char* err, size_t n, const std::string& m) {
  if (!err || !n) return;
  const size_t k = std::min(n - 1, m.size());
  std::memcpy(err, m.data(), k);
  err[k] = '\0';
}
template <typename F>
int guarded(char* err, size_t n, F&& f) {
  try {
    f();
    return PMMF_OK;
  } catch (const Error& e) {
    set_err(err, n, e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_err(err, n, e.what());
    return PMMF_INTERNAL;
  }
}
}  // namespace

extern "C" {

int pmmf_oracle_factorize(const pmmf_b200_coo* a, const pmmf_b200_params* pp, void** out, char* err,
                          size_t errlen) {
  return guarded(err, errlen, [&] {
    if (a->on_device) fail(PMMF_INVALID_ARGUMENT, "oracle takes host buffers only");
    Params p{pp->k, pp->n_stages, pp->eta, pp->m_target, pp->c_min, pp->c_max, pp->d_max, pp->bypass_enabled != 0,
             pp->core_min, pp->core_cap, pp->seed};
    *out = new Result(factorize(a, p));
  });
}
int pmmf_oracle_result_summary(void* h, pmmf_b200_summary* o) {
  auto* r = static_cast<Result*>(h);
  o->n = r->n;
  o->n_stages = static_cast<int64_t>(r->stages.size());
  o->k = r->k;
  o->core_size = static_cast<int64_t>(r->core_idx.size());
  o->n_diagonal = static_cast<int64_t>(r->diag.size());
  o->trivial = r->trivial;
  o->residual_sq = r->residual_sq;
  return PMMF_OK;
}
int pmmf_oracle_result_active_history(void* h, int64_t* o) {
  auto* r = static_cast<Result*>(h);
  std::copy(r->hist.begin(), r->hist.end(), o);
  return PMMF_OK;
}
int pmmf_oracle_result_stage_sizes(void* h, int64_t s, pmmf_b200_stage_sizes* o) {
  auto* r = static_cast<Result*>(h);
  if (s < 0 || s >= static_cast<int64_t>(r->stages.size())) return PMMF_OUT_OF_RANGE;
  const Stage& st = r->stages[s];
  o->n_clusters = static_cast<int64_t>(st.off.size()) - 1;
  o->partition_size = static_cast<int64_t>(st.members.size());
  o->n_rotations = static_cast<int64_t>(st.rots.size());
  o->n_eliminated = static_cast<int64_t>(st.elim.size());
  o->n_bypassed = static_cast<int64_t>(st.bypassed.size());
  return PMMF_OK;
}
int pmmf_oracle_result_stage(void* h, int64_t s, int64_t* offs, int64_t* mem, int64_t* ri, double* rq,
                             int64_t* ei, double* ed, double* em, int64_t* by) {
  auto* r = static_cast<Result*>(h);
  if (s < 0 || s >= static_cast<int64_t>(r->stages.size())) return PMMF_OUT_OF_RANGE;
  const Stage& st = r->stages[s];
  std::copy(st.off.begin(), st.off.end(), offs);
  std::copy(st.members.begin(), st.members.end(), mem);
  const int64_t k = r->k;
  for (size_t t = 0; t < st.rots.size(); ++t)
    for (int64_t a = 0; a < k; ++a) {
      ri[t * k + a] = st.rots[t].idx[a];
      for (int64_t b = 0; b < k; ++b) rq[(t * k + a) * k + b] = st.rots[t].q(a, b);
    }
  for (size_t e = 0; e < st.elim.size(); ++e) {
    ei[e] = st.elim[e].index;
    ed[e] = st.elim[e].diag;
    em[e] = st.elim[e].mass;
  }
  std::copy(st.bypassed.begin(), st.bypassed.end(), by);
  return PMMF_OK;
}
int pmmf_oracle_result_core(void* h, int64_t* ci, double* core, int64_t* di, double* dv) {
  auto* r = static_cast<Result*>(h);
  const int64_t g = static_cast<int64_t>(r->core_idx.size());
  std::copy(r->core_idx.begin(), r->core_idx.end(), ci);
  for (int64_t i = 0; i < g * g; ++i) core[i] = r->core.d[i];
  for (size_t i = 0; i < r->diag.size(); ++i) {
    di[i] = r->diag[i].first;
    dv[i] = r->diag[i].second;
  }
  return PMMF_OK;
}
int pmmf_oracle_result_stats(void* h, double* phases, int64_t* info) {
  auto* r = static_cast<Result*>(h);
  std::copy(r->phases, r->phases + 6, phases);
  for (size_t s = 0; s < r->info.size(); ++s) std::copy(r->info[s].begin(), r->info[s].end(), info + 7 * s);
  return PMMF_OK;
}
void pmmf_oracle_result_free(void* h) { delete static_cast<Result*>(h); }

int pmmf_oracle_operator_create(void* result, double thr, void** op, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto* o = new Operator();
    o->f = std::make_shared<Result>(*static_cast<Result*>(result));
    o->thr = thr;
    Mat a = o->f->core;  // jacobi_eigensystem, dense.hpp:191-199
    Mat q = jacobi_diagonalize(a);
    o->eval.resize(a.r);
    for (i64 i = 0; i < a.r; ++i) o->eval[i] = a(i, i);
    o->evec = transposed(q);
    for (double l : o->eval)
      if (l < -thr) ++o->neg;
    for (const auto& [i, d] : o->f->diag)
      if (d < -thr) ++o->neg;
    *op = o;
  });
}
int pmmf_oracle_operator_apply(void* op, int32_t mode, int64_t nrhs, const double* in, double* out,
                               int32_t on_device, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (on_device) fail(PMMF_INVALID_ARGUMENT, "oracle takes host buffers only");
    auto* o = static_cast<Operator*>(op);
    const i64 n = o->f->n;
    for (int64_t r = 0; r < nrhs; ++r) o->apply(mode, in + r * n, out + r * n);
  });
}
int pmmf_oracle_operator_zeroed_negatives(void* op, int64_t* out) {
  *out = static_cast<Operator*>(op)->neg;
  return PMMF_OK;
}
void pmmf_oracle_operator_free(void* op) { delete static_cast<Operator*>(op); }

// run_solve_experiment + pcg_symmetric (solver.hpp:112-167, :368-416).
static void solve_with(const pmmf_b200_coo* a, const Pre* pc, const pmmf_b200_solve_config* cfg, int32_t* iters,
                       int32_t* conv, int32_t* brk, double* res, double* wall_ms) {
  {
    if (!(cfg->tol > 0.0)) fail(PMMF_INVALID_ARGUMENT, "SolveConfig: tol must be positive");
    if (cfg->max_iter < 1) fail(PMMF_INVALID_ARGUMENT, "SolveConfig: max_iter < 1");
    if (cfg->rhs_count < 1) fail(PMMF_INVALID_ARGUMENT, "SolveConfig: rhs_count < 1");
    const auto start = clk::now();
    SpMat S = make_spmat(a);
    const i64 n = a->n;
    auto pre = [&](int side, const std::vector<double>& x, std::vector<double>& y) {
      if (pc)
        pc->apply(side, x.data(), y.data());
      else
        y = x;
    };
    const i64 stride = cfg->max_iter + 1;
    for (int rhs = 0; rhs < cfg->rhs_count; ++rhs) {
      Rng rng(derive(cfg->seed, {0xB0u, static_cast<uint64_t>(rhs)}));
      std::vector<double> b(static_cast<size_t>(n));
      {  // Rng::normal (rng.hpp:56-71), polar method with spare
        bool has = false;
        double spare = 0.0;
        for (auto& v : b) {
          if (has) {
            has = false;
            v = spare;
            continue;
          }
          double u, w, s;
          do {
            u = 2.0 * (static_cast<double>(rng.next() >> 11) * 0x1.0p-53) - 1.0;
            w = 2.0 * (static_cast<double>(rng.next() >> 11) * 0x1.0p-53) - 1.0;
            s = u * u + w * w;
          } while (s >= 1.0 || s == 0.0);
          const double f = std::sqrt(-2.0 * std::log(s) / s);
          spare = w * f;
          has = true;
          v = u * f;
        }
      }
      const double nb = std::sqrt(vdot(b, b));
      if (nb > 0.0)
        for (auto& v : b) v /= nb;
      double* trace = res + static_cast<i64>(rhs) * stride;
      for (i64 i = 0; i < stride; ++i) trace[i] = NAN;
      iters[rhs] = 0;
      conv[rhs] = 0;
      brk[rhs] = 0;
      const double bnorm = std::sqrt(vdot(b, b));
      trace[0] = bnorm;
      if (bnorm == 0.0) {
        conv[rhs] = 1;
        continue;
      }
      std::vector<double> y(n, 0.0), r(n), p(n), w(n), t1(n), t2(n), x(n), tr(n);
      pre(0, b, r);
      p = r;
      double rr = vdot(r, r);
      for (int k = 1; k <= cfg->max_iter; ++k) {
        pre(1, p, t1);
        spmv(S, t1, t2);
        pre(0, t2, w);
        const double pap = vdot(p, w);
        if (!(pap > 0.0)) {
          brk[rhs] = 1;
          break;
        }
        const double alpha = rr / pap;
        for (i64 i = 0; i < n; ++i) y[i] += alpha * p[i];
        for (i64 i = 0; i < n; ++i) r[i] -= alpha * w[i];
        pre(1, y, x);
        spmv(S, x, t2);
        for (i64 i = 0; i < n; ++i) tr[i] = b[i] - t2[i];
        const double rs = std::sqrt(vdot(tr, tr));
        trace[k] = rs;
        iters[rhs] = k;
        if (rs / bnorm <= cfg->tol) {
          conv[rhs] = 1;
          break;
        }
        const double rn = vdot(r, r);
        const double beta = rn / rr;
        rr = rn;
        for (i64 i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
      }
    }
    *wall_ms = ms_since(start);
  }
}

int pmmf_oracle_solve(const pmmf_b200_coo* a, void* op, const pmmf_b200_solve_config* cfg, int32_t* iters,
                      int32_t* conv, int32_t* brk, double* res, double* wall_ms, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    std::unique_ptr<Pre> pc;
    if (op) {
      pc = std::make_unique<Pre>();
      pc->kind = PMMF_PRECOND_PMMF;
      pc->n = a->n;
      pc->op = static_cast<Operator*>(op);
    }
    solve_with(a, pc.get(), cfg, iters, conv, brk, res, wall_ms);
  });
}

int pmmf_oracle_solve_precond(const pmmf_b200_coo* a, void* pc, const pmmf_b200_solve_config* cfg, int32_t* iters,
                              int32_t* conv, int32_t* brk, double* res, double* wall_ms, char* err, size_t errlen) {
  return guarded(err, errlen,
                 [&] { solve_with(a, static_cast<const Pre*>(pc), cfg, iters, conv, brk, res, wall_ms); });
}

int pmmf_oracle_precond_create(const pmmf_b200_coo* a, int32_t kind, double omega, void** out, char* err,
                               size_t errlen) {
  return guarded(err, errlen, [&] { *out = make_pre(a, kind, omega).release(); });
}

int pmmf_oracle_precond_from_operator(void* op, void** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto p = std::make_unique<Pre>();
    p->kind = PMMF_PRECOND_PMMF;
    p->op = static_cast<Operator*>(op);
    p->n = p->op->f->n;
    *out = p.release();
  });
}

int pmmf_oracle_precond_apply(void* pc, int32_t side, int64_t nrhs, const double* in, double* out, int32_t on_device,
                              char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (on_device) fail(PMMF_INVALID_ARGUMENT, "oracle takes host buffers only");
    const auto* p = static_cast<const Pre*>(pc);
    for (int64_t r = 0; r < nrhs; ++r) p->apply(side, in + r * p->n, out + r * p->n);
  });
}

int pmmf_oracle_precond_info(void* pc, int32_t* kind, int32_t* compensated, double* alpha) {
  const auto* p = static_cast<const Pre*>(pc);
  *kind = p->kind;
  *compensated = p->compensated;
  *alpha = p->alpha;
  return PMMF_OK;
}

void pmmf_oracle_precond_free(void* pc) { delete static_cast<Pre*>(pc); }

// nystrom_uniform (transform_ops.hpp:252-307)
int pmmf_oracle_nystrom_uniform(const pmmf_b200_coo* a, int64_t m, uint64_t seed, int64_t cap, double* fro,
                                int64_t* columns, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const i64 n = a->n;
    if (m < 1 || m > n) fail(PMMF_INVALID_ARGUMENT, "nystrom_uniform: m out of range");
    if (n > cap) fail(PMMF_NUMERIC, "dense_from_blocked: dimension exceeds cap");
    Mat dense(n, n);
    for (const Trip& e : to_triplets_kept(a)) dense(e.r, e.c) = e.v;
    std::vector<i64> ids(static_cast<size_t>(n));
    std::iota(ids.begin(), ids.end(), i64{0});
    Rng rng(seed);
    for (i64 t = 0; t < m; ++t) {
      const i64 pick = t + static_cast<i64>(rng.below(static_cast<uint64_t>(n - t)));
      std::swap(ids[t], ids[pick]);
    }
    std::vector<i64> sel(ids.begin(), ids.begin() + m);
    std::sort(sel.begin(), sel.end());
    std::copy(sel.begin(), sel.end(), columns);
    Mat c(n, m), w(m, m);
    for (i64 j = 0; j < m; ++j) {
      for (i64 i = 0; i < n; ++i) c(i, j) = dense(i, sel[j]);
      for (i64 i = 0; i < m; ++i) w(i, j) = dense(sel[i], sel[j]);
    }
    Mat q = jacobi_diagonalize(w);  // jacobi_eigensystem: values = diag(w), vectors = q^T
    double max_mag = 0.0;
    for (i64 e = 0; e < m; ++e) max_mag = std::max(max_mag, std::abs(w(e, e)));
    const double threshold = 1e-10 * max_mag;
    Mat pinv(m, m);
    for (i64 e = 0; e < m; ++e) {
      const double lambda = w(e, e);
      if (std::abs(lambda) <= threshold) continue;
      const double inv = 1.0 / lambda;
      for (i64 i = 0; i < m; ++i)
        for (i64 j = 0; j < m; ++j) pinv(i, j) += inv * q(e, i) * q(e, j);
    }
    Mat approx = multiply(multiply(c, pinv), transposed(c));
    double s = 0.0;
    for (i64 i = 0; i < n; ++i)
      for (i64 j = 0; j < n; ++j) {
        const double d = dense(i, j) - approx(i, j);
        s += d * d;
      }
    *fro = std::sqrt(s);
  });
}

int pmmf_oracle_rotation_from_gram(int32_t k, const double* g, double* q, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    Mat gs(k, k);
    std::copy(g, g + k * k, gs.d.begin());
    Mat qm = rotation_from_gram(gs);
    std::copy(qm.d.begin(), qm.d.end(), q);
  });
}

}  // extern "C"
