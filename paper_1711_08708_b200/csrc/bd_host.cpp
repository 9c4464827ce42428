// Host-side setup of the inner preconditioners (compiled with
// -ffp-contract=off so the IC(0) sweep rounds exactly like the numpy scalar
// arithmetic of the reference).
#include "bd_host.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <numeric>
#include <unordered_map>

namespace bd {

namespace {

// Sorted-merge dot product of two sparse row prefixes
// (_sparse_row_dot, bd/precond.py:201-216): products accumulated left to
// right in ascending column order, starting from 0.0.
double merge_dot(const int32_t* ca, const double* va, int64_t na, const int32_t* cb,
                 const double* vb, int64_t nb) {
  int64_t ia = 0, ib = 0;
  double out = 0.0;
  while (ia < na && ib < nb) {
    const int32_t a = ca[ia], b = cb[ib];
    if (a == b) {
      const double prod = va[ia] * vb[ib];
      out = out + prod;
      ++ia;
      ++ib;
    } else if (a < b) {
      ++ia;
    } else {
      ++ib;
    }
  }
  return out;
}

// One factorisation sweep over tril(A) (bd/precond.py:170-189); false on a
// non-positive pivot.  `val` holds the (possibly diagonal-scaled) copy.
bool ic0_sweep(const HostCsr& t, std::vector<double>& val) {
  const int64_t* ip = t.indptr.data();
  const int32_t* ci = t.indices.data();
  double* v = val.data();
  for (int64_t i = 0; i < t.n; ++i) {
    const int64_t rs = ip[i], re = ip[i + 1];
    for (int64_t idx = rs; idx < re; ++idx) {
      const int32_t j = ci[idx];
      const int64_t js = ip[j], je = ip[j + 1];
      const double s = merge_dot(ci + rs, v + rs, idx - rs, ci + js, v + js, (je - 1) - js);
      if (j == i) {
        const double pivot = v[idx] - s;
        if (pivot <= 0.0) return false;
        v[idx] = std::sqrt(pivot);
      } else {
        v[idx] = (v[idx] - s) / v[ip[j + 1] - 1];
      }
    }
  }
  return true;
}

}  // namespace

int ic0_factor(const HostCsr& a, int max_restarts, HostCsr* lower, int* restarts_used,
               std::string* msg) {
  // lower = tril(a) keeping stored entries (bd/precond.py:158)
  HostCsr t;
  t.n = a.n;
  t.indptr.assign(a.n + 1, 0);
  for (int64_t i = 0; i < a.n; ++i) {
    int64_t c = 0;
    for (int64_t p = a.indptr[i]; p < a.indptr[i + 1]; ++p)
      if (a.indices[p] <= i) ++c;
    t.indptr[i + 1] = t.indptr[i] + c;
  }
  t.indices.resize(t.indptr[a.n]);
  t.values.resize(t.indptr[a.n]);
  for (int64_t i = 0; i < a.n; ++i) {
    int64_t o = t.indptr[i];
    for (int64_t p = a.indptr[i]; p < a.indptr[i + 1]; ++p)
      if (a.indices[p] <= i) {
        t.indices[o] = a.indices[p];
        t.values[o] = a.values[p];
        ++o;
      }
  }
  // diagonal must be the last stored entry of every row (:160-166)
  std::vector<int64_t> diag_pos(a.n);
  for (int64_t i = 0; i < a.n; ++i) {
    const int64_t last = t.indptr[i + 1] - 1;
    if (last < t.indptr[i] || t.indices[last] != i) {
      char buf[96];
      std::snprintf(buf, sizeof buf, "missing diagonal entry in row %lld", (long long)i);
      *msg = buf;
      return 1;
    }
    diag_pos[i] = last;
  }
  double shift = 1.0;
  for (int attempt = 0; attempt <= max_restarts; ++attempt) {
    std::vector<double> val = t.values;
    if (shift != 1.0)
      for (int64_t i = 0; i < a.n; ++i) val[diag_pos[i]] = val[diag_pos[i]] * shift;
    if (ic0_sweep(t, val)) {
      lower->n = t.n;
      lower->indptr = t.indptr;
      lower->indices = t.indices;
      lower->values = std::move(val);
      if (restarts_used) *restarts_used = attempt;
      return 0;
    }
    shift = shift * (1.0 + 1e-3);
  }
  char buf[128];
  std::snprintf(buf, sizeof buf,
                "incomplete Cholesky failed after %d diagonal shift restarts", max_restarts);
  *msg = buf;
  return 2;
}

HostCsr transpose(const HostCsr& a) {
  HostCsr t;
  // square factors only on this path
  t.n = a.n;
  t.indptr.assign(a.n + 1, 0);
  const int64_t nnz = a.nnz();
  for (int64_t p = 0; p < nnz; ++p) t.indptr[a.indices[p] + 1]++;
  for (int64_t i = 0; i < a.n; ++i) t.indptr[i + 1] += t.indptr[i];
  t.indices.resize(nnz);
  t.values.resize(nnz);
  std::vector<int64_t> next(t.indptr.begin(), t.indptr.end() - 1);
  for (int64_t i = 0; i < a.n; ++i)
    for (int64_t p = a.indptr[i]; p < a.indptr[i + 1]; ++p) {
      const int64_t o = next[a.indices[p]]++;
      t.indices[o] = (int32_t)i;
      t.values[o] = a.values[p];
    }
  return t;
}

int64_t row_levels(const HostCsr& t, bool lower, std::vector<int32_t>* level) {
  level->assign(t.n, 0);
  int32_t depth = 0;
  auto visit = [&](int64_t i) {
    int32_t lv = 0;
    for (int64_t p = t.indptr[i]; p < t.indptr[i + 1]; ++p) {
      const int32_t j = t.indices[p];
      if (j != i) lv = std::max(lv, (*level)[j] + 1);
    }
    (*level)[i] = lv;
    depth = std::max(depth, lv + 1);
  };
  if (lower)
    for (int64_t i = 0; i < t.n; ++i) visit(i);
  else
    for (int64_t i = t.n - 1; i >= 0; --i) visit(i);
  return depth;
}

void build_schedule(const std::vector<int32_t>& level, int64_t depth, int pad,
                    std::vector<int32_t>* tasks) {
  std::vector<int64_t> count(depth + 1, 0);
  for (int32_t lv : level) count[lv + 1]++;
  std::vector<int64_t> start(depth + 1, 0);  // padded offsets
  for (int64_t l = 0; l < depth; ++l) {
    const int64_t c = count[l + 1];
    start[l + 1] = start[l] + (c + pad - 1) / pad * pad;
  }
  tasks->assign(start[depth], -1);
  std::vector<int64_t> fill(start.begin(), start.end() - 1);
  for (int64_t i = 0; i < (int64_t)level.size(); ++i) (*tasks)[fill[level[i]]++] = (int32_t)i;
}

// ---------------------------------------------------------------------------
// Nested dissection on the symmetric pattern.
namespace {

struct Graph {
  int64_t n;
  std::vector<int64_t> xadj;
  std::vector<int32_t> adj;
};

Graph symmetric_graph(const HostCsr& a) {
  // pattern of A + A^T without the diagonal
  std::vector<int64_t> deg(a.n, 0);
  for (int64_t i = 0; i < a.n; ++i)
    for (int64_t p = a.indptr[i]; p < a.indptr[i + 1]; ++p) {
      const int32_t j = a.indices[p];
      if (j == i) continue;
      deg[i]++;
      deg[j]++;
    }
  Graph g;
  g.n = a.n;
  g.xadj.assign(a.n + 1, 0);
  for (int64_t i = 0; i < a.n; ++i) g.xadj[i + 1] = g.xadj[i] + deg[i];
  g.adj.resize(g.xadj[a.n]);
  std::vector<int64_t> pos(g.xadj.begin(), g.xadj.end() - 1);
  for (int64_t i = 0; i < a.n; ++i)
    for (int64_t p = a.indptr[i]; p < a.indptr[i + 1]; ++p) {
      const int32_t j = a.indices[p];
      if (j == i) continue;
      g.adj[pos[i]++] = j;
      g.adj[pos[j]++] = (int32_t)i;
    }
  // dedupe each adjacency list
  std::vector<int64_t> nx(a.n + 1, 0);
  int64_t w = 0;
  for (int64_t i = 0; i < a.n; ++i) {
    auto b = g.adj.begin() + g.xadj[i], e = g.adj.begin() + g.xadj[i + 1];
    std::sort(b, e);
    auto u = std::unique(b, e);
    const int64_t len = u - b;
    std::copy(b, u, g.adj.begin() + w);
    nx[i] = w;
    w += len;
  }
  nx[a.n] = w;
  g.adj.resize(w);
  g.xadj = std::move(nx);
  return g;
}

struct NdState {
  const Graph* g;
  std::vector<int32_t> part;   // subset id of each node
  std::vector<int32_t> dist;   // BFS scratch
  std::vector<int32_t>* out;
  int32_t next_id = 1;
};

// BFS inside subset `id` from `root`; fills order (visited nodes) and dist.
void bfs(NdState& st, int32_t id, int32_t root, std::vector<int32_t>& order) {
  order.clear();
  order.push_back(root);
  st.dist[root] = 0;
  for (size_t h = 0; h < order.size(); ++h) {
    const int32_t u = order[h];
    for (int64_t p = st.g->xadj[u]; p < st.g->xadj[u + 1]; ++p) {
      const int32_t v = st.g->adj[p];
      if (st.part[v] == id && st.dist[v] < 0) {
        st.dist[v] = st.dist[u] + 1;
        order.push_back(v);
      }
    }
  }
}

void reset_dist(NdState& st, const std::vector<int32_t>& nodes) {
  for (int32_t u : nodes) st.dist[u] = -1;
}

void dissect(NdState& st, std::vector<int32_t> nodes, int32_t id) {
  const size_t kLeaf = 48;
  if (nodes.size() <= kLeaf) {
    std::sort(nodes.begin(), nodes.end());
    for (int32_t u : nodes) st.out->push_back(u);
    return;
  }
  // pseudo-peripheral root: repeated BFS to a farthest node
  std::vector<int32_t> order;
  int32_t root = *std::min_element(nodes.begin(), nodes.end());
  int32_t ecc = -1;
  for (int rep = 0; rep < 4; ++rep) {
    bfs(st, id, root, order);
    const int32_t far = order.back();
    const int32_t e = st.dist[far];
    reset_dist(st, order);
    if (e <= ecc) break;
    ecc = e;
    root = far;
  }
  bfs(st, id, root, order);
  if (order.size() < nodes.size()) {
    // disconnected: split off this component, recurse on both
    std::vector<int32_t> comp(order), rest;
    reset_dist(st, order);
    const int32_t id_c = st.next_id++, id_r = st.next_id++;
    for (int32_t u : comp) st.part[u] = id_c;
    for (int32_t u : nodes)
      if (st.part[u] == id) {
        st.part[u] = id_r;
        rest.push_back(u);
      }
    dissect(st, std::move(comp), id_c);
    dissect(st, std::move(rest), id_r);
    return;
  }
  const int32_t maxd = st.dist[order.back()];
  if (maxd < 2) {  // (near-)clique: no useful separator
    reset_dist(st, order);
    std::sort(nodes.begin(), nodes.end());
    for (int32_t u : nodes) st.out->push_back(u);
    return;
  }
  // level sizes; separator = the smallest level among those near the median
  std::vector<int64_t> lsize(maxd + 1, 0);
  for (int32_t u : order) lsize[st.dist[u]]++;
  int64_t acc = 0;
  int32_t mid = 1;
  for (int32_t l = 0; l <= maxd; ++l) {
    acc += lsize[l];
    if (2 * acc >= (int64_t)nodes.size()) {
      mid = l;
      break;
    }
  }
  mid = std::min(std::max(mid, 1), maxd - 1);
  int32_t best = mid;
  const int32_t span = std::max<int32_t>(1, maxd / 8);
  for (int32_t l = std::max(1, mid - span); l <= std::min(maxd - 1, mid + span); ++l)
    if (lsize[l] < lsize[best]) best = l;
  std::vector<int32_t> a, b, s;
  for (int32_t u : order) {
    const int32_t d = st.dist[u];
    if (d < best) a.push_back(u);
    else if (d > best) b.push_back(u);
    else s.push_back(u);
  }
  reset_dist(st, order);
  const int32_t ia = st.next_id++, ib = st.next_id++, is = st.next_id++;
  for (int32_t u : a) st.part[u] = ia;
  for (int32_t u : b) st.part[u] = ib;
  for (int32_t u : s) st.part[u] = is;
  dissect(st, std::move(a), ia);
  dissect(st, std::move(b), ib);
  std::sort(s.begin(), s.end());
  for (int32_t u : s) st.out->push_back(u);
}

}  // namespace

void nested_dissection(const HostCsr& a, std::vector<int32_t>* perm) {
  Graph g = symmetric_graph(a);
  NdState st;
  st.g = &g;
  st.part.assign(a.n, 0);
  st.dist.assign(a.n, -1);
  perm->clear();
  perm->reserve(a.n);
  st.out = perm;
  std::vector<int32_t> all(a.n);
  std::iota(all.begin(), all.end(), 0);
  dissect(st, std::move(all), 0);
}

// ---------------------------------------------------------------------------
// Up-looking sparse Cholesky of C = P A P^T.
int cholesky(const HostCsr& a, const std::vector<int32_t>& perm, HostCsr* lower,
             std::string* msg) {
  const int64_t n = a.n;
  std::vector<int32_t> inv(n);
  for (int64_t k = 0; k < n; ++k) inv[perm[k]] = (int32_t)k;
  // C rows, lower part (cols <= row) sorted
  std::vector<int64_t> cp(n + 1, 0);
  for (int64_t k = 0; k < n; ++k) {
    const int32_t r = perm[k];
    int64_t c = 0;
    for (int64_t p = a.indptr[r]; p < a.indptr[r + 1]; ++p)
      if (inv[a.indices[p]] <= k) ++c;
    cp[k + 1] = cp[k] + c;
  }
  std::vector<int32_t> ci(cp[n]);
  std::vector<double> cx(cp[n]);
  for (int64_t k = 0; k < n; ++k) {
    const int32_t r = perm[k];
    int64_t o = cp[k];
    for (int64_t p = a.indptr[r]; p < a.indptr[r + 1]; ++p) {
      const int32_t j = inv[a.indices[p]];
      if (j <= k) {
        ci[o] = j;
        cx[o] = a.values[p];
        ++o;
      }
    }
  }
  // elimination tree
  std::vector<int32_t> parent(n, -1), anc(n, -1);
  for (int64_t k = 0; k < n; ++k) {
    for (int64_t p = cp[k]; p < cp[k + 1]; ++p) {
      int32_t i = ci[p];
      while (i != -1 && i < k) {
        const int32_t nx = anc[i];
        anc[i] = (int32_t)k;
        if (nx == -1) parent[i] = (int32_t)k;
        i = nx;
      }
    }
  }
  // row patterns via ereach; first pass counts columns
  std::vector<int32_t> s(n), mark(n, -1);
  auto ereach = [&](int64_t k) -> int64_t {
    int64_t top = n;
    mark[k] = (int32_t)k;
    for (int64_t p = cp[k]; p < cp[k + 1]; ++p) {
      int32_t i = ci[p];
      if (i >= k) continue;
      int64_t len = 0;
      for (; mark[i] != k; i = parent[i]) {
        s[len++] = i;
        mark[i] = (int32_t)k;
      }
      while (len > 0) s[--top] = s[--len];
    }
    return top;
  };
  std::vector<int64_t> colcount(n, 1);
  for (int64_t k = 0; k < n; ++k) {
    const int64_t top = ereach(k);
    for (int64_t p = top; p < n; ++p) colcount[s[p]]++;
  }
  std::fill(mark.begin(), mark.end(), -1);
  // CSC of L, diagonal first in each column
  std::vector<int64_t> lp(n + 1, 0);
  for (int64_t j = 0; j < n; ++j) lp[j + 1] = lp[j] + colcount[j];
  std::vector<int32_t> li(lp[n]);
  std::vector<double> lx(lp[n]);
  std::vector<int64_t> c(lp.begin(), lp.end() - 1);
  std::vector<double> x(n, 0.0);
  for (int64_t k = 0; k < n; ++k) {
    const int64_t top = ereach(k);
    double d = 0.0;
    for (int64_t p = cp[k]; p < cp[k + 1]; ++p) {
      if (ci[p] == k) d += cx[p];
      else x[ci[p]] += cx[p];
    }
    for (int64_t p = top; p < n; ++p) {
      const int32_t i = s[p];
      const double lki = x[i] / lx[lp[i]];
      x[i] = 0.0;
      for (int64_t q = lp[i] + 1; q < c[i]; ++q) x[li[q]] -= lx[q] * lki;
      d -= lki * lki;
      const int64_t o = c[i]++;
      li[o] = (int32_t)k;
      lx[o] = lki;
    }
    if (!(d > 0.0)) {
      char buf[128];
      std::snprintf(buf, sizeof buf, "non-positive pivot %g at row %lld", d, (long long)k);
      *msg = buf;
      return 2;
    }
    const int64_t o = c[k]++;
    li[o] = (int32_t)k;
    lx[o] = std::sqrt(d);
  }
  // CSC(L) read as CSR is L^T; transpose gives CSR(L) with the diagonal last.
  HostCsr lt;
  lt.n = n;
  lt.indptr = std::move(lp);
  lt.indices = std::move(li);
  lt.values = std::move(lx);
  *lower = transpose(lt);
  return 0;
}

}  // namespace bd

// ---------------------------------------------------------------------------
// Tiled schedules for the cooperative triangular-solve kernel.
namespace bd {

namespace {

// BFS inside the node subset `nodes` (membership: mark[u] == id) from a
// pseudo-peripheral node; returns nodes sorted by BFS distance (unreached
// components appended).
void bfs_order(const Graph& g, std::vector<int32_t>& nodes, std::vector<int32_t>& mark,
               std::vector<int32_t>& dist, int32_t id, std::vector<int32_t>* out) {
  auto run = [&](int32_t root, std::vector<int32_t>& order) {
    order.clear();
    order.push_back(root);
    dist[root] = 0;
    for (size_t h = 0; h < order.size(); ++h) {
      const int32_t u = order[h];
      for (int64_t p = g.xadj[u]; p < g.xadj[u + 1]; ++p) {
        const int32_t v = g.adj[p];
        if (mark[v] == id && dist[v] < 0) {
          dist[v] = dist[u] + 1;
          order.push_back(v);
        }
      }
    }
  };
  std::vector<int32_t> order;
  int32_t root = *std::min_element(nodes.begin(), nodes.end());
  int32_t ecc = -1;
  for (int rep = 0; rep < 3; ++rep) {
    run(root, order);
    const int32_t far = order.back(), e = dist[far];
    for (int32_t u : order) dist[u] = -1;
    if (e <= ecc) break;
    ecc = e;
    root = far;
  }
  run(root, order);
  for (int32_t u : order) dist[u] = -1;
  out->swap(order);
  if (out->size() < nodes.size()) {  // disconnected remainder, appended in index order
    for (int32_t u : *out) mark[u] = -2 - id;
    std::vector<int32_t> rest;
    for (int32_t u : nodes)
      if (mark[u] == id) rest.push_back(u);
    for (int32_t u : *out) mark[u] = id;
    out->insert(out->end(), rest.begin(), rest.end());
  }
}

void bisect(const Graph& g, std::vector<int32_t> nodes, int parts, int32_t first_part,
            std::vector<int32_t>& mark, std::vector<int32_t>& dist, int32_t& next_id,
            std::vector<int32_t>* part) {
  if (parts <= 1 || nodes.size() <= 1) {
    for (int32_t u : nodes) (*part)[u] = first_part;
    return;
  }
  const int32_t id = next_id++;
  for (int32_t u : nodes) mark[u] = id;
  std::vector<int32_t> order;
  bfs_order(g, nodes, mark, dist, id, &order);
  const int pa = parts / 2, pb = parts - pa;
  const size_t cut = (size_t)((double)order.size() * pa / parts + 0.5);
  std::vector<int32_t> a(order.begin(), order.begin() + cut), b(order.begin() + cut, order.end());
  bisect(g, std::move(a), pa, first_part, mark, dist, next_id, part);
  bisect(g, std::move(b), pb, first_part + pa, mark, dist, next_id, part);
}

}  // namespace

void partition_rows(const HostCsr& a, int parts, std::vector<int32_t>* part) {
  Graph g = symmetric_graph(a);
  part->assign(a.n, 0);
  std::vector<int32_t> mark(a.n, -1), dist(a.n, -1);
  std::vector<int32_t> all(a.n);
  std::iota(all.begin(), all.end(), 0);
  int32_t next_id = 0;
  bisect(g, std::move(all), parts, 0, mark, dist, next_id, part);
}

namespace {
void rcb(int64_t lo_idx, std::vector<int32_t>& ids, size_t b, size_t e, int dim, const double* x,
         int parts, int32_t first, std::vector<int32_t>* part) {
  if (parts <= 1 || e - b <= 1) {
    for (size_t k = b; k < e; ++k) (*part)[ids[k]] = first;
    return;
  }
  int axis = 0;
  double best = -1.0;
  for (int d = 0; d < dim; ++d) {
    double mn = 1e300, mx = -1e300;
    for (size_t k = b; k < e; ++k) {
      const double v = x[(int64_t)ids[k] * dim + d];
      mn = std::min(mn, v);
      mx = std::max(mx, v);
    }
    if (mx - mn > best) {
      best = mx - mn;
      axis = d;
    }
  }
  const int pa = parts / 2, pb = parts - pa;
  const size_t cut = b + (size_t)((double)(e - b) * pa / parts + 0.5);
  std::nth_element(ids.begin() + b, ids.begin() + cut, ids.begin() + e, [&](int32_t u, int32_t v) {
    const double xu = x[(int64_t)u * dim + axis], xv = x[(int64_t)v * dim + axis];
    return xu < xv || (xu == xv && u < v);
  });
  rcb(lo_idx, ids, b, cut, dim, x, pa, first, part);
  rcb(lo_idx, ids, cut, e, dim, x, pb, first + pa, part);
}
}  // namespace

void partition_coords(int64_t n, int dim, const double* coords, int parts,
                      std::vector<int32_t>* part) {
  part->assign(n, 0);
  std::vector<int32_t> ids(n);
  std::iota(ids.begin(), ids.end(), 0);
  rcb(0, ids, 0, (size_t)n, dim, coords, parts, 0, part);
}

bool build_tile_schedule(const HostCsr& t, bool lower, const std::vector<int32_t>& part,
                         int parts, int G, int R, TileSchedule* out, bool entry_major) {
  const int64_t n = t.n;
  std::vector<int32_t> level;
  out->depth = row_levels(t, lower, &level);
  out->parts = parts;
  out->G = G;
  out->R = R;
  // rows of each part sorted by (level, row)
  std::vector<std::vector<int32_t>> rows(parts);
  for (int64_t i = 0; i < n; ++i) rows[part[i]].push_back((int32_t)i);
  out->part_task_ptr.assign(parts + 1, 0);
  out->part_step_ptr.assign(parts + 1, 0);
  out->step_task_ptr.clear();
  out->step_task_ptr.push_back(0);
  out->task_row.clear();
  out->task_row.reserve(n);
  std::vector<int32_t> slot(n, -1);
  out->max_part_rows = 0;
  for (int p = 0; p < parts; ++p) {
    auto& r = rows[p];
    std::stable_sort(r.begin(), r.end(),
                     [&](int32_t x, int32_t y) { return level[x] < level[y]; });
    const int32_t base = (int32_t)out->task_row.size();
    int32_t in_step = 0, cur_level = -1;
    for (size_t k = 0; k < r.size(); ++k) {
      const int32_t row = r[k];
      if (level[row] != cur_level || in_step == R) {
        if (k > 0) out->step_task_ptr.push_back(base + (int32_t)k);
        cur_level = level[row];
        in_step = 0;
      }
      slot[row] = (int32_t)k;
      out->task_row.push_back(row);
      ++in_step;
    }
    if (!r.empty()) out->step_task_ptr.push_back(base + (int32_t)r.size());
    out->part_task_ptr[p + 1] = (int32_t)out->task_row.size();
    out->part_step_ptr[p + 1] = (int32_t)out->step_task_ptr.size() - 1;
    out->max_part_rows = std::max<int>(out->max_part_rows, (int)r.size());
    out->max_part_steps = std::max<int>(out->max_part_steps,
                                        out->part_step_ptr[p + 1] - out->part_step_ptr[p]);
  }
  const int64_t nt = (int64_t)out->task_row.size();
  out->task_diag.assign(nt, 0.0);
  out->ell_col.assign(nt * G, 0);
  out->ell_val.assign(nt * G, 0.0);
  for (int p = 0; p < parts; ++p) {
    const int32_t zero_cell = -(int32_t)(out->part_task_ptr[p + 1] - out->part_task_ptr[p]) - 1;
    for (int32_t tk = out->part_task_ptr[p]; tk < out->part_task_ptr[p + 1]; ++tk) {
      const int32_t row = out->task_row[tk];
      int cnt = 0;
      for (int64_t q = t.indptr[row]; q < t.indptr[row + 1]; ++q) {
        const int32_t c = t.indices[q];
        if (c == row) {
          out->task_diag[tk] = t.values[q];
          continue;
        }
        if (cnt == G) return false;
        out->ell_col[tk * G + cnt] = (part[c] == p) ? -(slot[c] + 1) : c;
        out->ell_val[tk * G + cnt] = t.values[q];
        ++cnt;
      }
      for (; cnt < G; ++cnt) {
        out->ell_col[tk * G + cnt] = zero_cell;
        out->ell_val[tk * G + cnt] = 0.0;
      }
    }
  }
  if (entry_major) {
    // per step: [rows][G] -> [G][rows]
    std::vector<int32_t> col2(out->ell_col.size());
    std::vector<double> val2(out->ell_val.size());
    const int64_t nsteps = (int64_t)out->step_task_ptr.size() - 1;
    for (int64_t s = 0; s < nsteps; ++s) {
      const int64_t a = out->step_task_ptr[s], b = out->step_task_ptr[s + 1], ns = b - a;
      for (int64_t r = 0; r < ns; ++r)
        for (int e = 0; e < G; ++e) {
          col2[a * G + e * ns + r] = out->ell_col[(a + r) * G + e];
          val2[a * G + e * ns + r] = out->ell_val[(a + r) * G + e];
        }
    }
    out->ell_col.swap(col2);
    out->ell_val.swap(val2);
  }
  return true;
}

}  // namespace bd

// ---------------------------------------------------------------------------
namespace bd {

bool build_cluster_schedule(const HostCsr& t, bool lower, const std::vector<int32_t>& part,
                            int parts, int E, int W, int cap_rows, int cap_slots,
                            ClusterSchedule* out, std::string* why) {
  const int64_t n = t.n;
  std::vector<int32_t> level;
  const int64_t nl = row_levels(t, lower, &level);
  out->parts = parts;
  out->E = E;
  out->W = W;
  out->nlevels = (int)nl;
  // own rows per (part, level), in row order
  std::vector<std::vector<int32_t>> own((size_t)parts * nl);
  for (int64_t i = 0; i < n; ++i) own[(size_t)part[i] * nl + level[i]].push_back((int32_t)i);
  // dependency distance check and import sets
  std::vector<std::vector<int32_t>> imp((size_t)parts * nl);
  for (int64_t i = 0; i < n; ++i) {
    int cnt = 0;
    for (int64_t q = t.indptr[i]; q < t.indptr[i + 1]; ++q) {
      const int32_t j = t.indices[q];
      if (j == i) continue;
      if (++cnt > E) {
        *why = "row longer than the ELL width";
        return false;
      }
      const int d = level[i] - level[j];
      if (d < 1 || d >= W) {
        *why = "dependency outside the level window";
        return false;
      }
      if (part[j] != part[i]) imp[(size_t)part[i] * nl + level[j]].push_back(j);
    }
  }
  // window slots: own rows first, then imported rows (deduplicated, sorted)
  std::vector<int32_t> slot_own(n, -1);
  std::vector<std::unordered_map<int32_t, int32_t>> slot_imp((size_t)parts * nl);
  out->wmax = out->rmax = 0;
  for (int p = 0; p < parts; ++p)
    for (int64_t l = 0; l < nl; ++l) {
      auto& o = own[(size_t)p * nl + l];
      for (size_t k = 0; k < o.size(); ++k) slot_own[o[k]] = (int32_t)k;
      auto& im = imp[(size_t)p * nl + l];
      std::sort(im.begin(), im.end());
      im.erase(std::unique(im.begin(), im.end()), im.end());
      auto& m = slot_imp[(size_t)p * nl + l];
      for (size_t k = 0; k < im.size(); ++k) m[im[k]] = (int32_t)(o.size() + k);
      out->rmax = std::max<int>(out->rmax, (int)((o.size() + 7) / 8 * 8));
      out->wmax = std::max<int>(out->wmax, (int)(o.size() + im.size()));
    }
  if (out->rmax > cap_rows || out->wmax > cap_slots || (int64_t)W * out->wmax >= 32767) {
    *why = "level too wide for the shared-memory windows";
    return false;
  }
  const int wm = out->wmax;
  // task order: part-major, level-major, row order
  out->lvl_ptr.assign((size_t)parts * (nl + 1), 0);
  out->task_row.clear();
  for (int p = 0; p < parts; ++p) {
    out->lvl_ptr[(size_t)p * (nl + 1)] = (int32_t)out->task_row.size();
    for (int64_t l = 0; l < nl; ++l) {
      auto& o = own[(size_t)p * nl + l];
      out->task_row.insert(out->task_row.end(), o.begin(), o.end());
      while (out->task_row.size() % 8) out->task_row.push_back(-1);  // 16-byte aligned blocks
      out->lvl_ptr[(size_t)p * (nl + 1) + l + 1] = (int32_t)out->task_row.size();
    }
  }
  const int64_t nt = (int64_t)out->task_row.size();
  out->task_diag.assign(nt, 1.0);
  out->ell_val.assign(nt * E, 0.0);
  out->ell_code.assign(nt * E, (int16_t)-1);
  for (int64_t k = 0; k < nt; ++k) {
    const int32_t i = out->task_row[k];
    if (i < 0) continue;
    const int p = part[i];
    int cnt = 0;
    for (int64_t q = t.indptr[i]; q < t.indptr[i + 1]; ++q) {
      const int32_t j = t.indices[q];
      if (j == i) {
        out->task_diag[k] = t.values[q];
        continue;
      }
      const int32_t s = part[j] == p ? slot_own[j] : slot_imp[(size_t)p * nl + level[j]].at(j);
      out->ell_code[k * E + cnt] = (int16_t)((level[j] % W) * wm + s);
      out->ell_val[k * E + cnt] = t.values[q];
      ++cnt;
    }
  }
  // exports: owner p of row j pushes it to every part q that imports it
  std::vector<std::vector<std::pair<int32_t, int32_t>>> ex((size_t)parts * nl);
  for (int q = 0; q < parts; ++q)
    for (int64_t l = 0; l < nl; ++l)
      for (auto& kv : slot_imp[(size_t)q * nl + l]) {
        const int32_t j = kv.first;
        const int32_t dst = (int32_t)((l % W) * wm + kv.second);
        ex[(size_t)part[j] * nl + l].push_back({slot_own[j], (q << 16) | dst});
      }
  out->exp_ptr.assign((size_t)parts * (nl + 1), 0);
  out->exp_src.clear();
  out->exp_dst.clear();
  out->emax = 0;
  for (int p = 0; p < parts; ++p) {
    out->exp_ptr[(size_t)p * (nl + 1)] = (int32_t)out->exp_src.size();
    for (int64_t l = 0; l < nl; ++l) {
      auto& e = ex[(size_t)p * nl + l];
      std::sort(e.begin(), e.end());
      for (auto& pr : e) {
        out->exp_src.push_back(pr.first);
        out->exp_dst.push_back(pr.second);
      }
      while (out->exp_src.size() % 4) {
        out->exp_src.push_back(-1);
        out->exp_dst.push_back(0);
      }
      out->emax = std::max<int>(out->emax, (int)((e.size() + 3) / 4 * 4));
      out->exp_ptr[(size_t)p * (nl + 1) + l + 1] = (int32_t)out->exp_src.size();
    }
  }
  return true;
}

}  // namespace bd

// ---------------------------------------------------------------------------
#include <queue>
namespace bd {

bool build_dtile_schedule(const HostCsr& t, bool lower, const std::vector<int32_t>& tile,
                          int ntiles, int E, DTileSchedule* out, std::string* why) {
  const int64_t n = t.n;
  std::vector<int32_t> level;
  row_levels(t, lower, &level);
  std::vector<std::vector<int32_t>> rows(ntiles);
  for (int64_t i = 0; i < n; ++i) rows[tile[i]].push_back((int32_t)i);
  // tile DAG (edges from dependency tiles) and min level per tile
  std::vector<int32_t> minlv(ntiles, INT32_MAX), indeg(ntiles, 0);
  std::vector<std::vector<int32_t>> succ(ntiles);
  for (int64_t i = 0; i < n; ++i) {
    const int32_t ti = tile[i];
    minlv[ti] = std::min(minlv[ti], level[i]);
    int cnt = 0;
    for (int64_t q = t.indptr[i]; q < t.indptr[i + 1]; ++q) {
      const int32_t j = t.indices[q];
      if (j == i) continue;
      if (++cnt > E) {
        *why = "row longer than the ELL width";
        return false;
      }
      const int32_t tj = tile[j];
      if (tj != ti) succ[tj].push_back(ti);
    }
  }
  for (auto& s : succ) {
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
    for (int32_t v : s) indeg[v]++;
  }
  // priority topological order: smallest min level first, then tile id
  using Key = std::pair<int32_t, int32_t>;
  std::priority_queue<Key, std::vector<Key>, std::greater<Key>> pq;
  for (int32_t v = 0; v < ntiles; ++v)
    if (indeg[v] == 0) pq.push({minlv[v], v});
  std::vector<int32_t> order;
  order.reserve(ntiles);
  while (!pq.empty()) {
    const int32_t v = pq.top().second;
    pq.pop();
    order.push_back(v);
    for (int32_t w : succ[v])
      if (--indeg[w] == 0) pq.push({minlv[w], w});
  }
  if ((int)order.size() != ntiles) {
    *why = "tile graph has a cycle";
    return false;
  }
  out->E = E;
  out->tmax = out->smax = 0;
  out->tile_row_ptr.assign(1, 0);
  out->tile_step_ptr.assign(1, 0);
  out->step_row.clear();
  out->task_row.clear();
  std::vector<int32_t> slot(n, -1);
  for (int32_t v : order) {
    auto& r = rows[v];
    std::stable_sort(r.begin(), r.end(),
                     [&](int32_t a, int32_t b) { return level[a] < level[b]; });
    for (size_t k = 0; k < r.size(); ++k) {
      slot[r[k]] = (int32_t)k;
      if (k == 0 || level[r[k]] != level[r[k - 1]]) out->step_row.push_back((int32_t)k);
    }
    out->task_row.insert(out->task_row.end(), r.begin(), r.end());
    out->tile_row_ptr.push_back((int32_t)out->task_row.size());
    out->tile_step_ptr.push_back((int32_t)out->step_row.size());
    out->tmax = std::max<int>(out->tmax, (int)r.size());
    out->smax = std::max<int>(out->smax, out->tile_step_ptr.back() -
                                             out->tile_step_ptr[out->tile_step_ptr.size() - 2]);
  }
  const int64_t nt = (int64_t)out->task_row.size();
  out->task_diag.assign(nt, 1.0);
  out->ell_col.assign(nt * E, 0);
  out->ell_val.assign(nt * E, 0.0);
  const int32_t zero = -(out->tmax + 1);  // zero slot of every tile
  for (int64_t k = 0; k < nt; ++k) {
    const int32_t i = out->task_row[k];
    int cnt = 0;
    for (int64_t q = t.indptr[i]; q < t.indptr[i + 1]; ++q) {
      const int32_t j = t.indices[q];
      if (j == i) {
        out->task_diag[k] = t.values[q];
        continue;
      }
      out->ell_col[k * E + cnt] = tile[j] == tile[i] ? -(slot[j] + 1) : j;
      out->ell_val[k * E + cnt] = t.values[q];
      ++cnt;
    }
    for (; cnt < E; ++cnt) out->ell_col[k * E + cnt] = zero;
  }
  return true;
}

bool build_btile_schedule(const DTileSchedule& ds, BTileSchedule* out, std::string* why) {
  const int E = ds.E;
  const int ntiles = (int)ds.tile_row_ptr.size() - 1;
  const int64_t nt = (int64_t)ds.task_row.size();
  const int32_t zero = -(ds.tmax + 1);
  int ex = 1;
  for (int64_t k = 0; k < nt; ++k) {
    int c = 0;
    for (int e = 0; e < E; ++e) c += ds.ell_col[k * E + e] >= 0;
    ex = std::max(ex, c);
  }
  ex = ex <= 4 ? 4 : ex <= 8 ? 8 : ex;  // device kernels are instantiated for widths 4 and 8
  out->Ex = ex;
  out->tmax = ds.tmax;
  out->tile_row_ptr = ds.tile_row_ptr;
  out->task_row = ds.task_row;
  out->ext_col.assign(nt * ex, -1);
  out->ext_val.assign(nt * ex, 0.0);
  out->tile_inv_ptr.assign(1, 0);
  out->inv.clear();
  out->tile_in_ptr.assign(1, 0);
  out->in_col.clear();
  out->xmax = 0;
  std::vector<int32_t> loc;
  for (int t = 0; t < ntiles; ++t) {
    const int r0 = ds.tile_row_ptr[t], r1 = ds.tile_row_ptr[t + 1];
    loc.clear();
    for (int64_t k = r0; k < r1; ++k)
      for (int e = 0; e < E; ++e)
        if (ds.ell_col[k * E + e] >= 0) loc.push_back(ds.ell_col[k * E + e]);
    std::sort(loc.begin(), loc.end());
    loc.erase(std::unique(loc.begin(), loc.end()), loc.end());
    for (int64_t k = r0; k < r1; ++k) {
      int c = 0;
      for (int e = 0; e < E; ++e) {
        const int32_t code = ds.ell_col[k * E + e];
        if (code >= 0) {
          out->ext_col[k * ex + c] = (int32_t)(std::lower_bound(loc.begin(), loc.end(), code) - loc.begin());
          out->ext_val[k * ex + c] = ds.ell_val[k * E + e];
          ++c;
        }
      }
    }
    out->in_col.insert(out->in_col.end(), loc.begin(), loc.end());
    out->tile_in_ptr.push_back((int32_t)out->in_col.size());
    out->xmax = std::max<int>(out->xmax, (int)loc.size());
  }
  // packed sizes first (each block padded to an even length), then the
  // independent per-tile inverses in parallel (host threads)
  out->tile_inv_ptr.assign(ntiles + 1, 0);
  for (int t = 0; t < ntiles; ++t) {
    const int64_t nr = ds.tile_row_ptr[t + 1] - ds.tile_row_ptr[t];
    const int64_t len = nr * (nr + 1) / 2;
    out->tile_inv_ptr[t + 1] = out->tile_inv_ptr[t] + len + (len & 1);
  }
  out->inv.assign(out->tile_inv_ptr[ntiles], 0.0);
  int failed = 0;
  std::string fail_why;
#pragma omp parallel
  {
    std::vector<long double> x;
#pragma omp for schedule(dynamic, 16)
    for (int t = 0; t < ntiles; ++t) {
      if (failed) continue;
      const int r0 = ds.tile_row_ptr[t], nr = ds.tile_row_ptr[t + 1] - r0;
      // X = A^{-1} for the tile block A (lower triangular in slot order):
      // X[k][l] = (delta_kl - sum_{l<=j<k} A[k][j] X[j][l]) / A[k][k]
      x.assign((size_t)nr * nr, 0.0L);
      const char* err = nullptr;
      for (int k = 0; k < nr && !err; ++k) {
        const int64_t q = r0 + k;
        const long double d = ds.task_diag[q];
        if (!(d != 0.0L)) {
          err = "zero pivot in a tile block";
          break;
        }
        for (int e = 0; e < E; ++e) {
          const int32_t code = ds.ell_col[q * E + e];
          if (code >= 0 || code == zero) continue;
          const int j = -code - 1;
          if (j >= k) {
            err = "tile block is not triangular in slot order";
            break;
          }
          const long double a = ds.ell_val[q * E + e];
          for (int l = 0; l <= j; ++l) x[(size_t)k * nr + l] -= a * x[(size_t)j * nr + l];
        }
        if (err) break;
        x[(size_t)k * nr + k] += 1.0L;
        for (int l = 0; l <= k; ++l) x[(size_t)k * nr + l] /= d;
      }
      if (err) {
#pragma omp critical
        {
          failed = 1;
          fail_why = err;
        }
        continue;
      }
      double* dst = out->inv.data() + out->tile_inv_ptr[t];
      for (int k = 0; k < nr; ++k)
        for (int l = 0; l <= k; ++l) *dst++ = (double)x[(size_t)k * nr + l];
    }
  }
  if (failed) {
    *why = fail_why;
    return false;
  }
  return true;
}

int partition_grid(int64_t n, int dim, const double* coords, int target,
                   const std::vector<int32_t>* cls, std::vector<int32_t>* tile) {
  const int k = std::max(1, (int)std::lround(std::pow((double)target, 1.0 / dim)));
  std::vector<int64_t> bin(n, 0);
  int64_t stride = 1;
  for (int a = 0; a < dim; ++a) {
    std::vector<double> v(n);
    double lo = INFINITY, hi = -INFINITY;
    for (int64_t i = 0; i < n; ++i) {
      v[i] = coords[i * dim + a];
      lo = std::min(lo, v[i]);
      hi = std::max(hi, v[i]);
    }
    const double tol = 1e-9 * std::max(1.0, hi - lo);
    std::vector<double> u(v);
    std::sort(u.begin(), u.end());
    std::vector<double> uniq;
    for (double x : u)
      if (uniq.empty() || x - uniq.back() > tol) uniq.push_back(x);
    const double limit = 8.0 * std::pow((double)n, 1.0 / dim);
    int64_t nb;
    std::vector<int64_t> b(n);
    if ((double)uniq.size() <= limit) {  // structured axis: bin by layer rank
      for (int64_t i = 0; i < n; ++i) {
        const int64_t r = std::lower_bound(uniq.begin(), uniq.end(), v[i] - tol) - uniq.begin();
        b[i] = r / k;
      }
      nb = ((int64_t)uniq.size() + k - 1) / k;
    } else {  // unstructured: equal-width bins holding ~k layers of points
      nb = std::max<int64_t>(1, (int64_t)std::llround(std::pow((double)n, 1.0 / dim) / k));
      const double w = (hi - lo) / (double)nb;
      for (int64_t i = 0; i < n; ++i)
        b[i] = std::min<int64_t>(nb - 1, w > 0 ? (int64_t)((v[i] - lo) / w) : 0);
    }
    for (int64_t i = 0; i < n; ++i) bin[i] += b[i] * stride;
    stride *= nb;
  }
  if (cls)
    for (int64_t i = 0; i < n; ++i) bin[i] += stride * (int64_t)(*cls)[i];
  // compact to dense tile ids
  std::vector<int64_t> keys(bin);
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  tile->resize(n);
  for (int64_t i = 0; i < n; ++i)
    (*tile)[i] = (int32_t)(std::lower_bound(keys.begin(), keys.end(), bin[i]) - keys.begin());
  return (int)keys.size();
}


// Relaxed supernodes (exact inner): a row joins the current block of
// consecutive rows [c0, i) when the dense triangle the supernodal solves
// expect would miss at most frac·(i − c0) of the columns c0..i−1 in it; the
// missing entries are inserted as explicit zeros, which change no result
// (0·x adds nothing) but merge chains of small supernodes into fewer, larger
// ones (fewer levels of the supernodal task DAG).  Blocks stop at smax rows.
void relax_supernodes(HostCsr* L, double frac, int smax) {
  const int64_t n = L->n;
  if (n == 0 || !(frac > 0.0)) return;
  HostCsr out;
  out.n = n;
  out.indptr.assign(n + 1, 0);
  out.indices.reserve(L->indices.size() + L->indices.size() / 8);
  out.values.reserve(L->values.size() + L->values.size() / 8);
  int64_t c0 = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t b = L->indptr[i], e = L->indptr[i + 1];  // diagonal at e-1
    const int64_t k = i - c0;
    bool join = false;
    if (i > 0 && k > 0 && k < smax) {
      const int32_t* first = L->indices.data() + b;
      const int32_t* last = L->indices.data() + (e - 1);
      const int64_t present = last - std::lower_bound(first, last, (int32_t)c0);
      const int64_t miss = k - present;
      join = miss == 0 || (double)miss <= frac * (double)k;
    }
    if (!join) c0 = i;
    int64_t q = b;
    for (; q < e - 1 && L->indices[q] < c0; ++q) {  // external columns
      out.indices.push_back(L->indices[q]);
      out.values.push_back(L->values[q]);
    }
    for (int64_t j = c0; j < i; ++j) {  // the block's dense triangle row
      if (q < e - 1 && L->indices[q] == j) {
        out.indices.push_back((int32_t)j);
        out.values.push_back(L->values[q]);
        ++q;
      } else {
        out.indices.push_back((int32_t)j);
        out.values.push_back(0.0);
      }
    }
    out.indices.push_back((int32_t)i);  // diagonal last
    out.values.push_back(L->values[e - 1]);
    out.indptr[i + 1] = (int64_t)out.indices.size();
  }
  *L = std::move(out);
}

}  // namespace bd
