// Host setup: clean-up (D1), squared EDT (D2), immersion watershed (D3),
// saddle/peak merge (D4-D5), relabel (D6), interfaces (D7), floating-face
// repair (D7b), duals (D8), mask band (D9), face ownership and the W order
// (D10).  See DESIGN.md §3 for the readings; PAPER.md P:156 defers
// the watershed details, so these rules are this project's specification.
#include "setup.hpp"
#include <chrono>
#include <thread>
#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <numeric>
#include <queue>
#include <stdexcept>
#include <tuple>
#include <unordered_map>

namespace pmns {

// Parallel for over [0, n) in contiguous chunks (host threads; every body
// writes disjoint outputs, so results are independent of the thread count).
template <class F>
static void par_for(int64_t n, F fn) {
  unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (n < 4096 || nt == 1) {
    fn((int64_t)0, n);
    return;
  }
  std::vector<std::thread> th;
  int64_t chunk = (n + nt - 1) / nt;
  for (unsigned t = 0; t < nt; ++t) {
    int64_t a = t * chunk, b = std::min<int64_t>(n, a + chunk);
    if (a >= b) break;
    th.emplace_back([=]() { fn(a, b); });
  }
  for (auto &x : th) x.join();
}


namespace {
enum CellState { VOIDC = 0, SOLIDC = 1, OUTC = 2 };

struct Nbr {  // face neighbours of a voxel, -1 = none
  int64_t v[6];
  int n;
};

inline void face_nbrs(const Geometry &g, int64_t f, Nbr &out) {
  int i = (int)(f % g.nx);
  int64_t t = f / g.nx;
  int j = (int)(t % g.ny);
  int k = (int)(t / g.ny);
  out.n = 2 * g.dim;
  // order: x-, x+, y-, y+, z-, z+
  out.v[0] = i > 0 ? g.flat(k, j, i - 1) : -1;
  out.v[1] = i + 1 < g.nx ? g.flat(k, j, i + 1) : -1;
  if (g.py) {
    out.v[2] = g.flat(k, (j + g.ny - 1) % g.ny, i);
    out.v[3] = g.flat(k, (j + 1) % g.ny, i);
  } else {
    out.v[2] = j > 0 ? g.flat(k, j - 1, i) : -1;
    out.v[3] = j + 1 < g.ny ? g.flat(k, j + 1, i) : -1;
  }
  if (g.dim == 3) {
    if (g.pz) {
      out.v[4] = g.flat((k + g.nz - 1) % g.nz, j, i);
      out.v[5] = g.flat((k + 1) % g.nz, j, i);
    } else {
      out.v[4] = k > 0 ? g.flat(k - 1, j, i) : -1;
      out.v[5] = k + 1 < g.nz ? g.flat(k + 1, j, i) : -1;
    }
  }
}

// 26 (3D) / 8 (2D) neighbourhood, periodic-aware
inline int box_nbrs(const Geometry &g, int64_t f, int64_t *out) {
  int i = (int)(f % g.nx);
  int64_t t = f / g.nx;
  int j = (int)(t % g.ny);
  int k = (int)(t / g.ny);
  int n = 0;
  int kr = g.dim == 3 ? 1 : 0;
  for (int dk = -kr; dk <= kr; ++dk)
    for (int dj = -1; dj <= 1; ++dj)
      for (int di = -1; di <= 1; ++di) {
        if (!dk && !dj && !di) continue;
        int kk = k + dk, jj = j + dj, ii = i + di;
        if (g.py) jj = (jj % g.ny + g.ny) % g.ny;
        if (g.pz) kk = (kk % g.nz + g.nz) % g.nz;
        if (ii < 0 || ii >= g.nx || jj < 0 || jj >= g.ny || kk < 0 || kk >= g.nz)
          out[n++] = -1;
        else
          out[n++] = g.flat(kk, jj, ii);
      }
  return n;
}

inline int cell_state(const Geometry &g, int k, int j, int i) {
  if (i < 0 || i >= g.nx) {
    // x outside: OUT unless the lateral coordinate is outside a wall
    bool lat_ok = true;
    if (!g.py && (j < 0 || j >= g.ny)) lat_ok = false;
    if (g.dim == 3 && !g.pz && (k < 0 || k >= g.nz)) lat_ok = false;
    return lat_ok ? OUTC : SOLIDC;
  }
  if (g.py) j = (j % g.ny + g.ny) % g.ny;
  else if (j < 0 || j >= g.ny) return SOLIDC;
  if (g.dim == 3) {
    if (g.pz) k = (k % g.nz + g.nz) % g.nz;
    else if (k < 0 || k >= g.nz) return SOLIDC;
  } else if (k != 0) {
    return SOLIDC;
  }
  return g.is_void[g.flat(k, j, i)] ? VOIDC : SOLIDC;
}
}  // namespace

int32_t Geometry::face_code(int a, int k, int j, int i) const {
  if (a == 0 ? (i < 0 || i > nx) : (i < 0 || i >= nx)) return kMirror;
  int k0 = k, j0 = j, i0 = i;
  if (a == 0) i0 -= 1;
  else if (a == 1) j0 -= 1;
  else k0 -= 1;
  int s0 = cell_state(*this, k0, j0, i0), s1 = cell_state(*this, k, j, i);
  bool dof = (s0 == VOIDC && s1 == VOIDC) || (s0 == VOIDC && s1 == OUTC) || (s0 == OUTC && s1 == VOIDC);
  if (dof) {
    int kk = k, jj = j;
    if (py) jj = (jj % ny + ny) % ny;
    if (dim == 3 && pz) kk = (kk % nz + nz) % nz;
    return fmap[a][((int64_t)kk * fy[a] + jj) * fx[a] + i];
  }
  int ns = (s0 == SOLIDC) + (s1 == SOLIDC);
  return ns == 2 ? kGhost : kZero;   // ns == 1 -> zero face; OUT+OUT impossible
}

// ----------------------------------------------------------------------------
// D1 + numbering
// ----------------------------------------------------------------------------
void build_geometry(const uint8_t *solid, int dim, int nx, int ny, int nz, bool py, bool pz, Geometry &g) {
  g.dim = dim;
  g.nx = nx;
  g.ny = ny;
  g.nz = dim == 3 ? nz : 1;
  g.py = py;
  g.pz = dim == 3 && pz;
  int64_t nv = g.nvox();
  // D1: flood from void voxels on the x = 0 and x = nx-1 planes
  std::vector<uint8_t> keep(nv, 0);
  std::vector<int64_t> stack;
  for (int k = 0; k < g.nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i : {0, nx - 1}) {
        int64_t f = g.flat(k, j, i);
        if (!solid[f] && !keep[f]) {
          keep[f] = 1;
          stack.push_back(f);
        }
      }
  Nbr nb;
  g.is_void.assign(nv, 0);
  for (int64_t f = 0; f < nv; ++f) g.is_void[f] = solid[f] ? 0 : 1;
  while (!stack.empty()) {
    int64_t f = stack.back();
    stack.pop_back();
    face_nbrs(g, f, nb);
    for (int c = 0; c < nb.n; ++c) {
      int64_t q = nb.v[c];
      if (q >= 0 && g.is_void[q] && !keep[q]) {
        keep[q] = 1;
        stack.push_back(q);
      }
    }
  }
  int64_t nvoid = 0;
  for (int64_t f = 0; f < nv; ++f) {
    g.is_void[f] = keep[f];
    nvoid += keep[f];
  }
  if (nvoid == 0) throw std::runtime_error("ENONPERC: no void connected to the inlet/outlet planes");
  // face maps
  for (int a = 0; a < 3; ++a) {
    g.fx[a] = nx + (a == 0 ? 1 : 0);
    g.fy[a] = ny + ((a == 1 && !g.py) ? 1 : 0);
    g.fz[a] = g.nz + ((a == 2 && dim == 3 && !g.pz) ? 1 : 0);
    g.fmap[a].clear();
  }
  int64_t off = 0;
  for (int a = 0; a < dim; ++a) {
    g.fmap[a].assign((int64_t)g.fx[a] * g.fy[a] * g.fz[a], kGhost);
    // canonical numbering: C order over (nz, ny, nx(+1)) — the positions that
    // can be DOFs; the extra top-wall positions never are.
    int64_t cnt = 0;
    for (int k = 0; k < g.fz[a]; ++k)
      for (int j = 0; j < g.fy[a]; ++j)
        for (int i = 0; i < g.fx[a]; ++i) {
          int k0 = k, j0 = j, i0 = i;
          if (a == 0) i0 -= 1;
          else if (a == 1) j0 -= 1;
          else k0 -= 1;
          int s0 = cell_state(g, k0, j0, i0), s1 = cell_state(g, k, j, i);
          bool dof = (s0 == VOIDC && s1 == VOIDC) || (s0 == VOIDC && s1 == OUTC) || (s0 == OUTC && s1 == VOIDC);
          int64_t idx = ((int64_t)k * g.fy[a] + j) * g.fx[a] + i;
          if (dof) {
            g.fmap[a][idx] = (int32_t)(off + cnt);
            ++cnt;
          } else {
            int ns = (s0 == SOLIDC) + (s1 == SOLIDC);
            g.fmap[a][idx] = ns == 2 ? kGhost : kZero;
          }
        }
    g.n_face[a] = cnt;
    off += cnt;
  }
  g.n_f = off;
  g.cmap.assign(nv, -1);
  int64_t c = 0;
  for (int64_t f = 0; f < nv; ++f)
    if (g.is_void[f]) g.cmap[f] = (int32_t)(off + c++);
  g.n_c = c;
  g.N = off + c;
  if (g.N >= (int64_t)INT32_MAX) throw std::runtime_error("EINVAL: problem too large for int32 indices");
}

// ----------------------------------------------------------------------------
// D2: exact squared EDT (separable lower envelope with exact rational tests)
// ----------------------------------------------------------------------------
namespace {
const int64_t kInf = (int64_t)1 << 50;

// out[x] = min_q (f[q] + (x - pos[q])^2) over sample points (pos, f) (f < kInf),
// evaluated at x = 0..n-1.  Points must be sorted by pos (strictly increasing).
void envelope(const std::vector<int64_t> &pos, const std::vector<int64_t> &fv, int n, int64_t *out,
              int64_t stride) {
  int m = (int)pos.size();
  if (m == 0) {
    for (int x = 0; x < n; ++x) out[x * stride] = kInf;
    return;
  }
  std::vector<int> v(m);
  std::vector<int64_t> zn(m + 1), zd(m + 1);  // boundaries z[k] = zn/zd (zd > 0); z[0] = -inf
  int kk = 0;
  v[0] = 0;
  bool neg_inf0 = true;
  (void)neg_inf0;
  // intersection of parabolas q (new) and v (old): s = ((f_q + p_q^2) - (f_v + p_v^2)) / (2 (p_q - p_v))
  auto inter = [&](int q, int vv, int64_t &num, int64_t &den) {
    num = (fv[q] + pos[q] * pos[q]) - (fv[vv] + pos[vv] * pos[vv]);
    den = 2 * (pos[q] - pos[vv]);
  };
  // z[0] = -inf represented by flag
  std::vector<uint8_t> zinf(m + 1, 0);
  zinf[0] = 1;  // -inf
  for (int q = 1; q < m; ++q) {
    int64_t num, den;
    while (true) {
      inter(q, v[kk], num, den);
      // compare s <= z[kk]
      bool le;
      if (zinf[kk]) le = false;
      else le = (__int128)num * zd[kk] <= (__int128)zn[kk] * den;
      if (le && kk > 0) {
        --kk;
        continue;
      }
      if (le && kk == 0) {  // cannot happen with z[0] = -inf
        break;
      }
      break;
    }
    ++kk;
    v[kk] = q;
    zn[kk] = num;
    zd[kk] = den;
    zinf[kk] = 0;
  }
  // evaluate: for x, find last k with z[k] <= x
  int k = 0;
  for (int x = 0; x < n; ++x) {
    while (k + 1 <= kk && ((__int128)zn[k + 1] <= (__int128)x * zd[k + 1])) ++k;
    int q = v[k];
    int64_t d = x - pos[q];
    out[x * stride] = fv[q] + d * d;
  }
}

void edt_pass(const Geometry &g, std::vector<int64_t> &F, int axis, bool periodic, bool walls) {
  int n = axis == 0 ? g.nx : axis == 1 ? g.ny : g.nz;
  int64_t stride = axis == 0 ? 1 : axis == 1 ? g.nx : (int64_t)g.nx * g.ny;
  int64_t lines = g.nvox() / n;
  par_for(lines, [&](int64_t L0, int64_t L1) {
  std::vector<int64_t> pos, fv;
  pos.reserve(3 * n + 2);
  fv.reserve(3 * n + 2);
  std::vector<int64_t> tmp(n);
  for (int64_t L = L0; L < L1; ++L) {
    int64_t base;
    if (axis == 0) base = L * g.nx;
    else if (axis == 1) base = (L / g.nx) * (int64_t)g.nx * g.ny + (L % g.nx);
    else base = L;
    pos.clear();
    fv.clear();
    if (periodic) {
      for (int rep = -1; rep <= 1; ++rep)
        for (int q = 0; q < n; ++q) {
          int64_t val = F[base + q * stride];
          if (val < kInf) {
            pos.push_back((int64_t)rep * n + q);
            fv.push_back(val);
          }
        }
    } else {
      if (walls) {
        pos.push_back(-1);
        fv.push_back(0);
      }
      for (int q = 0; q < n; ++q) {
        int64_t val = F[base + q * stride];
        if (val < kInf) {
          pos.push_back(q);
          fv.push_back(val);
        }
      }
      if (walls) {
        pos.push_back(n);
        fv.push_back(0);
      }
    }
    envelope(pos, fv, n, tmp.data(), 1);
    for (int q = 0; q < n; ++q) F[base + q * stride] = tmp[q];
  }
  });
}
}  // namespace

static std::vector<int64_t> squared_edt(const Geometry &g) {
  int64_t nv = g.nvox();
  std::vector<int64_t> F(nv);
  for (int64_t f = 0; f < nv; ++f) F[f] = g.is_void[f] ? kInf : 0;
  edt_pass(g, F, 0, false, false);          // x: outside counts as void
  edt_pass(g, F, 1, g.py, !g.py);           // y: periodic or solid wall layer
  if (g.dim == 3) edt_pass(g, F, 2, g.pz, !g.pz);
  for (int64_t f = 0; f < nv; ++f) {
    if (!g.is_void[f]) F[f] = 0;
    else if (F[f] >= kInf) F[f] = (int64_t)1 << 40;   // no solid anywhere: same sentinel as the oracle
  }
  return F;
}

// ----------------------------------------------------------------------------
// D3: level-synchronous immersion
// ----------------------------------------------------------------------------
static int64_t watershed(const Geometry &g, const std::vector<int64_t> &D, std::vector<int64_t> &label) {
  int64_t nv = g.nvox();
  label.assign(nv, -1);
  std::vector<int64_t> vox;
  for (int64_t f = 0; f < nv; ++f)
    if (g.is_void[f]) vox.push_back(f);
  std::stable_sort(vox.begin(), vox.end(), [&](int64_t a, int64_t b) { return D[a] > D[b]; });
  int64_t nlab = 0;
  Nbr nb;
  std::vector<int64_t> remaining, next, newlab;
  std::vector<int64_t> comp_mark(nv, -1);
  size_t p = 0;
  while (p < vox.size()) {
    size_t q = p;
    while (q < vox.size() && D[vox[q]] == D[vox[p]]) ++q;
    remaining.assign(vox.begin() + p, vox.begin() + q);
    std::sort(remaining.begin(), remaining.end());
    while (!remaining.empty()) {
      newlab.assign(remaining.size(), -1);
      bool any = false;
      for (size_t r = 0; r < remaining.size(); ++r) {
        face_nbrs(g, remaining[r], nb);
        int64_t m = -1;
        for (int c = 0; c < nb.n; ++c) {
          int64_t u = nb.v[c];
          if (u >= 0 && g.is_void[u] && label[u] >= 0 && (m < 0 || label[u] < m)) m = label[u];
        }
        newlab[r] = m;
        if (m >= 0) any = true;
      }
      if (!any) break;
      next.clear();
      for (size_t r = 0; r < remaining.size(); ++r) {
        if (newlab[r] >= 0) label[remaining[r]] = newlab[r];
        else next.push_back(remaining[r]);
      }
      remaining.swap(next);
    }
    // leftover components at this level -> new basins by smallest index
    if (!remaining.empty()) {
      for (int64_t f : remaining) comp_mark[f] = -2;  // candidate marker
      std::vector<int64_t> st;
      for (int64_t f : remaining) {
        if (comp_mark[f] != -2) continue;
        int64_t id = nlab++;
        comp_mark[f] = id;
        label[f] = id;
        st.push_back(f);
        while (!st.empty()) {
          int64_t u = st.back();
          st.pop_back();
          face_nbrs(g, u, nb);
          for (int c = 0; c < nb.n; ++c) {
            int64_t w = nb.v[c];
            if (w >= 0 && comp_mark[w] == -2) {
              comp_mark[w] = id;
              label[w] = id;
              st.push_back(w);
            }
          }
        }
      }
      for (int64_t f : remaining) comp_mark[f] = -1;
    }
    p = q;
  }
  return nlab;
}

// ----------------------------------------------------------------------------
// D4-D6
// ----------------------------------------------------------------------------
typedef std::vector<std::map<int64_t, int64_t>> Adj;

static void saddles(const Geometry &g, const std::vector<int64_t> &lab, const std::vector<int64_t> &D, int64_t nl,
                    Adj &S) {
  S.assign(nl, {});
  Nbr nb;
  for (int64_t f = 0; f < g.nvox(); ++f) {
    if (!g.is_void[f]) continue;
    face_nbrs(g, f, nb);
    for (int c = 0; c < nb.n; ++c) {
      int64_t u = nb.v[c];
      if (u < 0 || !g.is_void[u]) continue;
      int64_t a = lab[f], b = lab[u];
      if (a >= b) continue;
      int64_t val = std::min(D[f], D[u]);
      auto it = S[a].find(b);
      if (it == S[a].end() || it->second < val) {
        S[a][b] = val;
        S[b][a] = val;
      }
    }
  }
}

static void relabel_by_first(const Geometry &g, std::vector<int64_t> &lab) {
  std::unordered_map<int64_t, int64_t> mp;
  int64_t next = 0;
  for (int64_t f = 0; f < g.nvox(); ++f) {
    if (lab[f] < 0) continue;
    auto it = mp.find(lab[f]);
    if (it == mp.end()) {
      mp.emplace(lab[f], next);
      lab[f] = next++;
    } else {
      lab[f] = it->second;
    }
  }
}

static void merge_basins(const Geometry &g, std::vector<int64_t> &lab, int64_t nl, const std::vector<int64_t> &D,
                         double h_m, int n_min) {
  std::vector<int64_t> P(nl, -1), size(nl, 0);
  for (int64_t f = 0; f < g.nvox(); ++f)
    if (g.is_void[f]) {
      P[lab[f]] = std::max(P[lab[f]], D[f]);
      size[lab[f]]++;
    }
  Adj S;
  saddles(g, lab, D, nl, S);
  std::vector<int64_t> parent(nl);
  std::iota(parent.begin(), parent.end(), 0);
  std::vector<uint8_t> alive(nl, 1);
  auto key = [&](int64_t a, int64_t b) {
    return std::sqrt((double)std::min(P[a], P[b])) - std::sqrt((double)S[a].at(b));
  };
  auto merge = [&](int64_t src, int64_t dst) {
    parent[src] = dst;
    alive[src] = 0;
    P[dst] = std::max(P[dst], P[src]);
    size[dst] += size[src];
    for (auto &kv : S[src]) {
      int64_t c = kv.first;
      if (c == dst) continue;
      auto it = S[dst].find(c);
      if (it == S[dst].end() || kv.second > it->second) {
        S[dst][c] = kv.second;
        S[c][dst] = kv.second;
      }
      S[c].erase(src);
    }
    S[dst].erase(src);
    S[src].clear();
  };
  typedef std::tuple<double, int64_t, int64_t> KE;
  std::priority_queue<KE, std::vector<KE>, std::greater<KE>> heap;
  for (int64_t a = 0; a < nl; ++a)
    for (auto &kv : S[a])
      if (a < kv.first) heap.emplace(key(a, kv.first), a, kv.first);
  while (!heap.empty()) {
    KE e = heap.top();
    heap.pop();
    double k;
    int64_t a, b;
    std::tie(k, a, b) = e;
    if (!(alive[a] && alive[b] && S[a].count(b))) continue;
    if (key(a, b) != k) continue;
    if (!(k < h_m)) break;
    int64_t src, dst;
    if (P[a] < P[b]) { src = a; dst = b; }
    else if (P[b] < P[a]) { src = b; dst = a; }
    else { src = std::max(a, b); dst = std::min(a, b); }
    merge(src, dst);
    for (auto &kv : S[dst]) heap.emplace(key(dst, kv.first), std::min(dst, kv.first), std::max(dst, kv.first));
  }
  typedef std::pair<int64_t, int64_t> SE;
  std::priority_queue<SE, std::vector<SE>, std::greater<SE>> h2;
  for (int64_t a = 0; a < nl; ++a)
    if (alive[a] && size[a] < n_min) h2.emplace(size[a], a);
  while (!h2.empty()) {
    SE e = h2.top();
    h2.pop();
    int64_t s = e.first, a = e.second;
    if (!alive[a] || size[a] != s || size[a] >= n_min) continue;
    if (S[a].empty()) continue;
    int64_t b = -1, bs = -1;
    for (auto &kv : S[a])
      if (kv.second > bs || (kv.second == bs && kv.first < b)) {
        bs = kv.second;
        b = kv.first;
      }
    merge(a, b);
    if (size[b] < n_min) h2.emplace(size[b], b);
  }
  auto find = [&](int64_t x) {
    while (parent[x] != x) x = parent[x];
    return x;
  };
  for (int64_t f = 0; f < g.nvox(); ++f)
    if (lab[f] >= 0) lab[f] = find(lab[f]);
  relabel_by_first(g, lab);
}

// host phase timer (PMNS_TRACE=1)
struct SetupTimer {
  bool on = getenv("PMNS_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void lap(const char *what) {
    if (!on) return;
    auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[pmns setup] %-14s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

// ----------------------------------------------------------------------------
// D7 interfaces
// ----------------------------------------------------------------------------
static int compute_interfaces(const Geometry &g, const std::vector<int64_t> &lab, std::vector<int32_t> &iface) {
  int64_t nv = g.nvox();
  iface.assign(nv, -1);
  std::vector<int64_t> pa(nv, -1);
  std::vector<int64_t> cand;
  Nbr nb;
  for (int64_t f = 0; f < nv; ++f) {
    if (!g.is_void[f]) continue;
    face_nbrs(g, f, nb);
    int64_t m = INT64_MAX;
    for (int c = 0; c < nb.n; ++c) {
      int64_t u = nb.v[c];
      if (u >= 0 && g.is_void[u] && lab[u] < m) m = lab[u];
    }
    if (m < lab[f]) {
      pa[f] = m;
      cand.push_back(f);
    }
  }
  // components (26/8-connectivity) among candidates with the same pair
  std::vector<int64_t> comp(nv, -1);
  std::vector<std::tuple<int64_t, int64_t, int64_t, int64_t>> comps;  // (a, b, first, id)
  int64_t bn[26];
  std::vector<int64_t> st;
  int64_t nc = 0;
  for (int64_t f : cand) {  // ascending flat order
    if (comp[f] >= 0) continue;
    int64_t id = nc++;
    comp[f] = id;
    comps.emplace_back(pa[f], lab[f], f, id);
    st.push_back(f);
    while (!st.empty()) {
      int64_t u = st.back();
      st.pop_back();
      int n = box_nbrs(g, u, bn);
      for (int c = 0; c < n; ++c) {
        int64_t w = bn[c];
        if (w >= 0 && pa[w] >= 0 && comp[w] < 0 && pa[w] == pa[u] && lab[w] == lab[u]) {
          comp[w] = id;
          st.push_back(w);
        }
      }
    }
  }
  std::sort(comps.begin(), comps.end());
  std::vector<int32_t> rank(nc);
  for (size_t r = 0; r < comps.size(); ++r) rank[std::get<3>(comps[r])] = (int32_t)r;
  for (int64_t f : cand) iface[f] = rank[comp[f]];
  return (int)nc;
}

// face ownership helpers (D10) on current (lab, iface)
struct FaceFlank {
  std::vector<int64_t> c0, c1;   // flank voxel indices (-1 if outside / solid)
};

static void face_flanks(const Geometry &g, FaceFlank &ff) {
  ff.c0.assign(g.n_f, -1);
  ff.c1.assign(g.n_f, -1);
  for (int a = 0; a < g.dim; ++a)
    for (int k = 0; k < g.fz[a]; ++k)
      for (int j = 0; j < g.fy[a]; ++j)
        for (int i = 0; i < g.fx[a]; ++i) {
          int32_t id = g.fmap[a][((int64_t)k * g.fy[a] + j) * g.fx[a] + i];
          if (id < 0) continue;
          int k0 = k, j0 = j, i0 = i;
          if (a == 0) i0 -= 1;
          else if (a == 1) j0 = g.py ? (j - 1 + g.ny) % g.ny : j - 1;
          else k0 = g.pz ? (k - 1 + g.nz) % g.nz : k - 1;
          if (i0 >= 0 && i0 < g.nx && j0 >= 0 && j0 < g.ny && k0 >= 0 && k0 < g.nz && g.is_void[g.flat(k0, j0, i0)])
            ff.c0[id] = g.flat(k0, j0, i0);
          if (i < g.nx && j < g.ny && k < g.nz && g.is_void[g.flat(k, j, i)]) ff.c1[id] = g.flat(k, j, i);
        }
}

// D7b floating faces.  fnb: per face, the codes of its 2*dim same-orientation
// neighbours at +-1 along each axis (geometry only, computed once).
static std::vector<int32_t> face_nbr_codes(const Geometry &g) {
  const int W = 2 * g.dim;
  std::vector<int32_t> fnb((size_t)g.n_f * W, kZero);
  for (int a = 0; a < g.dim; ++a)
    par_for(g.fz[a] * (int64_t)g.fy[a], [&](int64_t r0, int64_t r1) {
    for (int64_t r = r0; r < r1; ++r) {
      const int k = (int)(r / g.fy[a]), j = (int)(r % g.fy[a]);
        for (int i = 0; i < g.fx[a]; ++i) {
          int32_t id = g.fmap[a][((int64_t)k * g.fy[a] + j) * g.fx[a] + i];
          if (id < 0) continue;
          int q = 0;
          for (int b = 0; b < g.dim; ++b)
            for (int o = -1; o <= 1; o += 2) {
              int kk = k + (b == 2 ? o : 0), jj = j + (b == 1 ? o : 0), ii = i + (b == 0 ? o : 0);
              fnb[(size_t)id * W + q++] = g.face_code(a, kk, jj, ii);
            }
        }
    }
    });
  return fnb;
}

static std::vector<uint8_t> floating(const Geometry &g, const FaceFlank &ff, const std::vector<int32_t> &fnb,
                                     const std::vector<int64_t> &prim) {
  int64_t nf = g.n_f;
  const int W = 2 * g.dim;
  std::vector<int64_t> owner(nf, -1);
  for (int64_t f = 0; f < nf; ++f) {
    int64_t p = -1;
    if (ff.c0[f] >= 0 && prim[ff.c0[f]] >= 0) p = prim[ff.c0[f]];
    if (ff.c1[f] >= 0 && prim[ff.c1[f]] >= 0) p = prim[ff.c1[f]];
    owner[f] = p;
  }
  std::vector<int64_t> uf(nf);
  std::iota(uf.begin(), uf.end(), 0);
  auto find = [&](int64_t x) {
    while (uf[x] != x) {
      uf[x] = uf[uf[x]];
      x = uf[x];
    }
    return x;
  };
  std::vector<uint8_t> anch(nf, 0);
  for (int64_t id = 0; id < nf; ++id)
    for (int q = 0; q < W; ++q) {
      int32_t c = fnb[(size_t)id * W + q];
      if (c == kZero || c == kGhost) anch[id] = 1;
      if (c >= 0 && owner[id] >= 0 && owner[c] == owner[id]) {
        int64_t r1 = find(id), r2 = find(c);
        if (r1 != r2) uf[std::max(r1, r2)] = std::min(r1, r2);
      }
    }
  std::vector<uint8_t> canch(nf, 0);
  for (int64_t f = 0; f < nf; ++f)
    if (anch[f]) canch[find(f)] = 1;
  std::vector<uint8_t> flt(nf, 0);
  for (int64_t f = 0; f < nf; ++f) flt[f] = owner[f] >= 0 && !canch[find(f)];
  return flt;
}

static void repair_floating(const Geometry &g, const FaceFlank &ff, const std::vector<int32_t> &fnb,
                            const std::vector<int64_t> &lab, std::vector<int32_t> &iface) {
  int64_t bn[26];
  SetupTimer tm;
  int rounds = 0;
  while (true) {
    ++rounds;
    if (tm.on) fprintf(stderr, "[pmns setup] repair round %d\n", rounds);
    std::vector<int64_t> prim(g.nvox(), -1);
    for (int64_t f = 0; f < g.nvox(); ++f)
      if (g.is_void[f] && iface[f] < 0) prim[f] = lab[f];
    std::vector<uint8_t> flt = floating(g, ff, fnb, prim);
    std::vector<int64_t> cells;
    for (int64_t f = 0; f < g.n_f; ++f)
      if (flt[f]) {
        if (ff.c0[f] >= 0 && prim[ff.c0[f]] >= 0) cells.push_back(ff.c0[f]);
        if (ff.c1[f] >= 0 && prim[ff.c1[f]] >= 0) cells.push_back(ff.c1[f]);
      }
    if (cells.empty()) return;
    std::sort(cells.begin(), cells.end());
    cells.erase(std::unique(cells.begin(), cells.end()), cells.end());
    std::vector<std::pair<int64_t, int32_t>> upd;
    for (int64_t c : cells) {
      int n = box_nbrs(g, c, bn);
      int32_t m = INT32_MAX;
      for (int q = 0; q < n; ++q)
        if (bn[q] >= 0 && iface[bn[q]] >= 0 && iface[bn[q]] < m) m = iface[bn[q]];
      if (m != INT32_MAX) upd.emplace_back(c, m);
    }
    if (upd.empty()) throw std::runtime_error("EINVAL: D7b floating faces with no adjacent interface");
    for (auto &u : upd) iface[u.first] = u.second;
  }
}


void decompose(const Geometry &g, double h_m, int n_min, int dual_layers, int mask_band, Decomp &d) {
  SetupTimer tm;
  int64_t nv = g.nvox();
  std::vector<int64_t> D = squared_edt(g);
  tm.lap("edt");
  std::vector<int64_t> lab;
  int64_t nraw = watershed(g, D, lab);
  d.raw_basins = nraw;
  tm.lap("watershed");
  merge_basins(g, lab, nraw, D, h_m, n_min);
  tm.lap("merge");
  FaceFlank ff;
  face_flanks(g, ff);
  tm.lap("face flanks");
  const std::vector<int32_t> fnb = face_nbr_codes(g);
  tm.lap("face nbr codes");
  std::vector<int32_t> iface;
  int nc = 0;
  auto first_empty = [&](const std::vector<int32_t> &ifc) -> int64_t {
    int64_t nl = 0;
    for (int64_t f = 0; f < nv; ++f)
      if (lab[f] >= 0) nl = std::max(nl, lab[f] + 1);
    std::vector<int64_t> cnt(nl, 0);
    for (int64_t f = 0; f < nv; ++f)
      if (g.is_void[f] && ifc[f] < 0) cnt[lab[f]]++;
    for (int64_t a = 0; a < nl; ++a)
      if (cnt[a] == 0) return a;
    return -1;
  };
  int outer = 0;
  while (true) {
    ++outer;
    nc = compute_interfaces(g, lab, iface);
    tm.lap("iface pass");
    int64_t a = first_empty(iface);
    if (a < 0) {
      repair_floating(g, ff, fnb, lab, iface);
      a = first_empty(iface);
      if (a < 0) break;
    }
    int64_t nl = 0;
    for (int64_t f = 0; f < nv; ++f)
      if (lab[f] >= 0) nl = std::max(nl, lab[f] + 1);
    Adj S;
    saddles(g, lab, D, nl, S);
    if (S[a].empty()) throw std::runtime_error("EINVAL: empty primary without neighbours");
    int64_t b = -1, bs = -1;
    for (auto &kv : S[a])
      if (kv.second > bs || (kv.second == bs && kv.first < b)) {
        bs = kv.second;
        b = kv.first;
      }
    for (int64_t f = 0; f < nv; ++f)
      if (lab[f] == a) lab[f] = b;
    relabel_by_first(g, lab);
  }
  tm.lap("interfaces");
  int64_t np = 0;
  for (int64_t f = 0; f < nv; ++f)
    if (lab[f] >= 0) np = std::max(np, lab[f] + 1);
  d.n_p = (int)np;
  d.n_c = nc;
  d.label.assign(nv, -1);
  d.iface = iface;
  for (int64_t f = 0; f < nv; ++f)
    if (g.is_void[f] && iface[f] < 0) d.label[f] = (int32_t)lab[f];
  // D8 duals: geodesic dilation
  std::vector<std::vector<int64_t>> seeds(nc);
  for (int64_t f = 0; f < nv; ++f)
    if (iface[f] >= 0) seeds[iface[f]].push_back(f);
  d.duals.assign(nc, {});
  std::vector<int64_t> mark(nv, -1);
  Nbr nb;
  for (int j = 0; j < nc; ++j) {
    std::vector<int64_t> cur = seeds[j], front = seeds[j], nxt;
    for (int64_t f : cur) mark[f] = j;
    for (int s = 0; s < dual_layers; ++s) {
      nxt.clear();
      for (int64_t f : front) {
        face_nbrs(g, f, nb);
        for (int c = 0; c < nb.n; ++c) {
          int64_t u = nb.v[c];
          if (u >= 0 && g.is_void[u] && mark[u] != j) {
            mark[u] = j;
            nxt.push_back(u);
          }
        }
      }
      if (nxt.empty()) break;
      cur.insert(cur.end(), nxt.begin(), nxt.end());
      front = nxt;
    }
    std::sort(cur.begin(), cur.end());
    d.duals[j] = cur;
  }
  // D9 mask band
  std::vector<int32_t> dist(nv, -1);
  std::vector<int64_t> front, nxt;
  for (int64_t f = 0; f < nv; ++f)
    if (iface[f] >= 0) {
      dist[f] = 0;
      front.push_back(f);
    }
  for (int s = 1; s <= mask_band; ++s) {
    nxt.clear();
    for (int64_t f : front) {
      face_nbrs(g, f, nb);
      for (int c = 0; c < nb.n; ++c) {
        int64_t u = nb.v[c];
        if (u >= 0 && g.is_void[u] && dist[u] < 0) {
          dist[u] = s;
          nxt.push_back(u);
        }
      }
    }
    front.swap(nxt);
  }
  d.mask_cell.assign(nv, 0);
  for (int64_t f = 0; f < nv; ++f) d.mask_cell[f] = dist[f] >= 0;
  tm.lap("duals+mask");
}

// ----------------------------------------------------------------------------
// D10 and the W order
// ----------------------------------------------------------------------------
void make_layout(const Geometry &g, const Decomp &d, Layout &L) {
  FaceFlank ff;
  face_flanks(g, ff);
  int64_t N = g.N, nf = g.n_f;
  std::vector<int64_t> grp(N);
  L.face_owner_p.assign(nf, -1);
  L.face_mask.assign(nf, 0);
  for (int64_t f = 0; f < nf; ++f) {
    int64_t c0 = ff.c0[f], c1 = ff.c1[f];
    int32_t p = -1;
    if (c0 >= 0 && d.label[c0] >= 0) p = d.label[c0];
    if (c1 >= 0 && d.label[c1] >= 0) p = d.label[c1];
    L.face_owner_p[f] = p;
    if (p >= 0) {
      grp[f] = p;
    } else {
      int32_t m = INT32_MAX;
      if (c0 >= 0 && d.iface[c0] >= 0) m = std::min(m, d.iface[c0]);
      if (c1 >= 0 && d.iface[c1] >= 0) m = std::min(m, d.iface[c1]);
      if (m == INT32_MAX) throw std::runtime_error("EINVAL: face without owner");
      grp[f] = (int64_t)d.n_p + d.n_c + m;
    }
    L.face_mask[f] = (c0 >= 0 && d.mask_cell[c0]) || (c1 >= 0 && d.mask_cell[c1]);
  }
  for (int64_t v = 0; v < g.nvox(); ++v) {
    if (!g.is_void[v]) continue;
    int64_t id = g.cmap[v];
    grp[id] = d.label[v] >= 0 ? d.label[v] : (int64_t)d.n_p + d.iface[v];
  }
  int64_t ng = (int64_t)d.n_p + 2 * d.n_c;
  std::vector<int64_t> cnt(ng + 1, 0);
  for (int64_t u = 0; u < N; ++u) cnt[grp[u] + 1]++;
  for (int64_t q = 0; q < ng; ++q) cnt[q + 1] += cnt[q];
  L.seg = cnt;
  L.perm.assign(N, 0);
  std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
  for (int64_t u = 0; u < N; ++u) L.perm[pos[grp[u]]++] = u;   // stable: canonical order within group
  L.inv.assign(N, 0);
  for (int64_t w = 0; w < N; ++w) L.inv[L.perm[w]] = w;
  // dual unknown sets (cells + faces with >= 1 flank in the dual), device slots sorted
  std::vector<int64_t> mark(g.nvox(), -1);
  L.dual_unknowns.assign(d.n_c, {});
  // faces by flank voxel: build voxel -> faces adjacency
  std::vector<int64_t> vptr(g.nvox() + 1, 0);
  for (int64_t f = 0; f < nf; ++f) {
    if (ff.c0[f] >= 0) vptr[ff.c0[f] + 1]++;
    if (ff.c1[f] >= 0) vptr[ff.c1[f] + 1]++;
  }
  for (int64_t v = 0; v < g.nvox(); ++v) vptr[v + 1] += vptr[v];
  std::vector<int64_t> vf(vptr.back()), fill(vptr.begin(), vptr.end() - 1);
  for (int64_t f = 0; f < nf; ++f) {
    if (ff.c0[f] >= 0) vf[fill[ff.c0[f]]++] = f;
    if (ff.c1[f] >= 0) vf[fill[ff.c1[f]]++] = f;
  }
  for (int j = 0; j < d.n_c; ++j) {
    std::vector<int64_t> &out = L.dual_unknowns[j];
    for (int64_t v : d.duals[j]) {
      out.push_back(L.inv[g.cmap[v]]);
      for (int64_t q = vptr[v]; q < vptr[v + 1]; ++q) out.push_back(L.inv[vf[q]]);
    }
    std::sort(out.begin(), out.end());
    out.erase(std::unique(out.begin(), out.end()), out.end());
  }
}

}  // namespace pmns
