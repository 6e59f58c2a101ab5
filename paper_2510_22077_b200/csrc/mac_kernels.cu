// Matrix-free MAC operators on the compact void-only layout (SURVEY §8(a)
// rows a1, a2, a6, a8, a10 and the J~_w build operator).
//
//  a1  r(x)   = rho (u-u^n)/dt + rho N(u) - mu L u + grad p - rho b ; div u
//      (Eq. governing_eqs, Eq. Ax=b P:34-65; readings A3-A8)
//  a2  J(x) v = rho/dt v + rho sum_b [c_b(u) D_b v + c_b(v) D_b u] - mu L v + grad v_p ; div v
//      (reading A9: exact derivative with the upwind selector frozen)
//  JW  J~_w v = rho/dt v + [face not masked] rho sum_b c_b(w) D_b v - mu L v + grad v_p ; div v
//      (Eq. mod_res: inertia removed near interfaces)
//
// One thread per unknown (row).  Neighbours are found through dense int32
// position maps (face maps per orientation, cell map) holding device slots or
// the codes ZERO (one solid flank), GHOST (both flanks solid); MIRROR is
// implied beyond the inlet/outlet planes.
#include "kernels.cuh"

namespace pmns {

constexpr int kJacMinBlocks = 6;   // default of PMNS_JAC_MINB (measured: scripts/bench_jacobian.py)

namespace {

__device__ __forceinline__ int wrapi(int x, int n) {
  x %= n;
  return x < 0 ? x + n : x;
}

// code of face (a; k, j, i): device slot >= 0, or kDZero / kDGhost / kDMirror
__device__ __forceinline__ int32_t fcode(const DevGeom &G, int a, int k, int j, int i) {
  if (a == 0 ? (i < 0 || i > G.nx) : (i < 0 || i >= G.nx)) return kDMirror;
  if (G.py) j = wrapi(j, G.ny);
  else if (j < 0 || j >= G.fy[a]) return kDGhost;
  if (G.dim == 3) {
    if (G.pz) k = wrapi(k, G.nz);
    else if (k < 0 || k >= G.fz[a]) return kDGhost;
  } else if (k != 0) {
    return kDGhost;
  }
  return __ldg(G.fmap[a] + ((int64_t)k * G.fy[a] + j) * G.fx[a] + i);
}

// cell slot, -1 solid (incl. lateral outside), -3 outside in x
__device__ __forceinline__ int32_t ccode(const DevGeom &G, int k, int j, int i) {
  if (i < 0 || i >= G.nx) return kDMirror;
  if (G.py) j = wrapi(j, G.ny);
  else if (j < 0 || j >= G.ny) return -1;
  if (G.dim == 3) {
    if (G.pz) k = wrapi(k, G.nz);
    else if (k < 0 || k >= G.nz) return -1;
  } else if (k != 0) {
    return -1;
  }
  return __ldg(G.cmap + ((int64_t)k * G.ny + j) * G.nx + i);
}

// neighbour value rule (reading A5/A6)
__device__ __forceinline__ double vrule(int32_t code, const double *__restrict__ v, double vf) {
  if (code >= 0) return __ldg(v + code);
  if (code == kDZero) return 0.0;
  if (code == kDGhost) return -vf;
  return vf;  // mirror
}

__device__ __forceinline__ void shift(int b, int o, int &k, int &j, int &i) {
  if (b == 0) i += o;
  else if (b == 1) j += o;
  else k += o;
}

// advecting velocity c_b at an a-face (reading A5), for two vectors at once
__device__ __forceinline__ void cadv(const DevGeom &G, int a, int b, int k, int j, int i,
                                     const double *__restrict__ s, const double *__restrict__ v, double &cs,
                                     double &cv) {
  // flank cells: low = pos - e_a (in cell coordinates), high = pos
  int kl = k, jl = j, il = i;
  shift(a, -1, kl, jl, il);
  double ss = 0.0, sv = 0.0;
  int nin = 0;
  for (int side = 0; side < 2; ++side) {
    int kc = side ? k : kl, jc = side ? j : jl, ic = side ? i : il;
    int32_t c = ccode(G, kc, jc, ic);
    if (c < 0) continue;
    ++nin;
    int32_t f0 = fcode(G, b, kc, jc, ic);
    int kh = kc, jh = jc, ih = ic;
    shift(b, 1, kh, jh, ih);
    int32_t f1 = fcode(G, b, kh, jh, ih);
    if (f0 >= 0) {
      ss += __ldg(s + f0);
      if (v) sv += __ldg(v + f0);
    }
    if (f1 >= 0) {
      ss += __ldg(s + f1);
      if (v) sv += __ldg(v + f1);
    }
  }
  double w = 1.0 / (2.0 * nin);
  cs = ss * w;
  cv = sv * w;
}

// Per-row stencil codes (built once by stencil_kernel; SoA, kTab x N int32):
//   face rows (orientation a): q = 4b + {0,1,2,3} -> neighbour position of
//   orientation a at offset {-2,-1,+1,+2} e_b (slot or ZERO/GHOST/MIRROR);
//   q = 12 + 4 bi + 2 side + lh -> the b-face (low/high) of the low/high flank
//   cell, for the bi-th direction b != a (slot, or -1 if not a DOF or the
//   flank is not void); q = 20, 21 -> low / high flank cell (ccode).
//   cell rows: q = 2b + {0,1} -> low / high b-face (slot or negative).
__global__ void stencil_kernel(DevGeom G, int32_t *__restrict__ tab) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= G.N) return;
  uint32_t pp = __ldg(G.rowpos + r);
  int t = pp >> 30, k = (pp >> 20) & 1023, j = (pp >> 10) & 1023, i = pp & 1023;
  const int64_t N = G.N;
  for (int q = 0; q < kTab; ++q) tab[q * N + r] = -1;
  if (t == 3) {
    for (int bb = 0; bb < G.dim; ++bb) {
      int kh = k, jh = j, ih = i;
      shift(bb, 1, kh, jh, ih);
      tab[(2 * bb) * N + r] = fcode(G, bb, k, j, i);
      tab[(2 * bb + 1) * N + r] = fcode(G, bb, kh, jh, ih);
    }
    return;
  }
  const int a = t;
  for (int bb = 0; bb < G.dim; ++bb)
    for (int oi = 0; oi < 4; ++oi) {
      const int o = oi < 2 ? oi - 2 : oi - 1;
      int k1 = k, j1 = j, i1 = i;
      shift(bb, o, k1, j1, i1);
      tab[(4 * bb + oi) * N + r] = fcode(G, a, k1, j1, i1);
    }
  int kl = k, jl = j, il = i;
  shift(a, -1, kl, jl, il);
  int32_t c0 = ccode(G, kl, jl, il), c1 = ccode(G, k, j, i);
  tab[20 * N + r] = c0;
  tab[21 * N + r] = c1;
  int bi = 0;
  for (int bb = 0; bb < G.dim; ++bb) {
    if (bb == a) continue;
    for (int side = 0; side < 2; ++side) {
      int kc = side ? k : kl, jc = side ? j : jl, ic = side ? i : il;
      if ((side ? c1 : c0) < 0) continue;
      int kh = kc, jh = jc, ih = ic;
      shift(bb, 1, kh, jh, ih);
      int32_t f0 = fcode(G, bb, kc, jc, ic), f1 = fcode(G, bb, kh, jh, ih);
      tab[(12 + 4 * bi + 2 * side) * N + r] = f0 >= 0 ? f0 : -1;
      tab[(12 + 4 * bi + 2 * side + 1) * N + r] = f1 >= 0 ? f1 : -1;
    }
    ++bi;
  }
}

// Operand accessors of the row evaluation: a device vector, or the unit
// vector e_q (direct Jacobian assembly: the coefficient of column q is the
// row evaluated on e_q, with the same operations as the apply).
struct VGlob {
  const double *__restrict__ v;
  __device__ __forceinline__ double operator()(int64_t i) const { return __ldg(v + i); }
};
struct VUnit {
  int64_t q;
  __device__ __forceinline__ double operator()(int64_t i) const { return i == q ? 1.0 : 0.0; }
};
template <class VA>
__device__ __forceinline__ double vrule_a(int32_t code, const VA &va, double vf) {
  if (code >= 0) return va(code);
  if (code == kDZero) return 0.0;
  if (code == kDGhost) return -vf;
  return vf;  // mirror
}

// Momentum row of face slot r (orientation a) given its stencil codes (the
// arithmetic shared by the per-row-table and the cell-record evaluations).
template <int MODE, class VA>
__device__ __forceinline__ void face_row(const DevGeom &G, int64_t r, int a, const int32_t (&nb)[3][4],
                                         int32_t c0, int32_t c1, const int32_t (&fl)[8],
                                         const double *__restrict__ st, const double *__restrict__ up,
                                         const VA &va, double &out, double &out2) {
  constexpr bool kDual = MODE == MODE_DUAL;
  constexpr bool kRes = MODE == MODE_RES || MODE == MODE_RESM;
  constexpr bool kJac = MODE == MODE_JAC || MODE == MODE_JACM || kDual;
  constexpr bool kMasked = MODE == MODE_JW || MODE == MODE_JACM || MODE == MODE_RESM;
  out2 = 0.0;
  const double inv_h = 1.0 / G.h;
  const double vf = va(r);
  // viscous Laplacian (A6)
  double lap = 0.0;
#pragma unroll
  for (int bb = 0; bb < 3; ++bb)
    if (bb < G.dim) lap += vrule_a(nb[bb][1], va, vf) + vrule_a(nb[bb][2], va, vf) - 2.0 * vf;
  lap *= inv_h * inv_h;
  // pressure gradient (A3): flanks low = pos - e_a, high = pos
  double p0, p1;
  if (kRes) {
    p0 = c0 >= 0 ? __ldg(st + c0) : (c0 == kDMirror ? G.p_in : 0.0);
    p1 = c1 >= 0 ? __ldg(st + c1) : (c1 == kDMirror ? G.p_out : 0.0);
  } else {
    p0 = c0 >= 0 ? va(c0) : 0.0;
    p1 = c1 >= 0 ? va(c1) : 0.0;
  }
  double grad = (p1 - p0) * inv_h;
  // inertia (A5 / A9 / A10)
  double conv = 0.0, convA = 0.0;   // convA: the Oseen part (dual mode)
  bool do_conv = G.rho != 0.0 && (!kMasked || !G.mask[r]);
  if (do_conv) {
    const double sf = __ldg(st + r);
    const double w = 1.0 / (2.0 * ((c0 >= 0) + (c1 >= 0)));
    int bi = 0;
#pragma unroll
    for (int bb = 0; bb < 3; ++bb) {
      if (bb >= G.dim) break;
      double cs, cv;
      if (bb == a) {
        cs = sf;
        cv = vf;
      } else {
        // advecting velocity: mean of the b-faces of the void flank cells
        double ss = 0.0, sv = 0.0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          int32_t f = bi == 0 ? fl[e] : fl[4 + e];   // (register select: bi is data-dependent)
          if (f >= 0) {
            ss += __ldg(st + f);
            if (kJac) sv += va(f);
          }
        }
        cs = ss * w;
        cv = sv * w;
        ++bi;
      }
      const int sg = cs >= 0.0 ? 1 : -1;
      const int32_t m1 = sg > 0 ? nb[bb][1] : nb[bb][2], m2 = sg > 0 ? nb[bb][0] : nb[bb][3];
      const bool use2 = (m2 >= 0) || (m2 == kDZero);
      double Ds;
      {
        double s1 = vrule(m1, st, sf);
        Ds = use2 ? (3.0 * sf - 4.0 * s1 + vrule(m2, st, sf)) * (0.5 * inv_h) : (sf - s1) * inv_h;
        Ds *= (double)sg;
      }
      if (kRes) {
        conv += cs * Ds;
      } else {
        double v1 = vrule_a(m1, va, vf);
        double Dv = use2 ? (3.0 * vf - 4.0 * v1 + vrule_a(m2, va, vf)) * (0.5 * inv_h) : (vf - v1) * inv_h;
        Dv *= (double)sg;
        conv += cs * Dv;
        if (kDual) convA += cs * Dv;
        if (kJac) conv += cv * Ds;
      }
    }
    conv *= G.rho;
    convA *= G.rho;
  }
  double tt = 0.0;
  if (G.dt > 0.0) {
    if (kRes) tt = G.rho * (vf - (up ? __ldg(up + r) : 0.0)) / G.dt;
    else tt = G.rho / G.dt * vf;
  }
  out = tt + conv - G.mu * lap + grad;
  if (kDual) out2 = tt + (G.mask[r] ? 0.0 : convA) - G.mu * lap + grad;
  if (kRes) out -= G.rho * G.bf[a];
}


// One row of the operator (Eq. navstokes_mom / navstokes_mass on the MAC grid,
// readings A3-A10): out = row r of Op(v) (MODE_RES/RESM: of r(state)); in
// MODE_DUAL also out2 = row r of J~_w v (masked Oseen, w = state).
template <int MODE, class VA>
__device__ __forceinline__ void row_eval(const DevGeom &G, int64_t r, const double *__restrict__ st,
                                         const double *__restrict__ up, const VA &va, double &out,
                                         double &out2) {
  out2 = 0.0;
  const int64_t N = G.N;
  // the row's codes are read once: streamed (evict-first) so that L1 keeps the gathered operands
  const int32_t *__restrict__ T = G.tab + r;
  const int t = __ldcs(G.rowpos + r) >> 30;
  const double inv_h = 1.0 / G.h;
  if (t == 3) {
    // mass row: div (Eq. navstokes_mass; A8 sign +div)
    double d = 0.0;
    for (int bb = 0; bb < G.dim; ++bb) {
      int32_t f0 = __ldcs(T + (2 * bb) * N), f1 = __ldcs(T + (2 * bb + 1) * N);
      double v0 = f0 >= 0 ? va(f0) : 0.0;
      double v1 = f1 >= 0 ? va(f1) : 0.0;
      d += v1 - v0;
    }
    out = d * inv_h;
    out2 = out;   // mass rows are the same in J and J~_w (dual mode)
    return;
  }
  const int a = t;
  int32_t nb[3][4];
#pragma unroll
  for (int bb = 0; bb < 3; ++bb)
#pragma unroll
    for (int oi = 0; oi < 4; ++oi) nb[bb][oi] = bb < G.dim ? __ldcs(T + (4 * bb + oi) * N) : -1;
  const int32_t c0 = __ldcs(T + 20 * N), c1 = __ldcs(T + 21 * N);
  // flank-face codes of the advecting velocity, loaded with the other codes
  // (one dependent memory round trip fewer per row)
  int32_t fl[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) fl[e] = (G.rho != 0.0 && e < 4 * (G.dim - 1)) ? __ldcs(T + (12 + e) * N) : -1;
  // (specialising the orientation per branch was measured: no faster, and the
  // direct assembly then no longer reproduces the probed matrices bit for bit)
  face_row<MODE>(G, r, a, nb, c0, c1, fl, st, up, va, out, out2);
}

template <int MODE, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) apply_kernel(DevGeom G, const double *__restrict__ st,
                                                    const double *__restrict__ up, const double *__restrict__ v,
                                                    double *__restrict__ y, double alpha,
                                                    const double *__restrict__ b, double beta, int64_t vstride,
                                                    double *__restrict__ y2, int64_t r0 = 0, int64_t r1 = -1) {
  int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (r1 < 0 ? G.N : r1)) return;
  // gridDim.y > 1: a batch of vectors (probing), vector q at v + q*vstride, y + q*vstride
  v += (int64_t)blockIdx.y * vstride;
  y += (int64_t)blockIdx.y * vstride;
  constexpr bool kDual = MODE == MODE_DUAL;
  if (kDual) y2 += (int64_t)blockIdx.y * vstride;
  double out, out2;
  row_eval<MODE>(G, r, st, up, VGlob{v}, out, out2);   // RES modes: v = state
  double res = alpha * out;
  if (b) res += beta * __ldg(b + r);
  y[r] = res;
  if (kDual) y2[r] = alpha * out2;
}

// ---------------------------------------------------------------------------
// Krylov-phase J apply over cell records (K2).  One
// thread per (void cell, row role) evaluates the cell's mass row and the momentum
// rows of the faces stored with it (its low a-faces); stencil slots are reached
// through the records' neighbour indices (second neighbours by a second hop,
// L1/L2-resident), non-DOF positions come from 2 class bits each, so a cell
// costs 52 bytes of index data instead of ~3.7 x 88 bytes of per-row codes.
// The arithmetic is face_row<MODE_JAC>, the same as the per-row path, so both
// give the same bits.  Rows the record chase cannot reproduce (bit 31; e.g. a
// second neighbour behind a one-voxel wall) and the x-max boundary faces are
// evaluated from the per-row table by jrow_list_kernel (a second, small launch).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int32_t rec_step(const DevGeom &G, int32_t X, int d) {
  return X >= 0 ? __ldg(G.rec_n + (int64_t)d * G.n_rec + X) : -1;
}
// slot of the low a-face at record position X (x-max code: the boundary face)
__device__ __forceinline__ int32_t rec_face(const DevGeom &G, int a, int32_t X) {
  if (X >= 0) return __ldg(G.rec_f + (int64_t)a * G.n_rec + X);
  if (X <= -4 && a == 0) return __ldg(G.xm_slot + (-4 - X));
  return -1;
}

__device__ __forceinline__ void jrec_store(double *__restrict__ y, int64_t r, double out, double alpha,
                                           const double *__restrict__ b, double beta) {
  double res = alpha * out;
  if (b) res += beta * __ldg(b + r);
  y[r] = res;
}

// momentum row of record c's low A-face (A compile-time: all stencil arrays
// stay in registers)
template <int A>
__device__ __forceinline__ void jrec_face(const DevGeom &G, int64_t c, const double *__restrict__ st,
                                          const double *__restrict__ v, double *__restrict__ y, double alpha,
                                          const double *__restrict__ b, double beta) {
  constexpr int a = A;
  const int64_t R = G.n_rec;
  const VGlob va{v};
  double out, out2;
  const int32_t f = __ldg(G.rec_f + a * R + c);
  if (f < 0) return;
  const uint32_t cw = __ldg(G.rec_c + a * R + c);
  if (cw >> 31) return;   // flagged: jrow_list_kernel
  int32_t nbr[6];
#pragma unroll
  for (int d = 0; d < 6; ++d) nbr[d] = d < 2 * G.dim ? __ldg(G.rec_n + d * R + c) : -1;
  int32_t nb[3][4];
#pragma unroll
  for (int bb = 0; bb < 3; ++bb)
#pragma unroll
    for (int oi = 0; oi < 4; ++oi) {
      if (bb >= G.dim) {
        nb[bb][oi] = -1;
        continue;
      }
      const uint32_t k = (cw >> (2 * (4 * bb + oi))) & 3u;
      if (k) {
        nb[bb][oi] = -(int32_t)k;   // 1 ZERO, 2 GHOST, 3 MIRROR (kDZero/kDGhost/kDMirror)
      } else {
        const int d = 2 * bb + (oi >= 2);
        int32_t X = nbr[d];
        if (oi == 0 || oi == 3) X = rec_step(G, X, d);
        nb[bb][oi] = rec_face(G, a, X);
      }
    }
  const int32_t L = nbr[2 * a];   // low flank record (-3: beyond the inlet)
  const int32_t c0 = L >= 0 ? __ldg(G.rec_p + L) : L;
  const int32_t ps = __ldg(G.rec_p + c);
  int32_t fl[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) fl[e] = -1;
  if (G.rho != 0.0) {
    int bi = 0;
#pragma unroll
    for (int bb = 0; bb < 3; ++bb) {
      if (bb >= G.dim || bb == a) continue;
      if (L >= 0) {
        fl[4 * bi + 0] = rec_face(G, bb, L);
        fl[4 * bi + 1] = rec_face(G, bb, rec_step(G, L, 2 * bb + 1));
      }
      fl[4 * bi + 2] = __ldg(G.rec_f + bb * R + c);
      fl[4 * bi + 3] = rec_face(G, bb, nbr[2 * bb + 1]);
      ++bi;
    }
  }
  face_row<MODE_JAC>(G, f, a, nb, c0, ps, fl, st, nullptr, va, out, out2);
  jrec_store(y, f, out, alpha, b, beta);
}

__global__ void __launch_bounds__(256) jrec_kernel(DevGeom G, const double *__restrict__ st,
                                                   const double *__restrict__ v, double *__restrict__ y,
                                                   double alpha, const double *__restrict__ b, double beta) {
  // one grid row per role (warps stay uniform; record loads coalesced):
  // role 0 = the mass row, role 1 + a = the momentum row of the low a-face
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int role = (int)blockIdx.y;
  if (c >= G.n_rec) return;
  const int64_t R = G.n_rec;
  const VGlob va{v};
  double out, out2;
  if (role == 0) {
    const uint32_t cw0 = __ldg(G.rec_c + c);
    if (cw0 & (1u << 30)) return;   // flagged: jrow_list_kernel
    // mass row (Eq. navstokes_mass, A8): high b-face = low b-face of the +b neighbour
    double dsum = 0.0;
#pragma unroll
    for (int bb = 0; bb < 3; ++bb) {
      if (bb >= G.dim) break;
      const int32_t f0 = __ldg(G.rec_f + bb * R + c);
      const int32_t f1 = rec_face(G, bb, __ldg(G.rec_n + (2 * bb + 1) * R + c));
      double v0 = f0 >= 0 ? va(f0) : 0.0;
      double v1 = f1 >= 0 ? va(f1) : 0.0;
      dsum += v1 - v0;
    }
    out = dsum * (1.0 / G.h);
    jrec_store(y, __ldg(G.rec_p + c), out, alpha, b, beta);
    return;
  }
  if (role == 1) jrec_face<0>(G, c, st, v, y, alpha, b, beta);
  else if (role == 2) jrec_face<1>(G, c, st, v, y, alpha, b, beta);
  else jrec_face<2>(G, c, st, v, y, alpha, b, beta);
}

// The rows jrec_kernel leaves out (flagged records, x-max boundary faces),
// evaluated from the per-row table.
__global__ void __launch_bounds__(128) jrow_list_kernel(DevGeom G, const int32_t *__restrict__ rows, int64_t n,
                                                        const double *__restrict__ st, const double *__restrict__ v,
                                                        double *__restrict__ y, double alpha,
                                                        const double *__restrict__ b, double beta) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int32_t r = __ldg(rows + q);
  double out, out2;
  row_eval<MODE_JAC>(G, r, st, nullptr, VGlob{v}, out, out2);
  jrec_store(y, r, out, alpha, b, beta);
}

// Direct ELL assembly of the operator's matrix (replaces colour probing; the
// same entries bit for bit): row r's candidate columns are the slots its
// stencil codes name; each coefficient is the row evaluated on e_q.  Entries
// are emitted in the order colour probing with periods (px, py, pz) would
// produce (ascending colour index), exact zeros skipped.  MODE_DUAL fills E
// with J and E2 with J~_w; other modes fill E only.
template <int MODE>
__global__ void __launch_bounds__(128) assemble_kernel(DevGeom G, const double *__restrict__ st, int px, int py,
                                                       int pz, int32_t *__restrict__ col1, double *__restrict__ val1,
                                                       int32_t *__restrict__ cnt1, int32_t *__restrict__ col2,
                                                       double *__restrict__ val2, int32_t *__restrict__ cnt2,
                                                       int width, int *overflow) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= G.N) return;
  const int64_t N = G.N;
  const int32_t *__restrict__ T = G.tab + r;
  const int t = __ldg(G.rowpos + r) >> 30;
  int32_t cand[24];
  uint32_t key[24] = {};
  int nc = 0;
  auto add = [&](int32_t q) {
    if (q < 0) return;
    for (int e = 0; e < nc; ++e)
      if (cand[e] == q) return;
    const uint32_t pp = __ldg(G.rowpos + q);
    const int tq = (int)(pp >> 30);
    const uint32_t ti = tq == 3 ? (uint32_t)G.dim : (uint32_t)tq;
    const uint32_t kq = (pp >> 20) & 1023, jq = (pp >> 10) & 1023, iq = pp & 1023;
    const uint32_t kk = ((ti * pz + kq % pz) * py + jq % py) * px + iq % px;
    int e = nc++;
    while (e > 0 && key[e - 1] > kk) {   // insertion by colour index
      key[e] = key[e - 1];
      cand[e] = cand[e - 1];
      --e;
    }
    key[e] = kk;
    cand[e] = q;
  };
  add((int32_t)r);
  if (t == 3) {
    for (int q = 0; q < 2 * G.dim; ++q) add(__ldg(T + q * N));
  } else {
    for (int bb = 0; bb < G.dim; ++bb)
      for (int oi = 0; oi < 4; ++oi) add(__ldg(T + (4 * bb + oi) * N));
    add(__ldg(T + 20 * N));
    add(__ldg(T + 21 * N));
    for (int e = 12; e < 20; ++e) add(__ldg(T + e * N));
  }
  int n1 = 0, n2 = 0;
  for (int e = 0; e < nc; ++e) {
    double o, o2;
    row_eval<MODE>(G, r, st, nullptr, VUnit{cand[e]}, o, o2);
    if (o != 0.0) {
      if (n1 < width) {
        col1[r * (int64_t)width + n1] = cand[e];
        val1[r * (int64_t)width + n1] = o;
        ++n1;
      } else {
        atomicOr(overflow, 1);
      }
    }
    if (MODE == MODE_DUAL && o2 != 0.0) {
      if (n2 < width) {
        col2[r * (int64_t)width + n2] = cand[e];
        val2[r * (int64_t)width + n2] = o2;
        ++n2;
      } else {
        atomicOr(overflow, 1);
      }
    }
  }
  cnt1[r] = n1;
  if (MODE == MODE_DUAL) cnt2[r] = n2;
}

}  // namespace

// Resident CTAs per SM the Krylov-phase J apply is compiled for (register cap):
// PMNS_JAC_MINB = 1 (64 registers, 4 CTAs), 5 (48 registers), 6 (40 registers, the default: 0.68 ms against
// 0.73 ms at N = 15.25M) or 8 (32 registers)
static int jac_min_blocks() {
  static const int mb = [] {
    const char *e = getenv("PMNS_JAC_MINB");
    return e ? atoi(e) : kJacMinBlocks;
  }();
  return mb;
}

// y = J(state) v and y2 = J~_w v (w = state), nvec vectors (build-time probing)
void launch_apply_dual(const DevGeom &G, const double *state, const double *v, double *y, double *y2,
                       cudaStream_t s, int nvec) {
  int64_t nb = (G.N + 255) / 256;
  if (nb == 0) return;
  apply_kernel<MODE_DUAL><<<dim3((unsigned)nb, (unsigned)nvec), 256, 0, s>>>(G, state, nullptr, v, y, 1.0, nullptr,
                                                                           0.0, G.N, y2);
}

void launch_assemble(const DevGeom &G, int mode, const double *state, int px, int py, int pz, int32_t *col1,
                     double *val1, int32_t *cnt1, int32_t *col2, double *val2, int32_t *cnt2, int width,
                     int *overflow, cudaStream_t s) {
  int64_t nb = (G.N + 127) / 128;
  if (nb == 0) return;
  if (mode == MODE_DUAL)
    assemble_kernel<MODE_DUAL><<<(unsigned)nb, 128, 0, s>>>(G, state, px, py, pz, col1, val1, cnt1, col2, val2, cnt2,
                                                            width, overflow);
  else if (mode == MODE_JW)
    assemble_kernel<MODE_JW><<<(unsigned)nb, 128, 0, s>>>(G, state, px, py, pz, col1, val1, cnt1, nullptr, nullptr,
                                                          nullptr, width, overflow);
  else if (mode == MODE_JACM)
    assemble_kernel<MODE_JACM><<<(unsigned)nb, 128, 0, s>>>(G, state, px, py, pz, col1, val1, cnt1, nullptr,
                                                            nullptr, nullptr, width, overflow);
  else
    assemble_kernel<MODE_JAC><<<(unsigned)nb, 128, 0, s>>>(G, state, px, py, pz, col1, val1, cnt1, nullptr, nullptr,
                                                           nullptr, width, overflow);
}

void launch_apply_jrec(const DevGeom &G, const double *state, const double *v, double *y, double alpha,
                       const double *b, double beta, cudaStream_t s) {
  const int64_t nb = (G.n_rec + 255) / 256;
  if (nb) jrec_kernel<<<dim3((unsigned)nb, (unsigned)(G.dim + 1)), 256, 0, s>>>(G, state, v, y, alpha, b, beta);
  const int64_t nl = (G.n_rec_rows + 127) / 128;
  if (nl) jrow_list_kernel<<<(unsigned)nl, 128, 0, s>>>(G, G.rec_rows, G.n_rec_rows, state, v, y, alpha, b, beta);
}

void launch_apply_range(const DevGeom &G, int mode, const double *state, const double *uprev, const double *v,
                        double *y, double alpha, const double *b, double beta, cudaStream_t s, int64_t r0,
                        int64_t r1) {
  const int bs = 256;
  const int64_t nb = (r1 - r0 + bs - 1) / bs;
  if (nb <= 0) return;
  if (mode == MODE_JAC) {
    const int mb = jac_min_blocks();
    if (mb == 5)
      apply_kernel<MODE_JAC, 5><<<(unsigned)nb, bs, 0, s>>>(G, state, uprev, v, y, alpha, b, beta, G.N, nullptr, r0, r1);
    else if (mb == 6)
      apply_kernel<MODE_JAC, 6><<<(unsigned)nb, bs, 0, s>>>(G, state, uprev, v, y, alpha, b, beta, G.N, nullptr, r0, r1);
    else if (mb == 8)
      apply_kernel<MODE_JAC, 8><<<(unsigned)nb, bs, 0, s>>>(G, state, uprev, v, y, alpha, b, beta, G.N, nullptr, r0, r1);
    else
      apply_kernel<MODE_JAC><<<(unsigned)nb, bs, 0, s>>>(G, state, uprev, v, y, alpha, b, beta, G.N, nullptr, r0, r1);
  }
  else if (mode == MODE_RES)
    apply_kernel<MODE_RES><<<(unsigned)nb, bs, 0, s>>>(G, state, uprev, state, y, alpha, b, beta, G.N, nullptr, r0,
                                                       r1);
  else
    throw std::runtime_error("EINVAL: launch_apply_range mode");
}

void launch_stencil(const DevGeom &G, int32_t *tab, cudaStream_t s) {
  int64_t nb = (G.N + 255) / 256;
  if (nb) stencil_kernel<<<(unsigned)nb, 256, 0, s>>>(G, tab);
}

void launch_apply(const DevGeom &G, int mode, const double *state, const double *uprev, const double *v,
                  double *y, double alpha, const double *b, double beta, cudaStream_t s, int nvec) {
  int bs = 256;
  int64_t nb = (G.N + bs - 1) / bs;
  if (nb == 0) return;
  dim3 grid((unsigned)nb, (unsigned)nvec);
  if (mode == MODE_JAC) {
    const int mb = jac_min_blocks();
    if (mb == 5) apply_kernel<MODE_JAC, 5><<<grid, bs, 0, s>>>(G, state, uprev, v, y, alpha, b, beta, G.N, nullptr);
    else if (mb == 6) apply_kernel<MODE_JAC, 6><<<grid, bs, 0, s>>>(G, state, uprev, v, y, alpha, b, beta, G.N, nullptr);
    else if (mb == 8) apply_kernel<MODE_JAC, 8><<<grid, bs, 0, s>>>(G, state, uprev, v, y, alpha, b, beta, G.N, nullptr);
    else apply_kernel<MODE_JAC><<<grid, bs, 0, s>>>(G, state, uprev, v, y, alpha, b, beta, G.N, nullptr);
  }
  else if (mode == MODE_JW)
    apply_kernel<MODE_JW><<<grid, bs, 0, s>>>(G, state, uprev, v, y, alpha, b, beta, G.N, nullptr);
  else if (mode == MODE_JACM)
    apply_kernel<MODE_JACM><<<grid, bs, 0, s>>>(G, state, uprev, v, y, alpha, b, beta, G.N, nullptr);
  else if (mode == MODE_RESM)
    apply_kernel<MODE_RESM><<<grid, bs, 0, s>>>(G, state, uprev, state, y, alpha, b, beta, G.N, nullptr);
  else
    apply_kernel<MODE_RES><<<grid, bs, 0, s>>>(G, state, uprev, state, y, alpha, b, beta, G.N, nullptr);
}

}  // namespace pmns
