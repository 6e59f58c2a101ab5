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

template <int MODE>
__global__ void __launch_bounds__(256) apply_kernel(DevGeom G, const double *__restrict__ st,
                                                    const double *__restrict__ up, const double *__restrict__ v,
                                                    double *__restrict__ y, double alpha,
                                                    const double *__restrict__ b, double beta, int64_t vstride) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= G.N) return;
  // gridDim.y > 1: a batch of vectors (probing), vector q at v + q*vstride, y + q*vstride
  v += (int64_t)blockIdx.y * vstride;
  y += (int64_t)blockIdx.y * vstride;
  constexpr bool kRes = MODE == MODE_RES || MODE == MODE_RESM;
  constexpr bool kJac = MODE == MODE_JAC || MODE == MODE_JACM;
  constexpr bool kMasked = MODE == MODE_JW || MODE == MODE_JACM || MODE == MODE_RESM;
  uint32_t pp = __ldg(G.rowpos + r);
  int t = pp >> 30, k = (pp >> 20) & 1023, j = (pp >> 10) & 1023, i = pp & 1023;
  const double inv_h = 1.0 / G.h;
  double out;
  if (t == 3) {
    // mass row: div (Eq. navstokes_mass; A8 sign +div)
    double d = 0.0;
    for (int bb = 0; bb < G.dim; ++bb) {
      int kh = k, jh = j, ih = i;
      shift(bb, 1, kh, jh, ih);
      int32_t f0 = fcode(G, bb, k, j, i), f1 = fcode(G, bb, kh, jh, ih);
      double v0 = f0 >= 0 ? __ldg(v + f0) : 0.0;
      double v1 = f1 >= 0 ? __ldg(v + f1) : 0.0;
      d += v1 - v0;
    }
    out = d * inv_h;
  } else {
    const int a = t;
    const double vf = __ldg(v + r);
    // viscous Laplacian (A6)
    double lap = 0.0;
    for (int bb = 0; bb < G.dim; ++bb) {
      int km = k, jm = j, im = i, kp = k, jp = j, ip = i;
      shift(bb, -1, km, jm, im);
      shift(bb, 1, kp, jp, ip);
      lap += vrule(fcode(G, a, km, jm, im), v, vf) + vrule(fcode(G, a, kp, jp, ip), v, vf) - 2.0 * vf;
    }
    lap *= inv_h * inv_h;
    // pressure gradient (A3): flanks low = pos - e_a, high = pos
    int kl = k, jl = j, il = i;
    shift(a, -1, kl, jl, il);
    int32_t c0 = ccode(G, kl, jl, il), c1 = ccode(G, k, j, i);
    const double *vp = kRes ? st : v;
    double p0, p1;
    if (kRes) {
      p0 = c0 >= 0 ? __ldg(vp + c0) : (c0 == kDMirror ? G.p_in : 0.0);
      p1 = c1 >= 0 ? __ldg(vp + c1) : (c1 == kDMirror ? G.p_out : 0.0);
    } else {
      p0 = c0 >= 0 ? __ldg(vp + c0) : 0.0;
      p1 = c1 >= 0 ? __ldg(vp + c1) : 0.0;
    }
    double grad = (p1 - p0) * inv_h;
    // inertia (A5 / A9 / A10)
    double conv = 0.0;
    bool do_conv = G.rho != 0.0 && (!kMasked || !G.mask[r]);
    if (do_conv) {
      const double sf = __ldg(st + r);
      for (int bb = 0; bb < G.dim; ++bb) {
        double cs, cv;
        if (bb == a) {
          cs = sf;
          cv = vf;
        } else {
          cadv(G, a, bb, k, j, i, st, kJac ? v : nullptr, cs, cv);
        }
        const int s = cs >= 0.0 ? 1 : -1;
        int k1 = k, j1 = j, i1 = i, k2 = k, j2 = j, i2 = i;
        shift(bb, -s, k1, j1, i1);
        shift(bb, -2 * s, k2, j2, i2);
        int32_t m1 = fcode(G, a, k1, j1, i1), m2 = fcode(G, a, k2, j2, i2);
        bool use2 = (m2 >= 0) || (m2 == kDZero);
        // D_b applied to the state (for RES and the reaction term) and to v
        double Ds, Dv;
        {
          double s1 = vrule(m1, st, sf);
          Ds = use2 ? (3.0 * sf - 4.0 * s1 + vrule(m2, st, sf)) * (0.5 * inv_h) : (sf - s1) * inv_h;
          Ds *= (double)s;
        }
        if (kRes) {
          conv += cs * Ds;
        } else {
          double v1 = vrule(m1, v, vf);
          Dv = use2 ? (3.0 * vf - 4.0 * v1 + vrule(m2, v, vf)) * (0.5 * inv_h) : (vf - v1) * inv_h;
          Dv *= (double)s;
          conv += cs * Dv;
          if (kJac) conv += cv * Ds;
        }
      }
      conv *= G.rho;
    }
    double tt = 0.0;
    if (G.dt > 0.0) {
      if (kRes) tt = G.rho * (vf - (up ? __ldg(up + r) : 0.0)) / G.dt;
      else tt = G.rho / G.dt * vf;
    }
    out = tt + conv - G.mu * lap + grad;
    if (kRes) out -= G.rho * G.bf[a];
  }
  double res = alpha * out;
  if (b) res += beta * __ldg(b + r);
  y[r] = res;
}

}  // namespace

void launch_apply(const DevGeom &G, int mode, const double *state, const double *uprev, const double *v,
                  double *y, double alpha, const double *b, double beta, cudaStream_t s, int nvec) {
  int bs = 256;
  int64_t nb = (G.N + bs - 1) / bs;
  if (nb == 0) return;
  dim3 grid((unsigned)nb, (unsigned)nvec);
  if (mode == MODE_JAC)
    apply_kernel<MODE_JAC><<<grid, bs, 0, s>>>(G, state, uprev, v, y, alpha, b, beta, G.N);
  else if (mode == MODE_JW)
    apply_kernel<MODE_JW><<<grid, bs, 0, s>>>(G, state, uprev, v, y, alpha, b, beta, G.N);
  else if (mode == MODE_JACM)
    apply_kernel<MODE_JACM><<<grid, bs, 0, s>>>(G, state, uprev, v, y, alpha, b, beta, G.N);
  else if (mode == MODE_RESM)
    apply_kernel<MODE_RESM><<<grid, bs, 0, s>>>(G, state, uprev, state, y, alpha, b, beta, G.N);
  else
    apply_kernel<MODE_RES><<<grid, bs, 0, s>>>(G, state, uprev, state, y, alpha, b, beta, G.N);
}

}  // namespace pmns
