// Linear-algebra kernels of the gPLMM apply and FGMRES (SURVEY §8(a) rows
// a3, a4, a5, a7, a9, a10) and the build-time block extraction (B1, B2).
#include <cuda_runtime.h>

#include <cstdint>


namespace pmns {

// ---------------------------------------------------------------------------
// Batched dense GEMV  y_i = A_i x_i  (row-major, ld even, 16-byte aligned).
// a7/a9 local solves (Eq. Mp_Md) with the stored local inverses,
// and the coarse solve (a4, Eq. coarse_prob).  HBM-bound: one CTA per task
// (a tile of rows of one block), x staged in shared memory, one warp per row,
// 128-bit loads with 4 independent accumulators per lane.
// Epilogue: y[r] = acc                          (mode 0)
//           y[r] = acc + e0[r] + e1[r]          (mode 1: z = z_G + z_d + M_p^{-1} t)
//           y[r] = e0[r] - acc                  (mode 2: x_I = y_I - W x_S)
// x is X[xoff + q], or X[xidx[xoff + q]] when xidx is given.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512) gemv_tasks_kernel(const GemvTask *__restrict__ tasks, int ntasks,
                                                          const double *__restrict__ A,
                                                          const double *__restrict__ X, double *__restrict__ Y,
                                                          const double *__restrict__ E0,
                                                          const double *__restrict__ E1, int mode,
                                                          int smem_cap, const int64_t *__restrict__ xidx) {
  extern __shared__ double2 xs2[];
  double *xs = reinterpret_cast<double *>(xs2);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (blockIdx.x < ntasks) {   // the stored operator is constant: pull the first 32 KB of this CTA's tile into L2
    const GemvTask T = tasks[blockIdx.x];    // while the predecessor drains (PDL launch)
    const int64_t bytes = (int64_t)(T.r1 - T.r0) * T.ld * 8;
    const int64_t off = (int64_t)threadIdx.x * 128;
    if (off < bytes && off < 32768)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(A + T.aoff + (int64_t)T.r0 * T.ld + off / 8));
  }
  pdl_wait();
  pdl_trigger();
  for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
    GemvTask T = tasks[t];
    const int n = T.n;
    const int ld = T.ld;
    const bool staged = n + 1 <= smem_cap;
    __syncthreads();
    if (staged) {
      if (xidx) {   // x gathered through an index list (nested-dissection fronts)
        const int64_t *ix = xidx + T.xoff;
        for (int q = threadIdx.x; q < n; q += blockDim.x) xs[q] = __ldg(X + __ldg(ix + q));
      } else {
        const double *xsrc = X + T.xoff;
        for (int q = threadIdx.x; q < n; q += blockDim.x) xs[q] = __ldg(xsrc + q);
      }
      if (threadIdx.x == 0 && (n & 1)) xs[n] = 0.0;
    }
    __syncthreads();
    const double *xg = X + T.xoff;
    const int npair = (n + 1) >> 1;
    for (int r = T.r0 + warp; r < T.r1; r += nw) {
      const double2 *row = reinterpret_cast<const double2 *>(A + T.aoff + (int64_t)r * ld);
      double acc8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc8[u] = 0.0;
      int q = lane;
      if (staged) {
        // 8 independent 16-byte streaming loads per lane in flight (4 KB per
        // warp), predicated so the row tail keeps the same memory parallelism
        for (; q < npair; q += 256) {
          double2 m[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int qq = q + 32 * u;
            m[u] = qq < npair ? __ldcs(row + qq) : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int qq = q + 32 * u;
            if (qq < npair) {
              double2 xv = xs2[qq];
              acc8[u] = fma(m[u].x, xv.x, fma(m[u].y, xv.y, acc8[u]));
            }
          }
        }
      } else {
        for (; q < npair; q += 32) {
          double2 m0 = __ldcs(row + q);
          double x0, x1;
          if (xidx) {
            x0 = __ldg(X + __ldg(xidx + T.xoff + 2 * q));
            x1 = (2 * q + 1 < n) ? __ldg(X + __ldg(xidx + T.xoff + 2 * q + 1)) : 0.0;
          } else {
            x0 = __ldg(xg + 2 * q);
            x1 = (2 * q + 1 < n) ? __ldg(xg + 2 * q + 1) : 0.0;
          }
          acc8[0] = fma(m0.x, x0, fma(m0.y, x1, acc8[0]));
        }
      }
      double a0 = acc8[0] + acc8[4], a1 = acc8[1] + acc8[5], a2 = acc8[2] + acc8[6], a3 = acc8[3] + acc8[7];
      double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) {
        int64_t yi = T.yoff + r;
        if (mode == 1) acc += E0[yi] + E1[yi];
        else if (mode == 2) acc = E0[yi] - acc;
        Y[yi] = acc;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Batched GEMV for many-task sets of short rows (nested-dissection fronts,
// nd.inc): each warp keeps RPW rows in flight (2 x 16-byte streaming loads
// per row per lane per step), 256-thread CTAs, several CTAs per SM.  Same
// task / epilogue contract as gemv_tasks_kernel (modes 0 and 2).
// ---------------------------------------------------------------------------
template <int RPW>
__global__ void __launch_bounds__(256) gemv_rows_kernel(const GemvTask *__restrict__ tasks, int ntasks,
                                                         const double *__restrict__ A,
                                                         const double *__restrict__ X, double *__restrict__ Y,
                                                         const double *__restrict__ E0, int mode, int smem_cap,
                                                         const int64_t *__restrict__ xidx, GemvFuse fz) {
  extern __shared__ double2 xs2[];
  double *xs = reinterpret_cast<double *>(xs2);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (blockIdx.x < ntasks) {   // the stored operator is constant: pull the first 32 KB of this CTA's tile into L2
    const GemvTask T = tasks[blockIdx.x];    // while the predecessor drains (PDL launch)
    const int64_t bytes = (int64_t)(T.r1 - T.r0) * T.ld * 8;
    const int64_t off = (int64_t)threadIdx.x * 128;
    if (off < bytes && off < 32768)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(A + T.aoff + (int64_t)T.r0 * T.ld + off / 8));
  }
  pdl_wait();
  pdl_trigger();
  for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
    const GemvTask T = tasks[t];
    const int n = T.n, ld = T.ld;
    const bool staged = n + 1 <= smem_cap;
    __syncthreads();
    if (staged) {
      if (xidx) {
        const int64_t *ix = xidx + T.xoff;
        for (int q = threadIdx.x; q < n; q += blockDim.x) {
          double xv = __ldg(X + __ldg(ix + q));
          if (fz.uptr) {   // pending boundary updates of the descendants (fixed order)
            const int64_t p = T.xoff + q;
            for (int64_t e = __ldg(fz.uptr + p); e < __ldg(fz.uptr + p + 1); ++e) xv -= fz.U[__ldg(fz.usrc + e)];
          }
          xs[q] = xv;
        }
      } else {
        for (int q = threadIdx.x; q < n; q += blockDim.x) xs[q] = __ldg(X + T.xoff + q);
      }
      if (threadIdx.x == 0 && (n & 1)) xs[n] = 0.0;
    }
    __syncthreads();
    const int npair = (n + 1) >> 1;
    for (int r0 = T.r0 + warp * RPW; r0 < T.r1; r0 += nw * RPW) {
      double acc[RPW];
      const double2 *row[RPW];
      bool rv[RPW];
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr) {
        acc[rr] = 0.0;
        rv[rr] = r0 + rr < T.r1;
        row[rr] = reinterpret_cast<const double2 *>(A + T.aoff + (int64_t)(rv[rr] ? r0 + rr : r0) * ld);
      }
      for (int q = lane; q < npair; q += 64) {
        double2 m[RPW][2];
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr)
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int qq = q + 32 * u;
            m[rr][u] = (rv[rr] && qq < npair) ? __ldcs(row[rr] + qq) : make_double2(0.0, 0.0);
          }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int qq = q + 32 * u;
          if (qq >= npair) continue;
          double x0, x1;
          if (staged) {
            double2 xv = xs2[qq];
            x0 = xv.x;
            x1 = xv.y;
          } else if (xidx) {
            x0 = __ldg(X + __ldg(xidx + T.xoff + 2 * qq));
            x1 = (2 * qq + 1 < n) ? __ldg(X + __ldg(xidx + T.xoff + 2 * qq + 1)) : 0.0;
          } else {
            x0 = __ldg(X + T.xoff + 2 * qq);
            x1 = (2 * qq + 1 < n) ? __ldg(X + T.xoff + 2 * qq + 1) : 0.0;
          }
#pragma unroll
          for (int rr = 0; rr < RPW; ++rr) acc[rr] = fma(m[rr][u].x, x0, fma(m[rr][u].y, x1, acc[rr]));
        }
      }
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[rr] += __shfl_xor_sync(0xffffffffu, acc[rr], o);
      if (lane < RPW) {
        double a = acc[0];
#pragma unroll
        for (int rr = 1; rr < RPW; ++rr)
          if (lane == rr) a = acc[rr];
        if (r0 + lane < T.r1) {
          const int64_t yi = T.yoff + r0 + lane;
          const double val = mode == 2 ? E0[yi] - a : a;
          if (fz.yidx) Y[fz.yidx[yi]] = val;
          else Y[yi] = val;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Multi-vector variant (KV right-hand sides, vector c at X + c*ldx and
// Y + c*ldy): each streamed matrix row serves all KV vectors (the multi-RHS
// solves of the folded Abar fronts, nd.inc).  Epilogue modes 0 and 2; x gathered
// through xidx; y scattered through fz.yidx when given.  Staging: KV*n doubles.
// ---------------------------------------------------------------------------
template <int RPW, int KV>
__global__ void __launch_bounds__(256) gemv_rows_multi_kernel(const GemvTask *__restrict__ tasks, int ntasks,
                                                               const double *__restrict__ A,
                                                               const double *__restrict__ X, int64_t ldx,
                                                               double *__restrict__ Y, int64_t ldy,
                                                               const double *__restrict__ E0, int64_t lde, int mode,
                                                               const int64_t *__restrict__ xidx,
                                                               const int64_t *__restrict__ yidx) {
  extern __shared__ double2 xs2m[];
  double *xs = reinterpret_cast<double *>(xs2m);   // xs[c * np2 + q]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
    const GemvTask T = tasks[t];
    const int n = T.n, ld = T.ld;
    const int np2 = (n + 1) & ~1;
    __syncthreads();
    for (int e = threadIdx.x; e < KV * np2; e += blockDim.x) {
      const int cc = e / np2, q = e % np2;
      double v = 0.0;
      if (q < n) {
        const int64_t ix = xidx ? __ldg(xidx + T.xoff + q) : T.xoff + q;
        v = __ldg(X + cc * ldx + ix);
      }
      xs[cc * np2 + q] = v;
    }
    __syncthreads();
    const int npair = np2 >> 1;
    for (int r0 = T.r0 + warp * RPW; r0 < T.r1; r0 += nw * RPW) {
      double acc[RPW][KV];
      const double2 *row[RPW];
      bool rv[RPW];
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr) {
        rv[rr] = r0 + rr < T.r1;
        row[rr] = reinterpret_cast<const double2 *>(A + T.aoff + (int64_t)(rv[rr] ? r0 + rr : r0) * ld);
#pragma unroll
        for (int cc = 0; cc < KV; ++cc) acc[rr][cc] = 0.0;
      }
      for (int q = lane; q < npair; q += 32) {
        double2 m[RPW];
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr) m[rr] = rv[rr] ? __ldcs(row[rr] + q) : make_double2(0.0, 0.0);
#pragma unroll
        for (int cc = 0; cc < KV; ++cc) {
          const double2 xv = reinterpret_cast<const double2 *>(xs + cc * np2)[q];
#pragma unroll
          for (int rr = 0; rr < RPW; ++rr) acc[rr][cc] = fma(m[rr].x, xv.x, fma(m[rr].y, xv.y, acc[rr][cc]));
        }
      }
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr)
#pragma unroll
        for (int cc = 0; cc < KV; ++cc)
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) acc[rr][cc] += __shfl_xor_sync(0xffffffffu, acc[rr][cc], o);
      if (lane == 0) {
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr) {
          if (!rv[rr]) continue;
          const int64_t yi = T.yoff + r0 + rr;
          const int64_t yo = yidx ? yidx[yi] : yi;
#pragma unroll
          for (int cc = 0; cc < KV; ++cc) {
            const double val = mode == 2 ? E0[cc * lde + yi] - acc[rr][cc] : acc[rr][cc];
            Y[cc * ldy + yo] = val;
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Restriction R^ (a3; Eq. restrict_FVM, Eq. iMG_PR; reading A15):
// bc[q] = sum of v over the contiguous slot range [lo_q, hi_q).
// ---------------------------------------------------------------------------
__global__ void segsum_kernel(const int64_t *__restrict__ lo, const int64_t *__restrict__ hi,
                              const double *__restrict__ v, double *__restrict__ out, int64_t ostride,
                              int64_t vstride = 0) {
  __shared__ double red[32];
  const int q = blockIdx.x;
  // gridDim.y > 1: vector k = blockIdx.y at v + k*vstride, result at out[q*ostride + k]
  v += (int64_t)blockIdx.y * vstride;
  out += blockIdx.y;
  double s = 0.0;
  for (int64_t r = lo[q] + threadIdx.x; r < hi[q]; r += blockDim.x) s += v[r];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) out[(int64_t)q * ostride] = s;
  }
}

// ---------------------------------------------------------------------------
// Prolongation P^ (a5; Eq. prolong_1, Eq. iMG_PR_a):
// primary rows: z[r] = sum_c B_i[c][lr] * xc[cidx_i[c]]  (B_i column-major)
// interface-cell rows: z[r] = xc[iface(r)]
// ---------------------------------------------------------------------------
__global__ void prolong_kernel(int64_t n_prim_rows, int64_t n_pc_rows, const int32_t *__restrict__ row_blk,
                               const int64_t *__restrict__ blk_row0, const int64_t *__restrict__ blk_boff,
                               const int32_t *__restrict__ blk_ncol, const int64_t *__restrict__ blk_coff,
                               const int32_t *__restrict__ cidx, const double *__restrict__ B,
                               const int32_t *__restrict__ cell_iface, const double *__restrict__ xc,
                               double *__restrict__ z, int64_t xstride = 0, int64_t zstride = 0) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_pc_rows) return;
  xc += (int64_t)blockIdx.y * xstride;   // batched columns (coarse-matrix assembly)
  z += (int64_t)blockIdx.y * zstride;
  if (r < n_prim_rows) {
    int bi = row_blk[r];
    int64_t r0 = blk_row0[bi], n = blk_row0[bi + 1] - r0;
    int64_t lr = r - r0;
    const double *Bi = B + blk_boff[bi];
    const int32_t *ci = cidx + blk_coff[bi];
    int nc = blk_ncol[bi];
    double s = 0.0;
    for (int c = 0; c < nc; ++c) s = fma(Bi[(int64_t)c * n + lr], __ldg(xc + ci[c]), s);
    z[r] = s;
  } else {
    z[r] = __ldg(xc + cell_iface[r - n_prim_rows]);
  }
}

// f-rows (Eq. xf, homogeneous; reading A14): t = A^f_{pc} z, then
// z_f = -(A^f_f)^{-1} t cluster by cluster (dense inverses).
__global__ void frows_t_kernel(int64_t nfr, int64_t f0, const int64_t *__restrict__ rp,
                               const int32_t *__restrict__ ci, const double *__restrict__ cv,
                               const double *__restrict__ z, double *__restrict__ t, int64_t zstride = 0) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nfr) return;
  z += (int64_t)blockIdx.y * zstride;
  t += (int64_t)blockIdx.y * nfr;
  double s = 0.0;
  for (int64_t e = rp[q]; e < rp[q + 1]; ++e) s = fma(cv[e], z[ci[e]], s);
  t[q] = s;
}

__global__ void frows_solve_kernel(int64_t nfr, int64_t f0, const int32_t *__restrict__ clus_of,
                                   const int32_t *__restrict__ loc_of, const int64_t *__restrict__ clus_ptr,
                                   const int32_t *__restrict__ members, const int64_t *__restrict__ clus_moff,
                                   const double *__restrict__ Minv, const double *__restrict__ t,
                                   double *__restrict__ z, int64_t zstride = 0) {
  // one warp per f-row: lanes stride over the cluster's members (coalesced row of Minv)
  const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= nfr) return;
  t += (int64_t)blockIdx.y * nfr;
  z += (int64_t)blockIdx.y * zstride;
  int c = clus_of[q];
  int64_t p0 = clus_ptr[c], n = clus_ptr[c + 1] - p0;
  const double *M = Minv + clus_moff[c] + (int64_t)loc_of[q] * n;
  double s = 0.0;
  for (int64_t m = lane; m < n; m += 32) s = fma(M[m], t[members[p0 + m]], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) z[f0 + q] = -s;
}

// gather / deterministic scatter for the overlapping dual grids (a7)
__global__ void gather_kernel(int64_t n, const int64_t *__restrict__ idx, const double *__restrict__ src,
                              double *__restrict__ dst) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) dst[q] = __ldg(src + idx[q]);
}

__global__ void scatter_sum_kernel(int64_t N, const int64_t *__restrict__ ptr, const int64_t *__restrict__ pos,
                                   const double *__restrict__ buf, double *__restrict__ z) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  double s = 0.0;
  for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) s += buf[pos[e]];   // ascending dual order
  z[r] = s;
}

// ---------------------------------------------------------------------------
// Vector kernels for FGMRES (a10) and Newton (a11)
// ---------------------------------------------------------------------------
// partial dot products of w with the K vectors V[0..K) (row stride ldv):
// part[blk*K + k].  One launch for all K: the vectors are taken KB at a time
// so the accumulators stay in registers (w is re-read from L2 per chunk).
template <int KB>
__global__ void __launch_bounds__(256) multidot_kernel(int64_t N, int K, const double *__restrict__ V, int64_t ldv,
                                                       const double *__restrict__ w, double *__restrict__ part) {
  __shared__ double red[8][KB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k0 = 0; k0 < K; k0 += KB) {
    const int KC = min(KB, K - k0);
    double acc[KB];
#pragma unroll
    for (int k = 0; k < KB; ++k) acc[k] = 0.0;
    const double *Vk = V + (int64_t)k0 * ldv;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < N; r += (int64_t)gridDim.x * blockDim.x) {
      double wr = __ldg(w + r);
#pragma unroll
      for (int k = 0; k < KB; ++k)
        if (k < KC) acc[k] = fma(__ldg(Vk + k * ldv + r), wr, acc[k]);
    }
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      double sacc = acc[k];
      for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
      if (lane == 0) red[warp][k] = sacc;
    }
    __syncthreads();
    if (threadIdx.x < KC) {
      double sacc = 0.0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) sacc += red[q][threadIdx.x];
      part[(int64_t)blockIdx.x * K + k0 + threadIdx.x] = sacc;
    }
    __syncthreads();
  }
}

// out[k] = sum_b part[b*K + k]  (+ optional accumulate into out2[k])
__global__ void reduce_parts_kernel(int nb, int K, const double *__restrict__ part, double *__restrict__ out,
                                    double *__restrict__ accum) {
  int k = blockIdx.x;
  __shared__ double red[32];
  double s = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) s += part[(int64_t)b * K + k];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (int)(blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) {
      out[k] = s;
      if (accum) accum[k] += s;
    }
  }
}

// w[r] += sgn * sum_k c[k] V[k][r]
__global__ void __launch_bounds__(256) update_kernel(int64_t N, int K, const double *__restrict__ V, int64_t ldv,
                                                     const double *__restrict__ c, double sgn,
                                                     double *__restrict__ w) {
  __shared__ double cs[kMaxK];
  for (int k = threadIdx.x; k < K; k += blockDim.x) cs[k] = c[k];
  __syncthreads();
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < N; r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
#pragma unroll 8
    for (int k = 0; k < K; ++k) s = fma(cs[k], __ldg(V + k * ldv + r), s);
    w[r] = fma(sgn, s, w[r]);
  }
}

// v_out = v_in / sqrt(nrm2[0]) ; also stores h = sqrt(nrm2) to hout
__global__ void normalize_kernel(int64_t N, const double *__restrict__ nrm2, const double *__restrict__ vin,
                                 double *__restrict__ vout, double *__restrict__ hout) {
  double nr = sqrt(nrm2[0]);
  if (blockIdx.x == 0 && threadIdx.x == 0 && hout) hout[0] = nr;
  double inv = nr > 0.0 ? 1.0 / nr : 0.0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < N; r += (int64_t)gridDim.x * blockDim.x)
    vout[r] = vin[r] * inv;
}

// out = a + b + c (z = z_G + z_d + M_p^{-1} t with the M_p part combined over ranks)
__global__ void add3_kernel(int64_t n, const double *__restrict__ a, const double *__restrict__ b,
                            const double *__restrict__ c, double *__restrict__ out) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) out[q] = a[q] + b[q] + c[q];
}

__global__ void axpby_kernel(int64_t N, double a, const double *__restrict__ x, double b,
                             const double *__restrict__ y, double *__restrict__ out) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < N) out[r] = a * x[r] + (y ? b * y[r] : 0.0);
}

__global__ void permute_kernel(int64_t N, const int64_t *__restrict__ map, const double *__restrict__ src,
                               double *__restrict__ dst, int dir) {
  int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= N) return;
  if (dir == 0) dst[w] = src[map[w]];   // canonical -> device: dst[slot] = src[perm[slot]]
  else dst[map[w]] = src[w];            // device -> canonical
}

// ---------------------------------------------------------------------------
// Build (B1/B2): probing extraction of the operator into a per-row ELL list.
// Probe vector = indicator of all unknowns of color (t, rx, ry, rz); the
// coloring period p >= 5 per axis (dividing n on periodic axes) guarantees at
// most one column of that color in each row (stencil reach 2).
// ---------------------------------------------------------------------------
// color index within a batch = blockIdx.y; colors enumerate (t, rz, ry, rx) from c0
__device__ __forceinline__ void color_decode(int col, int ntypes_first, int px, int py, int pz, int &t, int &rx,
                                             int &ry, int &rz) {
  rx = col % px;
  col /= px;
  ry = col % py;
  col /= py;
  rz = col % pz;
  col /= pz;
  t = col;
}

__global__ void probe_fill_kernel(int64_t N, const uint32_t *__restrict__ rowpos, int c0, int ncol, int dim, int px,
                                  int py, int pz, double *__restrict__ v) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  int cc = c0 + (int)blockIdx.y;
  int t, rx, ry, rz;
  color_decode(cc, 0, px, py, pz, t, rx, ry, rz);
  if (t >= dim) t = 3;   // type index dim encodes cells
  uint32_t pp = rowpos[r];
  int tt = pp >> 30, k = (pp >> 20) & 1023, j = (pp >> 10) & 1023, i = pp & 1023;
  v[(int64_t)blockIdx.y * N + r] = (tt == t && i % px == rx && j % py == ry && k % pz == rz) ? 1.0 : 0.0;
}

__device__ __forceinline__ int wrap_d(int x, int n) {
  x %= n;
  return x < 0 ? x + n : x;
}

// one thread per row, looping over the batch's colors in order (so each row's
// ELL list is appended by exactly one thread: deterministic, no atomics)
__global__ void probe_extract_kernel(ProbeGeom P, int c0, int ncol, int dim, const double *__restrict__ ybatch,
                                     int32_t *__restrict__ ell_col, double *__restrict__ ell_val,
                                     int32_t *__restrict__ ell_cnt, int width, int *overflow) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= P.N) return;
  for (int q = 0; q < ncol; ++q) {
  int t, rx, ry, rz;
  color_decode(c0 + q, 0, P.px, P.py, P.pz, t, rx, ry, rz);
  if (t >= dim) t = 3;
  double val = ybatch[(int64_t)q * P.N + r];
  if (val == 0.0) continue;
  uint32_t pp = P.rowpos[r];
  int k = (pp >> 20) & 1023, j = (pp >> 10) & 1023, i = pp & 1023;
  // unique offset d in [-R, R] with (x + d) % p == residue (R = stencil reach)
  int di = wrap_d(rx - i, P.px);
  if (di > P.reach) di -= P.px;
  int dj = wrap_d(ry - j, P.py);
  if (dj > P.reach) dj -= P.py;
  int dk = wrap_d(rz - k, P.pz);
  if (dk > P.reach) dk -= P.pz;
  int ii = i + di, jj = j + dj, kk = k + dk;
  int32_t col = -1;
  // map lookup for type t at (kk, jj, ii)
  if (t == 3) {
    if (ii >= 0 && ii < P.nx) {
      if (P.pyflag) jj = wrap_d(jj, P.ny);
      if (P.pzflag) kk = wrap_d(kk, P.nz);
      if (jj >= 0 && jj < P.ny && kk >= 0 && kk < P.nz) col = P.cmap[((int64_t)kk * P.ny + jj) * P.nx + ii];
    }
  } else {
    if (ii >= 0 && ii < P.fx[t]) {
      if (P.pyflag) jj = wrap_d(jj, P.ny);
      if (P.pzflag) kk = wrap_d(kk, P.nz);
      if (jj >= 0 && jj < P.fy[t] && kk >= 0 && kk < P.fz[t])
        col = P.fmap[t][((int64_t)kk * P.fy[t] + jj) * P.fx[t] + ii];
    }
  }
  if (col < 0) {
    atomicOr(overflow, 2);   // a nonzero with no column: coloring violated
    if (atomicCAS(overflow + 1, 0, 1) == 0) {   // first failure: row, colour, value (diagnostics)
      overflow[2] = (int)r;
      overflow[3] = c0 + q;
      reinterpret_cast<double *>(overflow + 4)[0] = val;
    }
    continue;
  }
  int c = ell_cnt[r];
  if (c >= width) {
    atomicOr(overflow, 1);
    continue;
  }
  ell_col[r * (int64_t)width + c] = col;
  ell_val[r * (int64_t)width + c] = val;
  ell_cnt[r] = c + 1;
  }
}

// Dense block extraction from the ELL: rows [r0, r1) of block b map to local
// rows; columns found by binary search in the block's sorted slot list.
// Mode 0 (M_p, M_d): D[lr*ld + lc] = val for cols in the set.
// Mode 1 (folded Abar, Eq. reduce_1/reduce_2): cols in set -> D; interface
//   cell cols -> rhs[(c)*n + lr] for the interface's local index (Abar^p_c =
//   A^p_c Q°); all other cols folded onto the diagonal (csum).
__global__ void dense_extract_kernel(int64_t nrows_total, const int64_t *__restrict__ rows,
                                     const int32_t *__restrict__ row_blk, const int64_t *__restrict__ row_local,
                                     const int64_t *__restrict__ set_off, const int64_t *__restrict__ set_slots,
                                     const int64_t *__restrict__ blk_doff, const int32_t *__restrict__ blk_ld,
                                     const int32_t *__restrict__ ell_col, const double *__restrict__ ell_val,
                                     const int32_t *__restrict__ ell_cnt, int width, double *__restrict__ D,
                                     int mode, const int32_t *__restrict__ slot_iface, int64_t iface_lo,
                                     int64_t iface_hi, const int64_t *__restrict__ blk_roff,
                                     const int32_t *__restrict__ blk_cptr, const int32_t *__restrict__ blk_clist,
                                     double *__restrict__ rhs) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nrows_total) return;
  int64_t r = rows[q];
  int b = row_blk[q];
  int64_t lr = row_local[q];
  const int64_t *S = set_slots + set_off[b];
  int64_t n = set_off[b + 1] - set_off[b];
  int ld = blk_ld[b];
  double *Db = D + blk_doff[b];
  double fold = 0.0;
  int cnt = ell_cnt[r];
  for (int e = 0; e < cnt; ++e) {
    int32_t col = ell_col[r * (int64_t)width + e];
    double val = ell_val[r * (int64_t)width + e];
    // binary search
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (S[mid] < col) lo = mid + 1;
      else hi = mid;
    }
    if (lo < n && S[lo] == col) {
      Db[lr * ld + lo] += val;
    } else if (mode == 1) {
      if (col >= iface_lo && col < iface_hi) {
        int jf = slot_iface[col - iface_lo];
        int cp0 = blk_cptr[b], cp1 = blk_cptr[b + 1];
        for (int cc = cp0; cc < cp1; ++cc)
          if (blk_clist[cc] == jf) {
            rhs[blk_roff[b] + (int64_t)(cc - cp0) * n + lr] += val;
            break;
          }
      } else {
        fold += val;
      }
    }
  }
  if (mode == 1) Db[lr * ld + lr] += fold;
}

// --- substructured local solves (Schur complement on a separator) ---------
// r_S[q] = t[Sslot[q]] - sum_e cv[e] * yI[ci[e]]   (A_SI y_I, flat I positions)
__global__ void schur_rhs_kernel(int64_t nS, const int64_t *__restrict__ Sslot, const double *__restrict__ t,
                                 const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                 const double *__restrict__ cv, const double *__restrict__ yI,
                                 double *__restrict__ rS) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nS) return;
  double s = t[Sslot[q]];
  for (int64_t e = rp[q]; e < rp[q + 1]; ++e) s = fma(-cv[e], yI[ci[e]], s);
  rS[q] = s;
}

// out[slot0 + q] = (src >= 0 ? xI[src] : xS[-src-1]) (+ e0 + e1)
__global__ void slot_scatter_kernel(int64_t nslots, int64_t slot0, const int64_t *__restrict__ src,
                                    const double *__restrict__ xI, const double *__restrict__ xS,
                                    const double *__restrict__ e0, const double *__restrict__ e1,
                                    double *__restrict__ out) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nslots) return;
  int64_t sidx = src[q];
  double v = sidx >= 0 ? xI[sidx] : xS[-sidx - 1];
  int64_t r = slot0 + q;
  if (e0) v += e0[r] + e1[r];
  out[r] = v;
}

// S[rows[a], cols[b]] -= T[a*ldt + b]   (Schur update of one part)
__global__ void schur_update_kernel(int nr, int nc, const double *__restrict__ T, int ldt,
                                    const int32_t *__restrict__ rows, const int32_t *__restrict__ cols,
                                    double *__restrict__ S, int lds, int tcm = 0) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (int64_t)nr * nc) return;
  int a = (int)(q / nc), b = (int)(q % nc);
  double tv = tcm ? T[(int64_t)b * ldt + a] : T[(int64_t)a * ldt + b];
  S[(int64_t)rows[a] * lds + cols[b]] -= tv;
}

// multi-column gather / scatter of rows (column-major, k columns):
// dst[c*ldd + q] = src[c*lds + idx[q]]   (to_idx = 0)
// dst[c*ldd + idx[q]] = src[c*lds + q]   (to_idx = 1)
__global__ void rows_copy_kernel(int64_t n, int k, const int64_t *__restrict__ idx, const double *__restrict__ src,
                                 int64_t lds, double *__restrict__ dst, int64_t ldd, int to_idx) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * k) return;
  int64_t q = t % n, c = t / n;
  if (to_idx) dst[c * ldd + idx[q]] = src[c * lds + q];
  else dst[c * ldd + q] = src[c * lds + idx[q]];
}

// R[q + c*m] -= sum_e cv[e] * Y_P[l + c*n_P]  (A_SI Y, k columns); Y holds the
// block's parts one after another, part P (n_P x k, column-major) starting at
// ypo*k, where (ypo, n_P, l) = (ypo[ci], ystride[ci], yl[ci]) of the column.
__global__ void schur_rhs_multi_kernel(int64_t m, int k, const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
                                       const double *__restrict__ cv, const int64_t *__restrict__ ypo,
                                       const int32_t *__restrict__ ystride, const int32_t *__restrict__ yl,
                                       const double *__restrict__ Y, double *__restrict__ R) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m * k) return;
  int64_t q = t % m, c = t / m;
  double acc = 0.0;
  for (int64_t e = rp[q]; e < rp[q + 1]; ++e) {
    int32_t col = ci[e];
    acc = fma(cv[e], Y[ypo[col] * k + c * ystride[col] + yl[col]], acc);
  }
  R[c * m + q] -= acc;
}

// D[rows[q]*ld + rows[q]] += v[q]   (folded diagonal, Eq. reduce_1/2)
__global__ void diag_add_kernel(int64_t n, const int32_t *__restrict__ rows, const double *__restrict__ v,
                                double *__restrict__ D, int64_t ld) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) D[(int64_t)rows[q] * ld + rows[q]] += v[q];
}

// vector over primary slots <-> column q of the per-primary column-major RHS store
__global__ void rhs_column_kernel(int64_t nrows, int q, const int32_t *__restrict__ row_blk,
                                  const int64_t *__restrict__ blk_row0, const int64_t *__restrict__ blk_boff,
                                  const int32_t *__restrict__ blk_ncol, double *__restrict__ B,
                                  double *__restrict__ vec, int to_vec) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  int bi = row_blk[r];
  int64_t n = blk_row0[bi + 1] - blk_row0[bi], lr = r - blk_row0[bi];
  bool has = q < blk_ncol[bi];
  double *p = B + blk_boff[bi] + (int64_t)q * n + lr;
  if (to_vec) vec[r] = has ? *p : 0.0;
  else if (has) *p = vec[r];
}

// Dense block from the ELL: D[q*ld + pos(col in set)] += val for each row rows[q];
// optional diagonal addition dadd[q] (square blocks, Eq. reduce_1/2 fold).
__global__ void extract_block_kernel(int64_t nrows, const int64_t *__restrict__ rows, const int64_t *__restrict__ set,
                                     int64_t nset, const int32_t *__restrict__ ell_col,
                                     const double *__restrict__ ell_val, const int32_t *__restrict__ ell_cnt, int width,
                                     double *__restrict__ D, int64_t ld, const double *__restrict__ dadd,
                                     int trans = 0) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nrows) return;
  int64_t r = rows[q];
  int cnt = ell_cnt[r];
  for (int e = 0; e < cnt; ++e) {
    int32_t col = ell_col[r * (int64_t)width + e];
    int64_t lo = 0, hi = nset;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (set[mid] < col) lo = mid + 1;
      else hi = mid;
    }
    if (lo < nset && set[lo] == col) {
      if (trans) D[lo * ld + q] += ell_val[r * (int64_t)width + e];   // column-major (nrows x nset, ld)
      else D[q * ld + lo] += ell_val[r * (int64_t)width + e];
    }
  }
  if (dadd) D[q * ld + q] += dadd[q];
}

__global__ void set_identity_kernel(int64_t n, int64_t ld, double *__restrict__ M) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n * ld) return;
  int64_t c = q / ld, r = q % ld;
  M[q] = (r == c) ? 1.0 : 0.0;
}

// c_i RHS: rhs column = b_B restricted to the primary's rows
__global__ void copy_kernel(int64_t n, const double *__restrict__ src, double *__restrict__ dst) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) dst[q] = src[q];
}

// columns k0 .. k0+gridDim.y-1 of the identity (n rows each, column-major)
__global__ void unit_cols_kernel(int64_t n, int64_t k0, double *__restrict__ x) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) x[(int64_t)blockIdx.y * n + q] = (q == k0 + blockIdx.y) ? 1.0 : 0.0;
}

// probe vector of colour k0 + blockIdx.y: 1 on the coarse columns of that colour
__global__ void colour_cols_kernel(int64_t n, int64_t k0, const int32_t *__restrict__ colour, double *__restrict__ x) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) x[(int64_t)blockIdx.y * n + q] = (colour[q] == k0 + blockIdx.y) ? 1.0 : 0.0;
}

// A°[k, owner] = restricted probe value of row k (row-major, leading dim ldc)
__global__ void colour_scatter_kernel(int64_t n, int64_t k0, int64_t rstride, const int32_t *__restrict__ owner,
                                      const double *__restrict__ R, double *__restrict__ Ac, int64_t ldc) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int32_t j = owner[(k0 + blockIdx.y) * n + k];
  if (j >= 0) Ac[k * ldc + j] = R[k * rstride + blockIdx.y];
}

__global__ void unit_kernel(int64_t n, int64_t k, double *__restrict__ x) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) x[q] = (q == k) ? 1.0 : 0.0;
}

__global__ void negate_kernel(int64_t n, double *__restrict__ x) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) x[q] = -x[q];
}

}  // namespace pmns
