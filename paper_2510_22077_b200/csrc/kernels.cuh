// Device kernels of the gPLMM Newton-FGMRES hot path (sm_100a, fp64).
// Each kernel cites the step of SURVEY §8(a) it implements and the paper
// passage that defines the operation.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pmns {

// Programmatic dependent launch (PTX griddepcontrol, sm_90+): a kernel launched
// with cudaLaunchAttributeProgrammaticStreamSerialization may become resident
// while its predecessor in the stream drains; pdl_wait() blocks until the
// predecessor grid has completed and its writes are visible, so everything
// before it may touch only data no earlier kernel writes.  Both are no-ops
// for a normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

constexpr int32_t kDZero = -1, kDGhost = -2, kDMirror = -3;
constexpr int kTab = 22;

// Geometry as seen by the kernels.  Face/cell maps hold DEVICE slots.
struct DevGeom {
  int dim, nx, ny, nz, py, pz;
  int fx[3], fy[3], fz[3];
  const int32_t *fmap[3];
  const int32_t *cmap;
  const uint32_t *rowpos;   // per slot: type (2 bits) | k (10) | j (10) | i (10)
  const uint8_t *mask;      // per slot: 1 if face masked (D9)
  const int32_t *tab;       // per-row stencil codes, kTab x N (stencil_kernel)
  int64_t N;
  // Cell records of the Krylov-phase J apply (jrec_kernel; SURVEY 8(a) layout):
  // one record per void cell, in the device order of its pressure slot.
  //   rec_p[c]           pressure slot
  //   rec_f[a*n_rec+c]   slot of the cell's low a-face if a DOF, else -1
  //   rec_n[d*n_rec+c]   neighbour record, d = 2b + (0: -e_b, 1: +e_b); -1 solid /
  //                      lateral wall, -3 beyond the inlet (x < 0), -4-q at i = nx-1
  //                      for +x: q indexes xm_slot (the x-max boundary face)
  //   rec_c[a*n_rec+c]   class word of the low a-face row: 2 bits per stencil
  //                      position (b, o in -2,-1,+1,+2): 0 DOF (reached through
  //                      rec_n / rec_f), 1 ZERO, 2 GHOST, 3 MIRROR; bit 31: the
  //                      record chase cannot reproduce this row -> per-row table
  //   xm_slot[q]         x-max boundary face of record q's cell (its row is evaluated
  //                      from the per-row table)
  //   rec_rows[n_rec_rows]  rows evaluated from the per-row table instead (flagged
  //                      rows and the x-max faces)
  const int32_t *rec_p, *rec_f, *rec_n, *xm_slot, *rec_rows;
  const uint32_t *rec_c;
  int64_t n_rec, n_rec_rows;
  double h, rho, mu, dt, p_in, p_out, bf[3];
};

__host__ __device__ inline uint32_t pack_pos(int t, int k, int j, int i) {
  return ((uint32_t)t << 30) | ((uint32_t)k << 20) | ((uint32_t)j << 10) | (uint32_t)i;
}

// JAC: J(x) v; JW: J~_w v; RES: r(x); JACM / RESM: J and r with the inertia
// removed on masked faces (J~^k, r~^k of the coarse-scale solver)
enum ApplyMode { MODE_JAC = 0, MODE_JW = 1, MODE_RES = 2, MODE_JACM = 3, MODE_RESM = 4, MODE_DUAL = 5 };

// J v and J~_w v in one pass (probing)
void launch_apply_dual(const DevGeom &G, const double *state, const double *v, double *y, double *y2,
                       cudaStream_t s, int nvec);
// Direct ELL assembly of Op (mode JAC / JW / JACM) or of J and J~_w at once
// (MODE_DUAL, second matrix in col2/val2/cnt2); entries ordered as colour
// probing with periods (px, py, pz) orders them.  overflow[0] |= 1 if a row
// has more than `width` entries.
void launch_assemble(const DevGeom &G, int mode, const double *state, int px, int py, int pz, int32_t *col1,
                     double *val1, int32_t *cnt1, int32_t *col2, double *val2, int32_t *cnt2, int width,
                     int *overflow, cudaStream_t s);
// y = alpha * J(state) v + beta * b over the cell records (same arithmetic, in
// the same order, as launch_apply(MODE_JAC); G.rec_* must be set)
void launch_apply_jrec(const DevGeom &G, const double *state, const double *v, double *y, double alpha,
                       const double *b, double beta, cudaStream_t s);
// Same as launch_apply (modes JAC / RES only) over the rows [r0, r1) (the
// owned rows of a multi-GPU rank)
void launch_apply_range(const DevGeom &G, int mode, const double *state, const double *uprev, const double *v,
                        double *y, double alpha, const double *b, double beta, cudaStream_t s, int64_t r0,
                        int64_t r1);
// per-row stencil code table (setup, once)
void launch_stencil(const DevGeom &G, int32_t *tab, cudaStream_t s);
// y = alpha * Op(v) + beta * b   (b may be null); Op chosen by mode.
void launch_apply(const DevGeom &G, int mode, const double *state, const double *uprev, const double *v,
                  double *y, double alpha, const double *b, double beta, cudaStream_t s, int nvec = 1);

}  // namespace pmns
