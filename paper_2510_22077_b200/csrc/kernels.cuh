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
// per-row stencil code table (setup, once)
void launch_stencil(const DevGeom &G, int32_t *tab, cudaStream_t s);
// y = alpha * Op(v) + beta * b   (b may be null); Op chosen by mode.
void launch_apply(const DevGeom &G, int mode, const double *state, const double *uprev, const double *v,
                  double *y, double alpha, const double *b, double beta, cudaStream_t s, int nvec = 1);

}  // namespace pmns
