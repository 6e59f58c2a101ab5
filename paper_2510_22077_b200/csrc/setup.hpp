// Host-side setup (S1/S2 of SURVEY §8(a)): clean-up, squared EDT, immersion
// watershed + merge, interfaces, floating-face repair, duals, mask band,
// canonical numbering and the device (W) order.  Integer-only, deterministic;
// it must agree bit for bit with the oracle (readings D1-D10 in DESIGN.md).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace pmns {

// face-position codes in the face maps (non-negative = canonical DOF index)
constexpr int32_t kZero = -1;   // exactly one solid flank: u = 0
constexpr int32_t kGhost = -2;  // both flanks solid: ghost value -u_f

struct Geometry {
  int dim = 3;
  int nx = 0, ny = 0, nz = 1;
  bool py = false, pz = false;
  std::vector<uint8_t> is_void;   // after clean-up (D1)
  // face maps per orientation: extents (fx,fy,fz); value = canonical id,
  // kZero or kGhost.  Non-periodic lateral axes include the top wall face.
  int fx[3], fy[3], fz[3];
  std::vector<int32_t> fmap[3];
  std::vector<int32_t> cmap;      // canonical id of cell (>= n_f) or -1
  int64_t n_face[3] = {0, 0, 0};
  int64_t n_f = 0, n_c = 0, N = 0;
  int64_t nvox() const { return (int64_t)nx * ny * nz; }
  int64_t flat(int k, int j, int i) const { return ((int64_t)k * ny + j) * nx + i; }
  // classify face (a, k, j, i) with arbitrary coordinates:
  //   returns canonical index >= 0, kZero, kGhost, or kMirror (beyond inlet/outlet)
  int32_t face_code(int a, int k, int j, int i) const;
};
constexpr int32_t kMirror = -3;

struct Decomp {
  int n_p = 0, n_c = 0;
  int64_t raw_basins = 0;
  std::vector<int32_t> label;       // per voxel: primary id or -1
  std::vector<int32_t> iface;       // per voxel: interface id or -1
  std::vector<std::vector<int64_t>> duals;  // per dual: sorted flat voxel indices
  std::vector<uint8_t> mask_cell;   // per voxel: within band of an interface cell
};

struct Layout {
  std::vector<int64_t> perm;        // device slot -> canonical index
  std::vector<int64_t> inv;         // canonical -> device slot
  std::vector<int64_t> seg;         // n_p + 2 n_c + 1 group boundaries (primaries, iface cells, iface faces)
  std::vector<uint8_t> face_mask;   // per canonical face: masked (D9)
  std::vector<std::vector<int64_t>> dual_unknowns;   // per dual: device slots, sorted
  std::vector<int32_t> face_owner_p;                 // per canonical face: primary or -1
};

// Throws std::runtime_error("ENONPERC: ...") etc. on failure.
void build_geometry(const uint8_t *solid, int dim, int nx, int ny, int nz, bool py, bool pz, Geometry &g);
void decompose(const Geometry &g, double h_m, int n_min, int dual_layers, int mask_band, Decomp &d);
void make_layout(const Geometry &g, const Decomp &d, Layout &L);

}  // namespace pmns
