// d3q19.cuh -- D3Q19 velocity set, weights, and the device storage layout.
//
// Velocity set and order: DESIGN.md reading R1 (PAPER.md names no lattice; the
// only D3Q19 mention in the reference is SPEC.md:366).  Rest first, then the 18
// moving velocities in descending lexicographic (cx, cy, cz); weights 1/3,
// 1/18 (faces), 1/36 (edges); c_s^2 = 1/3.
//
// Storage ("plane-major SoA"): one z-plane holds
// all 38 distribution components (19 f + 19 g), each as an ny x nx array with x
// fastest.  The 38 component slots of a plane are ordered
//     [ f:cz=+1 (5) | g:cz=+1 (5) | f:cz=0 (9) | g:cz=0 (9) | f:cz=-1 (5) | g:cz=-1 (5) ]
// so the halo message of each direction (the 10 components that cross a z-slab
// boundary) is ONE contiguous run of 10*nx*ny doubles: no pack kernel (P:185-193,
// halo regions; SoA because it "permits memory coalescing").
#pragma once

#include <cstdint>

namespace lbk {

constexpr int Q = 19;
constexpr int NSLOT = 38;       // f and g components per plane
constexpr int GZ = 1;           // ghost planes of the distribution buffers (each side)
constexpr int GP = 2;           // ghost planes of the phi buffer (each side)
constexpr int HALO_COMPS = 10;  // components crossing a z boundary per direction

__host__ __device__ constexpr int cx(int i) {
  constexpr int t[Q] = {0, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0, 0, -1, -1, -1, -1, -1};
  return t[i];
}
__host__ __device__ constexpr int cy(int i) {
  constexpr int t[Q] = {0, 1, 0, 0, 0, -1, 1, 1, 1, 0, 0, -1, -1, -1, 1, 0, 0, 0, -1};
  return t[i];
}
__host__ __device__ constexpr int cz(int i) {
  constexpr int t[Q] = {0, 0, 1, 0, -1, 0, 1, 0, -1, 1, -1, 1, 0, -1, 0, 1, 0, -1, 0};
  return t[i];
}
__host__ __device__ constexpr double wgt(int i) {
  return (cx(i) * cx(i) + cy(i) * cy(i) + cz(i) * cz(i)) == 0
             ? 1.0 / 3.0
             : ((cx(i) * cx(i) + cy(i) * cy(i) + cz(i) * cz(i)) == 1 ? 1.0 / 18.0 : 1.0 / 36.0);
}
__host__ __device__ constexpr int csq(int i) { return cx(i) * cx(i) + cy(i) * cy(i) + cz(i) * cz(i); }

// slot of canonical component i within a plane, for f (dist = 0) or g (dist = 1)
__host__ __device__ constexpr int slot(int dist, int i) {
  // rank of i among the components with the same cz
  constexpr int rank_in_group[Q] = {
      // cz=0 group {0,1,3,5,7,12,14,16,18}; cz=+1 {2,6,9,11,15}; cz=-1 {4,8,10,13,17}
      0, 1, 0, 2, 0, 3, 1, 4, 1, 2, 2, 3, 5, 3, 6, 4, 7, 4, 8};
  return cz(i) == 1 ? dist * 5 + rank_in_group[i]
                    : (cz(i) == 0 ? 10 + dist * 9 + rank_in_group[i] : 28 + dist * 5 + rank_in_group[i]);
}

constexpr int SLOT_UP_FIRST = 0;     // first slot of the +z halo run (cz = +1)
constexpr int SLOT_DOWN_FIRST = 28;  // first slot of the -z halo run (cz = -1)

}  // namespace lbk
