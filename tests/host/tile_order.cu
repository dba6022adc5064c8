// Host-only check of tile_of_block (lb_kernels.cuh): for every lattice shape and
// residency given on the command line, the block -> (tile, chunk) map is a
// bijection, and chunk c of a tile comes `resid` (or the last group's size)
// blocks after chunk c-1.  Prints "ok" or the first violation.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "lb_kernels.cuh"

int main(int argc, char** argv) {
  for (int a = 1; a + 3 < argc; a += 4) {
    const int ntx = atoi(argv[a]), nty = atoi(argv[a + 1]), nch = atoi(argv[a + 2]), resid = atoi(argv[a + 3]);
    const int n = ntx * nty * nch;
    std::vector<int> seen(n, 0), pos(n, -1);
    for (int L = 0; L < n; ++L) {
      const lbk::TileId t = lbk::tile_of_block(L, ntx, nty, nch, lbk::TileOrder{resid, 1});
      if (t.bx < 0 || t.bx >= ntx || t.by < 0 || t.by >= nty || t.bz < 0 || t.bz >= nch) {
        printf("out of range: L=%d -> (%d,%d,%d) for %d %d %d %d\n", L, t.bx, t.by, t.bz, ntx, nty, nch, resid);
        return 1;
      }
      const int id = (t.bz * nty + t.by) * ntx + t.bx;
      if (seen[id]++) {
        printf("duplicate: L=%d for %d %d %d %d\n", L, ntx, nty, nch, resid);
        return 1;
      }
      pos[id] = L;
    }
    for (int c = 1; c < nch; ++c)
      for (int t = 0; t < ntx * nty; ++t) {
        const int d = pos[c * ntx * nty + t] - pos[(c - 1) * ntx * nty + t];
        const int grp = t / resid, rg = ntx * nty - grp * resid < resid ? ntx * nty - grp * resid : resid;
        if (d != rg) {
          printf("chunk distance %d != %d for tile %d chunk %d\n", d, rg, t, c);
          return 1;
        }
      }
  }
  printf("ok\n");
  return 0;
}
