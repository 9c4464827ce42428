// Dev check (CPU): depth of the tile DAG (forward pass) for coordinate-bisection
// tiles on a Kuhn-stencil grid, vs the row-level depth.  Usage: tile_depth X Y Z rows
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include "../../paper_1711_08708_b200/csrc/bd_host.hpp"
using namespace bd;
int main(int argc, char** argv) {
  const int X = argc > 1 ? atoi(argv[1]) : 129, Y = argc > 2 ? atoi(argv[2]) : 129,
            Z = argc > 3 ? atoi(argv[3]) : 65, R = argc > 4 ? atoi(argv[4]) : 64;
  const int64_t n = (int64_t)X * Y * Z;
  HostCsr L;
  L.n = n;
  L.indptr.push_back(0);
  std::vector<double> coords(3 * n);
  const int off[7][3] = {{-1, -1, -1}, {0, -1, -1}, {-1, 0, -1}, {0, 0, -1}, {-1, -1, 0}, {0, -1, 0}, {-1, 0, 0}};
  for (int k = 0; k < Z; ++k)
    for (int j = 0; j < Y; ++j)
      for (int i = 0; i < X; ++i) {
        const int64_t r = i + (int64_t)X * (j + (int64_t)Y * k);
        coords[3 * r] = i; coords[3 * r + 1] = j; coords[3 * r + 2] = k;
        for (auto& o : off) {
          const int a = i + o[0], b = j + o[1], c = k + o[2];
          if (a < 0 || b < 0 || c < 0) continue;
          L.indices.push_back((int32_t)(a + (int64_t)X * (b + (int64_t)Y * c)));
          L.values.push_back(-0.1);
        }
        L.indices.push_back(r); L.values.push_back(2.0);
        L.indptr.push_back((int64_t)L.indices.size());
      }
  int ntiles = (int)(n / R);
  std::vector<int32_t> tile;
  if (argc > 5 && atoi(argv[5]) == 1)
    ntiles = partition_grid(n, 3, coords.data(), R, nullptr, &tile);
  else
    partition_coords(n, 3, coords.data(), ntiles, &tile);
  DTileSchedule ds;
  std::string why;
  build_dtile_schedule(L, true, tile, ntiles, 8, &ds, &why);
  // depth over task order
  std::vector<int> tpos(n), depth(ntiles, 0);
  const int nt = (int)ds.tile_row_ptr.size() - 1;
  for (int q = 0; q < nt; ++q)
    for (int k = ds.tile_row_ptr[q]; k < ds.tile_row_ptr[q + 1]; ++k) tpos[ds.task_row[k]] = q;
  int maxd = 0, maxdeps = 0;
  double avgdeps = 0;
  for (int q = 0; q < nt; ++q) {
    std::vector<int> deps;
    for (int k = ds.tile_row_ptr[q]; k < ds.tile_row_ptr[q + 1]; ++k)
      for (int e = 0; e < 8; ++e) {
        const int c = ds.ell_col[(int64_t)k * 8 + e];
        if (c >= 0) deps.push_back(tpos[c]);
      }
    std::sort(deps.begin(), deps.end());
    deps.erase(std::unique(deps.begin(), deps.end()), deps.end());
    int d = 0;
    for (int u : deps) d = std::max(d, depth[u] + 1);
    depth[q] = d;
    maxd = std::max(maxd, d);
    maxdeps = std::max<int>(maxdeps, (int)deps.size());
    avgdeps += deps.size();
  }
  std::vector<int> hist(maxd + 1, 0);
  for (int q = 0; q < nt; ++q) hist[depth[q]]++;
  int w = 0;
  for (int h : hist) w = std::max(w, h);
  std::printf("grid %dx%dx%d rows/tile %d: tiles %d tmax %d, tile-DAG depth %d (max width %d), deps/tile avg %.1f max %d\n",
              X, Y, Z, R, nt, ds.tmax, maxd + 1, w, avgdeps / nt, maxdeps);
}
