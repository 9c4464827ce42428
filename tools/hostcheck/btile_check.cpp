// Dev check (CPU): blocked-tile schedules on a 3D 7-point lower factor.
// (1) every external dependency of a tile lies in an earlier tile;
// (2) a pass simulated tile by tile (y = b - L_ext x ; x = inv * y) matches a
//     plain forward / backward substitution.
#include <cmath>
#include <cstdio>
#include "../../paper_1711_08708_b200/csrc/bd_host.hpp"
using namespace bd;

static bool check(const HostCsr& t, bool lower, const std::vector<int32_t>& tile, int ntiles) {
  DTileSchedule ds;
  BTileSchedule bs;
  std::string why;
  if (!build_dtile_schedule(t, lower, tile, ntiles, 8, &ds, &why) || !build_btile_schedule(ds, &bs, &why)) {
    std::printf("build failed: %s\n", why.c_str());
    return false;
  }
  const int64_t n = t.n;
  std::vector<int> pos(n);
  const int nt = (int)bs.tile_row_ptr.size() - 1;
  for (int q = 0; q < nt; ++q)
    for (int k = bs.tile_row_ptr[q]; k < bs.tile_row_ptr[q + 1]; ++k) pos[bs.task_row[k]] = q;
  for (int q = 0; q < nt; ++q)
    for (int k = bs.tile_row_ptr[q]; k < bs.tile_row_ptr[q + 1]; ++k)
      for (int e = 0; e < bs.Ex; ++e) {
        const int sl = bs.ext_col[(int64_t)k * bs.Ex + e];
        const int c = sl >= 0 ? bs.in_col[bs.tile_in_ptr[q] + sl] : -1;
        if (c >= 0 && pos[c] >= q) {
          std::printf("tile %d row %d depends on tile %d\n", q, bs.task_row[k], pos[c]);
          return false;
        }
      }
  std::vector<double> b(n), x(n, NAN), ref(n);
  for (int64_t i = 0; i < n; ++i) b[i] = std::sin(0.37 * i) + 0.1;
  // reference substitution
  for (int64_t ii = 0; ii < n; ++ii) {
    const int64_t i = lower ? ii : n - 1 - ii;
    double s = b[i], d = 0;
    for (int64_t q = t.indptr[i]; q < t.indptr[i + 1]; ++q) {
      const int j = t.indices[q];
      if (j == i) d = t.values[q]; else s -= t.values[q] * ref[j];
    }
    ref[i] = s / d;
  }
  for (int q = 0; q < nt; ++q) {
    const int r0 = bs.tile_row_ptr[q], nr = bs.tile_row_ptr[q + 1] - r0;
    std::vector<double> y(nr);
    for (int k = 0; k < nr; ++k) {
      double acc = 0;
      for (int e = 0; e < bs.Ex; ++e) {
        const int sl = bs.ext_col[(int64_t)(r0 + k) * bs.Ex + e];
        const int c = sl >= 0 ? bs.in_col[bs.tile_in_ptr[q] + sl] : -1;
        if (c >= 0) {
          if (std::isnan(x[c])) { std::printf("x[%d] not ready\n", c); return false; }
          acc += bs.ext_val[(int64_t)(r0 + k) * bs.Ex + e] * x[c];
        }
      }
      y[k] = b[bs.task_row[r0 + k]] - acc;
    }
    const double* iv = bs.inv.data() + bs.tile_inv_ptr[q];
    for (int k = 0; k < nr; ++k) {
      double s = 0;
      for (int l = 0; l <= k; ++l) s += iv[(int64_t)k * (k + 1) / 2 + l] * y[l];
      x[bs.task_row[r0 + k]] = s;
    }
  }
  double err = 0, nrm = 0;
  for (int64_t i = 0; i < n; ++i) { err = std::fmax(err, std::fabs(x[i] - ref[i])); nrm = std::fmax(nrm, std::fabs(ref[i])); }
  std::printf("%s: xmax %d tiles %d tmax %d Ex %d inv %zu max rel err %.3e\n", lower ? "fwd" : "bwd", bs.xmax, nt, bs.tmax,
              bs.Ex, bs.inv.size(), err / nrm);
  return err / nrm < 1e-12;
}

int main() {
  const int X = 24, Y = 20, Z = 12;
  const int64_t n = (int64_t)X * Y * Z;
  HostCsr L;
  L.n = n;
  L.indptr.push_back(0);
  std::vector<double> coords(3 * n);
  for (int k = 0; k < Z; ++k)
    for (int j = 0; j < Y; ++j)
      for (int i = 0; i < X; ++i) {
        const int64_t r = i + (int64_t)X * (j + (int64_t)Y * k);
        coords[3 * r] = i; coords[3 * r + 1] = j; coords[3 * r + 2] = k;
        if (k) { L.indices.push_back(r - X * Y); L.values.push_back(-0.3); }
        if (j) { L.indices.push_back(r - X); L.values.push_back(-0.25); }
        if (i && j) { L.indices.push_back(r - X - 1); L.values.push_back(-0.05); }
        if (i) { L.indices.push_back(r - 1); L.values.push_back(-0.2); }
        L.indices.push_back(r); L.values.push_back(1.5 + 0.01 * (r % 7));
        L.indptr.push_back((int64_t)L.indices.size());
      }
  HostCsr U = transpose(L);
  const int ntiles = (int)(n / 64);
  std::vector<int32_t> tile;
  partition_coords(n, 3, coords.data(), ntiles, &tile);
  const bool ok = check(L, true, tile, ntiles) && check(U, false, tile, ntiles);
  std::puts(ok ? "OK" : "FAIL");
  return ok ? 0 : 1;
}
