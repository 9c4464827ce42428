// P1 stiffness / lumped-mass assembly on the device (setup path, SURVEY §8f
// rank 1; restates bd/assembly.py:36-97 and the harmonic-mean monodomain
// tensor of bd/precond.py:34-47).
//
// Per element e (simplex with A = D+1 vertices): edge matrix E (rows
// x_{r+1} - x_0), vol = det(E)/D!, gradients G = [-1ᵀ Eᵀ⁻¹ ; Eᵀ⁻¹], tensor σ_e
// (or the harmonic mean sym(inv(inv σ_a + inv σ_b)) for the monodomain
// block), local K_e = vol · sym(G σ Gᵀ).  The A² (row, col) pairs of every
// element are keyed row·nv + col and radix-sorted with a STABLE sort, so the
// contributions of each CSR entry sit together in element order and are
// summed sequentially: deterministic, no floating-point atomics.  Lumped mass
// m_v = Σ vol_e/(D+1), summed in the reference's (local vertex, element)
// order (bd/assembly.py:93-96).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

namespace bd {
namespace asmk {

template <int D>
__device__ __forceinline__ double det_inv(const double (&m)[D][D], double (&inv)[D][D]) {
  if constexpr (D == 2) {
    const double det = m[0][0] * m[1][1] - m[0][1] * m[1][0];
    inv[0][0] = m[1][1] / det;
    inv[0][1] = -m[0][1] / det;
    inv[1][0] = -m[1][0] / det;
    inv[1][1] = m[0][0] / det;
    return det;
  } else {
    const double c00 = m[1][1] * m[2][2] - m[1][2] * m[2][1];
    const double c01 = m[1][2] * m[2][0] - m[1][0] * m[2][2];
    const double c02 = m[1][0] * m[2][1] - m[1][1] * m[2][0];
    const double det = m[0][0] * c00 + m[0][1] * c01 + m[0][2] * c02;
    inv[0][0] = c00 / det;
    inv[1][0] = c01 / det;
    inv[2][0] = c02 / det;
    inv[0][1] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) / det;
    inv[1][1] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) / det;
    inv[2][1] = (m[0][1] * m[2][0] - m[0][0] * m[2][1]) / det;
    inv[0][2] = (m[0][1] * m[1][2] - m[0][2] * m[1][1]) / det;
    inv[1][2] = (m[0][2] * m[1][0] - m[0][0] * m[1][2]) / det;
    inv[2][2] = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) / det;
    return det;
  }
}

// local matrices (ne × A²), volumes (ne); bad[0] = 1 on a non-positive volume
template <int D>
__global__ void __launch_bounds__(256) k_local(int64_t ne, const double* __restrict__ xv,
                                               const int64_t* __restrict__ el,
                                               const double* __restrict__ sa,
                                               const double* __restrict__ sb,
                                               double* __restrict__ local, double* __restrict__ vol,
                                               int* __restrict__ bad) {
  constexpr int A = D + 1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t v[A];
#pragma unroll
    for (int a = 0; a < A; ++a) v[a] = el[e * A + a];
    double m[D][D], mi[D][D];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int c = 0; c < D; ++c) m[r][c] = xv[v[r + 1] * D + c] - xv[v[0] * D + c];
    const double det = det_inv<D>(m, mi);
    if (!(det > 0.0)) atomicExch(bad, 1);
    double vl = det;
#pragma unroll
    for (int k = 2; k <= D; ++k) vl /= (double)k;  // det / D!
    vol[e] = vl;
    // G[0] = -sum of rows of tail, G[r+1][c] = inv(E)[c][r]
    double g[A][D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double s = 0.0;
#pragma unroll
      for (int r = 0; r < D; ++r) {
        g[r + 1][c] = mi[c][r];
        s += mi[c][r];
      }
      g[0][c] = -s;
    }
    double sg[D][D];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int c = 0; c < D; ++c) sg[r][c] = sa[e * D * D + r * D + c];
    if (sb) {  // harmonic mean: sym(inv(inv(a) + inv(b)))
      double ia[D][D], ib[D][D], b[D][D], s[D][D];
      det_inv<D>(sg, ia);
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) b[r][c] = sb[e * D * D + r * D + c];
      det_inv<D>(b, ib);
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) s[r][c] = ia[r][c] + ib[r][c];
      det_inv<D>(s, b);
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) sg[r][c] = 0.5 * (b[r][c] + b[c][r]);
    }
    double gs[A][D];  // G σ
#pragma unroll
    for (int i = 0; i < A; ++i)
#pragma unroll
      for (int k = 0; k < D; ++k) {
        double s = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) s += g[i][d] * sg[d][k];
        gs[i][k] = s;
      }
    double K[A][A];
#pragma unroll
    for (int i = 0; i < A; ++i)
#pragma unroll
      for (int j = 0; j < A; ++j) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) s += gs[i][k] * g[j][k];
        K[i][j] = s;
      }
#pragma unroll
    for (int i = 0; i < A; ++i)
#pragma unroll
      for (int j = 0; j < A; ++j) local[e * A * A + i * A + j] = (0.5 * (K[i][j] + K[j][i])) * vl;
  }
}

template <int D>
__global__ void __launch_bounds__(256) k_keys(int64_t ne, const int64_t* __restrict__ el, int64_t nv,
                                              unsigned long long* __restrict__ keys,
                                              unsigned long long* __restrict__ vals) {
  constexpr int A = D + 1;
  const int64_t np = ne * A * A;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = p / (A * A);
    const int ij = (int)(p - e * A * A);
    const int64_t r = el[e * A + ij / A], c = el[e * A + ij % A];
    keys[p] = (unsigned long long)(r * nv + c);
    vals[p] = (unsigned long long)p;
  }
}

__global__ void __launch_bounds__(256) k_heads(int64_t np, const unsigned long long* __restrict__ keys,
                                               long long* __restrict__ head) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np;
       p += (int64_t)gridDim.x * blockDim.x)
    head[p] = (p == 0 || keys[p] != keys[p - 1]) ? 1 : 0;
}

__global__ void __launch_bounds__(256) k_seg_start(int64_t np, const long long* __restrict__ head,
                                                   const long long* __restrict__ pos,
                                                   long long* __restrict__ start) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np;
       p += (int64_t)gridDim.x * blockDim.x)
    if (head[p]) start[pos[p]] = p;
}

// (Entries whose contributions cancel in exact arithmetic come out as rounding
// residues here; the host side, assembly.py DeviceAssembler._reference_zeros,
// gives them the reference's own value, exact zero or residue.)

// one thread per CSR entry: sequential sum of its contributions (element
// order); diagonal entries also form the lumped mass in (local vertex, element)
// order
template <int D>
__global__ void __launch_bounds__(256) k_segsum(int64_t nnz, int64_t np, int64_t nv,
                                                const long long* __restrict__ start,
                                                const unsigned long long* __restrict__ keys,
                                                const unsigned long long* __restrict__ vals,
                                                const double* __restrict__ local,
                                                const double* __restrict__ vol,
                                                int* __restrict__ col, double* __restrict__ data,
                                                unsigned long long* __restrict__ ukey,
                                                double* __restrict__ mass) {
  constexpr int A = D + 1;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < nnz;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s0 = start[u], s1 = u + 1 < nnz ? start[u + 1] : np;
    const unsigned long long key = keys[s0];
    const int64_t r = (int64_t)(key / (unsigned long long)nv), c = (int64_t)(key % (unsigned long long)nv);
    double s = 0.0;
    for (int64_t q = s0; q < s1; ++q) s += local[vals[q]];
    data[u] = s;
    col[u] = (int)c;
    ukey[u] = key;
    if (r == c) {
      double ms = 0.0;
      for (int k = 0; k < A; ++k)
        for (int64_t q = s0; q < s1; ++q) {
          const unsigned long long p = vals[q];
          const int ij = (int)(p % (A * A));
          if (ij / A == k) ms += vol[p / (A * A)] / (double)A;
        }
      mass[r] = ms;
    }
  }
}

// rowptr[r] = first entry with row >= r (binary search over the sorted keys)
__global__ void __launch_bounds__(256) k_rowptr(int64_t nv, int64_t nnz,
                                                const unsigned long long* __restrict__ ukey,
                                                long long* __restrict__ rowptr) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= nv;
       r += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long target = (unsigned long long)r * (unsigned long long)nv;
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ukey[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    rowptr[r] = lo;
  }
}

// Heart tensors of the transmural-rotation fibre model (configs 2/3,
// conductivity.py TransmuralRotation + TensorField._heart_tensors) per
// element on the device: centroid, fibre angle linear in z, frame
// (f, s, n) = ((c, s, 0), (-s, c, 0), e_z), and sigma = sum_k g_k e_k e_k^T
// (orthotropic) or g_l f f^T + g_t (I - f f^T) (transversely isotropic),
// in the host's term order.
__global__ void __launch_bounds__(256) k_tensors_transmural(
    int64_t ne, const double* __restrict__ xv, const int64_t* __restrict__ el, double z0,
    double z1, double a0, double a1, double gi0, double gi1, double gi2, double ge0, double ge1,
    double ge2, int ortho, double* __restrict__ out_i, double* __restrict__ out_e) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    double cz = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a) cz += xv[el[e * 4 + a] * 3 + 2];
    cz /= 4.0;
    double z = (cz - z0) / (z1 - z0);
    z = z < 0.0 ? 0.0 : (z > 1.0 ? 1.0 : z);
    const double th = (a0 + (a1 - a0) * z) * (3.141592653589793 / 180.0);
    double sn, cs;
    sincos(th, &sn, &cs);
    const double fr[3][3] = {{cs, sn, 0.0}, {-sn, cs, 0.0}, {0.0, 0.0, 1.0}};
    for (int w = 0; w < 2; ++w) {
      const double g0 = w ? ge0 : gi0, g1 = w ? ge1 : gi1, g2 = w ? ge2 : gi2;
      double* o = (w ? out_e : out_i) + e * 9;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          double v;
          if (ortho) {  // sum_k g_k (e_k e_k^T), no contraction (numpy order)
            v = __dadd_rn(0.0, __dmul_rn(g0, __dmul_rn(fr[0][r], fr[0][q])));
            v = __dadd_rn(v, __dmul_rn(g1, __dmul_rn(fr[1][r], fr[1][q])));
            v = __dadd_rn(v, __dmul_rn(g2, __dmul_rn(fr[2][r], fr[2][q])));
          } else {
            const double pr = __dmul_rn(fr[0][r], fr[0][q]);
            v = __dadd_rn(__dmul_rn(g0, pr), __dmul_rn(g1, __dsub_rn(r == q ? 1.0 : 0.0, pr)));
          }
          o[r * 3 + q] = v;
        }
    }
  }
}

// host: device scratch buffers freed when the owner goes out of scope
struct DevScratch {
  std::vector<void*> p;
  ~DevScratch() {
    for (void* q : p) cudaFree(q);
  }
  template <class T>
  cudaError_t get(T** out, int64_t n) {
    const cudaError_t e = cudaMalloc((void**)out, sizeof(T) * (size_t)std::max<int64_t>(n, 1));
    if (e == cudaSuccess) p.push_back(*out);
    return e;
  }
};

}  // namespace asmk
}  // namespace bd
