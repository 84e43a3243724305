// vn.cuh — von Neumann entropy -sum lambda ln lambda of rho (spinmc.cpp:165-169) for a
// Hermitian n x n rho (n = d_a <= 64) resident in shared memory, computed by the 256 step
// threads of one CTA between two GEMMs (the FP64 pipe is free then).
//
// The reference diagonalises rho with cyclic complex Jacobi (linalg.cpp:161-232): n(n-1)/2
// strictly sequential rotations per sweep, a poor fit for 256 threads. Our rho already
// differs from the reference's in the last bits (DMMA summation order), so vN parity is
// a tolerance statement either way; we use the parallel textbook route instead:
//   1. Hermitian part W = (rho + rho^H)/2 (linalg.cpp:179-185, same as the reference);
//   2. Householder reduction to a Hermitian tridiagonal (n-2 reflections; each is one
//      matrix-vector product and one rank-2 update spread over the CTA); the off-diagonal
//      moduli |e_k| give a real symmetric tridiagonal with the same eigenvalues;
//   3. all eigenvalues by multisection on Sturm counts: G = 256/n threads per eigenvalue,
//      two interleaved count chains per thread, each round shrinks every eigenvalue's
//      bracket by 2G+1 until it is ~1 ulp of ||T|| wide;
//   4. entropy = -sum_{lambda > 1e-15} lambda ln lambda over the eigenvalues in ascending
//      order (the reference sums its sorted eigenvalues in that order), clamped at 0.
// Eigenvalue error ~ 1e-16 * ||rho|| absolute, so the entropy error is ~1e-13 at n = 64,
// inside the 1e-10 tolerance (tests/test_device_parity.py).
#pragma once
#include "tg_device.cuh"

namespace tg {
namespace vn {

constexpr int kMaxN = 64;
constexpr int kThreads = 256;
constexpr int kGroups = kThreads / kMaxN;  // column groups of the matrix-vector product

struct Scratch {
  double vr[kMaxN], vi[kMaxN];               // Householder vector v
  double wr[kMaxN], wi[kMaxN];               // w = p - K v
  double pp[kGroups][2][kMaxN];              // p = tau B v, partial over column groups
  double d[kMaxN], e2[kMaxN];                // tridiagonal: diagonal, |off-diagonal|^2
  double lam[kMaxN];                         // eigenvalues, ascending
  double tau, lo, hi, pivmin;
};

// Pitch (doubles) of rho's planes: odd, so a warp reading one row across columns, or
// 32 columns at one row, hits distinct banks.
template <int N>
struct Layout {
  static constexpr int P = N + 1;
  static constexpr int PLANE = N * P;
};

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Steps 1-2. On return W.d[0..n), W.e2[0..n-1) hold the tridiagonal.
template <class Sync>
__device__ void tridiagonalize(double* Ar, double* Ai, int n, int P, Scratch& W, int tid,
                               Sync sync) {
  const int warp = tid >> 5, lane = tid & 31;
  // Hermitian part (linalg.cpp:179-185): diagonal real, W(j,i) = conj(W(i,j))
  for (int j = warp; j < n; j += kThreads / 32) {
    for (int i = lane; i < n; i += 32) {
      if (i > j) {
        const double re = 0.5 * (Ar[i + j * P] + Ar[j + i * P]);
        const double im = 0.5 * (Ai[i + j * P] - Ai[j + i * P]);
        Ar[i + j * P] = re;
        Ai[i + j * P] = im;
        Ar[j + i * P] = re;
        Ai[j + i * P] = -im;
      } else if (i == j) {
        Ai[i + i * P] = 0.0;
      }
    }
  }
  sync();
  for (int k = 0; k + 2 < n; ++k) {
    const int m = n - k - 1;  // length of the column below the diagonal
    const int c0 = (k + 1) + k * P;
    if (warp == 0) {
      double xr0 = 0.0, xi0 = 0.0, xr1 = 0.0, xi1 = 0.0;
      if (lane < m) { xr0 = Ar[c0 + lane]; xi0 = Ai[c0 + lane]; }
      if (lane + 32 < m) { xr1 = Ar[c0 + lane + 32]; xi1 = Ai[c0 + lane + 32]; }
      double s = (lane == 0 ? 0.0 : fma(xr0, xr0, xi0 * xi0)) + fma(xr1, xr1, xi1 * xi1);
      s = warp_sum(s);  // |x|^2 without the first element
      const double a0r = __shfl_sync(0xffffffffu, xr0, 0), a0i = __shfl_sync(0xffffffffu, xi0, 0);
      const double ax0 = hypot(a0r, a0i);
      double tau = 0.0, v0r = a0r, v0i = a0i;
      if (s > 0.0) {
        // H = I - tau v v^H, v = x - alpha e1, alpha = -phase(x0) |x|: H x = alpha e1
        const double xx = fma(ax0, ax0, s), xnorm = sqrt(xx);
        const double phr = ax0 > 0.0 ? a0r / ax0 : 1.0, phi = ax0 > 0.0 ? a0i / ax0 : 0.0;
        const double mag = ax0 + xnorm;
        v0r = phr * mag;
        v0i = phi * mag;
        tau = 1.0 / (xnorm * mag);  // 2 / (v^H v)
        if (lane == 0) W.e2[k] = xx;
      } else if (lane == 0) {
        W.e2[k] = fma(a0r, a0r, a0i * a0i);  // column already reduced
      }
      if (lane < m) {
        W.vr[lane] = lane == 0 ? v0r : xr0;
        W.vi[lane] = lane == 0 ? v0i : xi0;
      }
      if (lane + 32 < m) {
        W.vr[lane + 32] = xr1;
        W.vi[lane + 32] = xi1;
      }
      if (lane == 0) {
        W.tau = tau;
        W.d[k] = Ar[k + k * P];
      }
    }
    sync();
    const double tau = W.tau;
    if (tau == 0.0) continue;  // block-uniform
    // p_r = sum_c B(r,c) v_c = sum_c conj(B(c,r)) v_c: thread (r, g) walks column k+1+r
    // (contiguous) over c = g, g+4, ...; lanes differ in r -> stride P (odd): no conflicts
    {
      const int r = tid & (kMaxN - 1), g = tid / kMaxN;
      if (r < m) {
        const double* cr = Ar + (k + 1) + (k + 1 + r) * P;
        const double* ci = Ai + (k + 1) + (k + 1 + r) * P;
        double sr = 0.0, si = 0.0;
        for (int c = g; c < m; c += kGroups) {
          const double br = cr[c], bi = ci[c], vr = W.vr[c], vi = W.vi[c];
          sr = fma(br, vr, fma(bi, vi, sr));
          si = fma(br, vi, fma(-bi, vr, si));
        }
        W.pp[g][0][r] = sr;
        W.pp[g][1][r] = si;
      }
    }
    sync();
    if (warp == 0) {  // p = tau B v; K = tau/2 Re(v^H p); w = p - K v
      double pr[2], pi[2], dot = 0.0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = lane + 32 * h;
        pr[h] = pi[h] = 0.0;
        if (r < m) {
          pr[h] = tau * ((W.pp[0][0][r] + W.pp[1][0][r]) + (W.pp[2][0][r] + W.pp[3][0][r]));
          pi[h] = tau * ((W.pp[0][1][r] + W.pp[1][1][r]) + (W.pp[2][1][r] + W.pp[3][1][r]));
          dot = fma(W.vr[r], pr[h], fma(W.vi[r], pi[h], dot));
        }
      }
      const double K = 0.5 * tau * warp_sum(dot);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = lane + 32 * h;
        if (r < m) {
          W.wr[r] = fma(-K, W.vr[r], pr[h]);
          W.wi[r] = fma(-K, W.vi[r], pi[h]);
        }
      }
    }
    sync();
    // B -= v w^H + w v^H (thread: row i = tid % 64, columns j = tid / 64 + 4t)
    {
      const int i = tid & (kMaxN - 1);
      if (i < m) {
        const double vr = W.vr[i], vi = W.vi[i], wr = W.wr[i], wi = W.wi[i];
        for (int j = tid / kMaxN; j < m; j += kGroups) {
          const double vjr = W.vr[j], vji = W.vi[j], wjr = W.wr[j], wji = W.wi[j];
          // v_i conj(w_j) + w_i conj(v_j)
          const double re = fma(vr, wjr, fma(vi, wji, fma(wr, vjr, wi * vji)));
          const double im = fma(vi, wjr, fma(-vr, wji, fma(wi, vjr, -wr * vji)));
          const int o = (k + 1 + i) + (k + 1 + j) * P;
          Ar[o] -= re;
          Ai[o] -= im;
        }
      }
    }
    sync();
  }
  if (tid == 0) {
    if (n >= 2) {
      const int a = n - 2, b = n - 1;
      if (n == 2) W.d[0] = Ar[0];
      W.d[a] = Ar[a + a * P];
      W.d[b] = Ar[b + b * P];
      const double er = Ar[b + a * P], ei = Ai[b + a * P];
      W.e2[a] = fma(er, er, ei * ei);
    } else {
      W.d[0] = Ar[0];
    }
  }
  sync();
}

// Sturm count: number of eigenvalues of the tridiagonal (d, e2) below x, two x at once.
__device__ __forceinline__ void sturm2(const Scratch& W, int n, double x0, double x1,
                                       double pivmin, int& c0, int& c1) {
  double q0 = W.d[0] - x0, q1 = W.d[0] - x1;
  if (fabs(q0) < pivmin) q0 = -pivmin;
  if (fabs(q1) < pivmin) q1 = -pivmin;
  c0 = q0 < 0.0;
  c1 = q1 < 0.0;
  for (int i = 1; i < n; ++i) {
    const double di = W.d[i], e = W.e2[i - 1];
    q0 = (di - x0) - e / q0;
    q1 = (di - x1) - e / q1;
    if (fabs(q0) < pivmin) q0 = -pivmin;
    if (fabs(q1) < pivmin) q1 = -pivmin;
    c0 += q0 < 0.0;
    c1 += q1 < 0.0;
  }
}

// Step 3: W.lam[0..n) ascending.
template <class Sync>
__device__ void eigenvalues(int n, Scratch& W, int tid, Sync sync) {
  const int lane = tid & 31;
  if (tid < 32) {  // Gershgorin bracket and pivot guard (LAPACK dstebz convention)
    double lo = 1e300, hi = -1e300, emax = 0.0;
    for (int i = lane; i < n; i += 32) {
      const double el = i > 0 ? sqrt(W.e2[i - 1]) : 0.0, er = i + 1 < n ? sqrt(W.e2[i]) : 0.0;
      lo = fmin(lo, W.d[i] - el - er);
      hi = fmax(hi, W.d[i] + el + er);
      if (i + 1 < n) emax = fmax(emax, W.e2[i]);
    }
    lo = warp_min(lo);
    hi = warp_max(hi);
    emax = warp_max(emax);
    if (lane == 0) {
      const double bnorm = fmax(fabs(lo), fabs(hi));
      const double pad = 2.0 * 2.220446049250313e-16 * bnorm * n + 2.0 * 2.2250738585072014e-308;
      W.lo = lo - pad;
      W.hi = hi + pad;
      W.pivmin = 2.2250738585072014e-308 * fmax(1.0, emax);
    }
  }
  sync();
  const int G = n >= 8 ? kThreads / n : 32;  // threads per eigenvalue (power of two, <= 32)
  const int j = tid / G, gl = tid % G;
  const int M = 2 * G;  // points per eigenvalue per round
  double lo = W.lo, hi = W.hi;
  const double pivmin = W.pivmin;
  const double tol = 2.220446049250313e-16 * fmax(fmax(fabs(lo), fabs(hi)), 1e-300);
  const int rounds = min(64, static_cast<int>(ceil(log((hi - lo) / tol) / log(static_cast<double>(M + 1)))));
  const double inv = 1.0 / (M + 1);
  for (int it = 0; it < rounds; ++it) {
    const double w = hi - lo;
    const double x0 = fma(w, (2 * gl + 1) * inv, lo), x1 = fma(w, (2 * gl + 2) * inv, lo);
    int c0, c1;
    sturm2(W, n, x0, x1, pivmin, c0, c1);
    double nlo = lo, nhi = hi;
    if (c0 <= j) nlo = fmax(nlo, x0); else nhi = fmin(nhi, x0);
    if (c1 <= j) nlo = fmax(nlo, x1); else nhi = fmin(nhi, x1);
    for (int o = G >> 1; o > 0; o >>= 1) {  // reduce over the eigenvalue's G lanes
      nlo = fmax(nlo, __shfl_xor_sync(0xffffffffu, nlo, o));
      nhi = fmin(nhi, __shfl_xor_sync(0xffffffffu, nhi, o));
    }
    lo = nlo;
    hi = nhi;
  }
  if (gl == 0 && j < n) W.lam[j] = 0.5 * (lo + hi);
  sync();
}

// Steps 1-4 (all kThreads threads). Returns the entropy in thread 0 (other threads: 0).
template <class Sync>
__device__ double entropy(double* Ar, double* Ai, int n, int P, Scratch& W, int tid, Sync sync) {
  tridiagonalize(Ar, Ai, n, P, W, tid, sync);
  eigenvalues(n, W, tid, sync);
  double e = 0.0;
  if (tid < 32) {
    for (int i = tid; i < n; i += 32) {
      const double l = W.lam[i];
      W.pp[0][0][i] = l > 1e-15 ? l * log(l) : 0.0;  // spinmc.cpp:166-168
    }
    __syncwarp();
    if (tid == 0)
      for (int i = 0; i < n; ++i) e -= W.pp[0][0][i];  // ascending order, as the reference
  }
  return (e < 0.0) ? 0.0 : e;  // std::max(entropy, 0.0)
}

}  // namespace vn
}  // namespace tg
