// vn_large.cuh — von Neumann entropy -sum lambda ln lambda of rho (spinmc.cpp:165-169) for a
// Hermitian n x n rho with n = d_a in [256, 1024] (16 <= S <= 21), too large for shared
// memory: rho lives in global memory (full column-major planes Re / Im, pitch n, written
// by the work queue's TILE items), and the 256 consumer threads of one CTA reduce it.
//
// The reference diagonalises with cyclic complex Jacobi (linalg.cpp:161-232). As for
// n <= 128 (vn.cuh, vn_packed.cuh) we take the parallel textbook route, parity being a
// tolerance statement either way:
//   1. Hermitian part W = (rho + rho^H)/2 (linalg.cpp:179-185);
//   2. Householder reduction to tridiagonal form, ONE pass over the trailing block per
//      reflector: reflector k's rank-2 update B -= v w^H + w v^H (w = tau B v - K v) is
//      applied to column k+1 first, reflector k+1 is formed from it, and a single sweep
//      over the remaining columns applies update k and accumulates B' v' for reflector k+1
//      (thread <-> row, column loop: coalesced);
//   3. eigenvalues by bisection on the division-free Sturm counts of vn.cuh (two points per
//      thread and round, every eigenvalue to ~1 ulp of ||T||);
//   4. entropy over the eigenvalues in ascending order (the reference's summation order),
//      clamped at 0 (std::max keeps -0.0: (e < 0) ? 0 : e).
// The scratch vectors live in the work queue's stage buffers, idle while a DEC item runs.
#pragma once
#include "vn.cuh"

namespace tg {
namespace vnl {

constexpr int kMinN = 256, kMaxN = 1024;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRowsPerThread = kMaxN / kThreads;  // 4

struct Scratch {
  double vr[2][kMaxN], vi[2][kMaxN];  // reflector v (double-buffered by k & 1)
  double pr[2][kMaxN], pi[2][kMaxN];  // B v
  double d[kMaxN], e2[kMaxN], lam[kMaxN];
  double red[2][kWarps][2];
  double tau[2];
  double lo, hi;
};

template <class Sync>
__device__ __forceinline__ double block_sum(double v, Scratch& W, int slot, int tid, Sync sync) {
  v = warp_sum(v);
  if ((tid & 31) == 0) W.red[slot][tid >> 5][0] = v;
  sync();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) t += W.red[slot][w][0];
  return t;
}

// Reflector from x = column c, rows r0 .. n-1 (m = n - r0 entries), H = I - tau v v^H with
// v = x + phase(x0) |x| e1 (vn.cuh's convention): v -> W.v*[b][0..m), tau -> W.tau[b],
// e2 = |x|^2. Every thread returns after a barrier.
template <class Sync>
__device__ void reflector(const double* Ar, const double* Ai, int n, int c, int r0, int b, Scratch& W,
                          int& k_e2_idx, int tid, Sync sync) {
  const int m = n - r0;
  double s = 0.0;
  for (int i = tid; i < m; i += kThreads) {
    const double xr = __ldcg(Ar + (r0 + i) + static_cast<size_t>(c) * n);
    const double xi = __ldcg(Ai + (r0 + i) + static_cast<size_t>(c) * n);
    W.vr[b][i] = xr;
    W.vi[b][i] = xi;
    if (i > 0) s = fma(xr, xr, fma(xi, xi, s));
  }
  s = block_sum(s, W, b, tid, sync);
  const double a0r = W.vr[b][0], a0i = W.vi[b][0];
  const double ax2 = fma(a0r, a0r, a0i * a0i);
  sync();  // every thread has read v[0] and the partial sums
  if (tid == 0) {
    if (s > 0.0) {
      const double inv0 = ax2 > 0.0 ? rsqrt(ax2) : 0.0;  // 1/|x0|
      const double ax0 = ax2 * inv0, xx = ax2 + s, xnorm = sqrt(xx), mag = ax0 + xnorm;
      const double phr = ax2 > 0.0 ? a0r * inv0 : 1.0, phi = a0i * inv0;
      W.vr[b][0] = phr * mag;
      W.vi[b][0] = phi * mag;
      W.tau[b] = 1.0 / (xnorm * mag);
      W.e2[k_e2_idx] = xx;
    } else {
      W.tau[b] = 0.0;
      W.e2[k_e2_idx] = ax2;
    }
  }
  sync();
  if (W.tau[b] == 0.0)
    for (int i = tid; i < m; i += kThreads) W.vr[b][i] = W.vi[b][i] = 0.0;
  sync();
}

// Phase 2 of reflector step k (trailing block rows/cols o .. n-1, size m): columns j >= 1,
// rows i >= 1 get update k; B' v' (reflector k+1, in W.v*[nb]) accumulates into W.p*[nb].
// R rows per thread (n <= 256 R, rows i = 1 + tid + h * 256) and JB = 16 / R columns per
// block: every block has 2 R JB = 32 loads in flight before any store (the sweep is bound by
// the latency of the L2 / HBM round trip, not by bandwidth).
template <int R>
__device__ __forceinline__ void phase2(double* Ar, double* Ai, int n, int m, int o, int b, int nb, double tau,
                                       double K, Scratch& W, int tid) {
  constexpr int JB = 16 / R;
  auto wr = [&](int i) { return fma(tau, W.pr[b][i], -K * W.vr[b][i]); };
  auto wi = [&](int i) { return fma(tau, W.pi[b][i], -K * W.vi[b][i]); };
  double pr[R], pim[R], vr_i[R], vi_i[R], wr_i[R], wi_i[R];
#pragma unroll
  for (int h = 0; h < R; ++h) {
    const int i = 1 + tid + h * kThreads;
    const bool ok = i < m;
    pr[h] = pim[h] = 0.0;
    vr_i[h] = ok ? W.vr[b][i] : 0.0;
    vi_i[h] = ok ? W.vi[b][i] : 0.0;
    wr_i[h] = ok ? wr(i) : 0.0;
    wi_i[h] = ok ? wi(i) : 0.0;
  }
  for (int j0 = 1; j0 < m; j0 += JB) {
    double ar[JB][R], ai[JB][R];
#pragma unroll
    for (int jj = 0; jj < JB; ++jj) {
      const int j = j0 + jj;
      const double* cr = Ar + o + static_cast<size_t>(o + (j < m ? j : 0)) * n;
      const double* ci = Ai + o + static_cast<size_t>(o + (j < m ? j : 0)) * n;
#pragma unroll
      for (int h = 0; h < R; ++h) {
        const int i = 1 + tid + h * kThreads;
        const bool ok = j < m && i < m;
        ar[jj][h] = ok ? __ldcg(cr + i) : 0.0;
        ai[jj][h] = ok ? __ldcg(ci + i) : 0.0;
      }
    }
#pragma unroll
    for (int jj = 0; jj < JB; ++jj) {
      const int j = j0 + jj;
      if (j >= m) break;
      const double vjr = W.vr[b][j], vji = W.vi[b][j], wjr = wr(j), wji = wi(j);
      const double ur = W.vr[nb][j - 1], ui = W.vi[nb][j - 1];  // v' of reflector k+1
      double* cr = Ar + o + static_cast<size_t>(o + j) * n;
      double* ci = Ai + o + static_cast<size_t>(o + j) * n;
#pragma unroll
      for (int h = 0; h < R; ++h) {
        const int i = 1 + tid + h * kThreads;
        if (i < m) {
          const double nr = fma(-vr_i[h], wjr, fma(-vi_i[h], wji, fma(-wr_i[h], vjr, fma(-wi_i[h], vji, ar[jj][h]))));
          const double ni = fma(-vi_i[h], wjr, fma(vr_i[h], wji, fma(-wi_i[h], vjr, fma(wr_i[h], vji, ai[jj][h]))));
          __stcg(cr + i, nr);
          __stcg(ci + i, ni);
          pr[h] = fma(nr, ur, fma(-ni, ui, pr[h]));
          pim[h] = fma(nr, ui, fma(ni, ur, pim[h]));
        }
      }
    }
  }
#pragma unroll
  for (int h = 0; h < R; ++h) {
    const int i = tid + h * kThreads;  // row 1 + i of the block = row i of the next block
    if (i < m - 1) {
      W.pr[nb][i] = pr[h];
      W.pi[nb][i] = pim[h];
    }
  }
}

// Steps 1-2: on return W.d[0..n), W.e2[0..n-1) hold the real symmetric tridiagonal with
// rho's eigenvalues. Ar / Ai are overwritten.
template <class Sync>
__device__ void tridiagonalize(double* Ar, double* Ai, int n, Scratch& W, int tid, Sync sync) {
  // Hermitian part (linalg.cpp:179-185): diagonal real, W(j,i) = conj(W(i,j))
  for (size_t q = tid; q < static_cast<size_t>(n) * n; q += kThreads) {
    const int i = static_cast<int>(q % n), j = static_cast<int>(q / n);
    if (i > j) {
      const size_t a = i + static_cast<size_t>(j) * n, t = j + static_cast<size_t>(i) * n;
      const double re = 0.5 * (__ldcg(Ar + a) + __ldcg(Ar + t));
      const double im = 0.5 * (__ldcg(Ai + a) - __ldcg(Ai + t));
      __stcg(Ar + a, re);
      __stcg(Ai + a, im);
      __stcg(Ar + t, re);
      __stcg(Ai + t, -im);
    } else if (i == j) {
      __stcg(Ai + q, 0.0);
    }
  }
  __threadfence_block();
  sync();
  // reflector 0 from column 0 (rows 1..), then B v for the trailing block (1..n-1)^2
  int k = 0;
  if (tid == 0) W.d[0] = __ldcg(Ar);
  reflector(Ar, Ai, n, 0, 1, 0, W, k, tid, sync);
  {
    const int m = n - 1;
    double pr[kRowsPerThread] = {0, 0, 0, 0}, pim[kRowsPerThread] = {0, 0, 0, 0};
    for (int j = 0; j < m; ++j) {
      const double vr = W.vr[0][j], vi = W.vi[0][j];
      const double* cr = Ar + 1 + static_cast<size_t>(1 + j) * n;
      const double* ci = Ai + 1 + static_cast<size_t>(1 + j) * n;
#pragma unroll
      for (int h = 0; h < kRowsPerThread; ++h) {
        const int i = tid + h * kThreads;
        if (i < m) {
          const double br = __ldcg(cr + i), bi = __ldcg(ci + i);
          pr[h] = fma(br, vr, fma(-bi, vi, pr[h]));
          pim[h] = fma(br, vi, fma(bi, vr, pim[h]));
        }
      }
    }
#pragma unroll
    for (int h = 0; h < kRowsPerThread; ++h) {
      const int i = tid + h * kThreads;
      if (i < m) {
        W.pr[0][i] = pr[h];
        W.pi[0][i] = pim[h];
      }
    }
  }
  sync();
  for (k = 0; k + 2 < n; ++k) {
    const int b = k & 1, nb = b ^ 1, m = n - k - 1, o = k + 1;  // trailing block rows/cols o .. n-1
    // K = tau^2/2 Re(v^H B v); w = tau B v - K v
    double part = 0.0;
    for (int i = tid; i < m; i += kThreads) part = fma(W.vr[b][i], W.pr[b][i], fma(W.vi[b][i], W.pi[b][i], part));
    const double tau = W.tau[b];
    const double K = 0.5 * tau * tau * block_sum(part, W, b, tid, sync);
    auto wr = [&](int i) { return fma(tau, W.pr[b][i], -K * W.vr[b][i]); };
    auto wi = [&](int i) { return fma(tau, W.pi[b][i], -K * W.vi[b][i]); };
    // phase 1: column o (block column 0) with update k: B(i,0) -= v_i conj(w_0) + w_i conj(v_0)
    {
      const double v0r = W.vr[b][0], v0i = W.vi[b][0], w0r = wr(0), w0i = wi(0);
      double* cr = Ar + o + static_cast<size_t>(o) * n;
      double* ci = Ai + o + static_cast<size_t>(o) * n;
      for (int i = tid; i < m; i += kThreads) {
        const double vr = W.vr[b][i], vi = W.vi[b][i], wri = wr(i), wii = wi(i);
        double ar = __ldcg(cr + i), ai = __ldcg(ci + i);
        ar = fma(-vr, w0r, fma(-vi, w0i, fma(-wri, v0r, fma(-wii, v0i, ar))));
        ai = fma(-vi, w0r, fma(vr, w0i, fma(-wii, v0r, fma(wri, v0i, ai))));
        __stcg(cr + i, ar);
        __stcg(ci + i, ai);
      }
    }
    __threadfence_block();
    sync();
    if (tid == 0) W.d[o] = __ldcg(Ar + o + static_cast<size_t>(o) * n);
    if (k + 3 < n) {
      // reflector k+1 from column o, rows o+1 ..
      int e2i = o;
      reflector(Ar, Ai, n, o, o + 1, nb, W, e2i, tid, sync);
      // phase 2: block columns j = 1 .. m-1, rows 1 .. m-1: update k, and B' v' (reflector k+1)
      // (rows per thread follow the shrinking block: more columns in flight as it shrinks)
      if (m <= kThreads + 1) phase2<1>(Ar, Ai, n, m, o, b, nb, tau, K, W, tid);
      else if (m <= 2 * kThreads + 1) phase2<2>(Ar, Ai, n, m, o, b, nb, tau, K, W, tid);
      else phase2<4>(Ar, Ai, n, m, o, b, nb, tau, K, W, tid);
      __threadfence_block();
      sync();
    } else {
      // last 2 x 2: update the remaining element (o+1, o+1) and (o+1, o) was done in phase 1
      if (tid == 0) {
        const int a = o + 1;
        const size_t idx = a + static_cast<size_t>(a) * n;
        const double v1r = W.vr[b][1], v1i = W.vi[b][1], w1r = wr(1), w1i = wi(1);
        double ar = __ldcg(Ar + idx);
        ar = fma(-v1r, w1r, fma(-v1i, w1i, fma(-w1r, v1r, fma(-w1i, v1i, ar))));
        W.d[a] = ar;
        const double er = __ldcg(Ar + a + static_cast<size_t>(o) * n), ei = __ldcg(Ai + a + static_cast<size_t>(o) * n);
        W.e2[o] = fma(er, er, ei * ei);
      }
      sync();
    }
  }
}

// Step 3: W.lam[0..n) ascending; thread t takes eigenvalues t, t + 256, ..., each by
// bisection with two Sturm points per round (the bracket shrinks 3x per round).
template <class Sync>
__device__ void eigenvalues(int n, Scratch& W, int tid, Sync sync) {
  const int lane = tid & 31;
  if (tid < 32) {  // Gershgorin bracket (LAPACK dstebz convention)
    double lo = 1e300, hi = -1e300;
    for (int i = lane; i < n; i += 32) {
      const double el = i > 0 ? sqrt(W.e2[i - 1]) : 0.0, er = i + 1 < n ? sqrt(W.e2[i]) : 0.0;
      lo = fmin(lo, W.d[i] - el - er);
      hi = fmax(hi, W.d[i] + el + er);
    }
    lo = vn::warp_min(lo);
    hi = vn::warp_max(hi);
    if (lane == 0) {
      const double bnorm = fmax(fabs(lo), fabs(hi));
      const double pad = 2.0 * 2.220446049250313e-16 * bnorm * n + 2.0 * 2.2250738585072014e-308;
      W.lo = lo - pad;
      W.hi = hi + pad;
    }
  }
  sync();
  const double tol = 2.220446049250313e-16 * fmax(fmax(fabs(W.lo), fabs(W.hi)), 1e-300);
  for (int j = tid; j < n; j += kThreads) {
    double lo = W.lo, hi = W.hi;
    for (int it = 0; it < 80 && hi - lo > tol; ++it) {
      const double x0 = fma(hi - lo, 1.0 / 3.0, lo), x1 = fma(hi - lo, 2.0 / 3.0, lo);
      int c0, c1;
      vn::sturm2(W, n, x0, x1, c0, c1);
      if (c0 > j) {
        hi = x0;
      } else if (c1 > j) {
        lo = x0;
        hi = x1;
      } else {
        lo = x1;
      }
    }
    W.lam[j] = 0.5 * (lo + hi);
  }
  sync();
}

// Steps 1-4 (the 256 consumer threads). Returns the entropy in thread 0 (others: 0).
template <class Sync>
__device__ double entropy(double* Ar, double* Ai, int n, Scratch& W, int tid, Sync sync) {
  tridiagonalize(Ar, Ai, n, W, tid, sync);
  eigenvalues(n, W, tid, sync);
  for (int i = tid; i < n; i += kThreads) {
    const double l = W.lam[i];
    W.pr[0][i] = l > 1e-15 ? l * log(l) : 0.0;  // spinmc.cpp:166-168
  }
  sync();
  double e = 0.0;
  if (tid == 0)
    for (int i = 0; i < n; ++i) e -= W.pr[0][i];  // ascending order, as the reference
  return (e < 0.0) ? 0.0 : e;                     // std::max(entropy, 0.0)
}

}  // namespace vnl
}  // namespace tg
