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
//      matrix-vector product and one rank-2 update spread over the CTA, two barriers per
//      reflection); the off-diagonal moduli |e_k| give a real symmetric tridiagonal with
//      the same eigenvalues;
//   3. all eigenvalues by multisection on division-free Sturm counts: G = 256/n threads
//      per eigenvalue, each round shrinks every eigenvalue's bracket by G+1 until it is
//      ~1 ulp of ||T|| wide;
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
constexpr int kWarps = kThreads / 32;

struct Scratch {
  double vr[2][kMaxN], vi[2][kMaxN];         // Householder vector v (double-buffered by k&1)
  double pr[2][kMaxN], pi[2][kMaxN];         // B v (double-buffered)
  double part[2][kWarps];                    // per-warp partials of Re(v^H B v)
  double tau[2];
  double d[kMaxN], e2[kMaxN];                // tridiagonal: diagonal, |off-diagonal|^2
  double lam[kMaxN];                         // eigenvalues, ascending
  double lo, hi;
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

// Warp 0: Householder reflector of column k (rows k+1..n-1), H = I - tau v v^H with
// v = x - alpha e1, alpha = -phase(x0) |x| (H x = alpha e1, tau = 2 / v^H v); records
// d_k = A(k,k) and e2_k = |alpha|^2. A column that is already reduced gets tau = v = 0.
__device__ __forceinline__ void reflector(const double* Ar, const double* Ai, int n, int P, int k,
                                          Scratch& W, int lane) {
  const int m = n - k - 1, c0 = (k + 1) + k * P, b = k & 1;
  double xr0 = 0.0, xi0 = 0.0, xr1 = 0.0, xi1 = 0.0;
  if (lane < m) { xr0 = Ar[c0 + lane]; xi0 = Ai[c0 + lane]; }
  if (lane + 32 < m) { xr1 = Ar[c0 + lane + 32]; xi1 = Ai[c0 + lane + 32]; }
  const double s = warp_sum((lane == 0 ? 0.0 : fma(xr0, xr0, xi0 * xi0)) + fma(xr1, xr1, xi1 * xi1));
  const double a0r = __shfl_sync(0xffffffffu, xr0, 0), a0i = __shfl_sync(0xffffffffu, xi0, 0);
  const double ax2 = fma(a0r, a0r, a0i * a0i);
  if (s > 0.0) {
    const double inv0 = ax2 > 0.0 ? rsqrt(ax2) : 0.0;  // 1/|x0|
    const double ax0 = ax2 * inv0, xx = ax2 + s, xnorm = sqrt(xx), mag = ax0 + xnorm;
    const double phr = ax2 > 0.0 ? a0r * inv0 : 1.0, phi = a0i * inv0;
    if (lane < m) {
      W.vr[b][lane] = lane == 0 ? phr * mag : xr0;
      W.vi[b][lane] = lane == 0 ? phi * mag : xi0;
    }
    if (lane + 32 < m) {
      W.vr[b][lane + 32] = xr1;
      W.vi[b][lane + 32] = xi1;
    }
    if (lane == 0) {
      W.tau[b] = 1.0 / (xnorm * mag);
      W.e2[k] = xx;
    }
  } else {
    if (lane < m) W.vr[b][lane] = W.vi[b][lane] = 0.0;
    if (lane + 32 < m) W.vr[b][lane + 32] = W.vi[b][lane + 32] = 0.0;
    if (lane == 0) {
      W.tau[b] = 0.0;
      W.e2[k] = ax2;
    }
  }
  if (lane == 0) W.d[k] = Ar[k + k * P];
}

// Rank-2 update of the trailing block (rows/cols k+1..n-1) with reflector k:
// B -= v w^H + w v^H, w = tau B v - K v, K = tau^2/2 Re(v^H B v). Warp 0 takes the first
// column (it feeds reflector k+1, which warp 0 computes right after); warps 1..7 the rest.
__device__ __forceinline__ void update(double* Ar, double* Ai, int n, int P, int k, const Scratch& W,
                                       int warp, int lane) {
  const int m = n - k - 1, o = k + 1, b = k & 1;
  const double tau = W.tau[b];
  double vhbv = 0.0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) vhbv += W.part[b][w];
  const double K = 0.5 * tau * tau * vhbv;
  double vr[2], vi[2], wr[2], wi[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int i = lane + 32 * h;
    vr[h] = vi[h] = wr[h] = wi[h] = 0.0;
    if (i < m) {
      vr[h] = W.vr[b][i];
      vi[h] = W.vi[b][i];
      wr[h] = fma(tau, W.pr[b][i], -K * vr[h]);
      wi[h] = fma(tau, W.pi[b][i], -K * vi[h]);
    }
  }
  // A -= v_i conj(w_j) + w_i conj(v_j), four chained DFMAs per component. All loads of a
  // group of columns are issued before any store (the compiler cannot reorder SMEM
  // loads across stores that may alias), so the chains of a group overlap.
  auto cols = [&](int j0, int nc) {  // columns j0, j0 + (kWarps-1), ... (nc <= 2)
    double ar[2][2], ai[2][2], wjr[2], wji[2], vjr[2], vji[2];
    int idx[2][2];
    bool ok[2][2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int jj = j0 + c * (kWarps - 1);
      const bool cv = c < nc;
      const int j = cv ? jj : j0;
      vjr[c] = W.vr[b][j];
      vji[c] = W.vi[b][j];
      wjr[c] = fma(tau, W.pr[b][j], -K * vjr[c]);
      wji[c] = fma(tau, W.pi[b][j], -K * vji[c]);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = lane + 32 * h;
        ok[c][h] = cv && i < m;
        idx[c][h] = ok[c][h] ? (o + i) + (o + j) * P : 0;
        ar[c][h] = Ar[idx[c][h]];
        ai[c][h] = Ai[idx[c][h]];
      }
    }
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        ar[c][h] = fma(-vr[h], wjr[c], fma(-vi[h], wji[c], fma(-wr[h], vjr[c], fma(-wi[h], vji[c], ar[c][h]))));
        ai[c][h] = fma(-vi[h], wjr[c], fma(vr[h], wji[c], fma(-wi[h], vjr[c], fma(wr[h], vji[c], ai[c][h]))));
      }
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (ok[c][h]) {
          Ar[idx[c][h]] = ar[c][h];
          Ai[idx[c][h]] = ai[c][h];
        }
  };
  if (warp == 0) {  // column 0 only: it feeds reflector k+1 (warp 0, right after)
    cols(0, 1);
  } else {          // warps 1..7: columns 1, 2, ... round robin, two per group
    for (int j = warp; j < m; j += 2 * (kWarps - 1)) cols(j, j + (kWarps - 1) < m ? 2 : 1);
  }
}

// B v (rows/cols k+1..n-1) for reflector k: warp w owns rows r = 8w + lane/4, the four
// lanes of a row split the columns c = g, g+4, ... (g = lane % 4) of column r
// (B(r,c) = conj(B(c,r)), so the walk is contiguous); two shuffle levels finish each row.
// With pitch P = 4 (mod 16) the 16 lanes of a half-warp hit distinct banks. Also the
// warp's partial of Re(v^H B v).
__device__ __forceinline__ void matvec(const double* Ar, const double* Ai, int n, int P, int k, Scratch& W,
                                       int warp, int lane) {
  const int m = n - k - 1, o = k + 1, b = k & 1;
  const int r = 8 * warp + (lane >> 2), g = lane & 3;
  double ar[4] = {0.0, 0.0, 0.0, 0.0}, ai[4] = {0.0, 0.0, 0.0, 0.0};  // 4 chains
  if (r < m) {
    const double* cr = Ar + o + (o + r) * P;
    const double* ci = Ai + o + (o + r) * P;
#pragma unroll
    for (int t = 0; t < kMaxN / 4; ++t) {
      const int c = g + 4 * t;
      if (c < m) {
        const double br = cr[c], bi = ci[c], vr = W.vr[b][c], vi = W.vi[b][c];
        ar[t & 3] = fma(br, vr, fma(bi, vi, ar[t & 3]));
        ai[t & 3] = fma(br, vi, fma(-bi, vr, ai[t & 3]));
      }
    }
  }
  double sr = (ar[0] + ar[1]) + (ar[2] + ar[3]), si = (ai[0] + ai[1]) + (ai[2] + ai[3]);
  sr += __shfl_xor_sync(0xffffffffu, sr, 1);
  si += __shfl_xor_sync(0xffffffffu, si, 1);
  sr += __shfl_xor_sync(0xffffffffu, sr, 2);
  si += __shfl_xor_sync(0xffffffffu, si, 2);
  double part = 0.0;
  if (g == 0 && r < m) {
    W.pr[b][r] = sr;
    W.pi[b][r] = si;
    part = fma(W.vr[b][r], sr, W.vi[b][r] * si);
  }
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
  if (lane == 0) W.part[b][warp] = part;
}

// Steps 1-2. On return W.d[0..n), W.e2[0..n-1) hold the tridiagonal. Two CTA barriers
// per reflector: [update k-1 (warp 0: first column, then reflector k)] | [B v] |.
template <class Sync>
__device__ void tridiagonalize(double* Ar, double* Ai, int n, int P, Scratch& W, int tid,
                               Sync sync) {
  const int warp = tid >> 5, lane = tid & 31;
  // Hermitian part (linalg.cpp:179-185): diagonal real, W(j,i) = conj(W(i,j))
  for (int j = warp; j < n; j += kWarps) {
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
    if (k > 0) update(Ar, Ai, n, P, k - 1, W, warp, lane);
    if (warp == 0) {
      __syncwarp();
      reflector(Ar, Ai, n, P, k, W, lane);
    }
    sync();
    matvec(Ar, Ai, n, P, k, W, warp, lane);
    sync();
  }
  if (n >= 3) {
    update(Ar, Ai, n, P, n - 3, W, warp, lane);
    sync();
  }
  if (tid == 0) {
    if (n >= 2) {
      const int a = n - 2, c = n - 1;
      W.d[a] = Ar[a + a * P];
      W.d[c] = Ar[c + c * P];
      const double er = Ar[c + a * P], ei = Ai[c + a * P];
      W.e2[a] = fma(er, er, ei * ei);
    } else {
      W.d[0] = Ar[0];
    }
  }
  sync();
}

// Sturm counts (number of eigenvalues of the tridiagonal below x) at two points by the
// three-term recurrence of the leading minors p_i = (d_i - x) p_{i-1} - e2_{i-1} p_{i-2}:
// the count is the number of sign changes p_{i-1} -> p_i (= negative LDL^T pivots
// p_i / p_{i-1}). Division-free, 3 FP64 ops per row and point (the FP64 pipe is the
// scarce resource); signs and zero pivots (replaced by a tiny value of the opposite sign,
// i.e. pivot -tiny, LAPACK dstebz) are integer work; every 4 rows the pair (p_{i-1}, p_i)
// is rescaled by a power of two when it leaves [2^-300, 2^300] (|p_i| can shrink by ~eps
// per row inside clusters of tiny eigenvalues, grows at most 3x per row for ||rho|| <= 1).
struct Minors {
  double pm, pc;
  int cnt;
  __device__ __forceinline__ void init(double d0, double x) {
    pm = 1.0;
    pc = d0 - x;
    if (pc == 0.0) pc = -0x1p-900;
    cnt = pc < 0.0;
  }
  __device__ __forceinline__ void row(double di, double e, double x) {
    double pn = fma(di - x, pc, -e * pm);
    const int hc = __double2hiint(pc);
    if (pn == 0.0) pn = hc < 0 ? 0x1p-900 : -0x1p-900;  // zero pivot -> -tiny
    cnt += static_cast<int>(static_cast<unsigned>(__double2hiint(pn) ^ hc) >> 31);
    pm = pc;
    pc = pn;
  }
  __device__ __forceinline__ void rescale() {
    const int ex = (__double2hiint(pc) >> 20) & 0x7ff;
    if (ex < 1023 - 300 || ex > 1023 + 300) {
      const double f = __hiloint2double((2046 - ex) << 20, 0);
      pm *= f;
      pc *= f;
    }
  }
};

template <class SW>  // vn::Scratch or vnp::Scratch
__device__ __forceinline__ void sturm2(const SW& W, int n, double x0, double x1, int& c0, int& c1) {
  Minors a, b;
  a.init(W.d[0], x0);
  b.init(W.d[0], x1);
  int i = 1;
  for (; i + 3 < n; i += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double di = W.d[i + u], e = W.e2[i + u - 1];
      a.row(di, e, x0);
      b.row(di, e, x1);
    }
    a.rescale();
    b.rescale();
  }
  for (; i < n; ++i) {
    const double di = W.d[i], e = W.e2[i - 1];
    a.row(di, e, x0);
    b.row(di, e, x1);
  }
  c0 = a.cnt;
  c1 = b.cnt;
}

// Step 3: W.lam[0..n) ascending, by multisection: G = 256/n threads per eigenvalue, two
// points each per round, the bracket shrinks by 2G+1 per round down to ~1 ulp of ||T||.
template <class SW, class Sync>
__device__ void eigenvalues(int n, SW& W, int tid, Sync sync) {
  const int lane = tid & 31;
  if (tid < 32) {  // Gershgorin bracket (LAPACK dstebz convention)
    double lo = 1e300, hi = -1e300;
    for (int i = lane; i < n; i += 32) {
      const double el = i > 0 ? sqrt(W.e2[i - 1]) : 0.0, er = i + 1 < n ? sqrt(W.e2[i]) : 0.0;
      lo = fmin(lo, W.d[i] - el - er);
      hi = fmax(hi, W.d[i] + el + er);
    }
    lo = warp_min(lo);
    hi = warp_max(hi);
    if (lane == 0) {
      const double bnorm = fmax(fabs(lo), fabs(hi));
      const double pad = 2.0 * 2.220446049250313e-16 * bnorm * n + 2.0 * 2.2250738585072014e-308;
      W.lo = lo - pad;
      W.hi = hi + pad;
    }
  }
  sync();
  const int G = n >= 8 ? kThreads / n : 32;  // threads per eigenvalue (power of two, <= 32)
  const int j = tid / G, gl = tid % G;
  const int M = 2 * G;                       // points per eigenvalue and round (2 per thread)
  double lo = W.lo, hi = W.hi;
  const double tol = 2.220446049250313e-16 * fmax(fmax(fabs(lo), fabs(hi)), 1e-300);
  const int rounds = min(80, static_cast<int>(ceil(log((hi - lo) / tol) / log(static_cast<double>(M + 1)))));
  const double f0 = static_cast<double>(2 * gl + 1) / (M + 1), f1 = static_cast<double>(2 * gl + 2) / (M + 1);
  for (int it = 0; it < rounds; ++it) {
    const double x0 = fma(hi - lo, f0, lo), x1 = fma(hi - lo, f1, lo);
    int c0, c1;
    sturm2(W, n, x0, x1, c0, c1);
    double nlo = lo, nhi = hi;  // x0 < x1: new bracket [max x with c <= j, min x with c > j]
    if (c0 > j) {
      nhi = x0;
    } else if (c1 > j) {
      nlo = x0;
      nhi = x1;
    } else {
      nlo = x1;
    }
    for (int off = G >> 1; off > 0; off >>= 1) {  // reduce over the eigenvalue's G lanes
      nlo = fmax(nlo, __shfl_xor_sync(0xffffffffu, nlo, off));
      nhi = fmin(nhi, __shfl_xor_sync(0xffffffffu, nhi, off));
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
      W.pr[0][i] = l > 1e-15 ? l * log(l) : 0.0;  // spinmc.cpp:166-168
    }
    __syncwarp();
    if (tid == 0)
      for (int i = 0; i < n; ++i) e -= W.pr[0][i];  // ascending order, as the reference
  }
  return (e < 0.0) ? 0.0 : e;  // std::max(entropy, 0.0)
}

}  // namespace vn
}  // namespace tg
