// vn_packed.cuh — von Neumann entropy -sum lambda ln lambda (spinmc.cpp:165-169) for
// 64 < n = d_a <= 128 (S = 14, 15): the HBM tier's GEMM leaves rho in a global scratch
// (its 64x64 tiles are written as they finish), and the Hermitian part is rebuilt in the
// drained stage buffers as a PACKED LOWER triangle, column-major:
//     A(i, j), i >= j, at cs(j) + i,   cs(j) = j*n - j(j+1)/2
// (n(n+1)/2 complex = 132 KB at n = 128; full storage, 256 KB, does not fit in SMEM).
// The method is vn.cuh's (same steps, same numerics): Householder tridiagonalisation with
// two CTA barriers per reflector (warp 0 builds reflector k+1 while warps 1..7 finish the
// rank-2 update of reflector k), then vn::eigenvalues (Sturm multisection, 2 threads per
// eigenvalue at n = 128) and the ascending-order entropy sum. On packed storage the
// update touches only the lower triangle (half the work of full storage); B v reads row r
// as A(r, c) for c <= r (strided) and conj(A(c, r)) for c > r (column r, contiguous).
#pragma once
#include "vn.cuh"

namespace tg {
namespace vnp {

constexpr int kMaxN = 128;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

struct Scratch {
  double vr[2][kMaxN], vi[2][kMaxN];  // Householder vector v (double-buffered by k&1)
  double pr[2][kMaxN], pi[2][kMaxN];  // B v (double-buffered)
  double part[2][kWarps];             // per-warp partials of Re(v^H B v)
  double tau[2];
  double d[kMaxN], e2[kMaxN];         // tridiagonal: diagonal, |off-diagonal|^2
  double lam[kMaxN];                  // eigenvalues, ascending
  double lo, hi;
};

__host__ __device__ constexpr int packed_size(int n) { return n * (n + 1) / 2; }
__device__ __forceinline__ int cs(int j, int n) { return j * n - ((j * (j + 1)) >> 1); }

// Hermitian part (linalg.cpp:179-185) of the full column-major rho (global, planes Rr/Ri,
// pitch n) into packed lower storage: W(i,j) = (rho(i,j) + conj(rho(j,i)))/2, W(i,i) real.
__device__ __forceinline__ void build(const double* Rr, const double* Ri, double* Ar, double* Ai, int n,
                                      int tid) {
  const int warp = tid >> 5, lane = tid & 31;
  for (int j = warp; j < n; j += kWarps) {
    const int c = cs(j, n);
    for (int i = j + lane; i < n; i += 32) {
      if (i == j) {
        Ar[c + i] = __ldcg(Rr + i + i * n);
        Ai[c + i] = 0.0;
      } else {
        Ar[c + i] = 0.5 * (__ldcg(Rr + i + j * n) + __ldcg(Rr + j + i * n));
        Ai[c + i] = 0.5 * (__ldcg(Ri + i + j * n) - __ldcg(Ri + j + i * n));
      }
    }
  }
}

// Warp 0: reflector of column k (rows k+1..n-1), as vn::reflector (4 rows per lane).
__device__ __forceinline__ void reflector(const double* Ar, const double* Ai, int n, int k, Scratch& W,
                                          int lane) {
  const int m = n - k - 1, c0 = cs(k, n) + k + 1, b = k & 1;
  double xr[4], xi[4], s = 0.0;
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const int i = lane + 32 * h;
    xr[h] = xi[h] = 0.0;
    if (i < m) {
      xr[h] = Ar[c0 + i];
      xi[h] = Ai[c0 + i];
    }
    if (i > 0) s += fma(xr[h], xr[h], xi[h] * xi[h]);
  }
  s = warp_sum(s);
  const double a0r = __shfl_sync(0xffffffffu, xr[0], 0), a0i = __shfl_sync(0xffffffffu, xi[0], 0);
  const double ax2 = fma(a0r, a0r, a0i * a0i);
  if (s > 0.0) {
    const double inv0 = ax2 > 0.0 ? rsqrt(ax2) : 0.0;  // 1/|x0|
    const double ax0 = ax2 * inv0, xx = ax2 + s, xnorm = sqrt(xx), mag = ax0 + xnorm;
    const double phr = ax2 > 0.0 ? a0r * inv0 : 1.0, phi = a0i * inv0;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int i = lane + 32 * h;
      if (i < m) {
        W.vr[b][i] = i == 0 ? phr * mag : xr[h];
        W.vi[b][i] = i == 0 ? phi * mag : xi[h];
      }
    }
    if (lane == 0) {
      W.tau[b] = 1.0 / (xnorm * mag);
      W.e2[k] = xx;
    }
  } else {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int i = lane + 32 * h;
      if (i < m) W.vr[b][i] = W.vi[b][i] = 0.0;
    }
    if (lane == 0) {
      W.tau[b] = 0.0;
      W.e2[k] = ax2;
    }
  }
  if (lane == 0) W.d[k] = Ar[cs(k, n) + k];
}

// Rank-2 update of the trailing lower triangle with reflector k: A(i,j) -= v_i conj(w_j) +
// w_i conj(v_j) for i >= j, w = tau B v - K v, K = tau^2/2 Re(v^H B v). Warp 0 takes the
// first column (it feeds reflector k+1), warps 1..7 the rest, two columns per group with
// all loads issued before the stores.
__device__ __forceinline__ void update(double* Ar, double* Ai, int n, int k, const Scratch& W, int warp,
                                       int lane) {
  const int m = n - k - 1, o = k + 1, b = k & 1;
  const double tau = W.tau[b];
  double vhbv = 0.0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) vhbv += W.part[b][w];
  const double K = 0.5 * tau * tau * vhbv;
  double vr[4], vi[4], wr[4], wi[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const int i = lane + 32 * h;
    vr[h] = vi[h] = wr[h] = wi[h] = 0.0;
    if (i < m) {
      vr[h] = W.vr[b][i];
      vi[h] = W.vi[b][i];
      wr[h] = fma(tau, W.pr[b][i], -K * vr[h]);
      wi[h] = fma(tau, W.pi[b][i], -K * vi[h]);
    }
  }
  auto cols = [&](int j0, int nc) {  // columns j0, j0 + (kWarps-1) of the trailing block
    double ar[2][4], ai[2][4], wjr[2], wji[2], vjr[2], vji[2];
    int idx[2][4];
    bool ok[2][4];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int jj = j0 + c * (kWarps - 1);
      const bool cv = c < nc;
      const int j = cv ? jj : j0;
      vjr[c] = W.vr[b][j];
      vji[c] = W.vi[b][j];
      wjr[c] = fma(tau, W.pr[b][j], -K * vjr[c]);
      wji[c] = fma(tau, W.pi[b][j], -K * vji[c]);
      const int base = cs(o + j, n) + o;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int i = lane + 32 * h;
        ok[c][h] = cv && i >= j && i < m;
        idx[c][h] = ok[c][h] ? base + i : 0;
        ar[c][h] = Ar[idx[c][h]];
        ai[c][h] = Ai[idx[c][h]];
      }
    }
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        ar[c][h] = fma(-vr[h], wjr[c], fma(-vi[h], wji[c], fma(-wr[h], vjr[c], fma(-wi[h], vji[c], ar[c][h]))));
        ai[c][h] = fma(-vi[h], wjr[c], fma(vr[h], wji[c], fma(-wi[h], vjr[c], fma(wr[h], vji[c], ai[c][h]))));
      }
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int h = 0; h < 4; ++h)
        if (ok[c][h]) {
          Ar[idx[c][h]] = ar[c][h];
          Ai[idx[c][h]] = ai[c][h];
        }
  };
  if (warp == 0) {
    cols(0, 1);
  } else {
    for (int j = warp; j < m; j += 2 * (kWarps - 1)) cols(j, j + (kWarps - 1) < m ? 2 : 1);
  }
}

// B v for reflector k (trailing block, rows/cols k+1..n-1): 4 lanes per row, rows
// 8w + lane/4 and 64 + 8w + lane/4; row r reads A(r, c) for c <= r (B(r,c) = A(r,c)) and
// conj(A(c, r)) for c > r. Also the warp's partial of Re(v^H B v).
__device__ __forceinline__ void matvec(const double* Ar, const double* Ai, int n, int k, Scratch& W, int warp,
                                       int lane) {
  const int m = n - k - 1, o = k + 1, b = k & 1, g = lane & 3;
  double part = 0.0;
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
    const int rr = 64 * pass + 8 * warp + (lane >> 2);
    double ar[4] = {0.0, 0.0, 0.0, 0.0}, ai[4] = {0.0, 0.0, 0.0, 0.0};
    if (rr < m) {
      const int r = o + rr;
      const int colr = cs(r, n);  // column r: A(c, r) at colr + c
      for (int c0 = g; c0 < m; c0 += 16) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {  // chain t
          const int cc = c0 + 4 * t;
          if (cc < m) {
            const int c = o + cc;
            const bool low = cc <= rr;
            const int ix = low ? cs(c, n) + r : colr + c;
            const double br = Ar[ix], bi0 = Ai[ix];
            const double bi = low ? -bi0 : bi0;  // -Im B(r,c)
            const double vr = W.vr[b][cc], vi = W.vi[b][cc];
            ar[t] = fma(br, vr, fma(bi, vi, ar[t]));
            ai[t] = fma(br, vi, fma(-bi, vr, ai[t]));
          }
        }
      }
    }
    double sr = (ar[0] + ar[1]) + (ar[2] + ar[3]), si = (ai[0] + ai[1]) + (ai[2] + ai[3]);
    sr += __shfl_xor_sync(0xffffffffu, sr, 1);
    si += __shfl_xor_sync(0xffffffffu, si, 1);
    sr += __shfl_xor_sync(0xffffffffu, sr, 2);
    si += __shfl_xor_sync(0xffffffffu, si, 2);
    if (g == 0 && rr < m) {
      W.pr[b][rr] = sr;
      W.pi[b][rr] = si;
      part = fma(W.vr[b][rr], sr, fma(W.vi[b][rr], si, part));
    }
  }
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
  if (lane == 0) W.part[b][warp] = part;
}

// Householder reduction; on return W.d[0..n), W.e2[0..n-1) hold the tridiagonal.
template <class Sync>
__device__ void tridiagonalize(double* Ar, double* Ai, int n, Scratch& W, int tid, Sync sync) {
  const int warp = tid >> 5, lane = tid & 31;
  for (int k = 0; k + 2 < n; ++k) {
    if (k > 0) update(Ar, Ai, n, k - 1, W, warp, lane);
    if (warp == 0) {
      __syncwarp();
      reflector(Ar, Ai, n, k, W, lane);
    }
    sync();
    matvec(Ar, Ai, n, k, W, warp, lane);
    sync();
  }
  if (n >= 3) {
    update(Ar, Ai, n, n - 3, W, warp, lane);
    sync();
  }
  if (tid == 0) {
    const int a = n - 2, c = n - 1;
    W.d[a] = Ar[cs(a, n) + a];
    W.d[c] = Ar[cs(c, n) + c];
    const double er = Ar[cs(a, n) + c], ei = Ai[cs(a, n) + c];
    W.e2[a] = fma(er, er, ei * ei);
  }
  sync();
}

// Entropy of the packed Hermitian part (all kThreads threads; valid in thread 0).
template <class Sync>
__device__ double entropy(double* Ar, double* Ai, int n, Scratch& W, int tid, Sync sync) {
  tridiagonalize(Ar, Ai, n, W, tid, sync);
  vn::eigenvalues(n, W, tid, sync);
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

}  // namespace vnp
}  // namespace tg
