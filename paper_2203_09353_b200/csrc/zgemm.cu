// zgemm.cu — fixed-size batched complex GEMM on DMMA.8x8x4: the device side of the GEMM
// batcher (VirtualDevice::batched_gemm, exec.cpp:144-221; per-entry math linalg.cpp:79-113:
// out = alpha*A*B + beta*C, column-major interleaved complex128).
//
// grid = (tiles_m * tiles_n, batch); each CTA computes one 64x64 output tile of one batch
// entry with 8 warps (16x32 sub-tile each, 2x4 blocks). K streams in chunks of 32 through
// SMEM, de-interleaved into planar Re/Im tiles (A as [k][i], B transposed as [k][j], pitch
// 68 doubles: conflict-free fragments). Complex product by real split:
//   Re = Ar Br - Ai Bi,  Im = Ar Bi + Ai Br   (4 DMMA per block per k-chunk of 4).
// Edges (m, n, k not multiples of the tile) are zero-padded in SMEM.
#include "smem_tier.cuh"
#include "tg_internal.h"

namespace tg {
namespace {

constexpr int ZT = 64, ZK = 32, ZP = ZT + 4;
constexpr int ZThreads = 256;

__global__ void __launch_bounds__(ZThreads, 1)
    zgemm_kernel(int m, int n, int k, double ar, double ai, const double* __restrict__ A,
                 int64_t sA, const double* __restrict__ B, int64_t sB, double br, double bi,
                 const double* __restrict__ C, int64_t sC, double* __restrict__ out, int64_t sO,
                 int fault) {
  extern __shared__ __align__(16) double zsm[];
  double *sAr = zsm, *sAi = zsm + ZK * ZP, *sBr = zsm + 2 * ZK * ZP, *sBi = zsm + 3 * ZK * ZP;
  const int tiles_n = (n + ZT - 1) / ZT;
  const int i0 = (blockIdx.x / tiles_n) * ZT, j0 = (blockIdx.x % tiles_n) * ZT;
  const size_t e = blockIdx.y;
  const double* a = A + 2 * sA * e;
  const double* b = B + 2 * sB * e;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wr = warp >> 1, wc = warp & 1;  // warp grid 4 x 2
  const int mm = lane >> 2, kq = lane & 3;
  double cr[2][4][2], ci[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;

  for (int k0 = 0; k0 < k; k0 += ZK) {
    // A tile: rows i0..i0+63, cols k0..k0+31 -> sA*[kk][ii]
    for (int c = tid; c < ZT * ZK; c += ZThreads) {
      const int ii = c % ZT, kk = c / ZT;
      const int gi = i0 + ii, gk = k0 + kk;
      double vr = 0.0, vi = 0.0;
      if (gi < m && gk < k) {
        const double2 v = *reinterpret_cast<const double2*>(a + 2 * (gi + static_cast<size_t>(gk) * m));
        vr = v.x;
        vi = v.y;
      }
      sAr[kk * ZP + ii] = vr;
      sAi[kk * ZP + ii] = vi;
    }
    // B tile: rows k0..k0+31, cols j0..j0+63 -> sB*[kk][jj]
    for (int c = tid; c < ZT * ZK; c += ZThreads) {
      const int kk = c % ZK, jj = c / ZK;
      const int gk = k0 + kk, gj = j0 + jj;
      double vr = 0.0, vi = 0.0;
      if (gk < k && gj < n) {
        const double2 v = *reinterpret_cast<const double2*>(b + 2 * (gk + static_cast<size_t>(gj) * k));
        vr = v.x;
        vi = v.y;
      }
      sBr[kk * ZP + jj] = vr;
      sBi[kk * ZP + jj] = vi;
    }
    __syncthreads();
#pragma unroll
    for (int kb = 0; kb < ZK; kb += 4) {
      const int col = (kb + kq) * ZP;
      double xa[2], ya[2], yn[2], xb[4], yb[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int row = (wr * 2 + i) * 8 + mm;
        xa[i] = sAr[row + col];
        ya[i] = sAi[row + col];
        yn[i] = -ya[i];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int cc = (wc * 4 + j) * 8 + mm;
        xb[j] = sBr[cc + col];
        yb[j] = sBi[cc + col];
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dmma(cr[i][j][0], cr[i][j][1], xa[i], xb[j]);
          dmma(cr[i][j][0], cr[i][j][1], yn[i], yb[j]);
          dmma(ci[i][j][0], ci[i][j][1], xa[i], yb[j]);
          dmma(ci[i][j][0], ci[i][j][1], ya[i], xb[j]);
        }
    }
    __syncthreads();
  }
  // fault hook (linalg.cpp:94): sign of the first term of element (0,0) flipped
  if (fault && i0 == 0 && j0 == 0 && wr == 0 && wc == 0 && lane == 0) {
    const double2 a00 = *reinterpret_cast<const double2*>(a);
    const double2 b00 = *reinterpret_cast<const double2*>(b);
    const double tr = __dsub_rn(__dmul_rn(a00.x, b00.x), __dmul_rn(a00.y, b00.y));
    cr[0][0][0] -= 2.0 * tr;
  }
  // epilogue (linalg.cpp:98-101): out = alpha*sum + beta*C, reference operation order
  const double* c = C ? C + 2 * sC * e : nullptr;
  double* o = out + 2 * sO * e;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gi = i0 + (wr * 2 + i) * 8 + mm;
        const int gj = j0 + (wc * 4 + j) * 8 + 2 * kq + h;
        if (gi < m && gj < n) {
          const size_t idx = gi + static_cast<size_t>(gj) * m;
          double cvr = 0.0, cvi = 0.0;
          if (c) {
            const double2 v = *reinterpret_cast<const double2*>(c + 2 * idx);
            cvr = v.x;
            cvi = v.y;
          }
          const double sr = cr[i][j][h], si = ci[i][j][h];
          const double re = __dsub_rn(__dadd_rn(__dsub_rn(__dmul_rn(ar, sr), __dmul_rn(ai, si)),
                                                __dmul_rn(br, cvr)),
                                      __dmul_rn(bi, cvi));
          const double im = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(ar, si), __dmul_rn(ai, sr)),
                                                __dmul_rn(br, cvi)),
                                      __dmul_rn(bi, cvr));
          *reinterpret_cast<double2*>(o + 2 * idx) = make_double2(re, im);
        }
      }
}

}  // namespace

cudaError_t launch_zgemm_strided(int batch, int m, int n, int k, double ar, double ai,
                                 const double* A, int64_t sA, const double* B, int64_t sB,
                                 double br, double bi, const double* C, int64_t sC, double* out,
                                 int64_t sO, int inject_fault, cudaStream_t stream) {
  if (batch < 1 || m < 1 || n < 1 || k < 1) return cudaErrorInvalidValue;
  const int tiles = ((m + ZT - 1) / ZT) * ((n + ZT - 1) / ZT);
  dim3 grid(tiles, batch);
  constexpr int bytes = 4 * ZK * ZP * 8;
  cudaError_t e = cudaFuncSetAttribute(zgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  zgemm_kernel<<<grid, ZThreads, bytes, stream>>>(m, n, k, ar, ai, A, sA, B, sB, br, bi, C, sC, out,
                                              sO, inject_fault);
  return cudaGetLastError();
}

}  // namespace tg
