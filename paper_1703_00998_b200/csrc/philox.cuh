// Counter-based Philox4x32-10 (Salmon et al., SC'11) and the Box-Muller map
// that produce G at each randUTV step (PAPER.md:941 ``G = randn(m-b(i-1), b)``).
// Stream layout = DESIGN.md reading R2:
//   key = (lo32(seed), hi32(seed)), counter = (row/2, column, step, purpose)
//   u  = (2*((x1:x0) >> 12) + 1) 2^-53,  u' = (2*((x3:x2) >> 12) + 1) 2^-53
//   G[2p] = sqrt(-2 ln u) cos(2 pi u'),  G[2p+1] = sqrt(-2 ln u) sin(2 pi u')
#pragma once
#include <cstdint>

namespace rutv {

__device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0,
                                             uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
  uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
  uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
  c0 = n0;
  c1 = lo1;
  c2 = n2;
  c3 = lo0;
}

__device__ __forceinline__ void philox4x32_10(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0,
                                              uint32_t k1) {
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += W0;
      k1 += W1;
    }
    philox_round(c0, c1, c2, c3, k0, k1);
  }
}

__device__ __forceinline__ void philox_gaussian_pair(uint32_t pair, uint32_t col, uint32_t step, uint32_t purpose,
                                                     uint32_t k0, uint32_t k1, double& g0, double& g1) {
  uint32_t c0 = pair, c1 = col, c2 = step, c3 = purpose;
  philox4x32_10(c0, c1, c2, c3, k0, k1);
  uint64_t w01 = (uint64_t(c1) << 32) | c0;
  uint64_t w23 = (uint64_t(c3) << 32) | c2;
  double u = (2.0 * double(w01 >> 12) + 1.0) * 0x1p-53;
  double u2 = (2.0 * double(w23 >> 12) + 1.0) * 0x1p-53;
  double rho = sqrt(-2.0 * log(u));
  double theta = (2.0 * 3.141592653589793) * u2;
  double s, c;
  sincos(theta, &s, &c);
  g0 = rho * c;
  g1 = rho * s;
}

}  // namespace rutv
