// numpy's reduction orders on the device, for results that must match the
// reference's numpy arithmetic bit for bit (umath loops_utils.h pairwise_sum).
#pragma once

namespace fo {

template <typename T>
__device__ T pairwise_leaf(const T* p, int n) {
  if (n < 8) {
    T res = T(0);
    for (int i = 0; i < n; ++i) res += p[i];
    return res;
  }
  T r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = p[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] += p[i + j];
  T res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += p[i];
  return res;
}

// blocks of <= 128 with eight accumulators, larger runs split at n/2 rounded
// down to a multiple of 8; DEPTH bounds the recursion (n <= 128 * 2^DEPTH)
template <int DEPTH, typename T>
__device__ T pairwise_sum(const T* a, int n) {
  if constexpr (DEPTH == 0) {
    return pairwise_leaf(a, n);
  } else {
    if (n <= 128) return pairwise_leaf(a, n);
    int n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_sum<DEPTH - 1>(a, n2) + pairwise_sum<DEPTH - 1>(a + n2, n - n2);
  }
}

}  // namespace fo
