// prims.cu -- the device-wide primitives of prims.cuh behind the C ABI, so
// the parity tests can check them on their own against numpy (stable
// argsort, cumulative max, flatnonzero) besides their end-to-end use in the
// presort, the epilogue and the time-split pipeline.
#include "../../include/hull3d_b200.h"
#include "h3d_host.h"
#include "prims.cuh"

using namespace h3d;

extern "C" {

size_t h3d_prim_temp_bytes(int64_t n) {
  size_t m = prim::rs_temp_bytes<unsigned long long>(n);
  const size_t a = prim::rs_temp_bytes<unsigned>(n), b = prim::scan_temp_bytes<long long>(n),
               c = prim::select_temp_bytes(n);
  if (a > m) m = a;
  if (b > m) m = b;
  return m > c ? m : c;
}

int64_t h3d_radix_sort_pairs(void *keys, void *keys_alt, int32_t *vals, int32_t *vals_alt, int64_t n,
                             int32_t key_bytes, int32_t begin_bit, int32_t end_bit, int32_t iota_vals,
                             void *tmp, size_t tmp_bytes, void *stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n < 0 || begin_bit < 0 || end_bit > 8 * key_bytes || (key_bytes != 4 && key_bytes != 8))
    return H3D_E_ARG;
  bool alt = false;
  cudaError_t e;
  h3d_count_launches(1 + (end_bit - begin_bit + 7) / 8);
  if (key_bytes == 4)
    e = prim::rs_sort_pairs<unsigned>(tmp, tmp_bytes, static_cast<unsigned *>(keys), vals,
                                      static_cast<unsigned *>(keys_alt), vals_alt, n, begin_bit, end_bit, &alt,
                                      s, iota_vals != 0);
  else
    e = prim::rs_sort_pairs<unsigned long long>(tmp, tmp_bytes, static_cast<unsigned long long *>(keys), vals,
                                                static_cast<unsigned long long *>(keys_alt), vals_alt, n,
                                                begin_bit, end_bit, &alt, s, iota_vals != 0);
  if (h3d_check(e)) return H3D_E_CUDA;
  return alt ? 1 : 0;
}

int64_t h3d_scan_i64(const int64_t *in, int64_t *out, int64_t n, int32_t op_max, int32_t exclusive,
                     void *tmp, size_t tmp_bytes, void *stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long *a = reinterpret_cast<const long long *>(in);
  long long *b = reinterpret_cast<long long *>(out);
  const long long lo = static_cast<long long>(1ull << 63);
  cudaError_t e;
  h3d_count_launches(3);
  if (op_max)
    e = exclusive ? prim::scan<true, long long>(tmp, tmp_bytes, a, b, n, prim::OpMax(), lo, lo, s)
                  : prim::scan<false, long long>(tmp, tmp_bytes, a, b, n, prim::OpMax(), lo, lo, s);
  else
    e = exclusive ? prim::scan<true, long long>(tmp, tmp_bytes, a, b, n, prim::OpSum(), 0ll, 0ll, s)
                  : prim::scan<false, long long>(tmp, tmp_bytes, a, b, n, prim::OpSum(), 0ll, 0ll, s);
  return h3d_check(e) ? H3D_E_CUDA : 0;
}

int64_t h3d_select_flagged(const int32_t *flags, int64_t n, int64_t *out, int64_t *count_dev, void *tmp,
                           size_t tmp_bytes, void *stream) {
  h3d_count_launches(3);
  return h3d_check(prim::select_flagged(tmp, tmp_bytes, flags, n, reinterpret_cast<long long *>(out),
                                        reinterpret_cast<long long *>(count_dev),
                                        static_cast<cudaStream_t>(stream)))
             ? H3D_E_CUDA
             : 0;
}

}  // extern "C"
