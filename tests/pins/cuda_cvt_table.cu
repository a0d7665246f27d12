// tests/pins/cuda_cvt_table.cu -- host-only pin for the oracle's element encoder.
//
// Writes, for every one of the 65536 BF16 bit patterns taken as the (already
// scaled) input value, the code CUDA's own host conversion routines produce with
// round-to-nearest-even and saturation to the finite range:
//   __nv_cvt_double_to_fp4(x, __NV_E2M1, cudaRoundNearest)
//   __nv_cvt_double_to_fp6(x, __NV_E3M2 / __NV_E2M3, cudaRoundNearest)
//   __nv_cvt_double_to_fp8(x, __NV_SATFINITE, __NV_E4M3 / __NV_E5M2)
// Output: 5 x 65536 bytes (format order E2M1, E3M2, E2M3, E4M3, E5M2) to argv[1].
// The oracle's brute-force nearest-code rule must agree on every finite input
// (tests/test_oracle_formats.py).  Compiled with nvcc as host code; no GPU used.
#include <cuda_fp4.h>
#include <cuda_fp6.h>
#include <cuda_fp8.h>
#include <cstdint>
#include <cstdio>
#include <cstring>

static double bf16_bits_to_double(uint16_t b) {
  uint32_t u = uint32_t(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return double(f);
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  FILE* fp = std::fopen(argv[1], "wb");
  if (!fp) return 3;
  static uint8_t out[5][65536];
  for (uint32_t b = 0; b < 65536; ++b) {
    double x = bf16_bits_to_double(uint16_t(b));
    out[0][b] = uint8_t(__nv_cvt_double_to_fp4(x, __NV_E2M1, cudaRoundNearest));
    out[1][b] = uint8_t(__nv_cvt_double_to_fp6(x, __NV_E3M2, cudaRoundNearest));
    out[2][b] = uint8_t(__nv_cvt_double_to_fp6(x, __NV_E2M3, cudaRoundNearest));
    out[3][b] = uint8_t(__nv_cvt_double_to_fp8(x, __NV_SATFINITE, __NV_E4M3));
    out[4][b] = uint8_t(__nv_cvt_double_to_fp8(x, __NV_SATFINITE, __NV_E5M2));
  }
  std::fwrite(out, 1, sizeof(out), fp);
  std::fclose(fp);
  return 0;
}
