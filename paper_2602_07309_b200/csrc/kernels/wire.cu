// /score wire ingest on the device: embedding_b64 items
// (service.cpp:361-370) decoded straight into the engine's soft-row buffer.
// Reference: base64_decode / decode_f32_base64 (base64.cpp:60-108): standard
// alphabet, '=' only in the last two positions of the last quantum, any
// other character invalid; little-endian float32 payload.
//
// One CTA per item, one thread per 4-character quantum (consecutive threads
// read consecutive 4-byte groups: coalesced; payloads may sit anywhere in a
// JSON body, so no alignment is assumed), three bytes out. Errors are reported as the smallest failing text position
// (atomicMin of position << 2 | kind) so the host raises the error the
// reference's sequential decoder would have hit first.
#include <cstdint>

#include "launch.h"

namespace srk {

namespace {

__device__ __forceinline__ int b64_val(unsigned c) {
  if (c >= 'A' && c <= 'Z') return static_cast<int>(c - 'A');
  if (c >= 'a' && c <= 'z') return static_cast<int>(c - 'a' + 26);
  if (c >= '0' && c <= '9') return static_cast<int>(c - '0' + 52);
  if (c == '+') return 62;
  if (c == '/') return 63;
  return -1;
}

__global__ void b64_decode_kernel(const uint8_t* __restrict__ text,
                                  const int64_t* __restrict__ char_begin,
                                  const int64_t* __restrict__ char_end,
                                  const int64_t* __restrict__ byte_off, uint8_t* __restrict__ out,
                                  unsigned long long* __restrict__ first_err) {
  pdl_wait();
  const int item = blockIdx.x;
  const int64_t s = char_begin[item], e = char_end[item];
  const int64_t q = (e - s) >> 2;
  uint8_t* dst = out != nullptr ? out + byte_off[item] : nullptr;
  for (int64_t i = threadIdx.x; i < q; i += blockDim.x) {
    const uint8_t* src = text + s + 4 * i;
    const uint32_t w = static_cast<uint32_t>(src[0]) | (static_cast<uint32_t>(src[1]) << 8) |
                       (static_cast<uint32_t>(src[2]) << 16) | (static_cast<uint32_t>(src[3]) << 24);
    const bool last = i + 1 == q;
    int vals[4];
    int pad = 0;
    unsigned long long err = ~0ull;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const unsigned c = (w >> (8 * j)) & 0xffu;
      // item-major error key: the reference decodes items in order
      const unsigned long long pos =
          (static_cast<unsigned long long>(item) << 40) | static_cast<unsigned long long>(4 * i + j);
      if (c == '=') {
        if (!last || j < 2) {
          if (err == ~0ull) err = (pos << 2) | 1u;  // misplaced base64 padding
        }
        vals[j] = 0;
        ++pad;
      } else {
        vals[j] = b64_val(c);
        if ((vals[j] < 0 || pad > 0) && err == ~0ull) err = (pos << 2) | 2u;  // invalid char
        if (vals[j] < 0) vals[j] = 0;
      }
    }
    if (err != ~0ull) atomicMin(first_err, err);
    if (dst != nullptr) {
      const uint32_t n = (vals[0] << 18) | (vals[1] << 12) | (vals[2] << 6) | vals[3];
      uint8_t* o = dst + 3 * i;
      o[0] = static_cast<uint8_t>((n >> 16) & 0xff);
      if (pad < 2) o[1] = static_cast<uint8_t>((n >> 8) & 0xff);
      if (pad < 1) o[2] = static_cast<uint8_t>(n & 0xff);
    }
  }
  pdl_trigger();
}

}  // namespace

cudaError_t b64_decode(const uint8_t* text, const int64_t* char_begin, const int64_t* char_end,
                       const int64_t* byte_off, int n_items, uint8_t* out,
                       unsigned long long* first_err, cudaStream_t stream) {
  if (n_items <= 0) return cudaSuccess;
  return launch_k(b64_decode_kernel, dim3(n_items), dim3(256), 0, stream, text, char_begin,
                  char_end, byte_off, out, first_err);
}

}  // namespace srk
