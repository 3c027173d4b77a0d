// Zero-copy PCIe read micro-benchmark (pinned host memory read by a kernel):
//   * segment size per request (8 / 64 / 128 / 256 bytes at a row stride, like K2's quadrant rows)
//   * whether a second pass over the same bytes is served from L2 (no PCIe traffic)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 pciebench.cu -o pciebench
#include <cstdio>
#include <cstdint>
#include <sys/mman.h>
#include <cstdlib>
#include <cstring>

// each warp reads `seg` bytes at each of `rows` row starts (stride `stride` bytes): lanes read
// 4-byte words; grid-strided over `n_units` units of rows x seg bytes
__global__ void rd(const uint32_t *src, int64_t n_units, int rows, int seg, int64_t stride,
                   int64_t unit_stride, uint32_t *sink) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t acc = 0;
  const int words = seg / 4;
  for (int64_t u = wid; u < n_units; u += nw) {
    const char *base = reinterpret_cast<const char *>(src) + u * unit_stride;
    for (int r = 0; r < rows; r++)
      for (int w = lane; w < words; w += 32)
        acc += reinterpret_cast<const uint32_t *>(base + r * stride)[w];
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main(int argc, char **argv) {
  const size_t bytes = 256ull << 20;
  uint32_t *h, *d_sink;
  const bool thp = argc > 1 && !strcmp(argv[1], "thp");
  if (thp) {  // transparent huge pages, then pinned and mapped by cudaHostRegister
    void *m = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    int rc = madvise(m, bytes, MADV_HUGEPAGE);
    memset(m, 0, bytes);
    cudaError_t e = cudaHostRegister(m, bytes, cudaHostRegisterMapped);
    printf("THP: madvise rc=%d, cudaHostRegister %s\n", rc, cudaGetErrorString(e));
    h = (uint32_t *)m;
  } else {
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  }
  for (size_t i = 0; i < bytes / 4; i++) h[i] = (uint32_t)i;
  uint32_t *dh;
  cudaHostGetDevicePointer(&dh, h, 0);
  cudaMalloc(&d_sink, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char *name, int rows, int seg, int64_t stride, int grid) {
    const int64_t unit_stride = (int64_t)rows * stride;
    const int64_t n_units = (int64_t)(bytes / unit_stride) - 1;
    float best = 1e9;
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(a);
      rd<<<grid, 256>>>(dh, n_units, rows, seg, stride, unit_stride, d_sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    const double useful = (double)n_units * rows * seg;
    printf("%-34s %8.3f ms  %7.1f GB/s useful  %8.1f M req/s\n", name, best, useful / best / 1e6,
           (double)n_units * rows * (seg > 128 ? seg / 128 : 1) / best / 1e3);
  };
  // K2-like: 8 rows of 64 B at a 10816-byte row stride (1352 px x 8 B)
  run("8 rows x 64 B (targets), grid 148x8", 8, 64, 10816, 148 * 8);
  run("8 rows x 64 B (targets), grid 148x32", 8, 64, 10816, 148 * 32);
  run("8 rows x 8 B (valid), grid 148x32", 8, 8, 1352, 148 * 32);
  run("16 rows x 128 B (tile rows)", 16, 128, 10816, 148 * 32);
  run("16 rows x 256 B", 16, 256, 10816, 148 * 32);
  run("contiguous 4 KB units", 1, 4096, 4096, 148 * 32);
  // L2 reuse: a 32 MB region read by two launches back to back; the second pass is fast only
  // if the GPU L2 keeps the sysmem lines
  {
    const int64_t n_units = (32ll << 20) / 4096;
    for (int pass = 0; pass < 2; pass++) {
      cudaEventRecord(a);
      rd<<<148 * 32, 256>>>(dh, n_units, 1, 4096, 4096, 4096, d_sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("32 MB pass %d: %.3f ms (%.1f GB/s)\n", pass, ms, 32.0 * 1048576 / ms / 1e6);
    }
  }
  // half lines: 64 B at a 128-B stride (the sibling half is never read)
  run("64 B at 128-B stride", 1, 64, 128, 148 * 32);
  run("128 B at 128-B stride", 1, 128, 128, 148 * 32);
  return 0;
}
