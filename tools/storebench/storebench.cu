// Write-pattern micro-benchmark for the SoA outputs of K3 (motions: 73 B per gv in 7 arrays) and
// K1 (64 B records + side arrays):  nvcc -gencode arch=compute_100a,code=sm_100a -O3 storebench.cu
#include <cstdio>
#include <cstdint>

struct M { int8_t *st; double *a, *b, *w, *sw; int32_t *c, *sc; };

__global__ void soa(M m, int64_t n) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  m.st[g] = 2;
  reinterpret_cast<double2 *>(m.a)[2 * g] = make_double2(1.0, 0.0);
  reinterpret_cast<double2 *>(m.a)[2 * g + 1] = make_double2(0.0, 1.0);
  reinterpret_cast<double2 *>(m.b)[g] = make_double2(0.0, 0.0);
  m.w[g] = 0.0; m.c[g] = 0; m.sc[g] = 0; m.sw[g] = 0.0;
}
__global__ void soa_cs(M m, int64_t n) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  __stcs(m.st + g, (int8_t)2);
  __stcs(reinterpret_cast<double2 *>(m.a) + 2 * g, make_double2(1.0, 0.0));
  __stcs(reinterpret_cast<double2 *>(m.a) + 2 * g + 1, make_double2(0.0, 1.0));
  __stcs(reinterpret_cast<double2 *>(m.b) + g, make_double2(0.0, 0.0));
  __stcs(m.w + g, 0.0); __stcs(m.c + g, 0); __stcs(m.sc + g, 0); __stcs(m.sw + g, 0.0);
}
// grid-stride, 4 gvs per thread per iteration (more stores in flight per thread)
__global__ void soa_gs(M m, int64_t n) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x) {
    m.st[g] = 2;
    reinterpret_cast<double2 *>(m.a)[2 * g] = make_double2(1.0, 0.0);
    reinterpret_cast<double2 *>(m.a)[2 * g + 1] = make_double2(0.0, 1.0);
    reinterpret_cast<double2 *>(m.b)[g] = make_double2(0.0, 0.0);
    m.w[g] = 0.0; m.c[g] = 0; m.sc[g] = 0; m.sw[g] = 0.0;
  }
}
__global__ void copy_ref(const double4 *x, double4 *y, int64_t n4) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n4) y[i] = x[i];
}
__global__ void fill_ref(double4 *y, int64_t n4) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n4) y[i] = make_double4(0, 0, 0, 0);
}

int main() {
  const int64_t n = 48000000;
  M m;
  cudaMalloc(&m.st, n); cudaMalloc(&m.a, 32 * n); cudaMalloc(&m.b, 16 * n);
  cudaMalloc(&m.w, 8 * n); cudaMalloc(&m.sw, 8 * n); cudaMalloc(&m.c, 4 * n); cudaMalloc(&m.sc, 4 * n);
  double4 *x, *y; const int64_t n4 = 73 * n / 32;
  cudaMalloc(&x, 32 * n4); cudaMalloc(&y, 32 * n4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto t = [&](const char *name, auto launch, double bytes) {
    float best = 1e9;
    for (int r = 0; r < 5; r++) {
      cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (r) best = ms < best ? ms : best;
    }
    printf("%-28s %.3f ms  %.0f GB/s\n", name, best, bytes / best / 1e6);
  };
  const unsigned g256 = (unsigned)((n + 255) / 256);
  t("soa 7 arrays", [&] { soa<<<g256, 256>>>(m, n); }, 73.0 * n);
  t("soa 7 arrays .cs", [&] { soa_cs<<<g256, 256>>>(m, n); }, 73.0 * n);
  t("soa grid-stride 148x16", [&] { soa_gs<<<148 * 16, 256>>>(m, n); }, 73.0 * n);
  t("fill 73n bytes double4", [&] { fill_ref<<<(unsigned)((n4 + 255) / 256), 256>>>(y, n4); }, 32.0 * n4);
  t("copy 73n bytes double4", [&] { copy_ref<<<(unsigned)((n4 + 255) / 256), 256>>>(x, y, n4); }, 64.0 * n4);
  return 0;
}
