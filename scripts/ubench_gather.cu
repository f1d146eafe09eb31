// ubench_gather.cu — hardware ceilings for the BFS hot loop's access pattern on B200:
// a streamed index array (like cadj) driving random 4-byte gathers / atomics /
// stores into a table (like rmatch / pred). Prints G accesses/s per variant.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_gather scripts/ubench_gather.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void k_gather(const int* __restrict__ idx, long long n, const int* tab, int* out, int items) {
  long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, tot = (long long)gridDim.x * blockDim.x;
  int acc = 0;
  for (long long base = tid; base < n; base += tot * items) {
    int v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) if (k < items) { long long e = base + k * tot; v[k] = e < n ? __ldcs(idx + e) : -1; }
#pragma unroll
    for (int k = 0; k < 16; ++k) if (k < items && v[k] >= 0) acc += __ldcg(tab + v[k]);
  }
  if (acc == 0x7fffffff) out[0] = acc;
}
__global__ void k_atomic(const int* __restrict__ idx, long long n, int* tab, int* out, int items) {
  long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, tot = (long long)gridDim.x * blockDim.x;
  int acc = 0;
  for (long long base = tid; base < n; base += tot * items) {
    int v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) if (k < items) { long long e = base + k * tot; v[k] = e < n ? __ldcs(idx + e) : -1; }
#pragma unroll
    for (int k = 0; k < 16; ++k) if (k < items && v[k] >= 0) acc += atomicOr(tab + v[k], 1 << 30);
  }
  if (acc == 0x7fffffff) out[0] = acc;
}
__global__ void k_store(const int* __restrict__ idx, long long n, int* tab, int items) {
  long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, tot = (long long)gridDim.x * blockDim.x;
  for (long long base = tid; base < n; base += tot * items) {
#pragma unroll
    for (int k = 0; k < 16; ++k) if (k < items) { long long e = base + k * tot; if (e < n) { int v = __ldcs(idx + e); tab[v] = (int)e; } }
  }
}
__global__ void k_claim(const int* __restrict__ idx, long long n, int* tab, int items) {
  // the push claim: gather a row's word, store it back with the visited bit when it was clear
  long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, tot = (long long)gridDim.x * blockDim.x;
  for (long long base = tid; base < n; base += tot * items) {
    int v[16], w[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) if (k < items) { long long e = base + k * tot; v[k] = e < n ? __ldcs(idx + e) : -1; }
#pragma unroll
    for (int k = 0; k < 16; ++k) if (k < items && v[k] >= 0) w[k] = __ldcg(tab + v[k]);
#pragma unroll
    for (int k = 0; k < 16; ++k) if (k < items && v[k] >= 0 && !(w[k] & (1 << 30))) tab[v[k]] = w[k] | (1 << 30);
  }
}
__global__ void k_gather2(const int* __restrict__ idx, long long n, const int* tab, int* out, int items) {
  // dependent: gather then gather again at the value (like rmatch -> offs)
  long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, tot = (long long)gridDim.x * blockDim.x;
  int acc = 0;
  for (long long base = tid; base < n; base += tot * items) {
    int v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) if (k < items) { long long e = base + k * tot; v[k] = e < n ? __ldcs(idx + e) : -1; }
#pragma unroll
    for (int k = 0; k < 16; ++k) if (k < items && v[k] >= 0) v[k] = __ldcg(tab + v[k]);
#pragma unroll
    for (int k = 0; k < 16; ++k) if (k < items && v[k] >= 0) acc += __ldcg(tab + (v[k] & 0x3fffffff));
  }
  if (acc == 0x7fffffff) out[0] = acc;
}

int main() {
  const long long n = 160000000;  // edges
  int* idx; int* tab; int* out;
  cudaMalloc(&idx, n * 4); cudaMalloc(&out, 64);
  const long long tabmax = 200000000;  // up to 800 MB: the C5 row state (interleaved {mate, pred})
  cudaMalloc(&tab, tabmax * 4);
  std::vector<int> h(n);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  FILE* js = fopen("gpurun_out/ubench_gather.jsonl", "w");
  for (long long T : {10000000LL, 100000000LL, 200000000LL}) {
    uint64_t s = 12345;
    for (long long i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (int)(s % T); }
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    for (int items : {1, 4, 8, 16}) {
      for (int blocks_per_sm : {4, 8}) {
        const int grid = sms * blocks_per_sm, thr = 256;
        for (int kind = 0; kind < 5; ++kind) {
          cudaMemset(tab, 0, T * 4);
          float best = 1e9;
          for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            if (kind == 0) k_gather<<<grid, thr>>>(idx, n, tab, out, items);
            if (kind == 1) k_atomic<<<grid, thr>>>(idx, n, tab, out, items);
            if (kind == 2) k_store<<<grid, thr>>>(idx, n, tab, items);
            if (kind == 3) k_gather2<<<grid, thr>>>(idx, n, tab, out, items);
            if (kind == 4) k_claim<<<grid, thr>>>(idx, n, tab, items);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
          }
          const char* names[] = {"gather", "atomicOr", "store", "gather2dep", "claim"};
          printf("table %5lld MB items %2d bpsm %d %-10s %8.3f ms  %7.1f G/s\n", T * 4 >> 20, items, blocks_per_sm,
                 names[kind], best, n / best / 1e6);
          if (js) fprintf(js, "{\"table_mb\": %lld, \"items\": %d, \"blocks_per_sm\": %d, \"kind\": \"%s\", \"ms\": %.4f, \"gps\": %.2f}\n",
                          T * 4 >> 20, items, blocks_per_sm, names[kind], best, n / best / 1e6);
        }
      }
    }
  }
  if (js) fclose(js);
  cudaError_t e = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(e));
  return 0;
}
