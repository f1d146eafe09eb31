// Do two cooperative launches on two streams of one process co-run? Each grid
// arrives on a shared counter and spins until both grids have arrived.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void arrive_spin(unsigned* cnt, unsigned total, int* ok) {
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(cnt, 1u);
    long long t0 = clock64();
    while (atomicAdd(cnt, 0u) < total) {
      __nanosleep(100);
      if (clock64() - t0 > (1ll << 33)) { *ok = 0; return; }  // ~4 s
    }
  }
}
int main() {
  unsigned* cnt; int* ok; cudaMalloc(&cnt, 4); cudaMalloc(&ok, 4);
  cudaStream_t s[4]; for (int i = 0; i < 4; ++i) cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mode = 0; mode < 2; ++mode)
    for (int P = 2; P <= 4; P += 2) {
      cudaMemset(cnt, 0, 4); int one = 1; cudaMemcpy(ok, &one, 4, cudaMemcpyHostToDevice);
      unsigned G = sms * 4 / P, total = G * P;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0, s[0]);
      for (int r = 0; r < P; ++r) {
        if (r) cudaStreamWaitEvent(s[r], e0, 0);
        void* args[] = {&cnt, &total, &ok};
        cudaError_t e = mode ? cudaLaunchCooperativeKernel((void*)arrive_spin, dim3(G), dim3(256), args, 0, s[r])
                             : cudaLaunchKernel((void*)arrive_spin, dim3(G), dim3(256), args, 0, s[r]);
        if (e != cudaSuccess) printf("launch err %s\n", cudaGetErrorString(e));
      }
      for (int r = 1; r < P; ++r) { cudaEventRecord(e1, s[r]); cudaStreamWaitEvent(s[0], e1, 0); }
      cudaEventRecord(e1, s[0]);
      cudaError_t e = cudaDeviceSynchronize();
      int h = 0; cudaMemcpy(&h, ok, 4, cudaMemcpyDeviceToHost);
      float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
      printf("%s P=%d G=%u per grid: %s (%s) %.3f ms\n", mode ? "cooperative" : "plain", P, G, h ? "CO-RAN" : "TIMEOUT",
             cudaGetErrorString(e), ms);
    }
  return 0;
}
