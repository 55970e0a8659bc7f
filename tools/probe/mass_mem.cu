// Memory-pattern probe for k_mass (the atomic step's mass pass): the same
// per-mass loads / stores over 1 M masses, variants timed with CUDA events.
#include <cstdio>
#include <cuda_runtime.h>
struct B { float4 *pos0, *pos1, *vel, *fext; float2 *plo0, *plo1; float *pm, *acc; };
__global__ void k_copyish(B b, int n) {  // v0: all loads, simple update, all stores
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float4 v = b.vel[i], f = b.fext[i], p = b.pos0[i];
  float2 l = b.plo0[i];
  float m = b.pm[i];
  float r = 1.f / m;
  v.x += f.x * r; v.y += f.y * r; v.z += f.z * r;
  p.x += v.x; p.y += v.y; p.z += v.z;
  b.pos1[i] = p; b.plo1[i] = l; b.vel[i] = v;
  b.fext[i] = make_float4(0, 0, 0, 0);
  b.acc[3 * i] = f.x; b.acc[3 * i + 1] = f.y; b.acc[3 * i + 2] = f.z;
}
__global__ void k_dep(B b, int n) {  // v1: vel first, exit on flag, then rest
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float4 v = b.vel[i];
  if (!(__float_as_uint(v.w) & 1u)) return;
  float4 f = b.fext[i], p = b.pos0[i];
  float2 l = b.plo0[i];
  float m = b.pm[i];
  float r = 1.f / m;
  v.x += f.x * r; v.y += f.y * r; v.z += f.z * r;
  p.x += v.x; p.y += v.y; p.z += v.z;
  b.pos1[i] = p; b.plo1[i] = l; b.vel[i] = v;
  b.fext[i] = make_float4(0, 0, 0, 0);
  b.acc[3 * i] = f.x; b.acc[3 * i + 1] = f.y; b.acc[3 * i + 2] = f.z;
}
__global__ void k_nc(B b, int n) {  // v3: dep-exit with nc loads for plo / pm
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float4 v = b.vel[i];
  if (!(__float_as_uint(v.w) & 1u)) return;
  float4 f = b.fext[i], p = b.pos0[i];
  float2 l = __ldg(b.plo0 + i);
  float m = __ldg(b.pm + i);
  float r = 1.f / m;
  v.x += f.x * r; v.y += f.y * r; v.z += f.z * r;
  p.x += v.x; p.y += v.y; p.z += v.z;
  b.pos1[i] = p; b.plo1[i] = l; b.vel[i] = v;
  b.fext[i] = make_float4(0, 0, 0, 0);
  b.acc[3 * i] = f.x; b.acc[3 * i + 1] = f.y; b.acc[3 * i + 2] = f.z;
}
__global__ void k_copy(const float4 *a, float4 *b, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}
int main() {
  const int n = 1000000;
  B b;
  cudaMalloc(&b.pos0, 16 * (n + 64)); cudaMalloc(&b.pos1, 16 * (n + 64));
  cudaMalloc(&b.vel, 16 * (n + 64)); cudaMalloc(&b.fext, 16 * (n + 64));
  cudaMalloc(&b.plo0, 8 * (n + 64)); cudaMalloc(&b.plo1, 8 * (n + 64));
  cudaMalloc(&b.pm, 4 * (n + 64)); cudaMalloc(&b.acc, 12 * (n + 64));
  cudaMemset(b.vel, 0x01, 16 * (n + 64));
  cudaMemset(b.pm, 0x3f, 4 * (n + 64));
  float4 *big; cudaMalloc(&big, 512 << 20);  // L2 flush
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto flush = [&]() { cudaMemsetAsync(big, 0, 512 << 20); };
  for (int bs : {128, 256, 512}) {
    for (int var = 0; var < 4; var++) {
      float best = 1e9;
      for (int rep = 0; rep < 20; rep++) {
        flush();
        cudaEventRecord(e0);
        int g = (n + bs - 1) / bs;
        if (var == 0) k_copyish<<<g, bs>>>(b, n);
        else if (var == 1) k_dep<<<g, bs>>>(b, n);
        else if (var == 3) k_nc<<<g, bs>>>(b, n);
        else k_copy<<<(4 * n + bs - 1) / bs, bs>>>(big, big + (64 << 20) / 16 * 4, 4 * n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("bs %d %s %.1f us\n", bs, var == 0 ? "all-loads" : var == 1 ? "dep-exit" : var == 3 ? "nc" : "copy64MB", best * 1e3);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
