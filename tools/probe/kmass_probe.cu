// k_mass (sl_device.cuh) on a synthetic 1 M-mass state, timed with CUDA
// events after an L2 flush: does the real kernel reproduce its in-library
// time, and which part costs it (compile with -DMASS_* variants).
#include <cstdio>
#include <vector>
#include "sl_device.cuh"
using namespace sl;
int main() {
  const int64_t n = 1000000;
  KState S;
  memset(&S, 0, sizeof S);
  S.m_n = n;
  auto dm = [](size_t b) { void *p; cudaMalloc(&p, b); cudaMemset(p, 0, b); return p; };
  S.pos[0] = dm(16 * (n + 64)); S.pos[1] = dm(16 * (n + 64));
  S.plo[0] = dm(8 * (n + 64)); S.plo[1] = dm(8 * (n + 64));
  S.pmass = (const float *)dm(4 * (n + 64));
  S.vel = dm(16 * (n + 64)); S.acc = dm(12 * (n + 64)); S.fext = dm(16 * (n + 64));
  S.status = (unsigned long long *)dm(64);
  std::vector<float> h(4 * n);
  for (int64_t i = 0; i < n; i++) { h[4*i] = 0.01f * (i % 100); h[4*i+1] = 0.01f * ((i / 100) % 100); h[4*i+2] = 0.01f * (i / 10000) + 0.001f; h[4*i+3] = 0.f; }
  cudaMemcpy(S.pos[0], h.data(), 16 * n, cudaMemcpyHostToDevice);
  for (int64_t i = 0; i < n; i++) { h[4*i] = h[4*i+1] = h[4*i+2] = 0.f; h[4*i+3] = __builtin_bit_cast(float, 1u); }
  cudaMemcpy(S.vel, h.data(), 16 * n, cudaMemcpyHostToDevice);
  std::vector<float> pm(n, 0.05f);
  cudaMemcpy((void *)S.pmass, pm.data(), 4 * n, cudaMemcpyHostToDevice);
  EnvP E;
  memset(&E, 0, sizeof E);
  E.g[2] = -9.81; E.gf[2] = -9.81f; E.drag = 0; E.v_stick = 1e-3; E.v_stickf = 1e-3f;
  E.np = 1;
  double pl[7] = {0, 0, 1, 0, 1e5, 0.5, 0.4};
  for (int q = 0; q < 7; q++) { E.pl[0][q] = pl[q]; E.plf[0][q] = (float)pl[q]; }
  StepP T; memset(&T, 0, sizeof T); T.dt = 1e-4; T.write_acc = 1;
  float4 *big; cudaMalloc(&big, 512 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int rep = 0; rep < 30; rep++) {
    cudaMemsetAsync(big, 0, 512 << 20);
    T.cur = rep & 1; T.step = 0;
    cudaEventRecord(e0);
    k_mass<PREC_FP32><<<(unsigned)((n + 255) / 256), 256>>>(S, E, T);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  printf("k_mass probe: %.1f us  (%s)\n", best * 1e3, cudaGetErrorString(cudaGetLastError()));
}
