// Probe: fp64 mma.sync.m8n8k4 on sm_100a — (1) is D = A B + C bitwise equal to
// the sequential fma chain over k (k = 0..3), (2) throughput vs DFMA.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// A 8x4 row-major, B 4x8 (col-major fragment), C/D 8x8 row-major
__global__ void probe(const double *A, const double *B, const double *C, double *D, double *R) {
  const int lane = threadIdx.x;
  // fragments (PTX ISA m8n8k4 f64): a: row = lane/4, col = lane%4; b: row(k) = lane%4, col = lane/4;
  // c/d: row = lane/4, cols = 2*(lane%4) + {0,1}
  const double a = A[(lane / 4) * 4 + lane % 4];
  const double b = B[(lane % 4) * 8 + lane / 4];
  const int r = lane / 4, c = 2 * (lane % 4);
  double d0, d1;
  dmma(d0, d1, a, b, C[r * 8 + c], C[r * 8 + c + 1]);
  D[r * 8 + c] = d0;
  D[r * 8 + c + 1] = d1;
  if (lane < 8) {
    for (int col = 0; col < 8; col++) {
      double acc = C[lane * 8 + col];
      for (int k = 0; k < 4; k++) acc = fma(A[lane * 4 + k], B[k * 8 + col], acc);
      R[lane * 8 + col] = acc;
    }
  }
}

__global__ void tput_dmma(double *out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int t = 0; t < 8; t++) c[t][0] = c[t][1] = t;
  for (int i = 0; i < iters; i++)
#pragma unroll
    for (int t = 0; t < 8; t++) dmma(c[t][0], c[t][1], a, b, c[t][0], c[t][1]);
  double s = 0;
  for (int t = 0; t < 8; t++) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void tput_dfma(double *out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[16];
  for (int t = 0; t < 16; t++) c[t] = t;
  for (int i = 0; i < iters; i++)
#pragma unroll
    for (int t = 0; t < 16; t++) c[t] = fma(a, b, c[t]);
  double s = 0;
  for (int t = 0; t < 16; t++) s += c[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double hA[32], hB[32], hC[64], hD[64], hR[64];
  srand(1);
  int mism = 0;
  double *A, *B, *C, *D, *R, *o;
  cudaMalloc(&A, 256); cudaMalloc(&B, 256); cudaMalloc(&C, 512); cudaMalloc(&D, 512); cudaMalloc(&R, 512);
  for (int trial = 0; trial < 2000; trial++) {
    for (int i = 0; i < 32; i++) hA[i] = (rand() / (double)RAND_MAX) * pow(10.0, rand() % 8 - 4);
    for (int i = 0; i < 32; i++) hB[i] = (rand() / (double)RAND_MAX) * pow(10.0, rand() % 8 - 4);
    for (int i = 0; i < 64; i++) hC[i] = (rand() / (double)RAND_MAX) * pow(10.0, rand() % 8 - 4);
    cudaMemcpy(A, hA, 256, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
    cudaMemcpy(C, hC, 512, cudaMemcpyHostToDevice);
    probe<<<1, 32>>>(A, B, C, D, R);
    cudaMemcpy(hD, D, 512, cudaMemcpyDeviceToHost);
    cudaMemcpy(hR, R, 512, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 64; i++) mism += memcmp(&hD[i], &hR[i], 8) != 0;
  }
  printf("dmma vs sequential fma chain: %d mismatches of %d\n", mism, 2000 * 64);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaMalloc(&o, sizeof(double) * sms * 8 * 256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(e0);
    tput_dmma<<<sms * 4, 256>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 256 * 8 * (double)iters * sms * 4 * (256 / 32);
    printf("DMMA m8n8k4: %.1f TFLOP/s\n", flops / ms / 1e9);
    cudaEventRecord(e0);
    tput_dfma<<<sms * 4, 256>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double f2 = 2.0 * 16 * (double)iters * sms * 4 * 256;
    printf("DFMA: %.1f TFLOP/s\n", f2 / ms / 1e9);
  }
  return 0;
}
