// Which SM runs which CTA of a one-CTA-per-SM grid (the k_tmem launch shape),
// and the L2 round-trip latency from each SM to one global line: shows how
// consecutive blockIdx map onto SMs / dies.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe/smid_probe tools/probe/smid_probe.cu
#include <cstdio>
#include <vector>

__global__ void probe(int* smid, long long* lat, volatile unsigned* line) {
  extern __shared__ unsigned char pad[];
  if (threadIdx.x == 0) {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    smid[blockIdx.x] = (int)s;
    unsigned v = 0;
    long long t0 = clock64();
    for (int i = 0; i < 64; ++i) v += __ldcg((const unsigned*)line + (v & 1));  // dependent L2 loads
    lat[blockIdx.x] = (clock64() - t0) / 64 + (v == 12345 ? 1 : 0);
    pad[0] = (unsigned char)v;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int n = sms;
  int* d_s;
  long long* d_l;
  unsigned* line;
  cudaMalloc(&d_s, n * sizeof(int));
  cudaMalloc(&d_l, n * sizeof(long long));
  cudaMalloc(&line, 256);
  cudaMemset(line, 0, 256);
  const size_t smem = 200 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe<<<n, 512, smem>>>(d_s, d_l, line);
  cudaDeviceSynchronize();
  std::vector<int> s(n);
  std::vector<long long> l(n);
  cudaMemcpy(s.data(), d_s, n * sizeof(int), cudaMemcpyDeviceToHost);
  cudaMemcpy(l.data(), d_l, n * sizeof(long long), cudaMemcpyDeviceToHost);
  printf("block: smid (L2 round trip, cycles)\n");
  for (int b = 0; b < n; ++b) printf("%d:%d(%lld)%s", b, s[b], l[b], (b % 8 == 7) ? "\n" : "  ");
  printf("\n");
  return 0;
}
