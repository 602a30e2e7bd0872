// All-to-all NVLink store probe (N GPUs, one process): every GPU runs a kernel whose CTAs
// store 16-byte vectors round-robin into the other N-1 GPUs' buffers (the traffic pattern of
// the ring-position layout's relabelling stores), all GPUs at once.  Prints the outgoing
// payload bandwidth per GPU.  Also the pairwise (N = 2) case for comparison.
// Build: make -C tools/p2p a2a_bw   Run: ./tools/p2p/a2a_bw [ngpus] [MiB per destination]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

struct Dst {
  uint4* p[8];
  int n;
};

// CTA b writes chunk rows to destination b % n (512-byte rows, like the mix epilogue)
__global__ void k_a2a(Dst d, size_t per_dst_vecs) {
  const int dst = blockIdx.x % d.n;
  const size_t cta_in_dst = blockIdx.x / d.n, ctas_per_dst = gridDim.x / d.n;
  uint4* out = d.p[dst];
  for (size_t i = cta_in_dst * blockDim.x + threadIdx.x; i < per_dst_vecs;
       i += ctas_per_dst * blockDim.x)
    out[i] = make_uint4((uint32_t)i, dst, 2, 3);
}

int main(int argc, char** argv) {
  int ngpu = 0;
  CK(cudaGetDeviceCount(&ngpu));
  int n = argc > 1 ? atoi(argv[1]) : ngpu;
  size_t mib = argc > 2 ? atol(argv[2]) : 1024;
  if (n > ngpu) n = ngpu;
  if (n < 2) { printf("need >= 2 GPUs\n"); return 0; }
  for (int a = 0; a < n; a++) {
    CK(cudaSetDevice(a));
    for (int b = 0; b < n; b++)
      if (a != b) {
        cudaError_t pe = cudaDeviceEnablePeerAccess(b, 0);
        if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) CK(pe);
        cudaGetLastError();
      }
  }
  const size_t bytes = mib << 20, vecs = bytes / 16;
  // buf[g][s]: GPU g's landing zone for sender s
  std::vector<std::vector<uint4*>> buf(n, std::vector<uint4*>(n, nullptr));
  for (int g = 0; g < n; g++) {
    CK(cudaSetDevice(g));
    for (int s = 0; s < n; s++)
      if (s != g) CK(cudaMalloc(&buf[g][s], bytes));
  }
  std::vector<cudaEvent_t> e0(n), e1(n);
  for (int group = 2; group <= n; group *= 2) {
    for (int rep = 0; rep < 3; rep++) {
      for (int g = 0; g < group; g++) {
        CK(cudaSetDevice(g));
        CK(cudaEventCreate(&e0[g]));
        CK(cudaEventCreate(&e1[g]));
      }
      for (int g = 0; g < group; g++) {
        CK(cudaSetDevice(g));
        CK(cudaDeviceSynchronize());
      }
      for (int g = 0; g < group; g++) {
        CK(cudaSetDevice(g));
        Dst d{};
        d.n = 0;
        for (int t = 0; t < group; t++)
          if (t != g) d.p[d.n++] = buf[t][g];
        int sms = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g));
        const int grid = sms * 4 / d.n * d.n;
        CK(cudaEventRecord(e0[g]));
        k_a2a<<<grid, 512>>>(d, vecs);
        CK(cudaGetLastError());
        CK(cudaEventRecord(e1[g]));
      }
      for (int g = 0; g < group; g++) {
        CK(cudaSetDevice(g));
        CK(cudaEventSynchronize(e1[g]));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
        const double out_bytes = (double)bytes * (group - 1);
        printf("{\"gpus\": %d, \"rep\": %d, \"gpu\": %d, \"ms\": %.3f, \"out_GBs\": %.1f}\n", group,
               rep, g, ms, out_bytes / (ms * 1e-3) / 1e9);
        CK(cudaEventDestroy(e0[g]));
        CK(cudaEventDestroy(e1[g]));
      }
    }
  }
  return 0;
}
