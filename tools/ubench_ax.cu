// Tuning microbenchmark for the Ax kernel at N=7 (n=8): AX_ONLY over E elements
// with random D, G, u.  Built per configuration with -DSEM_AX8_NE/NSG/PPC.
#define SEM_AX_ONLY_N8 1
#include "../paper_2107_01243_b200/csrc/ax.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

int main(int argc, char** argv) {
  const int E = argc > 1 ? atoi(argv[1]) : 8192;
  const int n3 = 512;
  const size_t nl = (size_t)E * n3;
  std::vector<double> h(6 * nl);
  for (size_t q = 0; q < h.size(); q++) h[q] = (double)((q * 2654435761u) % 1000) / 1000.0;
  double *G, *u, *w, *D;
  cudaMalloc(&G, 6 * nl * 8); cudaMalloc(&u, nl * 8); cudaMalloc(&w, nl * 8); cudaMalloc(&D, 64 * 8);
  cudaMemcpy(G, h.data(), 6 * nl * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(u, h.data(), nl * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(D, h.data(), 64 * 8, cudaMemcpyHostToDevice);
  double* flush;
  size_t fl = 512ull << 20;
  cudaMalloc(&flush, fl);
  sem::DevPlan P{};
  P.N = 7; P.n = 8; P.nloc = E; P.n_local = nl; P.D = D;
  sem::AxLaunch a{};
  a.u = u; a.w = w; a.G = G; a.r0lo = 0; a.r0hi = E;
  for (int q = 0; q < 64; q++) a.Dm[q] = h[q];
  int occ = sem::ax_occupancy(7, sem::AX_ONLY);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid = sem::ax_groups(7, E);   // launcher caps at residency
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9, tot = 0;
  const int reps = 20;
  for (int r = 0; r < reps + 3; r++) {
    cudaMemsetAsync(flush, r, fl);
    cudaEventRecord(e0);
    sem::launch_ax(P, a, sem::AX_ONLY, grid, 0, false);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 3) { best = std::min(best, ms); tot += ms; }
  }
  cudaError_t err = cudaGetLastError();
  printf("NE=%d NSG=%d PPC=%d occ=%d grid=%d smem=%zu  best %.2f us  mean %.2f us  %.0f GB/s (64 B/pt)  %s\n",
         SEM_AX8_NE, SEM_AX8_NSG, SEM_AX8_PPC, occ, grid, sem::dev::AxShape<8>::smem_bytes, best * 1e3,
         tot / reps * 1e3, nl * 64.0 / (best * 1e-3) / 1e9, cudaGetErrorString(err));
  return 0;
}
