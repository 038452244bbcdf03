// trace_kernels.cu — pipeline timeline of the SpMM kernels (debug tool, not part of libvenom).
// Builds the library TU with -DVENOM_TRACE so the kernels record %globaltimer at pipeline events
// for CTAs 0/1, then prints per-k-stage event times (ns, relative to the first event).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DVENOM_TRACE \
//          -o tools/trace_kernels tools/trace_kernels.cu
// Run:   tools/trace_kernels R K T V M strategy tile_t pair pre(1: pre-ordered metadata) max_ctas
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2310_02065_b200/csrc/venom_api.cu"
// the SpMM instantiation units of libvenom (one program here)
#include "../paper_2310_02065_b200/csrc/tu_gather_pre_f16.cu"
#include "../paper_2310_02065_b200/csrc/tu_gather_pre_bf16.cu"
#include "../paper_2310_02065_b200/csrc/tu_gather_nopre_f16.cu"
#include "../paper_2310_02065_b200/csrc/tu_gather_nopre_bf16.cu"
#include "../paper_2310_02065_b200/csrc/tu_densek_f16.cu"
#include "../paper_2310_02065_b200/csrc/tu_densek_bf16.cu"

int main(int argc, char** argv) {
  const long R = argc > 1 ? atol(argv[1]) : 1024, K = argc > 2 ? atol(argv[2]) : 4096,
             T = argc > 3 ? atol(argv[3]) : 4096;
  const int V = argc > 4 ? atoi(argv[4]) : 64, M = argc > 5 ? atoi(argv[5]) : 8;
  const int strat = argc > 6 ? atoi(argv[6]) : 2, tile = argc > 7 ? atoi(argv[7]) : 0;
  const int pair = argc > 8 ? atoi(argv[8]) : 0;
  const long G = K / M;
  uint16_t *vals, *B, *C;
  uint8_t *meta, *cidx;
  cudaMalloc(&vals, R * G * 4);
  cudaMalloc(&meta, R * ((G + 1) / 2));
  cudaMalloc(&cidx, (R / V) * G * 4);
  cudaMalloc(&B, K * T * 2);
  cudaMalloc(&C, R * T * 2);
  cudaMemset(vals, 0x3c, R * G * 4);
  cudaMemset(meta, 0x44, R * ((G + 1) / 2));
  std::vector<uint32_t> cw((R / V) * G, 0x03020100u);
  cudaMemcpy(cidx, cw.data(), cw.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(B, 0, K * T * 2);
  unsigned long long* tr;
  const size_t ntr = 2 * 16 * 256;
  cudaMalloc(&tr, ntr * 8);
  cudaMemcpyToSymbol(g_venom_trace, &tr, sizeof(tr));
  const int pre = argc > 9 ? atoi(argv[9]) : 0;
  uint8_t* mtc = nullptr;
  if (pre) {
    const int64_t nb = venom_metadata_tc_bytes(R, K, venom_format_t{V, 2, M});
    cudaMalloc(&mtc, nb);
    cudaMemset(mtc, 0x44, nb);
  }
  const int max_ctas = argc > 10 ? atoi(argv[10]) : 0;
  venom_spmm_opts_t o{tile, 0, max_ctas, strat, pair, mtc};
  venom_format_t f{V, 2, M};
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(tr, 0, ntr * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    int st = venom_spmm_ex(vals, meta, cidx, R, K, f, B, T, T, C, T, nullptr, VENOM_F16, &o, 0);
    cudaEventRecord(b);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("rep %d status %d err %s time %.4f ms\n", rep, st, cudaGetErrorString(cudaGetLastError()), ms);
  }
  std::vector<unsigned long long> h(ntr);
  cudaMemcpy(h.data(), tr, ntr * 8, cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ull;
  for (int k = 0; k < 16; ++k)
    for (int i = 0; i < 256; ++i)
      if (h[k * 256 + i] && h[k * 256 + i] < t0) t0 = h[k * 256 + i];
  const char* names[13] = {"prodB", "mmaFull", "mmaCommit", "meta", "prodDone", "prodTop",
                           "prodA+", "prodB3d+", "mmaIssued", "epiAcc(tile)", "epiStored(tile)",
                           "kern(0start,1init,2end)", "epiRel(tile)"};
  for (int cta = 0; cta < 2; ++cta) {
    printf("CTA %d\nit ", cta);
    for (int k = 0; k < 13; ++k) printf("%11.11s", names[k]);
    printf("   (ns since first event)\n");
    for (int i = 0; i < 96; ++i) {
      bool any = false;
      for (int k = 0; k < 13; ++k) any |= h[(cta * 16 + k) * 256 + i] != 0;
      if (!any) continue;
      printf("%3d", i);
      for (int k = 0; k < 13; ++k) {
        const unsigned long long v = h[(cta * 16 + k) * 256 + i];
        if (v) printf("%11lld", (long long)(v - t0));
        else printf("%11s", "-");
      }
      printf("\n");
    }
  }
  return 0;
}
