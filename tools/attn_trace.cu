// Diagnostics: per-tile timestamps of the flash-attention forward (CTA 0) at the C2 shape.
// nvcc -gencode arch=compute_100a,code=sm_100a -DHY_ATTN_TRACE -Iinclude -Ipaper_2110_08633_b200/csrc/kernels
//      tools/attn_trace.cu -o tools/attn_trace -lcuda
#include <cstdio>
#include <vector>
#include "../paper_2110_08633_b200/csrc/kernels/attention_fa.cu"
int main() {
  const int B = 8, T = 512, H = 12, D = H * 64;
  float *qkv, *out, *lse;
  cudaMalloc(&qkv, sizeof(float) * B * T * 3 * D);
  cudaMalloc(&out, sizeof(float) * B * T * D);
  cudaMalloc(&lse, sizeof(float) * B * H * T);
  cudaMemset(qkv, 0, sizeof(float) * B * T * 3 * D);
  for (int r = 0; r < 3; ++r) hy::attention_fwd_fa(0, B, T, H, qkv, out, lse);
  cudaDeviceSynchronize();
  unsigned long long tr[8][256];
  cudaMemcpyFromSymbol(tr, hy::g_attn_trace, sizeof(tr));
  const char* names[8] = {"S issued", "PV issued", "sm: wait S", "sm: S landed", "sm: S loaded", "sm: softmax done",
                          "sm: PV(g-1) ok", "sm: P stored"};
  const unsigned long long t0 = tr[2][0];
  printf("g   ");
  for (int k = 0; k < 8; ++k) printf("%14s", names[k]);
  printf("\n");
  for (int g = 0; g < 12; ++g) {
    printf("%-4d", g);
    for (int k = 0; k < 8; ++k) printf("%14lld", (long long)(tr[k][g] - t0));
    printf("\n");
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
