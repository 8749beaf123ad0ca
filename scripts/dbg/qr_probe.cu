#define RT_DEBUG_QR 1
#include <cstdio>
#include "../../paper_1905_07311_b200/csrc/smallla.cu"
int main() {
  const int m = 8, n = 2;
  double hY[m * n];
  for (int i = 0; i < m * n; ++i) hY[i] = (double)((i * 7919) % 13) - 6.0;
  double *Y, *Q;
  cudaMalloc(&Y, sizeof hY); cudaMalloc(&Q, sizeof hY);
  cudaMemcpy(Y, hY, sizeof hY, cudaMemcpyHostToDevice);
  cudaMemset(Q, 0, sizeof hY);
  rt::Ctx c; cudaStreamCreate(&c.stream);
  setenv("RTUCKER_QR_NCTA", "2", 1);
  try { rt::householder_qr(c, Y, m, n, Q); } catch (std::exception &e) { printf("ERR %s\n", e.what()); }
  printf("sync: %s\n", cudaGetErrorString(cudaStreamSynchronize(c.stream)));
  double hQ[m * n]; cudaMemcpy(hQ, Q, sizeof hQ, cudaMemcpyDeviceToHost);
  for (int i = 0; i < m; ++i) printf("%8.4f %8.4f\n", hQ[i], hQ[i + m]);
  double dbg[1024]; cudaMemcpyFromSymbol(dbg, rt::g_dbg, sizeof dbg);
  for (int cta = 0; cta < 2; ++cta) for (int j = 0; j < n; ++j) for (int c = j; c < n; ++c) printf("Q cta %d j %d c %d f %g own %g Qlast %g i0nloc %g\n", cta, j, c, dbg[512+cta*64+4*j+c], dbg[768+cta*64+4*j+c], dbg[256+cta*64+8*j+2*c], dbg[256+cta*64+8*j+2*c+1]);
}
// (appended) 
