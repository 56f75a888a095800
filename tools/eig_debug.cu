// Debug harness: append a random symmetric tridiagonal (s=1) row by row and
// print the eigen-engine intermediates after each append.
#include "../paper_1602_05033_b200/csrc/eigen.cuh"
#include <cstdio>
#include <vector>
#include <cmath>
using namespace kry;
int main() {
  EigEngine e;
  const int s = 1, m = 6;
  if (e.init(s, s * m + 8, 0)) { printf("init fail\n"); return 1; }
  std::vector<double> dsym(m * 64, 0.0), sub(m * 64, 0.0);
  for (int j = 0; j < m; ++j) { dsym[j * 64] = -2.0 - 0.3 * j; sub[j * 64] = 0.5 + 0.1 * j; }
  double *dd, *ds;
  cudaMalloc(&dd, m * 64 * 8); cudaMalloc(&ds, m * 64 * 8);
  cudaMemcpy(dd, dsym.data(), m * 64 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(ds, sub.data(), m * 64 * 8, cudaMemcpyHostToDevice);
  for (int j = 0; j < m; ++j) {
    int rc = e.append_block(0, dd + j * 64, j ? ds + (j - 1) * 64 : nullptr);
    cudaError_t err = cudaDeviceSynchronize();
    int K = e.K;
    std::vector<double> lam(K), F(K), L(K), zh(K + 1), mu(K + 1), org(K + 1), tau(K + 1), zz(K + 1);
    int counts[2];
    cudaMemcpy(lam.data(), e.lam_cur(), K * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(F.data(), e.F_cur(), K * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(L.data(), e.L_cur(), K * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(zh.data(), e.zhat, K * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(zz.data(), e.zz, K * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(mu.data(), e.mu, K * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(org.data(), e.org, K * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(tau.data(), e.tau, K * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(counts, e.counts, 8, cudaMemcpyDeviceToHost);
    printf("append %d rc %d err %s K %d p %d nd %d\n", j, rc, cudaGetErrorString(err), K, counts[0], counts[1]);
    for (int i = 0; i < K; ++i)
      printf("  %d lam % .6f F % .6f L % .6f | zz % .4e zhat % .4e mu % .6f org % .6f tau % .3e\n", i, lam[i], F[i],
             L[i], zz[i], zh[i], mu[i], org[i], tau[i]);
  }
  return 0;
}
