// Probe: the d^F tree form's correctly rounded log (csrc/tree.cu cr_log) on a few values
// against the host libm.  Build (after python -m paper_0905_1744_b200.build):
//   O=paper_0905_1744_b200/lib/obj; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//     -o tools/crlog_probe tools/crlog_probe.cu $O/{api.cu,comm.cpp,exact.cpp,minsum.cu,minsum_tc.cu,order.cu,profiles.cu,tc_sparse.cu}.o -ldl -lcuda
#include "../paper_0905_1744_b200/csrc/tree.cu"
#include <cstdio>
int main() {
  using namespace sa;
  const int n = 2;
  double hF[4] = {1.0, 0.98, 0.98, 1.0};
  double *F, *S;
  unsigned long long* unc;
  cudaMalloc(&F, 32); cudaMalloc(&S, 32); cudaMalloc(&unc, 8); cudaMemset(unc, 0, 8);
  cudaMemcpy(F, hF, 32, cudaMemcpyHostToDevice);
  printf("table %d\n", (int)ensure_ln_table());
  dF_matrix_kernel<<<1, 256>>>(F, 2, n, 0.02, S, 2, unc);
  double hS[4];
  cudaMemcpy(hS, S, 32, cudaMemcpyDeviceToHost);
  printf("err %s S01 %.17g S10 %.17g\n", cudaGetErrorString(cudaGetLastError()), hS[1], hS[2]);
  double xs[6] = {0.5, 0.781117588817471, 0.605847029570968, 0.0, 1e-9, 0.9808107022244528};
  for (double f : xs) {
    hF[1] = hF[2] = f;
    cudaMemcpy(F, hF, 32, cudaMemcpyHostToDevice);
    dF_matrix_kernel<<<1, 256>>>(F, 2, n, 0.02, S, 2, unc);
    cudaMemcpy(hS, S, 32, cudaMemcpyDeviceToHost);
    printf("f %.17g ln(x) %.17g  host log %.17g\n", f, hS[1], std::log(0.02 + f));
  }
}
