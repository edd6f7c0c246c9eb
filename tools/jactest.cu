// Standalone check of the warp Jacobi (dev tool): reconstruct random faces.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2506_09594_b200/csrc/prox.cuh"
#include "../paper_2506_09594_b200/csrc/jacobi.cuh"
namespace tr { void set_error(const char*, ...) {} }
using namespace tr;
__global__ void k_probe(double2* faces, int r0, int r1, int* sweeps_out) {
  extern __shared__ double jac_smem[];
  int lane = threadIdx.x & 31;
  double* Vr = jac_smem; double* Vi = Vr + kJW * kVld; double* Wr = Vi + kJW * kVld; double* Wi = Wr + kJW * kVld;
  double xr[kJW], xi[kJW];
  for (int i = 0; i < kJW; ++i) { xr[i] = 0; xi[i] = 0; if (i < r0 && lane < r1) { xr[i] = faces[i + r0*lane].x; xi[i] = faces[i + r0*lane].y; } }
  long long t0 = clock64();
  warp_jacobi(xr, xi, Vr, Vi, Wr, Wi, r0, r1, *sweeps_out);
  long long t1 = clock64();
  if (lane == 0) printf("cycles %lld\n", t1 - t0);
  // reconstruct X V^H and store
  __syncwarp();
  for (int i = 0; i < r0; ++i) { Wr[i*kVld + lane] = xr[i]; Wi[i*kVld+lane] = xi[i]; }
  __syncwarp();
  if (lane < r1) for (int i = 0; i < r0; ++i) { double ar=0, ai=0; for (int j=0;j<r1;++j){ double yr=Wr[i*kVld+j], yi=Wi[i*kVld+j], vr=Vr[lane*kVld+j], vi=Vi[lane*kVld+j]; ar += yr*vr+yi*vi; ai += yi*vr-yr*vi;} faces[i + r0*lane] = make_double2(ar, ai); }
}
int main(int argc, char** argv) {
  int r0 = 25, r1 = 25; std::vector<double2> h(r0*r1), o;
  srand(1); for (auto& v : h) { v.x = rand()/(double)RAND_MAX - 0.5; v.y = rand()/(double)RAND_MAX - 0.5; }
  double2* d; cudaMalloc(&d, sizeof(double2)*r0*r1); cudaMemcpy(d, h.data(), sizeof(double2)*r0*r1, cudaMemcpyHostToDevice);
  int* sw; cudaMalloc(&sw, 4);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 4*kJW*kVld*8);
  int ms = argc > 1 ? atoi(argv[1]) : 40; cudaMemcpy(sw, &ms, 4, cudaMemcpyHostToDevice);
  k_probe<<<1, 32, 4*kJW*kVld*8>>>(d, r0, r1, sw);
  o.resize(r0*r1); cudaMemcpy(o.data(), d, sizeof(double2)*r0*r1, cudaMemcpyDeviceToHost);
  double err = 0; for (int i = 0; i < r0*r1; ++i) err = fmax(err, fabs(o[i].x-h[i].x) + fabs(o[i].y-h[i].y));
  printf("recon err %g (%s)\n", err, cudaGetErrorString(cudaGetLastError()));
}
