// What cudaPointerGetAttributes / cudaHostGetFlags report for pageable host memory before and
// after first touch, page-locked memory and registered memory (driver 580: the resident pageable
// case decides which path mgp_resample_host takes).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
static void show(const char* what, const void* p) {
  cudaPointerAttributes at{};
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  unsigned fl = 0;
  cudaError_t e2 = cudaHostGetFlags(&fl, (void*)p);
  printf("%-34s attr=%d type=%d dev=%p host=%p | hostGetFlags=%d flags=%u\n", what, (int)e, (int)at.type, at.devicePointer,
         at.hostPointer, (int)e2, fl);
  cudaGetLastError();
}
int main() {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrPageableMemoryAccess, 0);
  int v2 = 0;
  cudaDeviceGetAttribute(&v2, cudaDevAttrPageableMemoryAccessUsesHostPageTables, 0);
  printf("pageableMemoryAccess=%d usesHostPageTables=%d\n", v, v2);
  const size_t n = 128u << 20;
  char* a = (char*)malloc(n);
  show("malloc untouched", a);
  memset(a, 1, n);
  show("malloc touched", a);
  show("malloc touched +4096", a + 4096);
  void* h = nullptr;
  cudaMallocHost(&h, n);
  show("cudaMallocHost", h);
  show("cudaMallocHost +12345", (char*)h + 12345);
  char* r = (char*)malloc(n);
  memset(r, 1, n);
  cudaHostRegister(r, n, 0);
  show("registered", r);
  show("registered +777", r + 777);
  return 0;
}
