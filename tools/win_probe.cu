// tools/win_probe.cu — feasibility probe (build: nvcc -gencode arch=compute_100a,code=sm_100a -I<nccl>/include
// win_probe.cu -l:libnccl.so.2): NCCL symmetric window on a 1-rank communicator, peer pointer from the device API,
// a kernel storing through it, and the bytes read back.
#include <cstdio>
#include <nccl.h>
#include <nccl_device.h>
__global__ void peer_ptrs(ncclWindow_t w, int G, unsigned char** out) {
  int d = threadIdx.x;
  if (d < G) out[d] = (unsigned char*)ncclGetPeerPointer(w, 0, d);
}
__global__ void fill(unsigned char** p, size_t n) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[0][i] = (unsigned char)(i * 7);
  __threadfence_system();
}
#define CK(x) do { auto r = (x); if ((int)r) { printf("FAIL %s -> %d\n", #x, (int)r); return 1; } } while (0)
int main() {
  ncclUniqueId id; CK(ncclGetUniqueId(&id));
  ncclComm_t c; CK(ncclCommInitRank(&c, 1, id, 0));
  size_t n = 64 << 20;
  void* buf; CK(ncclMemAlloc(&buf, n));
  ncclWindow_t w; CK(ncclCommWindowRegister(c, buf, n, &w, NCCL_WIN_COLL_SYMMETRIC));
  unsigned char** dp; CK(cudaMalloc(&dp, 64));
  peer_ptrs<<<1, 32>>>(w, 1, dp);
  unsigned char* hp[1]; CK(cudaMemcpy(hp, dp, 8, cudaMemcpyDeviceToHost));
  printf("buf %p peer0 %p\n", buf, hp[0]);
  fill<<<148, 256>>>(dp, n);
  CK(cudaDeviceSynchronize());
  unsigned char* h = new unsigned char[n];
  CK(cudaMemcpy(h, buf, n, cudaMemcpyDeviceToHost));
  size_t bad = 0; for (size_t i = 0; i < n; ++i) bad += h[i] != (unsigned char)(i * 7);
  printf("mismatches %zu\n", bad);
  // re-register bigger (the grow path)
  CK(ncclCommWindowDeregister(c, w)); CK(ncclMemFree(buf));
  CK(ncclMemAlloc(&buf, 2 * n)); CK(ncclCommWindowRegister(c, buf, 2 * n, &w, NCCL_WIN_COLL_SYMMETRIC));
  peer_ptrs<<<1, 32>>>(w, 1, dp); CK(cudaMemcpy(hp, dp, 8, cudaMemcpyDeviceToHost));
  printf("regrow buf %p peer0 %p\n", buf, hp[0]);
  CK(ncclCommWindowDeregister(c, w)); CK(ncclMemFree(buf)); CK(ncclCommDestroy(c));
  printf("ok\n");
  return 0;
}
