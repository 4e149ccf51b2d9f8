// TEST INFRASTRUCTURE ONLY: a minimal stand-in for libnccl (the handful of entry points libbipb
// dlopens) so that the multi-rank code path of the library can run with several processes on
// ONE GPU (real NCCL refuses two ranks on the same device).  Collectives are synchronous:
// each rank stages its send buffer into a CUDA-IPC-shared device buffer, ranks meet at a
// shared-memory barrier, and every rank reads all contributions in rank order (all-reduce:
// fixed-order sum, so results are bitwise identical on every rank).
// Selected by BIPB_NCCL_LIB=<path to libfakenccl.so>.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <nccl.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>

namespace {
constexpr int MAXR = 16;
constexpr size_t CAP = 256ull << 20;  // bytes per rank staging buffer
struct Shared {
  std::atomic<int> arrived[2];
  std::atomic<int> gen;
  std::atomic<int> ready;
  cudaIpcMemHandle_t h[MAXR];
};
struct Comm {
  int rank, n;
  Shared* sh;
  void* mine;
  void* peer[MAXR];
  int phase;
};
void barrier(Comm* c) {
  Shared* s = c->sh;
  const int g = s->gen.load();
  if (s->arrived[g & 1].fetch_add(1) + 1 == c->n) {
    s->arrived[g & 1].store(0);
    s->gen.store(g + 1);
  } else {
    while (s->gen.load() == g) sched_yield();
  }
}
__global__ void accumulate(double* dst, const double* src, size_t n, int first) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = first ? src[i] : dst[i] + src[i];
}
__global__ void accumulate_u64(unsigned long long* dst, const unsigned long long* src, size_t n, int first) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = first ? src[i] : dst[i] + src[i];
}
}  // namespace

extern "C" {
ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  memset(id, 0, sizeof(*id));
  snprintf(id->internal, sizeof(id->internal), "/bipb_fakenccl_%d_%ld", (int)getpid(), (long)time(nullptr));
  return ncclSuccess;
}
ncclResult_t ncclCommInitRank(ncclComm_t* out, int nranks, ncclUniqueId id, int rank) {
  if (nranks > MAXR) return ncclInvalidArgument;
  int fd = shm_open(id.internal, O_CREAT | O_RDWR, 0600);
  if (fd < 0 || ftruncate(fd, sizeof(Shared)) != 0) return ncclSystemError;
  Shared* s = (Shared*)mmap(nullptr, sizeof(Shared), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  Comm* c = new Comm();
  c->rank = rank;
  c->n = nranks;
  c->sh = s;
  if (cudaMalloc(&c->mine, CAP) != cudaSuccess) return ncclUnhandledCudaError;
  if (cudaIpcGetMemHandle(&s->h[rank], c->mine) != cudaSuccess) return ncclUnhandledCudaError;
  s->ready.fetch_add(1);
  while (s->ready.load() < nranks) sched_yield();
  for (int p = 0; p < nranks; ++p) {
    if (p == rank) {
      c->peer[p] = c->mine;
    } else if (cudaIpcOpenMemHandle(&c->peer[p], s->h[p], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      return ncclUnhandledCudaError;
    }
  }
  barrier(c);
  if (rank == 0) shm_unlink(id.internal);
  *out = (ncclComm_t)c;
  return ncclSuccess;
}
static size_t tsize(ncclDataType_t t) { return t == ncclFloat64 ? 8 : (t == ncclFloat32 ? 4 : 1); }
ncclResult_t ncclAllGather(const void* send, void* recv, size_t count, ncclDataType_t dt, ncclComm_t comm,
                           cudaStream_t st) {
  Comm* c = (Comm*)comm;
  const size_t bytes = count * tsize(dt);
  if (bytes > CAP) return ncclInvalidArgument;
  cudaMemcpyAsync(c->mine, send, bytes, cudaMemcpyDeviceToDevice, st);
  cudaStreamSynchronize(st);
  barrier(c);
  for (int p = 0; p < c->n; ++p)
    cudaMemcpyAsync((char*)recv + p * bytes, c->peer[p], bytes, cudaMemcpyDeviceToDevice, st);
  cudaStreamSynchronize(st);
  barrier(c);
  return ncclSuccess;
}
ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t dt, ncclRedOp_t op,
                           ncclComm_t comm, cudaStream_t st) {
  Comm* c = (Comm*)comm;
  const bool u64 = dt == ncclUint64 || dt == ncclInt64;  // exact sums (bipb_exact.cuh)
  if ((dt != ncclFloat64 && !u64) || op != ncclSum || count * 8 > CAP) return ncclInvalidArgument;
  cudaMemcpyAsync(c->mine, send, count * 8, cudaMemcpyDeviceToDevice, st);
  cudaStreamSynchronize(st);
  barrier(c);
  for (int p = 0; p < c->n; ++p)
    if (u64)
      accumulate_u64<<<256, 256, 0, st>>>((unsigned long long*)recv, (const unsigned long long*)c->peer[p], count,
                                          p == 0);
    else
      accumulate<<<256, 256, 0, st>>>((double*)recv, (const double*)c->peer[p], count, p == 0);
  cudaStreamSynchronize(st);
  barrier(c);
  return ncclSuccess;
}
ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  Comm* c = (Comm*)comm;
  barrier(c);
  for (int p = 0; p < c->n; ++p)
    if (p != c->rank) cudaIpcCloseMemHandle(c->peer[p]);
  cudaFree(c->mine);
  munmap(c->sh, sizeof(Shared));
  delete c;
  return ncclSuccess;
}
// abort: local teardown without the barrier (the peers may be gone or stuck)
ncclResult_t ncclCommAbort(ncclComm_t comm) {
  Comm* c = (Comm*)comm;
  for (int p = 0; p < c->n; ++p)
    if (p != c->rank) cudaIpcCloseMemHandle(c->peer[p]);
  cudaFree(c->mine);
  munmap(c->sh, sizeof(Shared));
  delete c;
  return ncclSuccess;
}
ncclResult_t ncclCommGetAsyncError(ncclComm_t, ncclResult_t* r) {
  *r = ncclSuccess;  // collectives are synchronous here: errors are returned directly
  return ncclSuccess;
}
const char* ncclGetErrorString(ncclResult_t r) { return r == ncclSuccess ? "fake nccl: success" : "fake nccl: error"; }
}
