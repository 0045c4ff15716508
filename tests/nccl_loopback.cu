// tests/nccl_loopback.cu -- TEST INFRASTRUCTURE: an in-process "NCCL" for the row-sharded mode's
// multi-rank test on ONE GPU (tests/test_sharded_loopback.py). Several ranks are host threads of one
// process, each with its own CUDA stream; a collective is a host rendezvous of all ranks followed by
// stream-ordered device work: every rank stages its send buffer (event-ordered after its prior work),
// then each rank builds its result from all staged buffers in rank order (deterministic sums), and no
// rank reuses its buffers before every rank has finished reading. No kernel ever waits on another
// rank's kernel (the ordering is by CUDA events between streams), so nothing can hang the GPU.
// Loaded by libpsdproj.so through PSDPROJ_NCCL_LIB; implements the six entry points it uses.
#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

namespace {

struct Slot {
  const void* send = nullptr;
  void* recv = nullptr;
  cudaStream_t stream = nullptr;
  double* stage = nullptr;
  cudaEvent_t staged = nullptr, done = nullptr;
};

struct Group {
  int nranks = 0, joined = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
  std::vector<Slot> slots;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long g = generation;
    if (++arrived == nranks) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != g; });
    }
  }
};

struct Comm {
  Group* g;
  int rank;
};

std::mutex g_mu;
std::map<unsigned long long, Group*> g_groups;
unsigned long long g_next = 1;

__global__ void sum_kernel(int nr, const double* const* src, double* dst, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int r = 0; r < nr; ++r) a += src[r][i];  // rank order: deterministic
    dst[i] = a;
  }
}

size_t elem_size(ncclDataType_t t) {
  switch (t) {
    case ncclFloat64: return 8;
    case ncclInt32: case ncclFloat32: case ncclUint32: return 4;
    default: return 8;
  }
}

// the common collective: kind 0 = all-reduce (sum, fp64), 1 = all-gather
ncclResult_t collective(int kind, const void* send, void* recv, size_t count, ncclDataType_t type, Comm* c,
                        cudaStream_t st) {
  Group* g = c->g;
  const int r = c->rank, nr = g->nranks;
  const size_t bytes = count * elem_size(type);
  Slot& me = g->slots[r];
  me.send = send;
  me.recv = recv;
  me.stream = st;
  if (cudaMalloc(&me.stage, bytes ? bytes : 8) != cudaSuccess) return ncclUnhandledCudaError;
  cudaEventCreateWithFlags(&me.staged, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&me.done, cudaEventDisableTiming);
  // (1) stage my send buffer behind my stream's prior work
  cudaMemcpyAsync(me.stage, send, bytes, cudaMemcpyDeviceToDevice, st);
  cudaEventRecord(me.staged, st);
  g->barrier();
  // (2) my result from every rank's staged buffer (rank order)
  for (int q = 0; q < nr; ++q) cudaStreamWaitEvent(st, g->slots[q].staged, 0);
  if (kind == 1) {
    for (int q = 0; q < nr; ++q)
      cudaMemcpyAsync((char*)recv + q * bytes, g->slots[q].stage, bytes, cudaMemcpyDeviceToDevice, st);
  } else {
    std::vector<const double*> h(nr);
    for (int q = 0; q < nr; ++q) h[q] = (const double*)g->slots[q].stage;
    const double** dsrc = nullptr;
    cudaMalloc(&dsrc, sizeof(double*) * nr);
    cudaMemcpyAsync(dsrc, h.data(), sizeof(double*) * nr, cudaMemcpyHostToDevice, st);
    sum_kernel<<<64, 256, 0, st>>>(nr, dsrc, (double*)recv, count);
    cudaStreamSynchronize(st);  // h and dsrc die here
    cudaFree(dsrc);
  }
  cudaEventRecord(me.done, st);
  g->barrier();
  // (3) nobody frees / reuses a staging buffer before every rank has read it
  for (int q = 0; q < nr; ++q) cudaStreamWaitEvent(st, g->slots[q].done, 0);
  g->barrier();
  cudaStreamSynchronize(st);
  cudaFree(me.stage);
  cudaEventDestroy(me.staged);
  cudaEventDestroy(me.done);
  g->barrier();
  return cudaGetLastError() == cudaSuccess ? ncclSuccess : ncclUnhandledCudaError;
}

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  std::lock_guard<std::mutex> lk(g_mu);
  std::memset(id, 0, sizeof(*id));
  const unsigned long long k = g_next++;
  std::memcpy(id->internal, "LOOPBACK", 8);
  std::memcpy(id->internal + 8, &k, sizeof(k));
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  unsigned long long k;
  std::memcpy(&k, id.internal + 8, sizeof(k));
  Group* g;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_groups.find(k);
    if (it == g_groups.end()) {
      g = new Group();
      g->nranks = nranks;
      g->slots.resize(nranks);
      g_groups[k] = g;
    } else {
      g = it->second;
    }
  }
  if (rank < 0 || rank >= g->nranks || nranks != g->nranks) return ncclInvalidArgument;
  auto* c = new Comm{g, rank};
  g->barrier();  // all ranks joined
  *comm = reinterpret_cast<ncclComm_t>(c);
  return ncclSuccess;
}

ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t type, ncclRedOp_t op,
                           ncclComm_t comm, cudaStream_t st) {
  if (type != ncclFloat64 || op != ncclSum) return ncclInvalidArgument;
  return collective(0, send, recv, count, type, reinterpret_cast<Comm*>(comm), st);
}

ncclResult_t ncclAllGather(const void* send, void* recv, size_t count, ncclDataType_t type, ncclComm_t comm,
                           cudaStream_t st) {
  return collective(1, send, recv, count, type, reinterpret_cast<Comm*>(comm), st);
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  delete reinterpret_cast<Comm*>(comm);
  return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t r) { return r == ncclSuccess ? "loopback: success" : "loopback: error"; }

}  // extern "C"
