// Loopback multi-rank transport (SURVEY.md 4.2 "loopback fake"): P rank
// contexts of ONE process on ONE device, each driven by its own host thread,
// exchange through device copies instead of NCCL.  It runs the NCCL
// transport's code path unchanged -- Alg. 1's pack of the shared partials,
// the neighbour exchange, the unpack that adds the rank partials in ascending
// rank order (reading Q10), and the CG allreduces summed
// in ascending rank order -- so the partition plan and the cross-rank
// arithmetic are verified on a single GPU.  It is a test transport, not a
// compute backend: every operation is still one of libsem's kernels.
//
// Protocol of one collective (every rank calls the same collectives in the
// same order, as with NCCL):
//   1. the rank records an "in" event on its stream after its input is ready
//      and posts (pointers, event) to the world;            -- host barrier --
//   2. it makes its stream wait for the peers' "in" events, copies / reduces,
//      records an "out" event and posts it;                 -- host barrier --
//   3. its stream waits for the peers' "out" events, so a later write into
//      this rank's buffers cannot overtake a peer still reading them.
// A rank can be at most one barrier ahead of another, so one pair of events
// per rank suffices; the posted records are double-buffered by barrier
// generation.  Every stream wait refers to work already submitted, so the
// device never waits on the host.  flags & 1 ("shuffle") processes the
// neighbours in reverse order and delays each rank's posts by a random
// 0-300 us: completion order changes, results must not (rank-ordered sums).
// flags >> 8 = collective timeout in seconds (default 120): a rank that does
// not arrive makes the collective fail with SEM_ENCCL instead of hanging.
#include <cuda_runtime.h>

#include <chrono>
#include <condition_variable>
#include <mutex>
#include <random>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "kernels.h"
#include "sem_internal.h"

namespace sem {

namespace {

struct Post {
  const void* a = nullptr;             // input / send buffer
  void* b = nullptr;                   // output / receive buffer
  const int32_t* nbr = nullptr;        // sendrecv: neighbour ranks
  const int64_t* off = nullptr;        // sendrecv: per-neighbour offsets
  int nnbr = 0;
  cudaEvent_t ev = nullptr;
};

__global__ void rank_sum_kernel(const double* __restrict__ stage, int64_t ld, int P, int64_t count,
                                double* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count;
       k += (int64_t)gridDim.x * blockDim.x) {
    double s = stage[k];
    for (int q = 1; q < P; q++) s += stage[q * ld + k];   // ascending rank order
    out[k] = s;
  }
}

}  // namespace

struct LoopWorld {
  int P = 0, flags = 0, timeout_s = 120;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<Post> posts[2];
  double* stage = nullptr;   // [P][stage_ld]: allreduce inputs
  int64_t stage_ld = 0;
  std::vector<LoopComm*> comms;
};

struct LoopComm {
  LoopWorld* w = nullptr;
  int rank = 0;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  std::mt19937 rng;
};

namespace {

std::mutex g_reg_mu;
std::set<const void*> g_registry;   // live LoopComm handles

// host barrier: post this rank's record, return every rank's record of this generation
int barrier(LoopComm* c, const Post& mine, std::vector<Post>* all) {
  LoopWorld* w = c->w;
  if (w->flags & 1) {   // shuffle: random arrival order
    std::uniform_int_distribution<int> d(0, 300);
    std::this_thread::sleep_for(std::chrono::microseconds(d(c->rng)));
  }
  std::unique_lock<std::mutex> lk(w->mu);
  const uint64_t g = w->gen;
  w->posts[g & 1][c->rank] = mine;
  if (++w->arrived == w->P) {
    w->arrived = 0;
    w->gen++;
    w->cv.notify_all();
  } else if (!w->cv.wait_for(lk, std::chrono::seconds(w->timeout_s), [&] { return w->gen != g; })) {
    set_error("loopback: a rank did not reach the collective (timeout)");
    return SEM_ENCCL;
  }
  *all = w->posts[g & 1];
  return SEM_OK;
}

int cuda_ok(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SEM_OK;
  set_error(std::string("loopback ") + what + ": " + cudaGetErrorString(e));
  return SEM_ECUDA;
}

#define LB_TRY(expr)              \
  do {                            \
    int _s = (expr);              \
    if (_s != SEM_OK) return _s;  \
  } while (0)
#define LB_CUDA(expr) LB_TRY(cuda_ok((expr), #expr))

// steps 2-3 of the protocol after the caller's copies / reduction
int finish(LoopComm* c, cudaStream_t s) {
  LB_CUDA(cudaEventRecord(c->ev_out, s));
  Post me;
  me.ev = c->ev_out;
  std::vector<Post> all;
  LB_TRY(barrier(c, me, &all));
  for (int q = 0; q < c->w->P; q++)
    if (q != c->rank) LB_CUDA(cudaStreamWaitEvent(s, all[q].ev, 0));
  return SEM_OK;
}

}  // namespace

LoopComm* loop_lookup(const void* handle) {
  if (!handle) return nullptr;
  std::lock_guard<std::mutex> lk(g_reg_mu);
  return g_registry.count(handle) ? static_cast<LoopComm*>(const_cast<void*>(handle)) : nullptr;
}
int loop_rank(const LoopComm* c) { return c->rank; }
int loop_size(const LoopComm* c) { return c->w->P; }

int loop_sendrecv(LoopComm* c, const double* send, double* recv, const std::vector<int32_t>& nbr,
                  const std::vector<int64_t>& off, const std::vector<int64_t>& cnt,
                  cudaStream_t s) {
  LB_CUDA(cudaEventRecord(c->ev_in, s));
  Post me;
  me.a = send;
  me.nbr = nbr.data();
  me.off = off.data();
  me.nnbr = (int)nbr.size();
  me.ev = c->ev_in;
  std::vector<Post> all;
  LB_TRY(barrier(c, me, &all));
  const int nn = (int)nbr.size();
  for (int t = 0; t < nn; t++) {
    const int k = (c->w->flags & 1) ? nn - 1 - t : t;
    const int q = nbr[k];
    const Post& pq = all[q];
    int kq = -1;   // my position in q's neighbour list
    for (int x = 0; x < pq.nnbr; x++)
      if (pq.nbr[x] == c->rank) kq = x;
    if (kq < 0) {
      set_error("loopback: asymmetric neighbour lists");
      return SEM_ENCCL;
    }
    LB_CUDA(cudaStreamWaitEvent(s, pq.ev, 0));
    LB_CUDA(cudaMemcpyAsync(recv + off[k], static_cast<const double*>(pq.a) + pq.off[kq],
                            sizeof(double) * (size_t)cnt[k], cudaMemcpyDeviceToDevice, s));
  }
  return finish(c, s);
}

int loop_allreduce(LoopComm* c, const double* in, double* out, size_t count, cudaStream_t s) {
  LoopWorld* w = c->w;
  if ((int64_t)count > w->stage_ld) {
    set_error("loopback: allreduce count exceeds the staging buffer");
    return SEM_EINVAL;
  }
  double* mine = w->stage + (int64_t)c->rank * w->stage_ld;
  if (count) LB_CUDA(cudaMemcpyAsync(mine, in, sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
  LB_CUDA(cudaEventRecord(c->ev_in, s));
  Post me;
  me.ev = c->ev_in;
  std::vector<Post> all;
  LB_TRY(barrier(c, me, &all));
  for (int q = 0; q < w->P; q++)
    if (q != c->rank) LB_CUDA(cudaStreamWaitEvent(s, all[q].ev, 0));
  if (count) {
    rank_sum_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(w->stage, w->stage_ld, w->P,
                                                                    (int64_t)count, out);
    LB_CUDA(cudaGetLastError());
  }
  return finish(c, s);
}

int loop_allgather(LoopComm* c, const void* in, void* out, size_t bytes, cudaStream_t s) {
  char* o = static_cast<char*>(out);
  char* mine = o + (size_t)c->rank * bytes;
  if (in != mine && bytes) LB_CUDA(cudaMemcpyAsync(mine, in, bytes, cudaMemcpyDeviceToDevice, s));
  LB_CUDA(cudaEventRecord(c->ev_in, s));
  Post me;
  me.a = mine;
  me.ev = c->ev_in;
  std::vector<Post> all;
  LB_TRY(barrier(c, me, &all));
  for (int q = 0; q < c->w->P; q++) {
    if (q == c->rank) continue;
    LB_CUDA(cudaStreamWaitEvent(s, all[q].ev, 0));
    if (bytes) LB_CUDA(cudaMemcpyAsync(o + (size_t)q * bytes, all[q].a, bytes, cudaMemcpyDeviceToDevice, s));
  }
  return finish(c, s);
}

}  // namespace sem

// ----------------------------------------------------------------- C ABI
extern "C" int sem_loopback_create(int nranks, int flags, void** world) {
  if (!world || nranks < 1 || nranks > 64) {
    sem::set_error("sem_loopback_create: need 1 <= nranks <= 64 and a handle pointer");
    return SEM_EINVAL;
  }
  *world = nullptr;
  sem::LoopWorld* w = new (std::nothrow) sem::LoopWorld();
  if (!w) return SEM_ENOMEM;
  w->P = nranks;
  w->flags = flags;
  if ((flags >> 8) > 0) w->timeout_s = flags >> 8;
  w->posts[0].resize(nranks);
  w->posts[1].resize(nranks);
  w->stage_ld = 4096;   // >= the largest allreduce of the solvers (GMRES: restart + 1)
  if (cudaMalloc(&w->stage, sizeof(double) * nranks * w->stage_ld) != cudaSuccess) {
    cudaGetLastError();
    delete w;
    sem::set_error("sem_loopback_create: cudaMalloc failed");
    return SEM_ECUDA;
  }
  for (int r = 0; r < nranks; r++) {
    sem::LoopComm* c = new sem::LoopComm();
    c->w = w;
    c->rank = r;
    c->rng.seed(1234u + 7u * r);
    if (cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming) != cudaSuccess) {
      sem::set_error("sem_loopback_create: cudaEventCreate failed");
      return SEM_ECUDA;
    }
    w->comms.push_back(c);
    std::lock_guard<std::mutex> lk(sem::g_reg_mu);
    sem::g_registry.insert(c);
  }
  *world = w;
  return SEM_OK;
}

extern "C" int sem_loopback_comm(void* world, int rank, void** comm) {
  sem::LoopWorld* w = static_cast<sem::LoopWorld*>(world);
  if (!w || !comm || rank < 0 || rank >= w->P) {
    sem::set_error("sem_loopback_comm: bad arguments");
    return SEM_EINVAL;
  }
  *comm = w->comms[rank];
  return SEM_OK;
}

extern "C" int sem_loopback_destroy(void* world) {
  sem::LoopWorld* w = static_cast<sem::LoopWorld*>(world);
  if (!w) return SEM_OK;
  cudaDeviceSynchronize();
  for (sem::LoopComm* c : w->comms) {
    {
      std::lock_guard<std::mutex> lk(sem::g_reg_mu);
      sem::g_registry.erase(c);
    }
    cudaEventDestroy(c->ev_in);
    cudaEventDestroy(c->ev_out);
    delete c;
  }
  cudaFree(w->stage);
  delete w;
  return SEM_OK;
}
