// comm.cu — the transport under the row-partitioned runs: grouped send/recv of halo rows,
// all-reduce of small coefficient blocks, all-gather of the row offsets.
//
// Production transport: NCCL over NVLink / NVSwitch (one process per GPU).
// LOOPBACK transport (tests only, flz_ctx_create_loopback): the ranks are host THREADS of one
// process that share one GPU — NCCL refuses two ranks on one device, and a gpurun box has one
// GPU, so this is how the multi-rank device code (halo packing, halo slots of the planar and
// interleaved blocks, interior / boundary launches, event fencing between the compute and the
// communication stream, replicated host logic) is executed and checked there.  A send posts
// {pointer, bytes, event recorded on the sender's stream}; the matching recv makes the
// receiver's stream wait for that event, copies device to device and posts an event back that
// the sender's stream waits for before the buffer may be reused — the stream ordering NCCL
// gives.  Collectives go through per-rank device slots and host barriers (simple, not fast).
#include <condition_variable>
#include <deque>
#include <mutex>
#include <vector>

#include "flz_internal.hpp"

namespace flz {

struct LoopHub {
  struct Post {
    const void* ptr;
    size_t bytes;
    cudaEvent_t ready;
  };
  int n;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<std::deque<Post>> posts;        // [src * n + dst]
  std::vector<std::deque<cudaEvent_t>> acks;  // [src * n + dst]: receiver's copy is enqueued
  std::vector<double*> slot;                  // per rank, kSlotBytes of device memory
  std::vector<int64_t> gathered;              // all-gather through the host
  int arrived = 0;
  uint64_t generation = 0;
  static constexpr size_t kSlotBytes = 8u << 20;
  explicit LoopHub(int nranks)
      : n(nranks), posts((size_t)nranks * nranks), acks((size_t)nranks * nranks),
        slot(nranks, nullptr), gathered(nranks, 0) {}
  void barrier() {
    std::unique_lock<std::mutex> lock(mu);
    const uint64_t gen = generation;
    if (++arrived == n) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lock, [&] { return generation != gen; });
    }
  }
};

LoopHub* loop_hub_create(int nranks) { return new LoopHub(nranks); }
void loop_hub_destroy(LoopHub* hub) {
  if (!hub) return;
  for (double* p : hub->slot)
    if (p) cudaFree(p);
  delete hub;
}

namespace {

__global__ void loop_sum_kernel(double* out, const double* s0, const double* s1, const double* s2,
                                const double* s3, const double* s4, const double* s5,
                                const double* s6, const double* s7, int n, size_t count) {
  const double* s[8] = {s0, s1, s2, s3, s4, s5, s6, s7};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int r = 0; r < n; ++r) acc += s[r][i];   // rank order: the same sum on every rank
    out[i] = acc;
  }
}

void loop_run(flz_ctx* ctx, std::vector<CommOp>& ops) {
  LoopHub* hub = ctx->hub;
  const int me = ctx->rank, n = hub->n;
  for (CommOp& op : ops) {   // 1: post the sends
    if (!op.send) continue;
    cudaEvent_t ready;
    FLZ_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    FLZ_CUDA(cudaEventRecord(ready, op.stream));
    std::lock_guard<std::mutex> lock(hub->mu);
    hub->posts[(size_t)me * n + op.peer].push_back({op.buf, op.bytes, ready});
    hub->cv.notify_all();
  }
  for (CommOp& op : ops) {   // 2: receive
    if (op.send) continue;
    LoopHub::Post post;
    {
      std::unique_lock<std::mutex> lock(hub->mu);
      auto& q = hub->posts[(size_t)op.peer * n + me];
      hub->cv.wait(lock, [&] { return !q.empty(); });
      post = q.front();
      q.pop_front();
    }
    if (post.bytes != op.bytes)
      throw ApiError(FLZ_ENCCL, "loopback transport: send and recv sizes differ");
    FLZ_CUDA(cudaStreamWaitEvent(op.stream, post.ready, 0));
    FLZ_CUDA(cudaMemcpyAsync(op.buf, post.ptr, op.bytes, cudaMemcpyDeviceToDevice, op.stream));
    cudaEvent_t done;
    FLZ_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    FLZ_CUDA(cudaEventRecord(done, op.stream));
    FLZ_CUDA(cudaEventDestroy(post.ready));
    std::lock_guard<std::mutex> lock(hub->mu);
    hub->acks[(size_t)op.peer * n + me].push_back(done);
    hub->cv.notify_all();
  }
  for (CommOp& op : ops) {   // 3: a send completes (in stream order) when its copy has run
    if (!op.send) continue;
    cudaEvent_t done;
    {
      std::unique_lock<std::mutex> lock(hub->mu);
      auto& q = hub->acks[(size_t)me * n + op.peer];
      hub->cv.wait(lock, [&] { return !q.empty(); });
      done = q.front();
      q.pop_front();
    }
    FLZ_CUDA(cudaStreamWaitEvent(op.stream, done, 0));
    FLZ_CUDA(cudaEventDestroy(done));
  }
}

double* loop_slot(flz_ctx* ctx) {
  LoopHub* hub = ctx->hub;
  if (!hub->slot[ctx->rank]) FLZ_CUDA(cudaMalloc(&hub->slot[ctx->rank], LoopHub::kSlotBytes));
  return hub->slot[ctx->rank];
}

}  // namespace

void comm_group_start(flz_ctx* ctx) {
  if (ctx->hub) {
    ctx->comm_grouped = true;
    ctx->comm_ops.clear();
  } else {
    FLZ_NCCL(ncclGroupStart());
  }
}
void comm_group_end(flz_ctx* ctx) {
  if (ctx->hub) {
    ctx->comm_grouped = false;
    loop_run(ctx, ctx->comm_ops);
    ctx->comm_ops.clear();
  } else {
    FLZ_NCCL(ncclGroupEnd());
  }
}
void comm_send(flz_ctx* ctx, const void* buf, size_t bytes, int peer, cudaStream_t stream) {
  if (ctx->hub) {
    ctx->comm_ops.push_back({true, const_cast<void*>(buf), bytes, peer, stream});
    if (!ctx->comm_grouped) comm_group_end(ctx);
  } else {
    FLZ_NCCL(ncclSend(buf, bytes, ncclChar, peer, ctx->comm, stream));
  }
}
void comm_recv(flz_ctx* ctx, void* buf, size_t bytes, int peer, cudaStream_t stream) {
  if (ctx->hub) {
    ctx->comm_ops.push_back({false, buf, bytes, peer, stream});
    if (!ctx->comm_grouped) comm_group_end(ctx);
  } else {
    FLZ_NCCL(ncclRecv(buf, bytes, ncclChar, peer, ctx->comm, stream));
  }
}

void comm_allreduce_sum(flz_ctx* ctx, double* buf, size_t count, cudaStream_t stream) {
  if (ctx->nranks == 1 || count == 0) return;
  if (!ctx->hub) {
    FLZ_NCCL(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, ctx->comm, stream));
    return;
  }
  LoopHub* hub = ctx->hub;
  if (count * sizeof(double) > LoopHub::kSlotBytes)
    throw ApiError(FLZ_ENCCL, "loopback transport: all-reduce larger than its slot");
  double* mine = loop_slot(ctx);
  FLZ_CUDA(cudaMemcpyAsync(mine, buf, count * sizeof(double), cudaMemcpyDeviceToDevice, stream));
  FLZ_CUDA(cudaStreamSynchronize(stream));
  hub->barrier();   // every slot is filled
  const double* s[8] = {};
  for (int r = 0; r < hub->n && r < 8; ++r) s[r] = hub->slot[r];
  loop_sum_kernel<<<(unsigned)std::min<size_t>(64, (count + 255) / 256), 256, 0, stream>>>(
      buf, s[0], s[1], s[2], s[3], s[4], s[5], s[6], s[7], hub->n, count);
  FLZ_CUDA(cudaGetLastError());
  FLZ_CUDA(cudaStreamSynchronize(stream));
  hub->barrier();   // every slot has been read
}

void comm_allgather_i64(flz_ctx* ctx, const int64_t* d_in, int64_t* d_out, cudaStream_t stream) {
  if (!ctx->hub) {
    FLZ_NCCL(ncclAllGather(d_in, d_out, 1, ncclInt64, ctx->comm, stream));
    return;
  }
  LoopHub* hub = ctx->hub;
  int64_t v = 0;
  FLZ_CUDA(cudaMemcpyAsync(&v, d_in, sizeof v, cudaMemcpyDeviceToHost, stream));
  FLZ_CUDA(cudaStreamSynchronize(stream));
  {
    std::lock_guard<std::mutex> lock(hub->mu);
    hub->gathered[ctx->rank] = v;
  }
  hub->barrier();
  std::vector<int64_t> all;
  {
    std::lock_guard<std::mutex> lock(hub->mu);
    all = hub->gathered;
  }
  FLZ_CUDA(cudaMemcpyAsync(d_out, all.data(), all.size() * sizeof(int64_t), cudaMemcpyHostToDevice,
                           stream));
  FLZ_CUDA(cudaStreamSynchronize(stream));
  hub->barrier();   // nobody overwrites `gathered` before everyone has copied it
}

}  // namespace flz
