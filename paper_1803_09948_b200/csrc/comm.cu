// comm.cu — the multi-GPU data plane of the handle: one process per GPU, Morton-partitioned targets.
//
// Stands in for the reference's simulated-rank layer (part::distributed_matvec, src/let.cpp:320-362):
// its sender-initiated locally essential trees (extract_let, let.cpp:150-253; graft_let, :255-318) become
// two exchanges per matvec — the bodies of the leaves a peer sums directly, and the multipoles of the
// cells a peer translates from — with index lists fixed at setup:
//
//      pack kernel -> ONE grouped ncclSend / ncclRecv over all peers -> unpack kernel
//
// on a communication stream of its own, overlapped with the work that does not need the remote rows:
//
//   main stream   own charges -> pack q ........ P2M + M2M (own cells) -> pack M ............ M2L -> L2L -> L2P
//   comm stream                   exchange q                               exchange M
//   near stream                              unpack q -> P2P of the owned leaves (beside the M exchange and M2L)
//
// GMRES inner products are device-side: the local FP64 partial is all-reduced in place on the main
// stream (ncclAllReduce on the scalars the next kernel reads), no host round trip per coefficient.
//
// NCCL is loaded at run time (dlopen of libnccl.so.2): a single-GPU user needs no NCCL at all, and a host
// that already carries one (torch) shares it.  A second transport moves the same packed buffers through
// pinned host memory and two caller callbacks (all-to-all-v and all-reduce on HOST buffers): that is the
// MPI escape hatch, and it is what lets two processes share one GPU in the tests (NCCL refuses two ranks
// on one device) — everything but the ncclSend / ncclRecv calls themselves is the code under test.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <numeric>

#include "engine.hpp"

namespace hfmm_b200 {

// ---- NCCL through dlopen -------------------------------------------------------------------------
struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (a.lib) break;
    }
    if (!a.lib) throw Error(HFMM_ERR_DEVICE, std::string("libnccl.so.2 cannot be loaded: ") + dlerror());
    auto sym = [&](const char* n) {
      void* p = dlsym(a.lib, n);
      if (!p) throw Error(HFMM_ERR_DEVICE, std::string("NCCL symbol missing: ") + n);
      return p;
    };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(sym("ncclBroadcast"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    return a;
  }();
  return api;
}

#define HFMM_NCCL_CHECK(expr)                                                                         \
  do {                                                                                                \
    ncclResult_t r__ = (expr);                                                                        \
    if (r__ != ncclSuccess)                                                                           \
      throw ::hfmm_b200::Error(HFMM_ERR_DEVICE, std::string(#expr) + ": " + nccl().GetErrorString(r__)); \
  } while (0)

void nccl_unique_id(void* out128) {
  ncclUniqueId id;
  HFMM_NCCL_CHECK(nccl().GetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof(id));
}

// ---- transports ----------------------------------------------------------------------------------
struct Engine::Transport {
  virtual ~Transport() = default;
  // rows of `elem_bytes` each: send[soff[p] .. soff[p+1]) goes to peer p, recv[roff[p] .. roff[p+1]) comes
  // from peer p; device buffers; enqueued on `s` (ordered after earlier work on s)
  virtual void alltoallv(const void* send, const std::vector<uint64_t>& soff, void* recv,
                         const std::vector<uint64_t>& roff, size_t elem_bytes, cudaStream_t s) = 0;
  // in-place sum over the ranks of `count` doubles in device memory, ordered on s
  virtual void allreduce(double* dev, int count, cudaStream_t s) = 0;
  // every rank contributes full[first[p] .. first[p] + count[p]) (float2 elements): all-gather in place
  virtual void allgather(float2* full, const std::vector<uint64_t>& first, const std::vector<uint64_t>& count,
                         cudaStream_t s) = 0;
  virtual const char* name() const = 0;
};

namespace {

struct NcclTransport final : Engine::Transport {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  ~NcclTransport() override {
    if (comm) nccl().CommDestroy(comm);
  }
  void alltoallv(const void* send, const std::vector<uint64_t>& soff, void* recv, const std::vector<uint64_t>& roff,
                 size_t elem_bytes, cudaStream_t s) override {
    // one group: every send and receive of this exchange progresses together (no ordering deadlocks)
    HFMM_NCCL_CHECK(nccl().GroupStart());
    for (int p = 0; p < nranks; ++p) {
      if (p == rank) continue;
      const uint64_t ns = soff[p + 1] - soff[p], nr = roff[p + 1] - roff[p];
      if (ns)
        HFMM_NCCL_CHECK(nccl().Send(static_cast<const char*>(send) + soff[p] * elem_bytes, ns * elem_bytes / 4,
                                    ncclFloat32, p, comm, s));
      if (nr)
        HFMM_NCCL_CHECK(nccl().Recv(static_cast<char*>(recv) + roff[p] * elem_bytes, nr * elem_bytes / 4, ncclFloat32,
                                    p, comm, s));
    }
    HFMM_NCCL_CHECK(nccl().GroupEnd());
  }
  void allreduce(double* dev, int count, cudaStream_t s) override {
    HFMM_NCCL_CHECK(nccl().AllReduce(dev, dev, size_t(count), ncclFloat64, ncclSum, comm, s));
  }
  void allgather(float2* full, const std::vector<uint64_t>& first, const std::vector<uint64_t>& count,
                 cudaStream_t s) override {
    HFMM_NCCL_CHECK(nccl().GroupStart());
    for (int p = 0; p < nranks; ++p)
      if (count[p])
        HFMM_NCCL_CHECK(nccl().Broadcast(full + first[p], full + first[p], 2 * count[p], ncclFloat32, p, comm, s));
    HFMM_NCCL_CHECK(nccl().GroupEnd());
  }
  const char* name() const override { return "nccl"; }
};

// packed buffers staged through pinned host memory, the collectives performed by the caller
struct HostTransport final : Engine::Transport {
  hfmm_host_transport cb{};
  int rank = 0, nranks = 1;
  void *h_send = nullptr, *h_recv = nullptr;
  size_t cap_send = 0, cap_recv = 0;
  ~HostTransport() override {
    if (h_send) cudaFreeHost(h_send);
    if (h_recv) cudaFreeHost(h_recv);
  }
  static void reserve(void*& p, size_t& cap, size_t bytes) {
    if (bytes <= cap) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    HFMM_CUDA_CHECK(cudaMallocHost(&p, bytes));
    cap = bytes;
  }
  void alltoallv(const void* send, const std::vector<uint64_t>& soff, void* recv, const std::vector<uint64_t>& roff,
                 size_t elem_bytes, cudaStream_t s) override {
    const size_t sb = soff[nranks] * elem_bytes, rb = roff[nranks] * elem_bytes;
    reserve(h_send, cap_send, std::max<size_t>(sb, 16));
    reserve(h_recv, cap_recv, std::max<size_t>(rb, 16));
    if (sb) HFMM_CUDA_CHECK(cudaMemcpyAsync(h_send, send, sb, cudaMemcpyDeviceToHost, s));
    HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
    std::vector<uint64_t> sbytes(nranks), rbytes(nranks);
    for (int p = 0; p < nranks; ++p) {
      sbytes[p] = (soff[p + 1] - soff[p]) * elem_bytes;
      rbytes[p] = (roff[p + 1] - roff[p]) * elem_bytes;
    }
    if (cb.alltoallv(cb.user, h_send, sbytes.data(), h_recv, rbytes.data()) != 0)
      throw Error(HFMM_ERR_DEVICE, "host transport: all-to-all callback failed");
    if (rb) HFMM_CUDA_CHECK(cudaMemcpyAsync(recv, h_recv, rb, cudaMemcpyHostToDevice, s));
  }
  void allreduce(double* dev, int count, cudaStream_t s) override {
    std::vector<double> v(count);
    HFMM_CUDA_CHECK(cudaMemcpyAsync(v.data(), dev, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
    HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
    if (cb.allreduce_sum(cb.user, v.data(), count) != 0)
      throw Error(HFMM_ERR_DEVICE, "host transport: all-reduce callback failed");
    HFMM_CUDA_CHECK(cudaMemcpyAsync(dev, v.data(), sizeof(double) * count, cudaMemcpyHostToDevice, s));
    HFMM_CUDA_CHECK(cudaStreamSynchronize(s));  // v leaves scope
  }
  void allgather(float2* full, const std::vector<uint64_t>& first, const std::vector<uint64_t>& count,
                 cudaStream_t s) override {
    // my slice to every peer, every peer's slice to me: an all-to-all-v with one repeated send block
    const uint64_t mine = count[rank];
    std::vector<uint64_t> soff(nranks + 1, 0), roff(nranks + 1, 0);
    for (int p = 0; p < nranks; ++p) {
      soff[p + 1] = soff[p] + (p == rank ? 0 : mine);
      roff[p + 1] = roff[p] + (p == rank ? 0 : count[p]);
    }
    const size_t sb = soff[nranks] * sizeof(float2), rb = roff[nranks] * sizeof(float2);
    reserve(h_send, cap_send, std::max<size_t>(sb, 16));
    reserve(h_recv, cap_recv, std::max<size_t>(rb, 16));
    for (int p = 0; p < nranks; ++p)
      if (p != rank && mine)
        HFMM_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(h_send) + soff[p] * sizeof(float2), full + first[rank],
                                        mine * sizeof(float2), cudaMemcpyDeviceToHost, s));
    HFMM_CUDA_CHECK(cudaStreamSynchronize(s));
    std::vector<uint64_t> sbytes(nranks), rbytes(nranks);
    for (int p = 0; p < nranks; ++p) {
      sbytes[p] = (soff[p + 1] - soff[p]) * sizeof(float2);
      rbytes[p] = (roff[p + 1] - roff[p]) * sizeof(float2);
    }
    if (cb.alltoallv(cb.user, h_send, sbytes.data(), h_recv, rbytes.data()) != 0)
      throw Error(HFMM_ERR_DEVICE, "host transport: all-to-all callback failed");
    for (int p = 0; p < nranks; ++p)
      if (p != rank && count[p])
        HFMM_CUDA_CHECK(cudaMemcpyAsync(full + first[p], static_cast<char*>(h_recv) + roff[p] * sizeof(float2),
                                        count[p] * sizeof(float2), cudaMemcpyHostToDevice, s));
  }
  const char* name() const override { return "host callbacks"; }
};

// ---- pack / unpack: rows of `width` float2 gathered from / scattered to the rows idx[i] --------------
__global__ void __launch_bounds__(256)
gather_rows_kernel(const float2* __restrict__ src, const uint32_t* __restrict__ idx, uint64_t n_rows, uint32_t width,
                   uint32_t src_stride, float2* __restrict__ out) {
  const uint64_t total = n_rows * width;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = i / width;
    const uint32_t c = uint32_t(i - r * width);
    out[i] = src[uint64_t(idx[r]) * src_stride + c];
  }
}
__global__ void __launch_bounds__(256)
scatter_rows_kernel(const float2* __restrict__ in, const uint32_t* __restrict__ idx, uint64_t n_rows, uint32_t width,
                    uint32_t dst_stride, float2* __restrict__ dst) {
  const uint64_t total = n_rows * width;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = i / width;
    const uint32_t c = uint32_t(i - r * width);
    dst[uint64_t(idx[r]) * dst_stride + c] = in[i];
  }
}
inline unsigned grid_of(uint64_t total) { return unsigned(std::min<uint64_t>((total + 255) / 256, 148 * 16)); }

}  // namespace

struct Engine::ExchangePlan {
  // per peer offsets into the packed buffers (rows), nranks + 1 entries each
  std::vector<uint64_t> cell_soff, cell_roff, body_soff, body_roff;
  DeviceBuffer<uint32_t> send_cells, recv_cells, send_slots, recv_slots;  // row indices, peers concatenated
  DeviceBuffer<float2> send_buf, recv_buf;                                // sized for the larger exchange
  std::vector<uint64_t> slice_first, slice_count;                         // Morton body ranges of all ranks
  cudaStream_t stream = nullptr;                                          // communication stream
  cudaEvent_t ev_q_packed = nullptr, ev_q_here = nullptr, ev_m_packed = nullptr, ev_m_here = nullptr;
  ~ExchangePlan() {
    for (cudaEvent_t e : {ev_q_packed, ev_q_here, ev_m_packed, ev_m_here})
      if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
  }
};

void Engine::release_comm() {
  exchange_.reset();
  transport_.reset();
}

void Engine::comm_init_nccl(const void* unique_id_128) {
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  if (!unique_id_128) throw Error(HFMM_ERR_CONFIG, "null NCCL unique id");
  auto t = std::make_shared<NcclTransport>();
  t->rank = rank_;
  t->nranks = nranks_;
  ncclUniqueId id;
  std::memcpy(&id, unique_id_128, sizeof(id));
  HFMM_NCCL_CHECK(nccl().CommInitRank(&t->comm, nranks_, id, rank_));
  transport_ = t;
  exchange_.reset();
}

void Engine::comm_init_host(const hfmm_host_transport& cb) {
  if (!cb.alltoallv || !cb.allreduce_sum) throw Error(HFMM_ERR_CONFIG, "host transport needs both callbacks");
  auto t = std::make_shared<HostTransport>();
  t->rank = rank_;
  t->nranks = nranks_;
  t->cb = cb;
  transport_ = t;
  exchange_.reset();
}

const char* Engine::comm_name() const { return transport_ ? transport_->name() : "none"; }

// Index lists of the locally-essential-tree exchange (let.cpp:150-253, sender-initiated): every rank holds
// all pairs of the global walk into and out of its own cells, so "my cells peer p translates from" here equals
// "the cells of mine that p expects" there, element for element (ascending cell order) — no handshake.
void Engine::build_exchange_plan() {
  require_points();
  if (!transport_) throw Error(HFMM_ERR_CONFIG, "no communicator: call hfmm_cuda_comm_init_nccl / _host first");
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  const size_t nc = tree_.n_cells();
  std::vector<uint64_t> far(nc), near(nc);
  std::vector<int32_t> owner(nc);
  get_exchange_masks(far.data(), near.data(), owner.data());
  auto plan = std::make_shared<ExchangePlan>();
  const int R = nranks_;
  const uint64_t me = uint64_t(1) << rank_;
  std::vector<uint32_t> sc, rc, ss, rs;
  plan->cell_soff.assign(R + 1, 0);
  plan->cell_roff.assign(R + 1, 0);
  plan->body_soff.assign(R + 1, 0);
  plan->body_roff.assign(R + 1, 0);
  for (int p = 0; p < R; ++p) {
    if (p != rank_) {
      const uint64_t bit = uint64_t(1) << p;
      for (uint32_t c = 0; c < nc; ++c) {
        if (owner[c] == rank_) {
          if (far[c] & bit) sc.push_back(c);
          if (near[c] & bit)
            for (uint32_t b = 0; b < tree_.body_count[c]; ++b) ss.push_back(tree_.body_first[c] + b);
        } else if (owner[c] == p) {
          if (far[c] & me) rc.push_back(c);
          if (near[c] & me)
            for (uint32_t b = 0; b < tree_.body_count[c]; ++b) rs.push_back(tree_.body_first[c] + b);
        }
      }
    }
    plan->cell_soff[p + 1] = sc.size();
    plan->cell_roff[p + 1] = rc.size();
    plan->body_soff[p + 1] = ss.size();
    plan->body_roff[p + 1] = rs.size();
  }
  plan->send_cells.upload(sc, stream_);
  plan->recv_cells.upload(rc, stream_);
  plan->send_slots.upload(ss, stream_);
  plan->recv_slots.upload(rs, stream_);
  const uint32_t dim = uint32_t(nm_total(cfg_.order));
  plan->send_buf.resize(std::max<uint64_t>({uint64_t(sc.size()) * dim, uint64_t(ss.size()), 1}));
  plan->recv_buf.resize(std::max<uint64_t>({uint64_t(rc.size()) * dim, uint64_t(rs.size()), 1}));
  // Morton slices of every rank (partition cuts are the same on all ranks: same global lists)
  plan->slice_first.assign(R, 0);
  plan->slice_count.assign(R, 0);
  {
    std::vector<uint64_t> lo(R, ~uint64_t(0)), hi(R, 0);
    for (uint32_t c : tree_.leaves) {
      const int o = owner[c];
      if (o < 0 || o >= R || !tree_.body_count[c]) continue;
      lo[o] = std::min<uint64_t>(lo[o], tree_.body_first[c]);
      hi[o] = std::max<uint64_t>(hi[o], uint64_t(tree_.body_first[c]) + tree_.body_count[c]);
    }
    for (int p = 0; p < R; ++p)
      if (hi[p] > 0 && lo[p] != ~uint64_t(0)) {
        plan->slice_first[p] = lo[p];
        plan->slice_count[p] = hi[p] - lo[p];
      }
  }
  HFMM_CUDA_CHECK(cudaStreamCreateWithFlags(&plan->stream, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&plan->ev_q_packed, &plan->ev_q_here, &plan->ev_m_packed, &plan->ev_m_here})
    HFMM_CUDA_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  HFMM_CUDA_CHECK(cudaStreamSynchronize(stream_));
  exchange_ = plan;
  exchange_bytes_[0] = rs.size() * sizeof(float2);
  exchange_bytes_[1] = uint64_t(rc.size()) * dim * sizeof(float2);
}

void Engine::get_exchange_volume(uint64_t* charge_bytes, uint64_t* multipole_bytes) {
  if (!exchange_) build_exchange_plan();
  *charge_bytes = exchange_bytes_[0];
  *multipole_bytes = exchange_bytes_[1];
}

// One distributed FMM evaluation.  body_q_ holds this rank's charges in its owned Morton slots (the other
// slots are stale); on return near_ / far_ hold the potentials of the owned slots.
void Engine::dist_far_and_near() {
  if (nranks_ == 1 && !transport_) {  // a world of one without a communicator: nothing to exchange
    run_far_and_near();
    return;
  }
  if (!exchange_) build_exchange_plan();
  ExchangePlan& x = *exchange_;
  const int R = nranks_;
  const uint32_t dim = uint32_t(nm_total(cfg_.order));
  const bool host = std::strcmp(transport_->name(), "nccl") != 0;
  cudaStream_t cs = x.stream;

  // charges the peers sum directly: pack -> exchange (comm stream) -> unpack (near stream)
  if (x.body_soff[R])
    gather_rows_kernel<<<grid_of(x.body_soff[R]), 256, 0, stream_>>>(body_q_.get(), x.send_slots.get(), x.body_soff[R], 1,
                                                                     1, x.send_buf.get());
  HFMM_CUDA_CHECK(cudaGetLastError());
  HFMM_CUDA_CHECK(cudaEventRecord(x.ev_q_packed, stream_));
  HFMM_CUDA_CHECK(cudaStreamWaitEvent(cs, x.ev_q_packed, 0));
  transport_->alltoallv(x.send_buf.get(), x.body_soff, x.recv_buf.get(), x.body_roff, sizeof(float2), cs);
  if (x.body_roff[R])
    scatter_rows_kernel<<<grid_of(x.body_roff[R]), 256, 0, cs>>>(x.recv_buf.get(), x.recv_slots.get(), x.body_roff[R], 1, 1,
                                                                 body_q_.get());
  HFMM_CUDA_CHECK(cudaGetLastError());
  HFMM_CUDA_CHECK(cudaEventRecord(x.ev_q_here, cs));

  // own upward pass beside the charge exchange (P2M / M2M read the owned charges only); the near field is
  // held back until the halo charges are in place
  near_gate_ = x.ev_q_here;
  phase_upward();

  if (have_far_) {
    // the send buffer is reused: the charge exchange must have consumed it
    HFMM_CUDA_CHECK(cudaStreamWaitEvent(stream_, x.ev_q_here, 0));
    if (x.cell_soff[R])
      gather_rows_kernel<<<grid_of(x.cell_soff[R] * dim), 256, 0, stream_>>>(multipole_.get(), x.send_cells.get(),
                                                                             x.cell_soff[R], dim, uint32_t(stride_),
                                                                             x.send_buf.get());
    HFMM_CUDA_CHECK(cudaGetLastError());
    HFMM_CUDA_CHECK(cudaEventRecord(x.ev_m_packed, stream_));
    HFMM_CUDA_CHECK(cudaStreamWaitEvent(cs, x.ev_m_packed, 0));
    transport_->alltoallv(x.send_buf.get(), x.cell_soff, x.recv_buf.get(), x.cell_roff, size_t(dim) * sizeof(float2), cs);
    if (x.cell_roff[R])
      scatter_rows_kernel<<<grid_of(x.cell_roff[R] * dim), 256, 0, cs>>>(x.recv_buf.get(), x.recv_cells.get(),
                                                                         x.cell_roff[R], dim, uint32_t(stride_),
                                                                         multipole_.get());
    HFMM_CUDA_CHECK(cudaGetLastError());
    HFMM_CUDA_CHECK(cudaEventRecord(x.ev_m_here, cs));
    HFMM_CUDA_CHECK(cudaStreamWaitEvent(stream_, x.ev_m_here, 0));
  }
  (void)host;
  phase_downward();
  near_gate_ = nullptr;
}

// distributed plain FMM matvec on owned Morton slices (device float2 in, device float2 out)
void Engine::dist_matvec(const void* q_owned_dev, void* out_owned_dev) {
  require_points();
  HFMM_CUDA_CHECK(cudaSetDevice(cfg_.device));
  HFMM_CUDA_CHECK(cudaEventRecord(ev_[8], stream_));
  if (own_count_)
    HFMM_CUDA_CHECK(cudaMemcpyAsync(body_q_.get() + own_first_, q_owned_dev, size_t(own_count_) * sizeof(float2),
                                    cudaMemcpyDeviceToDevice, stream_));
  dist_far_and_near();
  launch_combine_owned(near_.get() + own_first_, far_.get() + own_first_, nullptr, body_index_.get() + own_first_,
                       static_cast<float2*>(out_owned_dev), own_count_, stream_);
  HFMM_CUDA_CHECK(cudaEventRecord(ev_[9], stream_));
}

void Engine::comm_allreduce(double* dev, int count) {
  if (transport_) transport_->allreduce(dev, count, stream_);  // also in a world of one: the path is the same
}

void Engine::comm_allgather_morton(float2* full) {
  if (!transport_) return;
  if (!exchange_) build_exchange_plan();
  transport_->allgather(full, exchange_->slice_first, exchange_->slice_count, stream_);
}

}  // namespace hfmm_b200
