// Multi-GPU plumbing: one process per GPU, NCCL over NVLink 5 / NVSwitch.  The unique id is
// created here and broadcast by the caller (torch.distributed), so the library owns its own
// communicator and can put its collectives on its own streams / inside CUDA graphs.
#include <algorithm>

#include "hhg_internal.h"

namespace hhg {
// Host-staged transport (hhg_comm_create_host): the stream is drained, the device buffer copied to
// pinned host memory, the caller's callback moves the data between processes (e.g. a gloo process
// group), the result copied back.  Correct by construction for any number of ranks sharing a GPU (no
// kernel ever waits on another rank), not capturable into a CUDA graph (callers check comm_capturable).
static int host_stage(hhg_comm* c, size_t n) {
  if (c->hcap >= n) return HHG_OK;
  if (c->hbuf) cudaFreeHost(c->hbuf);
  c->hbuf = nullptr;
  c->hcap = 0;
  HHG_CUDA(cudaMallocHost(&c->hbuf, 2 * std::max<size_t>(n, 1) * sizeof(double)));
  c->hcap = n;
  return HHG_OK;
}

bool comm_capturable(const hhg_comm* c) { return !c || c->nranks == 1 || !c->host; }

int comm_allreduce_sum(hhg_comm* c, double* buf, int64_t n, cudaStream_t s) {
  if (!c || c->nranks == 1) return HHG_OK;
  if (c->host) {
    HHG_TRY(host_stage(c, (size_t)n));
    HHG_CUDA(cudaMemcpyAsync(c->hbuf, buf, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    HHG_CUDA(cudaStreamSynchronize(s));
    if (c->allreduce_fn(c->user, c->hbuf, n) != 0) return fail(HHG_ENCCL, "host transport: allreduce callback failed");
    HHG_CUDA(cudaMemcpyAsync(buf, c->hbuf, n * sizeof(double), cudaMemcpyHostToDevice, s));
    HHG_CUDA(cudaStreamSynchronize(s));
    return HHG_OK;
  }
  ncclResult_t r = ncclAllReduce(buf, buf, (size_t)n, ncclDouble, ncclSum, c->nccl, s);
  if (r != ncclSuccess) return fail(HHG_ENCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
  count_launch();
  return HHG_OK;
}

// Interface exchange of one level/space: every neighbor gets our partial sums of the nodes we share
// (halo.sbuf segment), we receive theirs into the matching halo.rbuf segment.  One NCCL group of
// point-to-point calls; both sides list the shared nodes in the same canonical order.
int comm_exchange(hhg_comm* c, const Halo& h, int nc, const double* sbuf, double* rbuf, cudaStream_t s) {
  if (!c || c->nranks == 1) return HHG_OK;
  if (c->host) {  // every rank calls the callback (also without neighbours): it may be collective
    const size_t n = (size_t)h.nslots * nc;
    HHG_TRY(host_stage(c, n));
    double* hs = c->hbuf;
    double* hr = c->hbuf + c->hcap;
    if (n) HHG_CUDA(cudaMemcpyAsync(hs, sbuf, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    HHG_CUDA(cudaStreamSynchronize(s));
    std::vector<int> nbr(h.nbr.begin(), h.nbr.end());
    std::vector<int64_t> off(h.off.begin(), h.off.end());
    if (off.empty()) off.push_back(0);
    if (c->exchange_fn(c->user, (int)nbr.size(), nbr.data(), off.data(), nc, hs, hr) != 0)
      return fail(HHG_ENCCL, "host transport: exchange callback failed");
    if (n) HHG_CUDA(cudaMemcpyAsync(rbuf, hr, n * sizeof(double), cudaMemcpyHostToDevice, s));
    HHG_CUDA(cudaStreamSynchronize(s));
    return HHG_OK;
  }
  if (h.nbr.empty()) return HHG_OK;
  ncclResult_t r = ncclGroupStart();
  for (size_t i = 0; i < h.nbr.size() && r == ncclSuccess; ++i) {
    const size_t cnt = (size_t)(h.off[i + 1] - h.off[i]) * nc;
    r = ncclSend(sbuf + h.off[i] * nc, cnt, ncclDouble, h.nbr[i], c->nccl, s);
    if (r == ncclSuccess) r = ncclRecv(rbuf + h.off[i] * nc, cnt, ncclDouble, h.nbr[i], c->nccl, s);
  }
  ncclResult_t r2 = ncclGroupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess)
    return fail(HHG_ENCCL, std::string("interface exchange: ") + ncclGetErrorString(r != ncclSuccess ? r : r2));
  count_launch();
  return HHG_OK;
}
}  // namespace hhg

using namespace hhg;

extern "C" {

int hhg_comm_unique_id(uint8_t id[128]) {
  if (!id) return fail(HHG_EINVAL, "NULL id");
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) return fail(HHG_ENCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(id, &u, 128);
  return HHG_OK;
}

int hhg_comm_create(const uint8_t id[128], int nranks, int rank, int device, hhg_comm** out) {
  if (!id || !out) return fail(HHG_EINVAL, "NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(HHG_EINVAL, "bad rank / nranks");
  HHG_CUDA(cudaSetDevice(device));
  auto* c = new hhg_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  ncclUniqueId u;
  memcpy(&u, id, 128);
  ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(HHG_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  *out = c;
  return HHG_OK;
}

int hhg_comm_create_host(int nranks, int rank, hhg_exchange_fn exchange, hhg_allreduce_fn allreduce, void* user,
                         hhg_comm** out) {
  if (!exchange || !allreduce || !out) return fail(HHG_EINVAL, "hhg_comm_create_host: NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(HHG_EINVAL, "bad rank / nranks");
  auto* c = new hhg_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->host = true;
  c->exchange_fn = exchange;
  c->allreduce_fn = allreduce;
  c->user = user;
  if (cudaGetDevice(&c->device) != cudaSuccess) c->device = 0;
  *out = c;
  return HHG_OK;
}

int hhg_comm_destroy(hhg_comm* comm) {
  if (!comm) return HHG_OK;
  if (comm->hbuf) cudaFreeHost(comm->hbuf);
  if (comm->nccl) ncclCommDestroy(comm->nccl);
  delete comm;
  return HHG_OK;
}

}  // extern "C"
