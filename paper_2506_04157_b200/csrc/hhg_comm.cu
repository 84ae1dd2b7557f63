// Multi-GPU plumbing: one process per GPU, NCCL over NVLink 5 / NVSwitch.  The unique id is
// created here and broadcast by the caller (torch.distributed), so the library owns its own
// communicator and can put its collectives on its own streams / inside CUDA graphs.
#include "hhg_internal.h"

namespace hhg {
int comm_allreduce_sum(hhg_comm* c, double* buf, int64_t n, cudaStream_t s) {
  if (!c || c->nranks == 1) return HHG_OK;
  ncclResult_t r = ncclAllReduce(buf, buf, (size_t)n, ncclDouble, ncclSum, c->nccl, s);
  if (r != ncclSuccess) return fail(HHG_ENCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
  count_launch();
  return HHG_OK;
}

// Interface exchange of one level/space: every neighbor gets our partial sums of the nodes we share
// (halo.sbuf segment), we receive theirs into the matching halo.rbuf segment.  One NCCL group of
// point-to-point calls; both sides list the shared nodes in the same canonical order.
int comm_exchange(hhg_comm* c, const Halo& h, int nc, const double* sbuf, double* rbuf, cudaStream_t s) {
  if (!c || c->nranks == 1 || h.nbr.empty()) return HHG_OK;
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

int hhg_comm_destroy(hhg_comm* comm) {
  if (!comm) return HHG_OK;
  if (comm->nccl) ncclCommDestroy(comm->nccl);
  delete comm;
  return HHG_OK;
}

}  // extern "C"
