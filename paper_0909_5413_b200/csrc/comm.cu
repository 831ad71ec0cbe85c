// comm.cu -- strip halos and scalar reductions over NCCL.
//
// The paper's ghost-vector scatters become two point-to-point
// exchanges with the strip neighbours per operator application: ceil(rc/c) cell
// rows for the matvec ("limited to a constant number of elements in the
// vicinity") and overlap_rings rows for RASM.  GMRES inner products are
// reduced by an all-gather of the per-rank partials summed in rank order, so every
// rank holds bit-identical scalars and runs are deterministic (reading Q14).
#include "common.cuh"

namespace rbf {

int comm_init(rbf_ctx *c, const rbf_dist *d) {
  if (c->nranks <= 1 || c->comm_mode != RBF_COMM_NCCL) return RBF_OK;
  ncclUniqueId id;
  static_assert(sizeof(id.internal) == 128, "nccl id size");
  memcpy(id.internal, d->nccl_id, 128);
  RBF_NCCL_TRY(ncclCommInitRank(&c->nccl, c->nranks, id, c->rank));
  return RBF_OK;
}

void comm_destroy(rbf_ctx *c) {
  if (c->nccl) {
    ncclCommDestroy(c->nccl);
    c->nccl = nullptr;
  }
}

int halo_exchange(rbf_ctx *c, const double *v_loc, double *v_ext, bool matvec_depth,
                  cudaStream_t s) {
  if (c->nranks <= 1) return RBF_OK;
  if (c->comm_mode != RBF_COMM_NCCL) {
    set_error("virtual strip context (RBF_COMM_NONE) has no communicator: use the *_ext calls");
    return RBF_EUNSUPPORTED;
  }
  const long long own_off = c->s.own_lo - c->s.ext_lo;
  RBF_CUDA_TRY(cudaMemcpyAsync(v_ext + own_off, v_loc, sizeof(double) * n_loc(c),
                               cudaMemcpyDeviceToDevice, s));
  const Halo *h = matvec_depth ? c->halo_mv : c->halo_pc;
  RBF_NCCL_TRY(ncclGroupStart());
  for (int dir = 0; dir < 2; ++dir) {
    const int peer = dir == 0 ? c->rank - 1 : c->rank + 1;
    if (peer < 0 || peer >= c->nranks) continue;
    if (h[dir].send_cnt > 0)
      RBF_NCCL_TRY(ncclSend(v_loc + h[dir].send_off, (size_t)h[dir].send_cnt, ncclDouble, peer,
                            c->nccl, s));
    if (h[dir].recv_cnt > 0)
      RBF_NCCL_TRY(ncclRecv(v_ext + h[dir].recv_off, (size_t)h[dir].recv_cnt, ncclDouble, peer,
                            c->nccl, s));
  }
  RBF_NCCL_TRY(ncclGroupEnd());
  return RBF_OK;
}

int allgather_scalars(rbf_ctx *c, const double *send, double *recv, int count, cudaStream_t s) {
  if (c->nranks <= 1) return RBF_OK;  // single rank: recv aliases send
  if (c->comm_mode != RBF_COMM_NCCL) {
    set_error("virtual strip context (RBF_COMM_NONE) cannot reduce across strips");
    return RBF_EUNSUPPORTED;
  }
  RBF_NCCL_TRY(ncclAllGather(send, recv, (size_t)count, ncclDouble, c->nccl, s));
  return RBF_OK;
}

}  // namespace rbf
