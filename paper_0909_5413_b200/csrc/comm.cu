// comm.cu -- strip halos and scalar reductions over NCCL.
//
// The paper's ghost-vector scatters become two point-to-point
// exchanges with the strip neighbours per operator application: ceil(rc/c) cell
// rows for the matvec ("limited to a constant number of elements in the
// vicinity") and overlap_rings rows for RASM.  GMRES inner products are
// reduced by an all-gather of the per-rank partials summed in rank order, so every
// rank holds bit-identical scalars and runs are deterministic (reading Q14).
//
// RBF_COMM_THREADS is a second transport with the same semantics for contexts that
// live in ONE process on ONE device, one host thread per strip: every exchange is a
// device-to-device copy out of the peer context's buffers, ordered by stream
// synchronisations and a host barrier (no kernel ever waits on another context).
// It exists so the multi-strip solve (halo plans, reduction order, control flow) can
// be run and checked on a single GPU; it is not a performance path.
#include "common.cuh"

#include <condition_variable>
#include <map>
#include <mutex>
#include <string>
#include <vector>

namespace rbf {

struct ThreadGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<const double *> ptr[2];  // published per rank
  std::vector<long long> cnt[2];

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

static std::mutex g_groups_mu;
static std::map<std::string, ThreadGroup *> g_groups;  // process lifetime (test transport)

static int thread_group_join(rbf_ctx *c, const rbf_dist *d) {
  const std::string key(reinterpret_cast<const char *>(d->nccl_id), 128);
  std::lock_guard<std::mutex> lk(g_groups_mu);
  ThreadGroup *&g = g_groups[key];
  if (!g) {
    g = new ThreadGroup();
    g->n = c->nranks;
    for (int k = 0; k < 2; ++k) {
      g->ptr[k].assign(c->nranks, nullptr);
      g->cnt[k].assign(c->nranks, 0);
    }
  }
  if (g->n != c->nranks) {
    set_error("RBF_COMM_THREADS: group key already used with %d ranks (this context: %d)", g->n,
              c->nranks);
    return RBF_EINVAL;
  }
  c->tgroup = g;
  return RBF_OK;
}

// NCCL communicators, one per unique id per process.  An ncclUniqueId seeds exactly one
// communicator (its bootstrap root serves one ncclCommInitRank round), so contexts set
// up later with the same id -- e.g. one context per benchmark step -- reuse the
// communicator instead of re-initialising from a spent id (which would hang), and the
// communicator's creation cost is paid once.  They live until the process exits.
struct NcclEntry {
  ncclComm_t comm;
  int rank, nranks, device;
};
static std::mutex g_nccl_mu;
static std::map<std::string, NcclEntry> g_nccl;

int comm_init(rbf_ctx *c, const rbf_dist *d) {
  if (c->nranks <= 1) return RBF_OK;
  if (c->comm_mode == RBF_COMM_THREADS) return thread_group_join(c, d);
  if (c->comm_mode != RBF_COMM_NCCL) return RBF_OK;
  // the halo exchange runs on its own stream, at the highest priority, so the NCCL kernel
  // gets SMs while the interior work fills the GPU
  int lo = 0, hi = 0;
  RBF_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  RBF_CUDA_TRY(cudaStreamCreateWithPriority(&c->s_comm, cudaStreamNonBlocking, hi));
  RBF_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
  RBF_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
  const std::string key(reinterpret_cast<const char *>(d->nccl_id), 128);
  int dev = 0;
  RBF_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  auto it = g_nccl.find(key);
  if (it != g_nccl.end()) {
    const NcclEntry &e = it->second;
    if (e.rank != c->rank || e.nranks != c->nranks || e.device != dev) {
      set_error("rbf_setup: nccl_id already seeded a communicator as rank %d of %d on device %d "
                "(this context: rank %d of %d on device %d)", e.rank, e.nranks, e.device, c->rank,
                c->nranks, dev);
      return RBF_EINVAL;
    }
    c->nccl = e.comm;
    return RBF_OK;
  }
  ncclUniqueId id;
  static_assert(sizeof(id.internal) == 128, "nccl id size");
  memcpy(id.internal, d->nccl_id, 128);
  RBF_NCCL_TRY(ncclCommInitRank(&c->nccl, c->nranks, id, c->rank));
  g_nccl[key] = NcclEntry{c->nccl, c->rank, c->nranks, dev};
  return RBF_OK;
}

void comm_destroy(rbf_ctx *c) {
  c->nccl = nullptr;  // the communicator stays with its id (process lifetime, above)
  if (c->s_comm) cudaStreamSynchronize(c->s_comm);
  if (c->ev_in) cudaEventDestroy(c->ev_in);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  if (c->s_comm) cudaStreamDestroy(c->s_comm);
  c->ev_in = c->ev_halo = nullptr;
  c->s_comm = nullptr;
}

// RBF_COMM_THREADS exchange: publish this rank's send regions, copy the peers'.
static int halo_exchange_threads(rbf_ctx *c, const double *v_loc, double *v_ext, const Halo *h,
                                 cudaStream_t s) {
  ThreadGroup *G = c->tgroup;
  RBF_CUDA_TRY(cudaStreamSynchronize(s));  // v_loc complete
  for (int dir = 0; dir < 2; ++dir) {
    G->ptr[dir][c->rank] = v_loc + h[dir].send_off;
    G->cnt[dir][c->rank] = h[dir].send_cnt;
  }
  G->barrier();
  int st = RBF_OK;
  for (int dir = 0; dir < 2 && st == RBF_OK; ++dir) {
    const int peer = dir == 0 ? c->rank - 1 : c->rank + 1;
    if (peer < 0 || peer >= c->nranks || h[dir].recv_cnt == 0) continue;
    // the peer's send towards this rank is its opposite direction
    if (G->cnt[1 - dir][peer] != h[dir].recv_cnt) {
      set_error("halo plan mismatch: rank %d expects %lld from rank %d, which sends %lld", c->rank,
                (long long)h[dir].recv_cnt, peer, G->cnt[1 - dir][peer]);
      st = RBF_EINVAL;
      break;
    }
    if (cudaMemcpyAsync(v_ext + h[dir].recv_off, G->ptr[1 - dir][peer],
                        sizeof(double) * (size_t)h[dir].recv_cnt, cudaMemcpyDeviceToDevice,
                        s) != cudaSuccess) {
      set_error("RBF_COMM_THREADS halo copy failed");
      st = RBF_ECUDA;
    }
  }
  if (cudaStreamSynchronize(s) != cudaSuccess && st == RBF_OK) st = RBF_ECUDA;
  G->barrier();  // peers may overwrite their v_loc from here on
  return st;
}

// NCCL send/recv of one halo (both neighbours) on stream `cs`: sends from the owned
// vector, receives into the ext vector's halo slots
static int nccl_halo(rbf_ctx *c, const double *v_loc, double *v_ext, const Halo *h, cudaStream_t cs) {
  RBF_NCCL_TRY(ncclGroupStart());
  for (int dir = 0; dir < 2; ++dir) {
    const int peer = dir == 0 ? c->rank - 1 : c->rank + 1;
    if (peer < 0 || peer >= c->nranks) continue;
    if (h[dir].send_cnt > 0)
      RBF_NCCL_TRY(ncclSend(v_loc + h[dir].send_off, (size_t)h[dir].send_cnt, ncclDouble, peer, c->nccl, cs));
    if (h[dir].recv_cnt > 0)
      RBF_NCCL_TRY(ncclRecv(v_ext + h[dir].recv_off, (size_t)h[dir].recv_cnt, ncclDouble, peer, c->nccl, cs));
  }
  RBF_NCCL_TRY(ncclGroupEnd());
  return RBF_OK;
}

int halo_exchange(rbf_ctx *c, const double *v_loc, double *v_ext, bool matvec_depth,
                  cudaStream_t s) {
  if (c->nranks <= 1) return RBF_OK;
  if (c->comm_mode == RBF_COMM_THREADS) {
    const long long own_off = c->s.own_lo - c->s.ext_lo;
    RBF_CUDA_TRY(cudaMemcpyAsync(v_ext + own_off, v_loc, sizeof(double) * n_loc(c),
                                 cudaMemcpyDeviceToDevice, s));
    return halo_exchange_threads(c, v_loc, v_ext, matvec_depth ? c->halo_mv : c->halo_pc, s);
  }
  if (c->comm_mode != RBF_COMM_NCCL) {
    set_error("virtual strip context (RBF_COMM_NONE) has no communicator: use the *_ext calls");
    return RBF_EUNSUPPORTED;
  }
  const long long own_off = c->s.own_lo - c->s.ext_lo;
  RBF_CUDA_TRY(cudaMemcpyAsync(v_ext + own_off, v_loc, sizeof(double) * n_loc(c),
                               cudaMemcpyDeviceToDevice, s));
  return nccl_halo(c, v_loc, v_ext, matvec_depth ? c->halo_mv : c->halo_pc, s);
}

// Start the halo exchange of v_loc into c->w_ext.  NCCL: on the context's comm stream
// after the work already queued on s (the producer of v_loc); finish_halo makes s wait
// for it.  THREADS: synchronous (host barrier + device copies on s).
static int start_halo(rbf_ctx *c, const double *v_loc, const Halo *h, cudaStream_t s) {
  if (c->comm_mode == RBF_COMM_THREADS) return halo_exchange_threads(c, v_loc, c->w_ext, h, s);
  if (c->comm_mode != RBF_COMM_NCCL) {
    set_error("virtual strip context (RBF_COMM_NONE) has no communicator: use the *_ext calls");
    return RBF_EUNSUPPORTED;
  }
  RBF_CUDA_TRY(cudaEventRecord(c->ev_in, s));
  RBF_CUDA_TRY(cudaStreamWaitEvent(c->s_comm, c->ev_in, 0));
  RBF_TRY(nccl_halo(c, v_loc, c->w_ext, h, c->s_comm));
  RBF_CUDA_TRY(cudaEventRecord(c->ev_halo, c->s_comm));
  return RBF_OK;
}

static int finish_halo(rbf_ctx *c, cudaStream_t s) {
  if (c->comm_mode == RBF_COMM_NCCL) RBF_CUDA_TRY(cudaStreamWaitEvent(s, c->ev_halo, 0));
  return RBF_OK;
}

// y = A_rc w across strips.  Overlapped: the owned records are packed from w_loc and
// the interior lanes run while the halo is exchanged (NCCL: concurrently; THREADS: the
// exchange follows them in stream order), then the halo records and the boundary lanes.
int dist_matvec(rbf_ctx *c, const double *w_loc, double *y_loc, cudaStream_t s) {
  const long long own_off = c->s.own_lo - c->s.ext_lo;
  if (!c->overlap) {
    RBF_TRY(halo_exchange(c, w_loc, c->w_ext, true, s));
    return launch_matvec(c, c->w_ext, y_loc, s);
  }
  const bool nccl = c->comm_mode == RBF_COMM_NCCL;
  if (nccl) RBF_TRY(start_halo(c, w_loc, c->halo_mv, s));
  RBF_TRY(launch_pack_range(c, w_loc, n_loc(c), own_off, s));
  RBF_TRY(launch_matvec(c, nullptr, y_loc, s, true, 1));
  if (!nccl) RBF_TRY(start_halo(c, w_loc, c->halo_mv, s));
  RBF_TRY(finish_halo(c, s));
  for (int dir = 0; dir < 2; ++dir) {
    const Halo &h = c->halo_mv[dir];
    if (h.recv_cnt > 0) RBF_TRY(launch_pack_range(c, c->w_ext + h.recv_off, h.recv_cnt, h.recv_off, s));
  }
  return launch_matvec(c, nullptr, y_loc, s, true, 2);
}

// z = M^-1 r across strips, the same way: the owned part of r into the ext vector and
// the interior cells while the halo (overlap_rings rows) is exchanged, then the cells
// next to the strip edges.
int dist_rasm_apply(rbf_ctx *c, const double *r_loc, double *z_loc, cudaStream_t s) {
  if (c->g.asm_full) {
    // Eq.(8) across strips: r's halo, the own cells' t_c, then the t of the rings rows
    // next to each strip edge both ways (a point near the edge sums subdomains of both
    // strips, in ascending cell order as on one strip: bitwise the same sums)
    RBF_TRY(halo_exchange(c, r_loc, c->w_ext, false, s));
    RBF_TRY(launch_asm_local(c, c->w_ext, s));
    if (c->comm_mode == RBF_COMM_THREADS) {
      RBF_TRY(halo_exchange_threads(c, c->asm_t + c->asm_sb, c->asm_t, c->halo_asm, s));
    } else if (c->comm_mode == RBF_COMM_NCCL) {
      RBF_TRY(nccl_halo(c, c->asm_t + c->asm_sb, c->asm_t, c->halo_asm, s));
    } else {
      set_error("virtual strip context (RBF_COMM_NONE) has no communicator: use the *_ext calls");
      return RBF_EUNSUPPORTED;
    }
    return launch_asm_gather(c, z_loc, s);
  }
  if (!c->overlap) {
    RBF_TRY(halo_exchange(c, r_loc, c->w_ext, false, s));
    return launch_rasm_apply(c, c->w_ext, z_loc, s);
  }
  const bool nccl = c->comm_mode == RBF_COMM_NCCL;
  if (nccl) RBF_TRY(start_halo(c, r_loc, c->halo_pc, s));
  const long long own_off = c->s.own_lo - c->s.ext_lo;
  RBF_CUDA_TRY(cudaMemcpyAsync(c->w_ext + own_off, r_loc, sizeof(double) * n_loc(c),
                               cudaMemcpyDeviceToDevice, s));
  RBF_TRY(launch_rasm_apply(c, c->w_ext, z_loc, s, 1));
  if (!nccl) RBF_TRY(start_halo(c, r_loc, c->halo_pc, s));
  RBF_TRY(finish_halo(c, s));
  return launch_rasm_apply(c, c->w_ext, z_loc, s, 2);
}

int allgather_scalars(rbf_ctx *c, const double *send, double *recv, int count, cudaStream_t s) {
  if (c->nranks <= 1) return RBF_OK;  // single rank: recv aliases send
  if (c->comm_mode == RBF_COMM_THREADS) {
    ThreadGroup *G = c->tgroup;
    RBF_CUDA_TRY(cudaStreamSynchronize(s));
    G->ptr[0][c->rank] = send;
    G->barrier();
    int st = RBF_OK;
    for (int r = 0; r < c->nranks && st == RBF_OK; ++r)
      if (cudaMemcpyAsync(recv + (long long)r * count, G->ptr[0][r], sizeof(double) * count,
                          cudaMemcpyDeviceToDevice, s) != cudaSuccess) {
        set_error("RBF_COMM_THREADS all-gather copy failed");
        st = RBF_ECUDA;
      }
    if (cudaStreamSynchronize(s) != cudaSuccess && st == RBF_OK) st = RBF_ECUDA;
    G->barrier();
    return st;
  }
  if (c->comm_mode != RBF_COMM_NCCL) {
    set_error("virtual strip context (RBF_COMM_NONE) cannot reduce across strips");
    return RBF_EUNSUPPORTED;
  }
  RBF_NCCL_TRY(ncclAllGather(send, recv, (size_t)count, ncclDouble, c->nccl, s));
  return RBF_OK;
}

}  // namespace rbf

namespace rbf {

__global__ void k_add_vec(double *__restrict__ v, const double *__restrict__ a, long long n, int first) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) v[i] = first ? a[i] : v[i] + a[i];
}

int allreduce_vector(rbf_ctx *c, double *v, long long count, cudaStream_t s) {
  if (c->nranks <= 1 || count == 0) return RBF_OK;
  if (c->comm_mode == RBF_COMM_NCCL) {
    RBF_NCCL_TRY(ncclAllReduce(v, v, (size_t)count, ncclDouble, ncclSum, c->nccl, s));
    return RBF_OK;
  }
  if (c->comm_mode != RBF_COMM_THREADS) {
    set_error("virtual strip context (RBF_COMM_NONE) cannot reduce across strips");
    return RBF_EUNSUPPORTED;
  }
  ThreadGroup *G = c->tgroup;
  ScratchGuard sg(s);
  double *tmp = nullptr;
  RBF_TRY(sg.alloc(nullptr, &tmp, sizeof(double) * (size_t)count));
  RBF_CUDA_TRY(cudaMemcpyAsync(tmp, v, sizeof(double) * (size_t)count, cudaMemcpyDeviceToDevice, s));
  RBF_CUDA_TRY(cudaStreamSynchronize(s));
  G->ptr[0][c->rank] = tmp;
  G->barrier();
  const int blocks = (int)((count + 255) / 256);
  for (int r = 0; r < c->nranks; ++r) {  // rank order
    k_add_vec<<<blocks, 256, 0, s>>>(v, G->ptr[0][r], count, r == 0);
    count_launch(1);
  }
  int st = cudaStreamSynchronize(s) == cudaSuccess ? RBF_OK : RBF_ECUDA;
  if (st != RBF_OK) set_error("RBF_COMM_THREADS vector all-reduce failed");
  G->barrier();  // the peers' tmp buffers may be freed from here on
  return st;
}

}  // namespace rbf
