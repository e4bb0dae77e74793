// dist.cu -- row-partitioned (multi-GPU) plumbing: halo pack/unpack kernels and
// the NCCL transport.
//
// Per outer loop a rank exchanges, with each slab neighbour, the ghost rows of
// p (= Y[:,0]), r (= Y[:,sigma+1]) and x it needs for the communication-avoiding
// matrix-powers levels (depth <= sigma), in ONE grouped ncclSend/ncclRecv, and
// takes part in exactly ONE ncclAllReduce: the packed Gram + the two residual
// norms (red_buf).  Both are captured into the per-outer-loop CUDA graph.
//
// NCCL is dlopen'ed (the torch-bundled libnccl.so.2 by default) so a single-GPU
// plan has no NCCL dependency at all.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <vector>

#include "internal.cuh"

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;
std::mutex g_nccl_mu;
// collective calls issued (per thread): capture_outer reads the difference
// across one capture = the collectives in one outer-loop graph
thread_local long long g_allreduce_calls = 0, g_halo_groups = 0;

template <class F>
bool sym(void* h, const char* name, F& f) {
  f = reinterpret_cast<F>(dlsym(h, name));
  return f != nullptr;
}

__global__ void k_halo_pack(const double* __restrict__ P0, const double* __restrict__ R0,
                            const double* __restrict__ x, const int* __restrict__ idx,
                            const int* __restrict__ dst, const int* __restrict__ cnt, int n,
                            double* __restrict__ buf, const int* __restrict__ done) {
  if (*done) return;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int i = idx[t], o = dst[t], k = cnt[t];
    SSCG_CHECK(i >= 0 && o >= 0 && o + 2 * k < 3 * n + 2 * k);
    buf[o] = P0[i];
    buf[o + k] = R0[i];
    buf[o + 2 * k] = x[i];
  }
}

__global__ void k_halo_unpack(double* __restrict__ P0, double* __restrict__ R0,
                              double* __restrict__ x, const int* __restrict__ idx,
                              const int* __restrict__ src, const int* __restrict__ cnt, int n,
                              const double* __restrict__ buf, const int* __restrict__ done) {
  if (*done) return;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int i = idx[t], o = src[t], k = cnt[t];
    P0[i] = buf[o];
    R0[i] = buf[o + k];
    x[i] = buf[o + 2 * k];
  }
}

// sum of nb equal-length buffers in fixed order, written back to every buffer
// (the virtual-rank group's allreduce: bitwise identical on all members)
__global__ void k_vsum(double* const* bufs, int nb, int len) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < len; e += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += bufs[b][e];
    for (int b = 0; b < nb; ++b) bufs[b][e] = s;
  }
}

// ||b||^2 partials -> red_buf[0] (start of a solve; allreduced on a partitioned plan)
__global__ void k_norm_pack(const double* part, int n, double* out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += 32) s += part[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) out[0] = s;
}

int grid_for(int n) {
  int g = (n + 255) / 256;
  return g < 1 ? 1 : (g > 4 * NUM_SMS ? 4 * NUM_SMS : g);
}

}  // namespace

int nccl_load(const char* path) {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.h) return SSCG_OK;
  const char* p = (path && path[0]) ? path : "libnccl.so.2";
  void* h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
  if (!h) return sscg_fail(SSCG_EINVAL, "cannot load NCCL from %s: %s", p, dlerror());
  NcclApi a;
  a.h = h;
  bool ok = sym(h, "ncclGetUniqueId", a.getUniqueId) && sym(h, "ncclCommInitRank", a.commInitRank) &&
            sym(h, "ncclCommDestroy", a.commDestroy) && sym(h, "ncclAllReduce", a.allReduce) &&
            sym(h, "ncclSend", a.send) && sym(h, "ncclRecv", a.recv) &&
            sym(h, "ncclGroupStart", a.groupStart) && sym(h, "ncclGroupEnd", a.groupEnd) &&
            sym(h, "ncclGetErrorString", a.errorString) && sym(h, "ncclCommInitAll", a.commInitAll);
  if (!ok) return sscg_fail(SSCG_EINVAL, "NCCL library %s lacks a required symbol", p);
  g_nccl = a;
  return SSCG_OK;
}

static int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return SSCG_OK;
  return sscg_fail(SSCG_ECUDA, "%s: %s", what, g_nccl.errorString ? g_nccl.errorString(r) : "?");
}

int nccl_unique_id(const char* path, unsigned char* id128) {
  int rc = nccl_load(path);
  if (rc) return rc;
  ncclUniqueId id;
  rc = nccl_check(g_nccl.getUniqueId(&id), "ncclGetUniqueId");
  if (rc) return rc;
  memcpy(id128, id.internal, NCCL_UNIQUE_ID_BYTES);
  return SSCG_OK;
}

int nccl_comm_init(void** comm, const unsigned char* id128, int rank, int world) {
  ncclUniqueId id;
  memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t c = nullptr;
  int rc = nccl_check(g_nccl.commInitRank(&c, world, id, rank), "ncclCommInitRank");
  if (rc) return rc;
  *comm = c;
  return SSCG_OK;
}

// one communicator per device of a single-process group (ncclCommInitAll:
// rank i on devs[i]; the devices must be distinct)
int nccl_comm_init_all(void** comms, int n, const int* devs) {
  std::vector<ncclComm_t> c((size_t)n, nullptr);
  int rc = nccl_check(g_nccl.commInitAll(c.data(), n, devs), "ncclCommInitAll");
  if (rc) return rc;
  for (int i = 0; i < n; ++i) comms[i] = c[(size_t)i];
  return SSCG_OK;
}

void collective_counts(long long* allreduce, long long* halo) {
  *allreduce = g_allreduce_calls;
  *halo = g_halo_groups;
}

void nccl_comm_destroy(void* comm) {
  if (comm && g_nccl.commDestroy) g_nccl.commDestroy(static_cast<ncclComm_t>(comm));
}

// one grouped halo exchange: pack -> per-peer send/recv -> unpack
int halo_exchange(const HaloPlan& h, const Ctx& c, void* comm, cudaStream_t s) {
  const int sigma_col = h.r_col;
  double* P0 = c.Y;
  double* R0 = c.Y + (int64_t)sigma_col * c.ld;
  const int* done = &c.st->done;
  if (h.n_send) {
    k_halo_pack<<<grid_for(h.n_send), 256, 0, s>>>(P0, R0, c.x, h.d_send_idx, h.d_send_dst,
                                                    h.d_send_cnt, h.n_send, h.d_sendbuf, done);
  }
  if (comm) {
    int rc = nccl_check(g_nccl.groupStart(), "ncclGroupStart");
    if (rc) return rc;
    for (int q = 0; q < h.n_peers; ++q) {
      const int64_t so = h.send_off[q], sn = h.send_off[q + 1] - so;
      const int64_t ro = h.recv_off[q], rn = h.recv_off[q + 1] - ro;
      ncclComm_t cm = static_cast<ncclComm_t>(comm);
      if (sn) {
        rc = nccl_check(g_nccl.send(h.d_sendbuf + 3 * so, 3 * sn, ncclFloat64, h.peer_rank[q], cm, s),
                        "ncclSend");
        if (rc) return rc;
      }
      if (rn) {
        rc = nccl_check(g_nccl.recv(h.d_recvbuf + 3 * ro, 3 * rn, ncclFloat64, h.peer_rank[q], cm, s),
                        "ncclRecv");
        if (rc) return rc;
      }
    }
    rc = nccl_check(g_nccl.groupEnd(), "ncclGroupEnd");
    if (rc) return rc;
    ++g_halo_groups;
  }
  return SSCG_OK;
}

void halo_unpack(const HaloPlan& h, const Ctx& c, cudaStream_t s) {
  if (!h.n_recv) return;
  double* P0 = c.Y;
  double* R0 = c.Y + (int64_t)h.r_col * c.ld;
  k_halo_unpack<<<grid_for(h.n_recv), 256, 0, s>>>(P0, R0, c.x, h.d_recv_idx, h.d_recv_src,
                                                    h.d_recv_cnt, h.n_recv, h.d_recvbuf,
                                                    &c.st->done);
}

int nccl_allreduce(void* comm, double* buf, int64_t count, cudaStream_t s) {
  if (!comm) return SSCG_OK;
  ++g_allreduce_calls;
  return nccl_check(g_nccl.allReduce(buf, buf, (size_t)count, ncclFloat64, ncclSum,
                                     static_cast<ncclComm_t>(comm), s),
                    "ncclAllReduce");
}

void launch_vsum(double* const* d_bufs, int nb, int len, cudaStream_t s) {
  k_vsum<<<grid_for(len), 256, 0, s>>>(d_bufs, nb, len);
}

void launch_norm_pack(const Ctx& c, cudaStream_t s) {
  k_norm_pack<<<1, 32, 0, s>>>(c.part_t, c.red_n, c.red_buf);
}
