// NCCL communicator behind the distributed LU's broadcast hook (config 5a,
// SURVEY.md 8(e)): one communicator per rank (one process per GPU), created
// from a 128-byte unique id that the host side passes around
// (torch.distributed, MPI, a file -- the library does not care).
//
// NCCL is bound at run time (dlopen of libnccl.so.2, preferring the copy the
// process has already loaded, e.g. PyTorch's): libmpir_gpu.so itself has no
// link-time NCCL dependency, and single-GPU users never touch it. The few
// declarations below are NCCL's stable C ABI (nccl.h: ncclUniqueId is 128
// opaque bytes passed by value; ncclChar = 0).
//
// The reference has no counterpart (single process).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "../../include/mpir_gpu.h"
#include "common.cuh"
#include "kernels.cuh"

namespace
{
struct NcclUniqueId
{
  char internal[128];
};
using ncclComm_t = void *;
using ncclResult_t = int;
constexpr int NCCL_CHAR = 0;

struct Nccl
{
  void *so = nullptr;
  ncclResult_t (*GetUniqueId)(NcclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, NcclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void *, void *, size_t, int, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int *) = nullptr;
  std::string why;
};

Nccl &nccl()
{
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *nm : names)
      if ((n.so = dlopen(nm, RTLD_NOW | RTLD_NOLOAD)))
        break;
    if (!n.so)
      for (const char *nm : names)
        if ((n.so = dlopen(nm, RTLD_NOW | RTLD_GLOBAL)))
          break;
    if (!n.so)
    {
      n.why = std::string("libnccl.so.2 not found: ") + (dlerror() ? dlerror() : "");
      return;
    }
    auto sym = [&](const char *s) { return dlsym(n.so, s); };
    n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
    n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
    n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
    n.Broadcast = reinterpret_cast<decltype(n.Broadcast)>(sym("ncclBroadcast"));
    n.Send = reinterpret_cast<decltype(n.Send)>(sym("ncclSend"));
    n.Recv = reinterpret_cast<decltype(n.Recv)>(sym("ncclRecv"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
    n.GetVersion = reinterpret_cast<decltype(n.GetVersion)>(sym("ncclGetVersion"));
    if (!n.GetUniqueId || !n.CommInitRank || !n.CommDestroy || !n.Broadcast || !n.Send ||
        !n.Recv || !n.GetErrorString)
    {
      n.why = "libnccl.so.2 lacks an expected symbol";
      n.so = nullptr;
    }
  });
  return n;
}

void fill(mpirg_error *err, int status, const std::string &msg)
{
  if (!err)
    return;
  err->status = status;
  err->column = -1;
  err->value = 0.0;
  std::snprintf(err->message, sizeof(err->message), "%s", msg.c_str());
}

int nccl_fail(mpirg_error *err, const char *what, ncclResult_t rc)
{
  fill(err, MPIRG_ERR_NCCL, std::string(what) + ": " + nccl().GetErrorString(rc));
  return MPIRG_ERR_NCCL;
}
}  // namespace

struct mpirg_comm
{
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0, device = 0;
};

extern "C" {

int mpirg_comm_unique_id(void *id128, mpirg_error *err)
{
  Nccl &n = nccl();
  if (!n.so)
  {
    fill(err, MPIRG_ERR_NCCL, n.why);
    return MPIRG_ERR_NCCL;
  }
  NcclUniqueId id;
  const ncclResult_t rc = n.GetUniqueId(&id);
  if (rc != 0)
    return nccl_fail(err, "ncclGetUniqueId", rc);
  std::memcpy(id128, id.internal, sizeof(id.internal));
  fill(err, MPIRG_OK, "");
  return MPIRG_OK;
}

int mpirg_comm_create(mpirg_comm **out, int nranks, int rank, const void *id128, int device,
                      mpirg_error *err)
{
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks || !id128)
  {
    fill(err, MPIRG_ERR_INVALID_PARAM, "rank must lie in [0, nranks) and the id must be given");
    return MPIRG_ERR_INVALID_PARAM;
  }
  Nccl &n = nccl();
  if (!n.so)
  {
    fill(err, MPIRG_ERR_NCCL, n.why);
    return MPIRG_ERR_NCCL;
  }
  if (device >= 0 && cudaSetDevice(device) != cudaSuccess)
  {
    fill(err, MPIRG_ERR_CUDA, "cudaSetDevice failed for the communicator's device");
    return MPIRG_ERR_CUDA;
  }
  auto *c = new mpirg_comm;
  c->nranks = nranks;
  c->rank = rank;
  cudaGetDevice(&c->device);
  NcclUniqueId id;
  std::memcpy(id.internal, id128, sizeof(id.internal));
  const ncclResult_t rc = n.CommInitRank(&c->comm, nranks, id, rank);
  if (rc != 0)
  {
    delete c;
    return nccl_fail(err, "ncclCommInitRank", rc);
  }
  *out = c;
  fill(err, MPIRG_OK, "");
  return MPIRG_OK;
}

void mpirg_comm_destroy(mpirg_comm *c)
{
  if (!c)
    return;
  if (c->comm)
    nccl().CommDestroy(c->comm);
  delete c;
}

int mpirg_comm_nranks(const mpirg_comm *c) { return c->nranks; }
int mpirg_comm_rank(const mpirg_comm *c) { return c->rank; }

int mpirg_comm_version(void)
{
  Nccl &n = nccl();
  int v = 0;
  if (n.so && n.GetVersion)
    n.GetVersion(&v);
  return v;
}

// The broadcast hook (mpirg_bcast_fn) over NCCL: ctx is the mpirg_comm.
int mpirg_comm_bcast(void *ctx, void *buf, size_t bytes, int root, void *stream)
{
  auto *c = static_cast<mpirg_comm *>(ctx);
  return nccl().Broadcast(buf, buf, bytes, NCCL_CHAR, root, c->comm,
                          static_cast<cudaStream_t>(stream)) == 0
             ? MPIRG_OK
             : MPIRG_ERR_NCCL;
}

int mpirg_comm_send(mpirg_comm *c, const void *buf, size_t bytes, int peer, void *stream)
{
  return nccl().Send(buf, bytes, NCCL_CHAR, peer, c->comm, static_cast<cudaStream_t>(stream)) ==
                 0
             ? MPIRG_OK
             : MPIRG_ERR_NCCL;
}

int mpirg_comm_recv(mpirg_comm *c, void *buf, size_t bytes, int peer, void *stream)
{
  return nccl().Recv(buf, bytes, NCCL_CHAR, peer, c->comm, static_cast<cudaStream_t>(stream)) ==
                 0
             ? MPIRG_OK
             : MPIRG_ERR_NCCL;
}

}  // extern "C"
