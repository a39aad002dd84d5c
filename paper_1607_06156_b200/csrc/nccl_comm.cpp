// nccl_comm.cpp -- library-owned NCCL communicator (see nccl_comm.h).
//
// The exchange steps of the sharded path are all-reduces of
// counters and partition slots, all-gathers of bitmap slices / count vectors, and
// all-to-all-v of arcs and ids.  Here they are NCCL calls on the library's stream: the
// device orders them after the kernels that produce their inputs and before the kernels
// that consume their outputs, so the host only waits where it reads a value (counters).
// The all-to-all-v is one NCCL group of ncclSend/ncclRecv pairs (one per peer, byte counts
// from the host), which NCCL runs as a single fused launch over NVLink/NVSwitch.
//
// Symbols come from dlopen: first the libnccl.so.2 already in the process (PyTorch's), else
// the one the loader finds; CC_NCCL_LIB overrides the path.  Only the types come from nccl.h.
#include "nccl_comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/cc.h"

namespace cc {
namespace nccl {
namespace {

struct Api {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    const char* path = std::getenv("CC_NCCL_LIB");
    if (path && *path) {
      h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
    } else {
      h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
      if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) {
      const char* e = dlerror();
      a.why = std::string("cannot load libnccl: ") + (e ? e : "?");
      return;
    }
    bool all = true;
    auto get = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) {
        all = false;
        a.why += std::string(a.why.empty() ? "" : ", ") + "missing " + name;
      }
    };
    get(a.get_unique_id, "ncclGetUniqueId");
    get(a.comm_init_rank, "ncclCommInitRank");
    get(a.comm_destroy, "ncclCommDestroy");
    get(a.all_reduce, "ncclAllReduce");
    get(a.all_gather, "ncclAllGather");
    get(a.send, "ncclSend");
    get(a.recv, "ncclRecv");
    get(a.group_start, "ncclGroupStart");
    get(a.group_end, "ncclGroupEnd");
    get(a.error_string, "ncclGetErrorString");
    a.ok = all;
  });
  return a;
}

int check(ncclResult_t r, const char* what, std::string* err) {
  if (r == ncclSuccess) return 0;
  if (err) {
    char buf[256];
    std::snprintf(buf, sizeof(buf), "%s: %s", what, api().error_string ? api().error_string(r) : "?");
    *err = buf;
  }
  return 1;
}

bool ready(std::string* err) {
  if (api().ok) return true;
  if (err) *err = api().why;
  return false;
}

ncclDataType_t dtype(int dt) {
  switch (dt) {
    case DT_I32: return ncclInt32;
    case DT_I64: return ncclInt64;
    case DT_U32: return ncclUint32;
    default: return ncclUint8;
  }
}

ncclRedOp_t redop(int op) {
  switch (op) {
    case CC_OP_MIN: return ncclMin;
    case CC_OP_MAX: return ncclMax;
    default: return ncclSum;
  }
}

}  // namespace

int unique_id(void* out128, std::string* err) {
  if (!ready(err)) return 1;
  ncclUniqueId id;
  if (check(api().get_unique_id(&id), "ncclGetUniqueId", err)) return 1;
  std::memcpy(out128, &id, sizeof(id));
  return 0;
}

int init(void** comm, const void* id128, int world, int rank, int device, std::string* err) {
  if (!ready(err)) return 1;
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    if (err) *err = "cudaSetDevice failed before ncclCommInitRank";
    return 1;
  }
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  if (check(api().comm_init_rank(&c, world, id, rank), "ncclCommInitRank", err)) return 1;
  *comm = c;
  return 0;
}

void destroy(void* comm) {
  if (comm && api().ok) api().comm_destroy(static_cast<ncclComm_t>(comm));
}

int allreduce(void* comm, void* buf, uint64_t count, int dt, int op, cudaStream_t st, std::string* err) {
  if (!ready(err)) return 1;
  if (count == 0) return 0;
  return check(api().all_reduce(buf, buf, count, dtype(dt), redop(op), static_cast<ncclComm_t>(comm), st),
               "ncclAllReduce", err);
}

int allgather(void* comm, const void* send, void* recv, uint64_t bytes, cudaStream_t st, std::string* err) {
  if (!ready(err)) return 1;
  if (bytes == 0) return 0;
  return check(api().all_gather(send, recv, bytes, ncclUint8, static_cast<ncclComm_t>(comm), st),
               "ncclAllGather", err);
}

int alltoallv(void* comm, int world, const void* send, const uint64_t* sb, void* recv, const uint64_t* rb,
              cudaStream_t st, std::string* err) {
  if (!ready(err)) return 1;
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  const char* s = static_cast<const char*>(send);
  char* r = static_cast<char*>(recv);
  if (check(api().group_start(), "ncclGroupStart", err)) return 1;
  int bad = 0;
  uint64_t so = 0, ro = 0;
  for (int k = 0; k < world && !bad; k++) {
    if (sb[k]) bad |= check(api().send(s + so, sb[k], ncclUint8, k, c, st), "ncclSend", err);
    if (rb[k] && !bad) bad |= check(api().recv(r + ro, rb[k], ncclUint8, k, c, st), "ncclRecv", err);
    so += sb[k];
    ro += rb[k];
  }
  const int e = check(api().group_end(), "ncclGroupEnd", err);
  return bad | e;
}

}  // namespace nccl
}  // namespace cc
