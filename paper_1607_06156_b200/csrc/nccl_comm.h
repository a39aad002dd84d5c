// nccl_comm.h -- the library-owned NCCL communicator (cc_get_unique_id +
// cc_config.nccl_id).  Every collective is enqueued on the library's stream: no host
// synchronisation, no re-entry into the caller.  libnccl is resolved at run time (dlopen;
// the copy PyTorch already loaded when there is one), so libcc.so has no link-time NCCL
// dependency and a single-GPU user never loads it.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace cc {
namespace nccl {

// element types of the native collectives: the cc_dtype values plus unsigned 32-bit (the
// partition slots' MIN needs no order-preserving sign flip on NCCL)
enum { DT_I32 = 0, DT_I64 = 1, DT_U8 = 2, DT_U32 = 3 };

int unique_id(void* out128, std::string* err);
int init(void** comm, const void* id128, int world, int rank, int device, std::string* err);
void destroy(void* comm);
// op: CC_OP_SUM / CC_OP_MIN / CC_OP_MAX; in place
int allreduce(void* comm, void* buf, uint64_t count, int dt, int op, cudaStream_t st, std::string* err);
// recv <- rank-major concatenation of every rank's `bytes` at send
int allgather(void* comm, const void* send, void* recv, uint64_t bytes, cudaStream_t st, std::string* err);
// send: world consecutive blocks of sb[k] bytes for rank k; recv: rb[k] bytes from rank k
int alltoallv(void* comm, int world, const void* send, const uint64_t* sb, void* recv, const uint64_t* rb,
              cudaStream_t st, std::string* err);

}  // namespace nccl
}  // namespace cc
