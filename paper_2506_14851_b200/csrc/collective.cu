// K5 across GPUs as one C entry (pdg_rank_allgather_sort).
//
// Every rank holds its shard's packed keys (float32 key bits << 32 | global
// arrival position, distributed.py); one ncclAllGather over NVLink/NVSwitch
// collects width keys per rank (shards padded with a sentinel that sorts
// last), then one radix sort orders them on every rank.  The rank-major
// gather of arrival-ordered shards is itself in arrival order, so begin_bit =
// 32 (a stable sort on the key bits alone) gives the (key, arrival) order with
// half the passes.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2 -- in a PyTorch
// process the copy torch already loaded), so the library has no link-time
// NCCL dependency; the communicator is the caller's (ncclComm_t as void*).
#include <dlfcn.h>


#include "common.cuh"

namespace {
typedef int (*AllGatherFn)(const void*, void*, size_t, int, void*, cudaStream_t);
constexpr int kNcclUint64 = 5;     // ncclDataType_t ncclUint64

AllGatherFn nccl_allgather() {
  static AllGatherFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) fn = reinterpret_cast<AllGatherFn>(dlsym(h, "ncclAllGather"));
  }
  return fn;
}
}  // namespace

using namespace pdg;

extern "C" size_t pdg_rank_allgather_sort_temp_bytes(int64_t width, int32_t world) {
  const int64_t n = width * int64_t(world);
  return order_temp_bytes(n > 0 ? n : 1) + 256;
}

extern "C" int pdg_rank_allgather_sort(void* nccl_comm, const uint64_t* local_keys,
                                       int64_t width, int32_t world, uint64_t* gathered,
                                       uint64_t* sorted_keys, int32_t begin_bit, void* temp,
                                       size_t temp_bytes, void* stream) {
  if (!nccl_comm || width < 0 || world < 1 ||
      (width > 0 && (!local_keys || !gathered || !sorted_keys || !temp))) {
    set_error("pdg_rank_allgather_sort: invalid arguments");
    return PDG_EINVAL;
  }
  if (begin_bit != 0 && begin_bit != 32) {
    set_error("pdg_rank_allgather_sort: begin_bit must be 0 or 32");
    return PDG_EINVAL;
  }
  if (width == 0) return PDG_OK;
  const size_t need = pdg_rank_allgather_sort_temp_bytes(width, world);
  if (temp_bytes < need) {
    set_error("pdg_rank_allgather_sort: temp_bytes %zu < %zu", temp_bytes, need);
    return PDG_EINVAL;
  }
  AllGatherFn ag = nccl_allgather();
  if (!ag) {
    set_error("pdg_rank_allgather_sort: libnccl.so.2 / ncclAllGather not found");
    return PDG_EUNSUPPORTED;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int r = ag(local_keys, gathered, size_t(width), kNcclUint64, nccl_comm, st);
  if (r != 0) {
    set_error("pdg_rank_allgather_sort: ncclAllGather failed (ncclResult_t %d)", r);
    return PDG_ECUDA;
  }
  return order_sort(gathered, sorted_keys, nullptr, nullptr, width * int64_t(world), begin_bit,
                    64, temp, temp_bytes, st);
}
