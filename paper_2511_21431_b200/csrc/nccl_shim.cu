// nccl_shim.cu — dlopen'ed NCCL (see nccl_shim.h).
#include <dlfcn.h>
#include <cstdlib>
#include <cstring>
#include <nccl.h>
#include "nccl_shim.h"

namespace {
struct Api {
  bool tried = false, ok = false;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
};
Api g_api;

Api* api() {
  if (g_api.tried) return g_api.ok ? &g_api : nullptr;
  g_api.tried = true;
  void* lib = nullptr;
  // Prefer the instance already in the process (torch's), then an explicit path, then the soname.
  lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
  if (!lib) {
    const char* p = getenv("MEMFINE_NCCL_LIBRARY");
    if (p && *p) lib = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
  }
  if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) return nullptr;
#define LOAD(f, s) g_api.f = (decltype(g_api.f))dlsym(lib, s); if (!g_api.f) return nullptr;
  LOAD(getUniqueId, "ncclGetUniqueId");
  LOAD(commInitRank, "ncclCommInitRank");
  LOAD(commDestroy, "ncclCommDestroy");
  LOAD(allGather, "ncclAllGather");
  LOAD(allReduce, "ncclAllReduce");
  LOAD(groupStart, "ncclGroupStart");
  LOAD(groupEnd, "ncclGroupEnd");
  LOAD(send, "ncclSend");
  LOAD(recv, "ncclRecv");
#undef LOAD
  g_api.ok = true;
  return &g_api;
}

ncclDataType_t dt(int d) { return d == 1 ? ncclInt32 : d == 2 ? ncclFloat32 : ncclUint8; }
}  // namespace

int nccl_get_unique_id(uint8_t out[128]) {
  Api* a = api();
  if (!a) return 1;
  ncclUniqueId id;
  if (a->getUniqueId(&id) != ncclSuccess) return 1;
  memcpy(out, &id, sizeof id);
  return 0;
}

int nccl_comm_init(NcclComm* c, const uint8_t idb[128], int nranks, int rank) {
  Api* a = api();
  if (!a) return 1;
  ncclUniqueId id;
  memcpy(&id, idb, sizeof id);
  ncclComm_t comm;
  if (a->commInitRank(&comm, nranks, id, rank) != ncclSuccess) return 1;
  c->comm = comm;
  c->nranks = nranks;
  c->rank = rank;
  return 0;
}

void nccl_comm_destroy(NcclComm* c) {
  Api* a = api();
  if (a && c->comm) a->commDestroy((ncclComm_t)c->comm);
  c->comm = nullptr;
}

int nccl_all_gather_int(NcclComm* c, const int* send, int* recv, size_t n, cudaStream_t st) {
  Api* a = api();
  if (!a || !c->comm) return 1;
  return a->allGather(send, recv, n, ncclInt32, (ncclComm_t)c->comm, st) != ncclSuccess;
}

int nccl_stream_barrier(NcclComm* c, int* dev_int, cudaStream_t st) {
  Api* a = api();
  if (!a || !c->comm) return 1;
  return a->allReduce(dev_int, dev_int, 1, ncclInt32, ncclSum, (ncclComm_t)c->comm, st) != ncclSuccess;
}

int nccl_all_gather_bytes(NcclComm* c, const void* send, void* recv, size_t n, cudaStream_t st) {
  Api* a = api();
  if (!a || !c->comm) return 1;
  return a->allGather(send, recv, n, ncclUint8, (ncclComm_t)c->comm, st) != ncclSuccess;
}

int nccl_group_start() { Api* a = api(); return !a || a->groupStart() != ncclSuccess; }
int nccl_group_end() { Api* a = api(); return !a || a->groupEnd() != ncclSuccess; }

int nccl_send(NcclComm* c, const void* buf, size_t count, int dtype, int peer, cudaStream_t st) {
  Api* a = api();
  if (!a || !c->comm) return 1;
  return a->send(buf, count, dt(dtype), peer, (ncclComm_t)c->comm, st) != ncclSuccess;
}

int nccl_recv(NcclComm* c, void* buf, size_t count, int dtype, int peer, cudaStream_t st) {
  Api* a = api();
  if (!a || !c->comm) return 1;
  return a->recv(buf, count, dt(dtype), peer, (ncclComm_t)c->comm, st) != ncclSuccess;
}
