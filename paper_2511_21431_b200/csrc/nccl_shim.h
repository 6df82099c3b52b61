// nccl_shim.h — NCCL loaded at run time (dlopen) so libmemfine.so links no NCCL and uses
// the one instance torch already loaded (the wheel's 2.28.9).  Types come from
// the wheel's nccl.h; symbols from dlsym.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

struct NcclComm {
  void* comm = nullptr;   // ncclComm_t
  int nranks = 1, rank = 0;
};

// All return 0 on success.
int nccl_get_unique_id(uint8_t out[128]);
int nccl_comm_init(NcclComm* c, const uint8_t id[128], int nranks, int rank);
void nccl_comm_destroy(NcclComm* c);
int nccl_all_gather_int(NcclComm* c, const int* send, int* recv, size_t count_per_rank, cudaStream_t st);
// all-reduce of one int (sum) on `st`: a stream barrier across the EP group
int nccl_stream_barrier(NcclComm* c, int* dev_int, cudaStream_t st);
int nccl_all_gather_bytes(NcclComm* c, const void* send, void* recv, size_t bytes_per_rank, cudaStream_t st);
int nccl_group_start();
int nccl_group_end();
// dtype: 0 = uint8 bytes, 1 = int32, 2 = float32
int nccl_send(NcclComm* c, const void* buf, size_t count, int dtype, int peer, cudaStream_t st);
int nccl_recv(NcclComm* c, void* buf, size_t count, int dtype, int peer, cudaStream_t st);
