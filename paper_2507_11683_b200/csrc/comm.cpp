// Distributed-index-batching's only device<->device exchange: the gradient all-reduce
// ("averaged across all workers through an all-reduce operation"; "aside from DDP
// calls to AllReduce").  NCCL over NVLink 5 / NVSwitch; one communicator per rank, created from
// a ncclUniqueId that rank 0 makes and the caller broadcasts (torch process group).
#include <nccl.h>

#include <cstring>

#include "common.cuh"
#include "profile.cuh"

struct pgti_comm {
  ncclComm_t comm;
  int rank, world, device;
};

#define PGTI_NCCL_TRY(call)                                                              \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess)                                                               \
      return ::pgti::fail(PGTI_ERR_NCCL, "%s failed: %s", #call, ncclGetErrorString(r_)); \
  } while (0)

extern "C" pgti_status pgti_comm_unique_id(uint8_t id[128]) {
  pgti::clear_error();
  PGTI_REQUIRE(id, PGTI_ERR_INVALID_ARG, "pgti_comm_unique_id: null id");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId u;
  PGTI_NCCL_TRY(ncclGetUniqueId(&u));
  std::memcpy(id, &u, 128);
  return PGTI_OK;
}

extern "C" pgti_status pgti_comm_init(pgti_comm **out, const uint8_t id[128], int rank, int world,
                                      int device) {
  pgti::clear_error();
  PGTI_REQUIRE(out && id && world >= 1 && rank >= 0 && rank < world && device >= 0,
               PGTI_ERR_INVALID_ARG, "pgti_comm_init: rank=%d world=%d device=%d", rank, world,
               device);
  PGTI_CUDA_TRY(cudaSetDevice(device));
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t c;
  PGTI_NCCL_TRY(ncclCommInitRank(&c, world, u, rank));
  *out = new pgti_comm{c, rank, world, device};
  return PGTI_OK;
}

extern "C" pgti_status pgti_allreduce_grads(pgti_comm *c, float *grads, size_t n, void *stream) {
  pgti::clear_error();
  PGTI_REQUIRE(c && grads, PGTI_ERR_INVALID_ARG, "pgti_allreduce_grads: null pointer");
  // bytes each rank must move in a ring all-reduce: 2 (R-1)/R n 4 (reported as "bus" bytes)
  pgti::ProfScope prof(pgti::kProfAllreduce, pgti::as_stream(stream),
                       2.0 * (c->world - 1) / c->world * double(n) * 4.0, double(n));
  PGTI_NCCL_TRY(ncclAllReduce(grads, grads, n, ncclFloat32, ncclSum, c->comm,
                              pgti::as_stream(stream)));
  return PGTI_OK;
}

extern "C" pgti_status pgti_allreduce_f64(pgti_comm *c, double *buf, size_t n, void *stream) {
  pgti::clear_error();
  PGTI_REQUIRE(c && buf, PGTI_ERR_INVALID_ARG, "pgti_allreduce_f64: null pointer");
  PGTI_NCCL_TRY(
      ncclAllReduce(buf, buf, n, ncclFloat64, ncclSum, c->comm, pgti::as_stream(stream)));
  return PGTI_OK;
}

extern "C" pgti_status pgti_comm_destroy(pgti_comm *c) {
  pgti::clear_error();
  if (!c) return PGTI_OK;
  // collective: every rank calls this (after its last enqueued all-reduce); finalize flushes
  // outstanding work, destroy frees the resources
  ncclResult_t r = ncclCommFinalize(c->comm);
  if (r == ncclSuccess) r = ncclCommDestroy(c->comm);
  delete c;
  PGTI_REQUIRE(r == ncclSuccess, PGTI_ERR_NCCL, "ncclCommDestroy: %s", ncclGetErrorString(r));
  return PGTI_OK;
}
