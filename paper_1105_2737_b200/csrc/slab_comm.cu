// Multi-GPU data plane of the slab decomposition:
// one 3D field over `world` GPUs, one process per GPU, NCCL over NVLink.
//
//   grfc_slab_generate = pass A (the rank's spectrum slab k1 in [r N1/G, ...):
//                        generation + axis-0 FFT, partners regenerated from the
//                        counter-based noise, never exchanged)
//                      -> all-to-all of the G blocks (grouped ncclSend/ncclRecv;
//                         the rank's own block is a device copy)
//                      -> pass B on the received blocks, read in place
//   (bit-identical to the single-GPU field for every world size).
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): inside a PyTorch process
// that is the NCCL torch already loaded, elsewhere the system library; the
// product library itself has no link-time NCCL dependency. The communicator is
// bootstrapped the standard way: rank 0 calls grfc_comm_unique_id, the host
// framework broadcasts the 128 bytes, every rank calls grfc_comm_create.
#include <dlfcn.h>
#include <nccl.h>  // types and enums only; the entry points come from dlopen

#include <cstring>
#include <mutex>
#include <string>

#include "../../include/grfc.h"
#include "grfc_internal.cuh"

namespace grfc {
grfc_status set_error(grfc_status s, const std::string& msg);  // api.cu
}

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string missing;  // why NCCL is unusable ("" = usable)
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.missing = std::string("NCCL not found: ") + dlerror();
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn && api.missing.empty()) api.missing = std::string("NCCL symbol missing: ") + name;
    };
    sym(api.get_unique_id, "ncclGetUniqueId");
    sym(api.comm_init_rank, "ncclCommInitRank");
    sym(api.comm_destroy, "ncclCommDestroy");
    sym(api.send, "ncclSend");
    sym(api.recv, "ncclRecv");
    sym(api.group_start, "ncclGroupStart");
    sym(api.group_end, "ncclGroupEnd");
    sym(api.error_string, "ncclGetErrorString");
  });
  return api;
}

grfc_status nccl_fail(ncclResult_t r, const char* what) {
  const NcclApi& n = nccl();
  return grfc::set_error(GRFC_ENCCL, std::string("NCCL: ") + what + ": " +
                                         (n.error_string ? n.error_string(r) : std::to_string((int)r)));
}

grfc_status cuda_fail(cudaError_t e, const char* what) {
  return grfc::set_error(GRFC_ECUDA, std::string("CUDA: ") + what + ": " + cudaGetErrorString(e));
}

}  // namespace

struct grfc_comm_s {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0, device = 0;
};

extern "C" {

grfc_status grfc_comm_unique_id(unsigned char* id) {
  if (!id) return grfc::set_error(GRFC_EINVAL, "grfc: null argument");
  const NcclApi& n = nccl();
  if (!n.missing.empty()) return grfc::set_error(GRFC_ENCCL, n.missing);
  ncclUniqueId u;
  const ncclResult_t r = n.get_unique_id(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  static_assert(sizeof(u.internal) == GRFC_UNIQUE_ID_BYTES, "ncclUniqueId size");
  std::memcpy(id, u.internal, GRFC_UNIQUE_ID_BYTES);
  return GRFC_OK;
}

grfc_status grfc_comm_create(grfc_comm* out, const unsigned char* id, int world, int rank, int device) {
  if (!out || !id) return grfc::set_error(GRFC_EINVAL, "grfc: null argument");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return grfc::set_error(GRFC_EINVAL, "grfc: bad world/rank");
  const NcclApi& n = nccl();
  if (!n.missing.empty()) return grfc::set_error(GRFC_ENCCL, n.missing);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  ncclUniqueId u;
  std::memcpy(u.internal, id, GRFC_UNIQUE_ID_BYTES);
  auto* c = new grfc_comm_s();
  c->world = world;
  c->rank = rank;
  c->device = device;
  const ncclResult_t r = n.comm_init_rank(&c->comm, world, u, rank);
  cudaSetDevice(prev);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  *out = c;
  return GRFC_OK;
}

void grfc_comm_destroy(grfc_comm c) {
  if (!c) return;
  if (c->comm && nccl().comm_destroy) nccl().comm_destroy(c->comm);
  delete c;
}

grfc_status grfc_comm_info(grfc_comm c, int* world, int* rank, int* device) {
  if (!c) return grfc::set_error(GRFC_EINVAL, "grfc: null communicator");
  if (world) *world = c->world;
  if (rank) *rank = c->rank;
  if (device) *device = c->device;
  return GRFC_OK;
}

grfc_status grfc_slab_exchange(grfc_plan plan, grfc_comm c, const void* d_send, void* d_recv, void* stream) {
  if (!plan || !c || !d_send || !d_recv) return grfc::set_error(GRFC_EINVAL, "grfc: null argument");
  uint64_t buf = 0, block = 0;
  grfc_status st = grfc_slab_sizes(plan, c->world, &buf, &block, nullptr);
  if (st != GRFC_OK) return st;
  int dtype = 0, device = 0;
  st = grfc_plan_grid(plan, nullptr, nullptr, nullptr, &dtype, &device);
  if (st != GRFC_OK) return st;
  if (device != c->device) return grfc::set_error(GRFC_EINVAL, "grfc: plan and communicator are on different devices");
  const size_t bytes = block * (dtype == GRFC_F64 ? 16 : 8);
  cudaStream_t s = (cudaStream_t)stream;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  // block q of this rank's send buffer -> rank q, stored there at block `rank`
  const char* src = static_cast<const char*>(d_send);
  char* dst = static_cast<char*>(d_recv);
  cudaError_t e = cudaMemcpyAsync(dst + (size_t)c->rank * bytes, src + (size_t)c->rank * bytes, bytes,
                                  cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) {
    cudaSetDevice(prev);
    return cuda_fail(e, "local block copy");
  }
  if (c->world > 1) {
    const NcclApi& n = nccl();
    ncclResult_t r = n.group_start();
    for (int q = 0; q < c->world && r == ncclSuccess; ++q) {
      if (q == c->rank) continue;
      r = n.send(src + (size_t)q * bytes, bytes, ncclUint8, q, c->comm, s);
      if (r == ncclSuccess) r = n.recv(dst + (size_t)q * bytes, bytes, ncclUint8, q, c->comm, s);
    }
    const ncclResult_t r2 = n.group_end();
    if (r == ncclSuccess) r = r2;
    if (r != ncclSuccess) {
      cudaSetDevice(prev);
      return nccl_fail(r, "grouped send/recv");
    }
  }
  cudaSetDevice(prev);
  return GRFC_OK;
}

grfc_status grfc_slab_generate(grfc_plan plan, grfc_comm c, uint64_t seed, uint64_t field, void* d_out,
                               void* stream) {
  if (!plan || !c || !d_out) return grfc::set_error(GRFC_EINVAL, "grfc: null argument");
  uint64_t buf = 0;
  grfc_status st = grfc_slab_sizes(plan, c->world, &buf, nullptr, nullptr);
  if (st != GRFC_OK) return st;
  int dtype = 0, device = 0;
  grfc_plan_grid(plan, nullptr, nullptr, nullptr, &dtype, &device);
  if (device != c->device) return grfc::set_error(GRFC_EINVAL, "grfc: plan and communicator are on different devices");
  const size_t bytes = buf * (dtype == GRFC_F64 ? 16 : 8);
  cudaStream_t s = (cudaStream_t)stream;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  void* ws = nullptr;  // send | recv, stream-ordered from the device pool
  // world 1: the exchange is the identity, pass B reads pass A's buffer
  cudaError_t e = cudaMallocAsync(&ws, (c->world > 1 ? 2 : 1) * bytes, s);
  if (e != cudaSuccess) {
    cudaSetDevice(prev);
    return cuda_fail(e, "slab buffers");
  }
  void* send = ws;
  void* recv = c->world > 1 ? static_cast<char*>(ws) + bytes : ws;
  st = grfc_slab_pass_a(plan, c->world, c->rank, seed, field, send, stream);
  if (st == GRFC_OK && c->world > 1) st = grfc_slab_exchange(plan, c, send, recv, stream);
  if (st == GRFC_OK) st = grfc_slab_pass_b(plan, c->world, recv, d_out, stream);
  cudaFreeAsync(ws, s);
  cudaSetDevice(prev);
  return st;
}

}  // extern "C"
