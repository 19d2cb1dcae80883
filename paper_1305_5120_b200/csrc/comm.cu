// In-process multi-GPU communicator: one NCCL clique over the GPUs of this process
// (ncclCommInitAll), one rank per device, driven by one host thread per device.
//
// This is the collective layer of SURVEY.md section 8b's `chfsi_ctx_create(ndev,
// devices)`: a drop-in caller of chfsi_solve(H, Y0, config) (reference core.py:385)
// gets every visible GPU from ONE process, the way the reference takes its
// parallelism in-process (linalg.py:49-64 set_workers). The sharded phases are the
// same as under torch.distributed (distributed.py); only all-gathers and broadcasts
// are used. NCCL is resolved with dlopen at first use, so the
// library loads (and every single-GPU entry point works) without it.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

#include "internal.h"

namespace chfsi {
namespace {

struct NcclApi {
  bool tried = false, ok = false;
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclCommAbort) abort = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclGetErrorString) err = nullptr;
  decltype(&ncclGetVersion) version = nullptr;
};

NcclApi g_nccl;
std::mutex g_nccl_mu;

const NcclApi* nccl() {
  std::lock_guard<std::mutex> lock(g_nccl_mu);
  if (g_nccl.tried) return g_nccl.ok ? &g_nccl : nullptr;
  g_nccl.tried = true;
  // the process's already-loaded libnccl (torch's) first, then the loader's search path
  void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) return nullptr;
  g_nccl.init_all = (decltype(g_nccl.init_all))dlsym(lib, "ncclCommInitAll");
  g_nccl.destroy = (decltype(g_nccl.destroy))dlsym(lib, "ncclCommDestroy");
  g_nccl.abort = (decltype(g_nccl.abort))dlsym(lib, "ncclCommAbort");
  g_nccl.all_gather = (decltype(g_nccl.all_gather))dlsym(lib, "ncclAllGather");
  g_nccl.broadcast = (decltype(g_nccl.broadcast))dlsym(lib, "ncclBroadcast");
  g_nccl.err = (decltype(g_nccl.err))dlsym(lib, "ncclGetErrorString");
  g_nccl.version = (decltype(g_nccl.version))dlsym(lib, "ncclGetVersion");
  g_nccl.ok = g_nccl.init_all && g_nccl.destroy && g_nccl.abort && g_nccl.all_gather &&
              g_nccl.broadcast && g_nccl.err && g_nccl.version;
  return g_nccl.ok ? &g_nccl : nullptr;
}

int nccl_status(const NcclApi* api, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return OK;
  set_error(std::string(what) + ": " + api->err(r));
  return ERR_CUDA;
}

}  // namespace
}  // namespace chfsi

using namespace chfsi;

struct chfsi_comm_s {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1, device = 0;
};

extern "C" {

int chfsi_comm_available(int* version) {
  const NcclApi* api = nccl();
  if (version) *version = 0;
  if (!api) return 0;
  int v = 0;
  if (version && api->version(&v) == ncclSuccess) *version = v;
  return 1;
}

int chfsi_comm_init_all(int ndev, const int* devices, chfsi_comm_s** out) {
  if (ndev < 1 || !devices || !out) {
    set_error("chfsi_comm_init_all: need ndev >= 1, a device list and an output array");
    return ERR_ARG;
  }
  for (int i = 0; i < ndev; ++i)
    for (int j = 0; j < i; ++j)
      if (devices[i] == devices[j]) {
        set_error("chfsi_comm_init_all: an NCCL clique needs distinct devices");
        return ERR_ARG;
      }
  const NcclApi* api = nccl();
  if (!api) {
    set_error("chfsi_comm_init_all: libnccl.so.2 could not be loaded");
    return ERR_ARG;
  }
  std::vector<ncclComm_t> comms((size_t)ndev, nullptr);
  CHFSI_TRY(nccl_status(api, api->init_all(comms.data(), ndev, devices), "ncclCommInitAll"));
  for (int i = 0; i < ndev; ++i) {
    auto* c = new chfsi_comm_s();
    c->comm = comms[(size_t)i];
    c->rank = i;
    c->world = ndev;
    c->device = devices[i];
    out[i] = c;
  }
  return OK;
}

int chfsi_comm_destroy(chfsi_comm_s* c) {
  if (!c) return OK;
  const NcclApi* api = nccl();
  int st = OK;
  if (api && c->comm) {
    cudaSetDevice(c->device);
    st = nccl_status(api, api->destroy(c->comm), "ncclCommDestroy");
  }
  delete c;
  return st;
}

int chfsi_comm_abort(chfsi_comm_s* c) {
  if (!c) return OK;
  const NcclApi* api = nccl();
  int st = OK;
  if (api && c->comm) st = nccl_status(api, api->abort(c->comm), "ncclCommAbort");
  c->comm = nullptr;
  return st;
}

// recv (world * bytes) <- every rank's send (bytes), in rank order, on `stream`
int chfsi_comm_allgather(chfsi_comm_s* c, const void* send, void* recv, size_t bytes,
                         void* stream) {
  if (!c || !c->comm) {
    set_error("chfsi_comm_allgather: communicator closed");
    return ERR_ARG;
  }
  const NcclApi* api = nccl();
  cudaSetDevice(c->device);
  return nccl_status(api, api->all_gather(send, recv, bytes, ncclUint8, c->comm,
                                          (cudaStream_t)stream),
                     "ncclAllGather");
}

int chfsi_comm_broadcast(chfsi_comm_s* c, void* buf, size_t bytes, int root, void* stream) {
  if (!c || !c->comm) {
    set_error("chfsi_comm_broadcast: communicator closed");
    return ERR_ARG;
  }
  const NcclApi* api = nccl();
  cudaSetDevice(c->device);
  return nccl_status(api, api->broadcast(buf, buf, bytes, ncclUint8, root, c->comm,
                                         (cudaStream_t)stream),
                     "ncclBroadcast");
}

}  // extern "C"
