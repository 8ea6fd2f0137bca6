// C++ host for the multi-GPU z-slab decomposition:
// one process drives n slab solvers (one per device) of a periodic 3D domain
// and exchanges one layer of vertex data per half step between ring
// neighbours, overlapped with the interior update:
//   before the pressure half step (advance_p, stepper1d.cpp:147-156) slab r
//   needs the previous slab's last v layer (3 components) in its ghost layer
//   z = -1; before the velocity half step (advance_v, :158-166) it needs the
//   next slab's first p layer as its layer Kz.
// Per half step and slab: the layers that do not read the halo are advanced
// on the solver stream while the halo moves on a per-slab exchange stream;
// the boundary layer follows the exchange (events); the time stamp is
// committed once (hlf_commit_half).  Transports:
//   NCCL  ncclSend / ncclRecv in one group over a communicator clique
//         (ncclCommInitAll, single process; NVLink / NVSwitch between B200s).
//         libnccl.so.2 is opened lazily (dlopen), so the product library has
//         no link-time NCCL dependency and shares the copy torch loaded.
//   COPY  cudaMemcpyPeerAsync between the slabs' layers (device-to-device
//         when two slabs share a device, which is how one GPU runs a
//         multi-slab decomposition in the tests).
// Everything sits on the public C-ABI (hlf_b200.h) of the slab solvers.
#include <dlfcn.h>
#include <nccl.h>

#include <string>
#include <vector>

#include "../../include/hlf_b200.h"

struct hlf_slab_group {
  int n = 0;
  int transport = HLF_TRANSPORT_COPY;
  std::vector<int> dev;
  std::vector<hlf_solver*> s;
  std::vector<cudaStream_t> xs;                 // exchange stream per slab (on its device)
  std::vector<cudaEvent_t> ready, done;         // per slab: layer final (solver stream) / halo landed (exchange stream)
  std::vector<ncclComm_t> comm;
  std::string err;
};

namespace {

thread_local std::string g_group_error;

hlf_status gfail(hlf_slab_group* g, hlf_status st, const std::string& msg) {
  if (g) g->err = msg;
  else g_group_error = msg;
  return st;
}

#define HLF_GCUDA(g, call)                                                                            \
  do {                                                                                                \
    cudaError_t e_ = (call);                                                                          \
    if (e_ != cudaSuccess) return gfail((g), HLF_CUDA_ERROR, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

// the few NCCL entry points, resolved from libnccl.so.2 at first use
struct Nccl {
  bool ok = false;
  std::string why;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl lib = [] {
    Nccl L;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      L.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return L;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    L.CommInitAll = reinterpret_cast<decltype(L.CommInitAll)>(sym("ncclCommInitAll"));
    L.CommDestroy = reinterpret_cast<decltype(L.CommDestroy)>(sym("ncclCommDestroy"));
    L.GroupStart = reinterpret_cast<decltype(L.GroupStart)>(sym("ncclGroupStart"));
    L.GroupEnd = reinterpret_cast<decltype(L.GroupEnd)>(sym("ncclGroupEnd"));
    L.Send = reinterpret_cast<decltype(L.Send)>(sym("ncclSend"));
    L.Recv = reinterpret_cast<decltype(L.Recv)>(sym("ncclRecv"));
    L.GetErrorString = reinterpret_cast<decltype(L.GetErrorString)>(sym("ncclGetErrorString"));
    L.ok = L.CommInitAll && L.CommDestroy && L.GroupStart && L.GroupEnd && L.Send && L.Recv && L.GetErrorString;
    if (!L.ok) L.why = "libnccl.so.2 lacks ncclSend / ncclRecv";
    return L;
  }();
  return lib;
}

hlf_status nccl_check(hlf_slab_group* g, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return HLF_OK;
  return gfail(g, HLF_NCCL_ERROR, std::string(what) + ": " + nccl().GetErrorString(r));
}

hlf_status solver_check(hlf_slab_group* g, int r, hlf_status st) {
  if (st == HLF_OK) return HLF_OK;
  return gfail(g, st, "slab " + std::to_string(r) + ": " + hlf_last_error(g->s[r]));
}

// one halo exchange: kind 0 = p layer (next slab's layer 0 -> my layer Kz),
// kind 1 = v layers (previous slab's layer Kz-1 -> my ghost z = -1)
hlf_status exchange(hlf_slab_group* g, int kind) {
  const int n = g->n;
  const int ncomp = kind == 0 ? 1 : 3;
  // the exchange of slab r starts once r's sent layer is final (and, for
  // COPY, once the sender's layer is final on the sender's stream)
  for (int r = 0; r < n; ++r) {
    HLF_GCUDA(g, cudaSetDevice(g->dev[r]));
    HLF_GCUDA(g, cudaEventRecord(g->ready[r], static_cast<cudaStream_t>(hlf_get_stream(g->s[r]))));
  }
  if (g->transport == HLF_TRANSPORT_NCCL) {
    const Nccl& L = nccl();
    for (int r = 0; r < n; ++r) {
      HLF_GCUDA(g, cudaSetDevice(g->dev[r]));
      HLF_GCUDA(g, cudaStreamWaitEvent(g->xs[r], g->ready[r], 0));
    }
    hlf_status st = nccl_check(g, L.GroupStart(), "ncclGroupStart");
    if (st != HLF_OK) return st;
    for (int r = 0; r < n && st == HLF_OK; ++r) {
      // p: send my layer 0 to the previous slab, receive the next slab's;
      // v: send my last layer to the next slab, receive the previous slab's
      const int to = kind == 0 ? (r + n - 1) % n : (r + 1) % n;
      const int from = kind == 0 ? (r + 1) % n : (r + n - 1) % n;
      for (int c = 0; c < ncomp && st == HLF_OK; ++c) {
        double *sp = nullptr, *rp = nullptr;
        int64_t cnt = 0, rcnt = 0;
        st = solver_check(g, r, hlf_halo_send_ptr(g->s[r], kind, c, &sp, &cnt));
        if (st == HLF_OK) st = solver_check(g, r, hlf_halo_recv_ptr(g->s[r], kind, c, &rp, &rcnt));
        if (st == HLF_OK) st = nccl_check(g, L.Send(sp, static_cast<size_t>(cnt), ncclFloat64, to, g->comm[r], g->xs[r]), "ncclSend");
        if (st == HLF_OK) st = nccl_check(g, L.Recv(rp, static_cast<size_t>(rcnt), ncclFloat64, from, g->comm[r], g->xs[r]), "ncclRecv");
      }
    }
    hlf_status st2 = nccl_check(g, L.GroupEnd(), "ncclGroupEnd");
    if (st != HLF_OK) return st;
    if (st2 != HLF_OK) return st2;
    // a slab's send buffer and its received halo are both free / final once
    // its exchange stream passes the group
    for (int r = 0; r < n; ++r) {
      HLF_GCUDA(g, cudaSetDevice(g->dev[r]));
      HLF_GCUDA(g, cudaEventRecord(g->done[r], g->xs[r]));
    }
    return HLF_OK;
  }
  // COPY: the receiver pulls on its own exchange stream
  for (int q = 0; q < n; ++q) {
    const int r = kind == 0 ? (q + 1) % n : (q + n - 1) % n;  // the sender of q's halo
    HLF_GCUDA(g, cudaSetDevice(g->dev[q]));
    HLF_GCUDA(g, cudaStreamWaitEvent(g->xs[q], g->ready[r], 0));
    HLF_GCUDA(g, cudaStreamWaitEvent(g->xs[q], g->ready[q], 0));
    for (int c = 0; c < ncomp; ++c) {
      double *sp = nullptr, *rp = nullptr;
      int64_t cnt = 0, rcnt = 0;
      hlf_status st = solver_check(g, r, hlf_halo_send_ptr(g->s[r], kind, c, &sp, &cnt));
      if (st == HLF_OK) st = solver_check(g, q, hlf_halo_recv_ptr(g->s[q], kind, c, &rp, &rcnt));
      if (st != HLF_OK) return st;
      HLF_GCUDA(g, cudaMemcpyPeerAsync(rp, g->dev[q], sp, g->dev[r], static_cast<size_t>(cnt) * sizeof(double),
                                       g->xs[q]));
    }
    HLF_GCUDA(g, cudaEventRecord(g->done[q], g->xs[q]));
  }
  return HLF_OK;
}

// slab r's solver stream waits for the exchange that fills r's halo and,
// for COPY, for the copy that reads r's sent layer (before it is rewritten)
hlf_status wait_exchange(hlf_slab_group* g, int r, int kind) {
  const int n = g->n;
  cudaStream_t st = static_cast<cudaStream_t>(hlf_get_stream(g->s[r]));
  HLF_GCUDA(g, cudaSetDevice(g->dev[r]));
  HLF_GCUDA(g, cudaStreamWaitEvent(st, g->done[r], 0));
  if (g->transport == HLF_TRANSPORT_COPY) {
    const int reader = kind == 0 ? (r + n - 1) % n : (r + 1) % n;
    HLF_GCUDA(g, cudaStreamWaitEvent(st, g->done[reader], 0));
  }
  return HLF_OK;
}

hlf_status slab_step(hlf_slab_group* g, int step_index) {
  const int n = g->n;
  int Kz = 0;
  {
    int64_t dummy = 0;
    double* p = nullptr;
    int layers = 0;
    hlf_status st = solver_check(g, 0, hlf_field_device(g->s[0], 0, &p, &dummy, &dummy, &layers));
    if (st != HLF_OK) return st;
    Kz = layers - 1;  // p has Kz + 1 layers (layer Kz = the next slab's layer 0)
  }
  // pressure half: v halo in flight while layers 1..Kz-1 update
  hlf_status st = exchange(g, 1);
  if (st != HLF_OK) return st;
  for (int r = 0; r < n && st == HLF_OK; ++r) st = solver_check(g, r, hlf_advance_layers(g->s[r], 0, step_index, 1, Kz));
  for (int r = 0; r < n && st == HLF_OK; ++r) {
    st = wait_exchange(g, r, 1);
    if (st == HLF_OK) st = solver_check(g, r, hlf_advance_layers(g->s[r], 0, step_index, 0, 1));
    if (st == HLF_OK) st = solver_check(g, r, hlf_commit_half(g->s[r], 0));
  }
  if (st != HLF_OK) return st;
  // velocity half: p halo (final layer 0) in flight while layers 0..Kz-2 update
  st = exchange(g, 0);
  if (st != HLF_OK) return st;
  for (int r = 0; r < n && st == HLF_OK; ++r)
    st = solver_check(g, r, hlf_advance_layers(g->s[r], 1, step_index, 0, Kz - 1));
  for (int r = 0; r < n && st == HLF_OK; ++r) {
    st = wait_exchange(g, r, 0);
    if (st == HLF_OK) st = solver_check(g, r, hlf_advance_layers(g->s[r], 1, step_index, Kz - 1, Kz));
    if (st == HLF_OK) st = solver_check(g, r, hlf_commit_half(g->s[r], 1));
  }
  return st;
}

}  // namespace

extern "C" {

hlf_status hlf_slabs_create(const hlf_desc* global, int n, const int* devices, int transport, hlf_slab_group** out) {
  if (!global || !out || n < 1 || !devices) return gfail(nullptr, HLF_INVALID_ARGUMENT, "bad slab group arguments");
  *out = nullptr;
  if (global->dim != 3 || global->boundary[2] != HLF_PERIODIC)
    return gfail(nullptr, HLF_CONFIG_ERROR, "z slabs need d = 3 with a periodic z axis");
  if (global->K[2] % n != 0 || global->K[2] / n < 2)
    return gfail(nullptr, HLF_CONFIG_ERROR, "the z cells must split into slabs of >= 2 layers");
  if (global->scheme != HLF_SCHEME_LEAPFROG || global->variable_ap)
    return gfail(nullptr, HLF_CONFIG_ERROR, "slab groups run the constant-coefficient leapfrog scheme");
  bool distinct = true;
  for (int a = 0; a < n; ++a)
    for (int b = a + 1; b < n; ++b) distinct = distinct && devices[a] != devices[b];
  if (transport == HLF_TRANSPORT_AUTO) transport = (distinct && nccl().ok) ? HLF_TRANSPORT_NCCL : HLF_TRANSPORT_COPY;
  if (transport == HLF_TRANSPORT_NCCL && !nccl().ok) return gfail(nullptr, HLF_NCCL_ERROR, nccl().why);
  if (transport == HLF_TRANSPORT_NCCL && !distinct)
    return gfail(nullptr, HLF_CONFIG_ERROR, "NCCL needs one device per slab (use the copy transport on one device)");
  if (transport != HLF_TRANSPORT_NCCL && transport != HLF_TRANSPORT_COPY)
    return gfail(nullptr, HLF_INVALID_ARGUMENT, "unknown transport");
  auto* g = new hlf_slab_group;
  g->n = n;
  g->transport = transport;
  g->dev.assign(devices, devices + n);
  const int kz = global->K[2] / n;
  auto bail = [&](hlf_status st) {
    const std::string msg = g->err;
    hlf_slabs_destroy(g);
    return gfail(nullptr, st, msg);
  };
  for (int r = 0; r < n; ++r) {
    hlf_desc d = *global;
    d.K[2] = kz;
    d.x_min[2] = global->x_min[2] + r * kz * global->h;
    d.device = devices[r];
    d.stream = nullptr;  // each slab solver owns its stream
    d.z_slab = 1;
    hlf_solver* s = nullptr;
    if (hlf_create(&d, &s) != HLF_OK) {
      g->err = std::string("slab ") + std::to_string(r) + ": " + hlf_last_error(nullptr);
      return bail(HLF_CONFIG_ERROR);
    }
    g->s.push_back(s);
    cudaSetDevice(devices[r]);
    cudaStream_t xs = nullptr;
    cudaEvent_t a = nullptr, b = nullptr;
    if (cudaStreamCreateWithFlags(&xs, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&a, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&b, cudaEventDisableTiming) != cudaSuccess) {
      g->err = "stream / event creation failed";
      return bail(HLF_CUDA_ERROR);
    }
    g->xs.push_back(xs);
    g->ready.push_back(a);
    g->done.push_back(b);
  }
  if (transport == HLF_TRANSPORT_NCCL) {
    g->comm.resize(n);
    const ncclResult_t r = nccl().CommInitAll(g->comm.data(), n, devices);
    if (r != ncclSuccess) {
      g->comm.clear();
      g->err = std::string("ncclCommInitAll: ") + nccl().GetErrorString(r);
      return bail(HLF_NCCL_ERROR);
    }
  }
  *out = g;
  return HLF_OK;
}

void hlf_slabs_destroy(hlf_slab_group* g) {
  if (!g) return;
  for (int r = 0; r < static_cast<int>(g->s.size()); ++r) {
    cudaSetDevice(g->dev[r]);
    hlf_synchronize(g->s[r]);
    if (r < static_cast<int>(g->xs.size())) cudaStreamSynchronize(g->xs[r]);
  }
  for (ncclComm_t c : g->comm)
    if (c) nccl().CommDestroy(c);
  for (size_t r = 0; r < g->xs.size(); ++r) {
    cudaSetDevice(g->dev[r]);
    cudaStreamDestroy(g->xs[r]);
    cudaEventDestroy(g->ready[r]);
    cudaEventDestroy(g->done[r]);
  }
  for (hlf_solver* s : g->s) hlf_destroy(s);
  delete g;
}

const char* hlf_slabs_last_error(const hlf_slab_group* g) { return g ? g->err.c_str() : g_group_error.c_str(); }
int hlf_slabs_count(const hlf_slab_group* g) { return g ? g->n : -1; }
int hlf_slabs_transport(const hlf_slab_group* g) { return g ? g->transport : -1; }
hlf_solver* hlf_slabs_solver(hlf_slab_group* g, int r) {
  return (g && r >= 0 && r < g->n) ? g->s[r] : nullptr;
}

hlf_status hlf_slabs_set_times(hlf_slab_group* g, double t_p, double t_v, double dt) {
  if (!g) return HLF_INVALID_ARGUMENT;
  for (int r = 0; r < g->n; ++r) {
    hlf_status st = solver_check(g, r, hlf_set_times(g->s[r], t_p, t_v, dt));
    if (st != HLF_OK) return st;
  }
  return HLF_OK;
}

hlf_status hlf_slabs_advance_n(hlf_slab_group* g, int steps, int first_step) {
  if (!g || steps < 0) return HLF_INVALID_ARGUMENT;
  for (int r = 0; r < g->n; ++r) {  // this call reports its own steps only
    hlf_status st = solver_check(g, r, hlf_clear_finite(g->s[r]));
    if (st != HLF_OK) return st;
  }
  for (int i = 0; i < steps; ++i) {
    hlf_status st = slab_step(g, first_step + i);
    if (st != HLF_OK) return st;
  }
  // the finite check of every slab (check_finite, stepper1d.cpp:121-129)
  int worst = -1;
  for (int r = 0; r < g->n; ++r) {
    int bad = -1;
    hlf_status st = solver_check(g, r, hlf_poll_finite(g->s[r], &bad));
    if (st != HLF_OK) return st;
    if (bad >= 0 && (worst < 0 || bad < worst)) worst = bad;
  }
  if (worst >= 0) return gfail(g, HLF_INSTABILITY, "solution became non-finite at step " + std::to_string(worst));
  return HLF_OK;
}

hlf_status hlf_slabs_synchronize(hlf_slab_group* g) {
  if (!g) return HLF_INVALID_ARGUMENT;
  for (int r = 0; r < g->n; ++r) {
    hlf_status st = solver_check(g, r, hlf_synchronize(g->s[r]));
    if (st != HLF_OK) return st;
    HLF_GCUDA(g, cudaSetDevice(g->dev[r]));
    HLF_GCUDA(g, cudaStreamSynchronize(g->xs[r]));
  }
  return HLF_OK;
}

}  // extern "C"
