// Device-backed admission controllers: the
// reference's standalone controller ABI (kvadmit.h:86-159, capi.cpp:172-292,
// controller.cpp) for N controllers at once, their state resident in HBM.
//
//   update_window   one thread per controller (controller.cpp:67-91)
//   admission_pass  one warp per controller: the pause victim (the newest
//                   active agent at a step boundary, controller.cpp:130-136)
//                   is a warp-wide reverse ballot scan over the active list,
//                   the erase a warp-wide in-order shift
//   events          one thread per controller over its slice of the event
//                   batch (add_pending / on_agent_finished /
//                   on_request_complete / on_tool_return, controller.cpp:
//                   162-193), in submission order
// Arithmetic is the reference's (IEEE double, -fmad=false), so windows are
// bit-identical.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "host_internal.h"
#include "kvg_device.h"

using kvg_host::set_error;

namespace kvg {
namespace {

struct CtlDev {
  kvg_policy policy;  // aimd.w_max / initial_window resolved (controller.cpp:55-65)
  double window, su, sh;
  u64 ticks;
  u32 total, act_n, pend_head, pend_n, paus_head, paus_n;
  u32 cap;  // list capacity: the reference's vector / deques are unbounded and
            // misuse (re-queueing an admitted agent) can hold an id twice, so
            // lists get max(4 x total, total + 256) slots; overflow = KVG_ERR_STATE
  int have_s, err;
  u32* active;  // [cap] insertion-ordered
  u32* pend;    // [cap] FIFO ring
  u32* paus;    // [cap] FIFO ring
};

constexpr unsigned FULLM = 0xffffffffu;

__device__ __forceinline__ double display_window(const CtlDev& c) {  // controller.cpp:106-117
  switch (c.policy.kind) {
    case KVG_POLICY_UNCONTROLLED: return static_cast<double>(c.total);
    case KVG_POLICY_AIMD: return c.window;
    default: return static_cast<double>(c.policy.cap);
  }
}

__device__ __forceinline__ u64 admission_limit(const CtlDev& c) {  // controller.cpp:93-104
  switch (c.policy.kind) {
    case KVG_POLICY_UNCONTROLLED: return ~0ull;
    case KVG_POLICY_AIMD: return static_cast<u64>(floor(c.window));
    default: return c.policy.cap;
  }
}

__global__ void k_update_window(CtlDev* cs, u32 n, const double* usage, const double* hit,
                                double* out) {
  const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  CtlDev& c = cs[i];
  ++c.ticks;
  if (c.policy.kind == KVG_POLICY_AIMD) {
    const kvg_controller_config& cfg = c.policy.aimd;
    double u = usage[i], h = hit[i];
    if (cfg.signal_smoothing > 0) {
      if (c.have_s) {
        u = cfg.signal_smoothing * c.su + (1 - cfg.signal_smoothing) * usage[i];
        h = cfg.signal_smoothing * c.sh + (1 - cfg.signal_smoothing) * hit[i];
      }
      c.su = u;
      c.sh = h;
      c.have_s = 1;
    }
    double w = c.window;
    if (u < cfg.u_low) w = w + cfg.alpha;
    else if (u > cfg.u_high && h < cfg.h_thresh) w = w * cfg.beta;
    c.window = w < cfg.w_min ? cfg.w_min : (cfg.w_max < w ? cfg.w_max : w);
  }
  if (out) out[i] = display_window(c);
}

__device__ __forceinline__ u32 ring(u32 head, u32 k, u32 cap) {
  const u32 i = head + k;
  return i >= cap ? i - cap : i;
}

// admission_pass, controller.cpp:124-160. One warp per controller; every
// lane tracks the list sizes in registers (identical values), lane 0 writes.
__global__ void k_admission(CtlDev* cs, u32 n, const uint8_t* at_boundary, const u64* agent_off,
                            const u64* cmd_off, kvg_command* cmds, u64* n_out) {
  const u32 ci = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (ci >= n) return;
  CtlDev& c = cs[ci];
  const uint8_t* bnd = at_boundary + agent_off[ci];
  kvg_command* out = cmds + cmd_off[ci];
  u32* const active = c.active;
  u32 act = c.act_n, paus_n = c.paus_n, paus_head = c.paus_head;
  u32 pend_n = c.pend_n, pend_head = c.pend_head;
  const u32 total = c.cap;
  u64 k = 0;
  const u64 kcap = cmd_off[ci + 1] - cmd_off[ci];  // scratch: the list capacity
  const u64 limit = admission_limit(c);
  const bool gated = c.policy.kind == KVG_POLICY_AGENT_CAP || c.policy.kind == KVG_POLICY_AIMD;
  if (gated) {
    while (act > limit && k < kcap) {
      // newest active agent at a step boundary: reverse scan, 32 at a time
      long long victim = -1;
      for (long long base = static_cast<long long>(act) - 1; base >= 0 && victim < 0;
           base -= 32) {
        const long long idx = base - lane;
        const bool hitb = idx >= 0 && bnd[active[idx]] != 0;
        const unsigned m = __ballot_sync(FULLM, hitb);
        if (m) victim = base - (__ffs(m) - 1);
      }
      if (victim < 0) break;
      const u32 id = active[victim];
      __syncwarp();
      for (u32 b = static_cast<u32>(victim); b + 1 < act; b += 32) {  // erase: shift left
        const u32 j = b + lane;
        u32 v = 0;
        if (j + 1 < act) v = active[j + 1];
        __syncwarp();
        if (j + 1 < act) active[j] = v;
        __syncwarp();
      }
      --act;
      if (lane == 0) {
        c.paus[ring(paus_head, paus_n, total)] = id;
        out[k] = kvg_command{KVG_CMD_PAUSE, {0, 0, 0}, id};
      }
      ++paus_n;
      ++k;
      __syncwarp();
    }
  }
  if (lane == 0) {
    while (act < limit) {
      if (k >= kcap) {  // more commands than agents: only after API misuse
        c.err = KVG_ERR_STATE;
        break;
      }
      u32 id;
      uint8_t kind;
      if (gated && paus_n > 0) {
        id = c.paus[paus_head];
        paus_head = ring(paus_head, 1, total);
        --paus_n;
        kind = KVG_CMD_RESUME;
      } else if (pend_n > 0) {
        id = c.pend[pend_head];
        pend_head = ring(pend_head, 1, total);
        --pend_n;
        kind = KVG_CMD_ADMIT;
      } else {
        break;
      }
      if (act >= total) {  // list full (API misuse re-queued ids)
        c.err = KVG_ERR_STATE;
        break;
      }
      active[act++] = id;
      out[k++] = kvg_command{kind, {0, 0, 0}, id};
    }
    c.act_n = act;
    c.paus_n = paus_n;
    c.paus_head = paus_head;
    c.pend_n = pend_n;
    c.pend_head = pend_head;
    n_out[ci] = k;
  }
}

__device__ bool erase_active(CtlDev& c, u32 id) {
  for (u32 i = 0; i < c.act_n; ++i) {
    if (c.active[i] != id) continue;
    for (u32 j = i; j + 1 < c.act_n; ++j) c.active[j] = c.active[j + 1];
    --c.act_n;
    return true;
  }
  return false;
}

__device__ bool add_pending(CtlDev& c, u32 id) {
  if (c.pend_n >= c.cap) return false;
  c.pend[ring(c.pend_head, c.pend_n, c.cap)] = id;
  ++c.pend_n;
  return true;
}

// controller.cpp:162-193, in submission order per controller.
__global__ void k_events(CtlDev* cs, u32 n, const kvg_ctl_event* ev, const u64* ev_off,
                         const u32* order, int32_t* status) {
  const u32 ci = blockIdx.x * blockDim.x + threadIdx.x;
  if (ci >= n) return;
  CtlDev& c = cs[ci];
  for (u64 t = ev_off[ci]; t < ev_off[ci + 1]; ++t) {
    const u32 e = order[t];
    const kvg_ctl_event& x = ev[e];
    int st = KVG_OK;
    if (x.agent >= c.total) {
      st = KVG_ERR_CONFIG;
    } else {
      switch (x.kind) {
        case KVG_CTL_ADD_PENDING:
          if (!add_pending(c, x.agent)) st = KVG_ERR_STATE;
          break;
        case KVG_CTL_AGENT_FINISHED:
          if (!erase_active(c, x.agent)) st = KVG_ERR_STATE;  // UnknownAgent
          break;
        case KVG_CTL_REQUEST_COMPLETE:
          if (c.policy.kind == KVG_POLICY_REQUEST_CAP && !erase_active(c, x.agent))
            st = KVG_ERR_STATE;
          break;
        case KVG_CTL_TOOL_RETURN:
          if (c.policy.kind == KVG_POLICY_REQUEST_CAP) {
            if (!add_pending(c, x.agent)) st = KVG_ERR_STATE;
          } else {
            bool found = false;
            for (u32 i = 0; i < c.act_n && !found; ++i) found = c.active[i] == x.agent;
            if (!found) st = KVG_ERR_STATE;
          }
          break;
        default: st = KVG_ERR_CONFIG;
      }
    }
    if (status) status[e] = st;
  }
}

}  // namespace
}  // namespace kvg

struct kvg_controllers {
  int device = 0;
  size_t n = 0;
  kvg::CtlDev* d = nullptr;
  kvg::u32* lists = nullptr;
  kvg::u64* agent_off = nullptr;  // device [n+1]
  kvg::u64* list_off = nullptr;   // device [n+1]
  std::vector<kvg::u64> h_off;    // host copy
  std::vector<kvg::u64> l_off;    // list offsets (capacity per controller)
  std::vector<kvg::u32> total;
};

#define CUDA_TRY2(x)                                                          \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) return (kvg_status)set_error(KVG_ERR_CUDA, cudaGetErrorString(e_)); \
  } while (0)

extern "C" {

KVG_API kvg_status kvg_controllers_create(int device, size_t n, const kvg_policy* policies,
                                          const uint32_t* total_agents,
                                          kvg_controllers** out) {
  if (out == nullptr || (n > 0 && (policies == nullptr || total_agents == nullptr)))
    return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  for (size_t i = 0; i < n; ++i) {
    std::string why;
    if (!kvg_host::validate_policy(policies[i], &why))
      return (kvg_status)set_error(KVG_ERR_CONFIG, "controller " + std::to_string(i) + ": " + why);
  }
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return (kvg_status)set_error(KVG_ERR_CUDA, "no CUDA device: the B200 engine has no CPU fallback");
  CUDA_TRY2(cudaSetDevice(device));
  auto* h = new kvg_controllers();
  h->device = device;
  h->n = n;
  h->h_off.assign(n + 1, 0);
  h->total.assign(total_agents, total_agents + n);
  h->l_off.assign(n + 1, 0);
  auto list_cap = [](kvg::u32 t) { return std::max<kvg::u64>(4ull * t, t + 256ull); };
  for (size_t i = 0; i < n; ++i) {
    h->h_off[i + 1] = h->h_off[i] + total_agents[i];
    h->l_off[i + 1] = h->l_off[i] + list_cap(total_agents[i]);
  }
  const kvg::u64 slots = h->l_off[n];
  std::vector<kvg::CtlDev> hs(n);
  cudaError_t e = cudaMalloc(&h->d, std::max<size_t>(1, n) * sizeof(kvg::CtlDev));
  if (e == cudaSuccess) e = cudaMalloc(&h->lists, std::max<kvg::u64>(1, 3 * slots) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&h->agent_off, (n + 1) * 8);
  if (e == cudaSuccess) e = cudaMalloc(&h->list_off, (n + 1) * 8);
  if (e != cudaSuccess) {
    kvg_controllers_free(h);
    return (kvg_status)set_error(KVG_ERR_CUDA, cudaGetErrorString(e));
  }
  for (size_t i = 0; i < n; ++i) {
    kvg::CtlDev& c = hs[i];
    std::memset(&c, 0, sizeof c);
    c.policy = policies[i];
    c.total = total_agents[i];
    c.window = 1.0;  // Controller::window_ default (controller.hpp:119)
    if (c.policy.kind == KVG_POLICY_AIMD) {  // Controller ctor, controller.cpp:55-65
      kvg_controller_config& cfg = c.policy.aimd;
      if (cfg.w_max == 0) cfg.w_max = std::max(cfg.w_min, static_cast<double>(c.total));
      if (cfg.initial_window == 0) cfg.initial_window = cfg.w_min;
      c.window = cfg.initial_window;
    }
    c.cap = static_cast<kvg::u32>(list_cap(c.total));
    c.active = h->lists + h->l_off[i];
    c.pend = h->lists + slots + h->l_off[i];
    c.paus = h->lists + 2 * slots + h->l_off[i];
  }
  if (n) {
    e = cudaMemcpy(h->d, hs.data(), n * sizeof(kvg::CtlDev), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
      e = cudaMemcpy(h->agent_off, h->h_off.data(), (n + 1) * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
      e = cudaMemcpy(h->list_off, h->l_off.data(), (n + 1) * 8, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      kvg_controllers_free(h);
      return (kvg_status)set_error(KVG_ERR_CUDA, cudaGetErrorString(e));
    }
  }
  *out = h;
  return KVG_OK;
}

KVG_API void kvg_controllers_free(kvg_controllers* h) {
  if (h == nullptr) return;
  cudaSetDevice(h->device);
  cudaFree(h->d);
  cudaFree(h->lists);
  cudaFree(h->agent_off);
  cudaFree(h->list_off);
  delete h;
}

KVG_API kvg_status kvg_controllers_update_window(kvg_controllers* h, const double* usage,
                                                 const double* hit_rate, double* window_out) {
  if (h == nullptr || (h->n > 0 && (usage == nullptr || hit_rate == nullptr)))
    return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  for (size_t i = 0; i < h->n; ++i)
    if (!std::isfinite(usage[i]) || !std::isfinite(hit_rate[i]))
      return (kvg_status)set_error(KVG_ERR_CONFIG, "signals must be finite");
  if (h->n == 0) return KVG_OK;
  CUDA_TRY2(cudaSetDevice(h->device));
  double* dbuf = nullptr;
  CUDA_TRY2(cudaMalloc(&dbuf, 3 * h->n * sizeof(double)));
  cudaMemcpy(dbuf, usage, h->n * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemcpy(dbuf + h->n, hit_rate, h->n * sizeof(double), cudaMemcpyHostToDevice);
  kvg::k_update_window<<<static_cast<unsigned>((h->n + 127) / 128), 128>>>(
      h->d, static_cast<kvg::u32>(h->n), dbuf, dbuf + h->n, dbuf + 2 * h->n);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && window_out)
    e = cudaMemcpy(window_out, dbuf + 2 * h->n, h->n * sizeof(double), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaFree(dbuf);
  if (e != cudaSuccess) return (kvg_status)set_error(KVG_ERR_CUDA, cudaGetErrorString(e));
  return KVG_OK;
}

KVG_API kvg_status kvg_controllers_admission_pass(kvg_controllers* h, const uint8_t* at_boundary,
                                                  kvg_command* commands, size_t* n_out,
                                                  int32_t* status) {
  if (h == nullptr || (h->n > 0 && (at_boundary == nullptr || commands == nullptr ||
                                    n_out == nullptr)))
    return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  if (h->n == 0) return KVG_OK;
  CUDA_TRY2(cudaSetDevice(h->device));
  const kvg::u64 slots = h->h_off[h->n], lslots = h->l_off[h->n];
  char* buf = nullptr;
  const size_t bb = (slots + 15) / 16 * 16;
  CUDA_TRY2(cudaMalloc(&buf, bb + lslots * sizeof(kvg_command) + h->n * 8 + 16));
  uint8_t* d_b = reinterpret_cast<uint8_t*>(buf);
  kvg_command* d_c = reinterpret_cast<kvg_command*>(buf + bb);
  kvg::u64* d_n = reinterpret_cast<kvg::u64*>(buf + bb + lslots * sizeof(kvg_command));
  cudaMemcpy(d_b, at_boundary, slots, cudaMemcpyHostToDevice);
  const unsigned warps_per_block = 4;
  kvg::k_admission<<<static_cast<unsigned>((h->n + warps_per_block - 1) / warps_per_block),
                     32 * warps_per_block>>>(h->d, static_cast<kvg::u32>(h->n), d_b,
                                             h->agent_off, h->list_off, d_c, d_n);
  cudaError_t e = cudaGetLastError();
  std::vector<kvg::u64> nn(h->n);
  std::vector<kvg_command> cc(lslots);
  if (e == cudaSuccess) e = cudaMemcpy(nn.data(), d_n, h->n * 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess)
    e = cudaMemcpy(cc.data(), d_c, lslots * sizeof(kvg_command), cudaMemcpyDeviceToHost);
  cudaFree(buf);
  if (e != cudaSuccess) return (kvg_status)set_error(KVG_ERR_CUDA, cudaGetErrorString(e));
  // A pass emits at most one command per agent unless the lists hold an id
  // twice (API misuse): the reference then fails the call after the pass has
  // run (capi.cpp:228-236); so does controller i here (status[i]).
  int worst = KVG_OK;
  for (size_t i = 0; i < h->n; ++i) {
    const kvg::u64 cap = h->h_off[i + 1] - h->h_off[i];
    int st = KVG_OK;
    if (nn[i] > cap) {
      st = KVG_ERR_STATE;
      n_out[i] = 0;
      if (worst == KVG_OK) worst = st;
    } else {
      n_out[i] = nn[i];
      std::copy(cc.begin() + h->l_off[i], cc.begin() + h->l_off[i] + nn[i],
                commands + h->h_off[i]);
    }
    if (status) status[i] = st;
  }
  if (worst != KVG_OK)
    return (kvg_status)set_error(worst, "admission pass emitted more commands than agents");
  return KVG_OK;
}

KVG_API kvg_status kvg_controllers_apply(kvg_controllers* h, const kvg_ctl_event* events,
                                         size_t n_events, int32_t* status) {
  if (h == nullptr || (n_events > 0 && events == nullptr))
    return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  if (n_events == 0 || h->n == 0) return KVG_OK;
  for (size_t i = 0; i < n_events; ++i)
    if (events[i].controller >= h->n)
      return (kvg_status)set_error(KVG_ERR_CONFIG, "event names an unknown controller");
  // bucket events by controller, keeping submission order (counting sort)
  std::vector<kvg::u64> off(h->n + 1, 0);
  for (size_t i = 0; i < n_events; ++i) ++off[events[i].controller + 1];
  for (size_t i = 0; i < h->n; ++i) off[i + 1] += off[i];
  std::vector<kvg::u32> order(n_events);
  std::vector<kvg::u64> fill(off.begin(), off.end() - 1);
  for (size_t i = 0; i < n_events; ++i) order[fill[events[i].controller]++] = static_cast<kvg::u32>(i);
  CUDA_TRY2(cudaSetDevice(h->device));
  char* buf = nullptr;
  const size_t eb = n_events * sizeof(kvg_ctl_event), ob = (h->n + 1) * 8, rb = n_events * 4;
  CUDA_TRY2(cudaMalloc(&buf, eb + ob + 2 * rb + 64));
  auto* d_e = reinterpret_cast<kvg_ctl_event*>(buf);
  auto* d_off = reinterpret_cast<kvg::u64*>(buf + eb);
  auto* d_ord = reinterpret_cast<kvg::u32*>(buf + eb + ob);
  auto* d_st = reinterpret_cast<int32_t*>(buf + eb + ob + rb);
  cudaMemcpy(d_e, events, eb, cudaMemcpyHostToDevice);
  cudaMemcpy(d_off, off.data(), ob, cudaMemcpyHostToDevice);
  cudaMemcpy(d_ord, order.data(), rb, cudaMemcpyHostToDevice);
  kvg::k_events<<<static_cast<unsigned>((h->n + 127) / 128), 128>>>(
      h->d, static_cast<kvg::u32>(h->n), d_e, d_off, d_ord, d_st);
  cudaError_t e = cudaGetLastError();
  std::vector<int32_t> st(n_events);
  if (e == cudaSuccess) e = cudaMemcpy(st.data(), d_st, rb, cudaMemcpyDeviceToHost);
  cudaFree(buf);
  if (e != cudaSuccess) return (kvg_status)set_error(KVG_ERR_CUDA, cudaGetErrorString(e));
  int worst = KVG_OK;
  for (size_t i = 0; i < n_events; ++i) {
    if (status) status[i] = st[i];
    if (st[i] != KVG_OK && worst == KVG_OK) worst = st[i];
  }
  if (worst != KVG_OK)
    return (kvg_status)set_error(worst, "controller event rejected (unknown agent or full queue)");
  return KVG_OK;
}

KVG_API kvg_status kvg_controllers_state(const kvg_controllers* h, double* window,
                                         double* display_window, uint64_t* ticks,
                                         size_t* active, size_t* pending, size_t* paused) {
  if (h == nullptr) return (kvg_status)set_error(KVG_ERR_CONFIG, "null argument");
  if (h->n == 0) return KVG_OK;
  CUDA_TRY2(cudaSetDevice(h->device));
  std::vector<kvg::CtlDev> hs(h->n);
  CUDA_TRY2(cudaMemcpy(hs.data(), h->d, h->n * sizeof(kvg::CtlDev), cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < h->n; ++i) {
    const kvg::CtlDev& c = hs[i];
    if (window) window[i] = c.window;
    if (display_window)
      display_window[i] = c.policy.kind == KVG_POLICY_UNCONTROLLED ? static_cast<double>(c.total)
                          : c.policy.kind == KVG_POLICY_AIMD       ? c.window
                                                                   : static_cast<double>(c.policy.cap);
    if (ticks) ticks[i] = c.ticks;
    if (active) active[i] = c.act_n;
    if (pending) pending[i] = c.pend_n;
    if (paused) paused[i] = c.paus_n;
  }
  return KVG_OK;
}

/* The active list of controller i, in admission order (controller.hpp:122). */
KVG_API kvg_status kvg_controllers_active(const kvg_controllers* h, size_t i, uint32_t* out,
                                          size_t cap, size_t* n_out) {
  if (h == nullptr || i >= h->n || n_out == nullptr)
    return (kvg_status)set_error(KVG_ERR_CONFIG, "bad argument");
  CUDA_TRY2(cudaSetDevice(h->device));
  kvg::CtlDev c;
  CUDA_TRY2(cudaMemcpy(&c, h->d + i, sizeof c, cudaMemcpyDeviceToHost));
  *n_out = c.act_n;
  if (out && cap)
    CUDA_TRY2(cudaMemcpy(out, c.active, std::min<size_t>(cap, c.act_n) * 4, cudaMemcpyDeviceToHost));
  return KVG_OK;
}

}  // extern "C"
