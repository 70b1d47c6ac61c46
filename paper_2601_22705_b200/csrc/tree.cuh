// Offload-mode radix tree (EvictionMode::kOffload) for the engine leader
// (included by leader.cuh after the Lead struct).
//
// Node-granular restatement of cache_tree.cpp, step for step with the CPU
// oracle's TreeCache (oracle/kvoracle.cpp), which is pinned per event to the
// unmodified reference. Everything here runs on the leader thread except the
// eviction frontier scan, which is a cooperative op (OP_FRONTIER, engine.cu):
// all warps of the CTA sweep the node pool and compact the frontier nodes
// (device, slots > 0, unpinned, children_with_device == 0) into a heap array.
// The flat sweep equals the reference's collect_frontier DFS (cache_tree.cpp:
// 236-249): checked on every offload fixture (KVO_CHECK_FLAT_FRONTIER).
#pragma once

namespace kvg {

// ------------------------------------------------------------ node pool

__device__ __forceinline__ u64 t_key(const Lead& L, u32 a, u64 k) {
  return ((k < L.S ? 0ull : static_cast<u64>(a) + 1) << 32) | k;
}
__device__ __forceinline__ u64 t_nkey(const Lead& L, const TNodeDev& n, u64 k) {
  return ((k < L.S ? 0ull : static_cast<u64>(n.tail)) << 32) | k;
}
__device__ __forceinline__ bool t_subdev(const TNodeDev& n) {
  return n.device_slots > 0 || n.cwd > 0;
}

// ------------------------------------------------------------ walk mirror

extern __shared__ __align__(16) unsigned char kvg_tw_smem[];  // the dynamic smem (engine_body)

// The walk loops keep the mirror's placement and the shared-prompt bound in
// registers (stores through generic pointers would otherwise force the Lead
// fields to be re-read from shared memory on every level).
struct TWc {
  u32 off, n;   // shared-memory part: ids [0, n) at kvg_tw_smem + off, pins after
  TWalk* g;     // HBM part
  TNodeDev* N;  // pins of ids >= n: the authoritative records
  u32 S, pad;   // shared-prompt pages
};
__device__ __forceinline__ TWc tw_ctx(const SimDev& D, const Lead& L) {
  return TWc{L.tw_off, L.tw_n, D.twalk, D.tnodes, static_cast<u32>(L.S), 0};
}
__device__ __forceinline__ uint4* tw_sm(const TWc& W) {
  return reinterpret_cast<uint4*>(kvg_tw_smem + W.off);
}
__device__ __forceinline__ TMeta* tw_sm_meta(const TWc& W) {
  return reinterpret_cast<TMeta*>(kvg_tw_smem + W.off + static_cast<size_t>(W.n) * sizeof(TWalk));
}
__device__ __forceinline__ TWalk tw_get(const TWc& W, u32 id) {
  uint4 v;
  if (id < W.n) v = tw_sm(W)[id];
  else v = reinterpret_cast<const uint4*>(W.g)[id];
  return TWalk{v.x, v.y, v.z, v.w};
}
__device__ __forceinline__ void tw_set(const TWc& W, u32 id, const TWalk& t) {
  const uint4 v = make_uint4(t.first_child, t.start, t.npages, t.tailh);
  if (id < W.n) tw_sm(W)[id] = v;
  else reinterpret_cast<uint4*>(W.g)[id] = v;
}
__device__ __forceinline__ TWalk* tw_ref(const TWc& W, u32 id) {  // single-field writes
  return id < W.n ? reinterpret_cast<TWalk*>(tw_sm(W)) + id : W.g + id;
}
__device__ __forceinline__ int tw_pin(const TWc& W, u32 id) {
  return id < W.n ? tw_sm_meta(W)[id].pin_count : W.N[id].pin_count;
}
__device__ __forceinline__ void tw_set_pin(const TWc& W, u32 id, int v) {
  if (id < W.n) tw_sm_meta(W)[id].pin_count = v;
  W.N[id].pin_count = v;
}
// the frontier twins: every write of device_slots / cwd / alive goes through these
__device__ __forceinline__ void tm_slots(const TWc& W, u32 id, u32 v) {
  if (id < W.n) tw_sm_meta(W)[id].device_slots = v;
  W.N[id].device_slots = v;
}
__device__ __forceinline__ void tm_cwd(const TWc& W, u32 id, int v) {
  if (id < W.n) tw_sm_meta(W)[id].cwd = v;
  W.N[id].cwd = v;
}
__device__ __forceinline__ void tm_alive(const TWc& W, u32 id, u32 v) {
  if (id < W.n) tw_sm_meta(W)[id].alive = v;
  W.N[id].alive = v;
}
__device__ __forceinline__ void tw_put(const TWc& W, u32 id, const TNodeDev& n) {
  tw_set(W, id, TWalk{n.first_child, n.start, n.npages, n.tail | (n.host ? 0x80000000u : 0u)});
  if (id < W.n) tw_sm_meta(W)[id] = TMeta{n.device_slots, n.pin_count, n.cwd, n.alive};
}
__device__ __forceinline__ void tw_host(const TWc& W, u32 id, u32 host) {
  TWalk* w = tw_ref(W, id);
  w->tailh = (w->tailh & 0x7fffffffu) | (host ? 0x80000000u : 0u);
}
__device__ __forceinline__ bool tw_is_host(const TWalk& w) { return (w.tailh >> 31) != 0; }

__device__ u32 h_find(const SimDev& D, u64 key) {
  u32 i = static_cast<u32>(hash64(key)) & D.hmask;
  for (;;) {
    const u64 k = D.hkeys[i];
    if (k == key) return D.hvals[i];
    if (k == kEmptyKey) return 0;
    i = (i + 1) & D.hmask;
  }
}
__device__ void h_insert(const SimDev& D, u64 key, u32 v) {
  u32 i = static_cast<u32>(hash64(key)) & D.hmask;
  for (;;) {
    const u64 k = D.hkeys[i];
    if (k == kEmptyKey || k == kTombKey) {
      D.hkeys[i] = key;
      D.hvals[i] = v;
      return;
    }
    i = (i + 1) & D.hmask;
  }
}
__device__ void h_erase(const SimDev& D, u64 key) {
  u32 i = static_cast<u32>(hash64(key)) & D.hmask;
  for (;;) {
    const u64 k = D.hkeys[i];
    if (k == key) {
      D.hkeys[i] = kTombKey;
      return;
    }
    if (k == kEmptyKey) return;
    i = (i + 1) & D.hmask;
  }
}

__device__ u32 t_alloc(const SimDev& D, Lead& L) {
  if (L.t_free_n > 0) return D.tfree[--L.t_free_n];
  if (L.t_alloc >= D.tcap) {
    fail(L, E_TABLE_FULL);
    return 0;
  }
  return L.t_alloc++;
}

__device__ void t_add_child(const SimDev& D, const Lead& L, u32 p, u32 c) {
  TNodeDev* N = D.tnodes;
  N[c].parent = p;
  N[c].prev_sib = 0;
  N[c].next_sib = N[p].first_child;
  if (N[p].first_child) N[N[p].first_child].prev_sib = c;
  N[p].first_child = c;
  tw_ref(tw_ctx(D, L), p)->first_child = c;
}
__device__ void t_remove_child(const SimDev& D, const Lead& L, u32 p, u32 c) {
  TNodeDev* N = D.tnodes;
  if (N[c].prev_sib) {
    N[N[c].prev_sib].next_sib = N[c].next_sib;
  } else {
    N[p].first_child = N[c].next_sib;
    tw_ref(tw_ctx(D, L), p)->first_child = N[c].next_sib;
  }
  if (N[c].next_sib) N[N[c].next_sib].prev_sib = N[c].prev_sib;
}

// find_child (cache_tree.cpp:56-66): a full page of the sequence is needed.
// Eviction tail-splits make the paths hundreds of nodes deep, nearly all of
// them single-child links, so the first child is tried before the hash: one
// dependent load per level instead of three. A node's children have distinct
// head keys (the reference's per-node map), so a first child whose head key
// matches IS the child; otherwise the head-key hash decides as before.
// Walk levels are 32-bit page arithmetic (contexts stay below 2^32 tokens:
// checked at batch create). `fc` is the first child of `node`, carried from
// the previous level's mirror load.
__device__ __noinline__ u32 w_find_slow(const SimDev& D, u32 node, u64 key) {
  const u32 c = h_find(D, key);
  return (c != 0 && D.tnodes[c].parent == node) ? c : 0;
}
__device__ __forceinline__ u32 w_find_child(const SimDev& D, const TWc& W, u32 node, u32 fc, u32 a,
                                             u32 p, u32 n_full) {
  if (p >= n_full) return 0;
  if (fc != 0) {
    const TWalk x = tw_get(W, fc);
    if (x.start == p && (p < W.S || (x.tailh & 0x7fffffffu) == a + 1)) return fc;
  }
  const u64 owner = p < W.S ? 0ull : static_cast<u64>(a) + 1;
  return w_find_slow(D, node, (owner << 32) | p);
}
__device__ u32 t_find_child(const SimDev& D, const Lead& L, u32 node, u32 a, u64 p, u64 n_full) {
  const TWc W = tw_ctx(D, L);
  return w_find_child(D, W, node, tw_get(W, node).first_child, a, static_cast<u32>(p),
                      static_cast<u32>(n_full));
}

// common_len in whole pages (a partial trailing page never counts).
__device__ __forceinline__ u32 w_common(const TWalk& n, u32 S, u32 a, u32 p, u32 n_full) {
  u32 k = n.npages < n_full - p ? n.npages : n_full - p;
  if ((n.tailh & 0x7fffffffu) != a + 1) {
    const u32 sh = S > p ? S - p : 0;
    k = k < sh ? k : sh;
  }
  return k;
}
__device__ __forceinline__ u64 t_common(const SimDev& D, const Lead& L, u32 c, u32 a, u64 p,
                                        u64 n_full) {
  const TWc W = tw_ctx(D, L);
  return w_common(tw_get(W, c), W.S, a, static_cast<u32>(p), static_cast<u32>(n_full));
}

// split_node, cache_tree.cpp:68-92 (offset in pages). Returns the suffix.
__device__ u32 t_split(const SimDev& D, Lead& L, u32 id, u64 off) {
  const u32 sid = t_alloc(D, L);
  if (sid == 0) return id;
  TNodeDev* N = D.tnodes;
  TNodeDev n = N[id];
  TNodeDev s;
  s.start = n.start + static_cast<u32>(off);
  s.npages = n.npages - static_cast<u32>(off);
  s.tail = n.tail;
  s.first_child = n.first_child;
  s.parent = id;
  s.next_sib = s.prev_sib = 0;
  s.last_access = n.last_access;
  s.ordinal = L.t_next_ord++;
  s.host = n.host;
  s.pin_count = n.pin_count;
  s.cwd = n.cwd;
  s.alive = 1;
  s.device_slots = 0;
  const TWc W = tw_ctx(D, L);
  if (!n.host) {
    s.device_slots = n.device_slots - static_cast<u32>(off);
    tm_slots(W, id, static_cast<u32>(off));
  }
  N[sid] = s;
  tw_put(W, sid, s);
  for (u32 c = s.first_child; c != 0; c = N[c].next_sib) N[c].parent = sid;
  N[id].npages = static_cast<u32>(off);
  N[id].first_child = 0;
  tm_cwd(W, id, t_subdev(s) ? 1 : 0);
  TWalk* w = tw_ref(W, id);
  w->npages = static_cast<u32>(off);
  w->first_child = 0;
  t_add_child(D, L, id, sid);
  h_insert(D, t_nkey(L, s, s.start), sid);
  return sid;
}

__device__ void t_gain(const SimDev& D, const Lead& L, u32 id) {  // propagate_gain, cache_tree.cpp:94-102
  TNodeDev* N = D.tnodes;
  const TWc W = tw_ctx(D, L);
  u32 p = N[id].parent;
  for (;;) {
    const bool had = t_subdev(N[p]);
    tm_cwd(W, p, N[p].cwd + 1);
    if (had || p == 0) break;
    p = N[p].parent;
  }
}
__device__ void t_loss(const SimDev& D, const Lead& L, u32 id) {  // propagate_loss, cache_tree.cpp:104-112
  TNodeDev* N = D.tnodes;
  const TWc W = tw_ctx(D, L);
  u32 p = N[id].parent;
  for (;;) {
    tm_cwd(W, p, N[p].cwd - 1);
    if (t_subdev(N[p]) || p == 0) break;
    p = N[p].parent;
  }
}

__device__ __forceinline__ bool t_frontier(const TNodeDev& n) {  // cache_tree.cpp:230-234
  return n.alive && !n.host && n.device_slots > 0 && n.pin_count == 0 && n.cwd == 0;
}

// OP_FRONTIER: the CTA sweeps the node pool and compacts the frontier nodes
// into op.fr with one atomic per warp (ballot + rank). Node ids below the
// shared-memory mirror bound are decided from the mirror (TWalk host bit +
// TMeta) and only the frontier ids then fetch (last_access, ordinal) from HBM,
// all at once after a barrier; ids above it read their 64 B records from HBM,
// one lane per record, kFrU records per lane in flight.
constexpr int kFrU = 4;
__device__ __forceinline__ void fr_emit(Op& op, int lane, bool f, const FrEnt& e) {
  const unsigned m = __ballot_sync(FULL, f);
  if (m == 0) return;
  u32 b0 = 0;
  if (lane == 0) b0 = atomicAdd(&op.fr_n, static_cast<unsigned>(__popc(m)));
  b0 = __shfl_sync(FULL, b0, 0);
  if (f) op.fr[b0 + __popc(m & ((1u << lane) - 1u))] = e;
}
__device__ __noinline__ void coop_frontier(Op& op, int warp, int lane, int nw) {
  static_assert(offsetof(TNodeDev, last_access) == 0 && offsetof(TNodeDev, ordinal) == 8 &&
                    offsetof(TNodeDev, device_slots) == 44 && offsetof(TNodeDev, pin_count) == 48 &&
                    offsetof(TNodeDev, cwd) == 52 && offsetof(TNodeDev, host) == 56 &&
                    offsetof(TNodeDev, alive) == 60,
                "coop_frontier reads TNodeDev as four 16 B quads");
  const uint4* N = reinterpret_cast<const uint4*>(op.tnodes);
  const u32 n = op.t_n;
  const u32 ns = n < op.tw_n ? n : op.tw_n;
  const int tid = warp * 32 + lane, nt = nw * 32;
  // 1) mirrored ids: frontier test from shared memory, ids only
  const TWalk* tws = reinterpret_cast<const TWalk*>(kvg_tw_smem + op.tw_off);
  const TMeta* tms = reinterpret_cast<const TMeta*>(kvg_tw_smem + op.tw_off +
                                                    static_cast<size_t>(op.tw_n) * sizeof(TWalk));
  for (u32 base = static_cast<u32>(warp) * 32u; base < ns; base += static_cast<u32>(nt)) {
    const u32 i = base + lane;
    bool f = false;
    if (i < ns) {
      const TMeta m = tms[i];
      f = m.alive != 0 && (tws[i].tailh >> 31) == 0 && m.device_slots != 0 && m.pin_count == 0 &&
          m.cwd == 0;
    }
    fr_emit(op, lane, f, FrEnt{0, 0, i, 0});
  }
  __syncthreads();
  const u32 n1 = op.fr_n;
  // 2a) their (last_access, ordinal), every load independent
  for (u32 k = tid; k < n1; k += nt) {
    const uint4 q0 = N[4 * static_cast<size_t>(op.fr[k].id)];
    op.fr[k].la = static_cast<u64>(q0.x) | static_cast<u64>(q0.y) << 32;
    op.fr[k].ord = static_cast<u64>(q0.z) | static_cast<u64>(q0.w) << 32;
  }
  // 2b) ids past the mirror: whole records from HBM
  for (u32 base = ns + static_cast<u32>(warp) * 32u; base < n; base += kFrU * static_cast<u32>(nt)) {
    uint4 q0[kFrU], q2[kFrU], q3[kFrU];
#pragma unroll
    for (int u = 0; u < kFrU; ++u) {
      const u32 i = base + u * nt + lane;
      q0[u] = q2[u] = q3[u] = make_uint4(0, 0, 0, 0);
      if (i < n) {
        q0[u] = N[4 * static_cast<size_t>(i)];
        q2[u] = N[4 * static_cast<size_t>(i) + 2];
        q3[u] = N[4 * static_cast<size_t>(i) + 3];
      }
    }
#pragma unroll
    for (int u = 0; u < kFrU; ++u) {
      // t_frontier: alive && !host && device_slots > 0 && pin_count == 0 && cwd == 0
      const bool f = q3[u].w != 0 && q3[u].z == 0 && q2[u].w != 0 && q3[u].x == 0 && q3[u].y == 0;
      fr_emit(op, lane, f,
              FrEnt{static_cast<u64>(q0[u].x) | static_cast<u64>(q0[u].y) << 32,
                    static_cast<u64>(q0[u].z) | static_cast<u64>(q0[u].w) << 32,
                    base + u * nt + lane, 0});
    }
  }
}

// ------------------------------------------------------------ operations

// match_prefix, cache_tree.cpp:114-142. Returns matched tokens.
__device__ __noinline__ u64 t_match(const SimDev& D, Lead& L, u32 a, u64 len, u64* host_matched) {
  const u64 now = ++L.cclock;
  const u32 n = static_cast<u32>(len / L.ps);
  TNodeDev* N = D.tnodes;
  const TWc W = tw_ctx(D, L);
  u32 node = 0, fc = tw_get(W, 0).first_child;
  u32 pos = 0, matched = 0, hm = 0;
  bool host_phase = false;
  while (pos < n) {
    const u32 c = w_find_child(D, W, node, fc, a, pos, n);
    if (c == 0) break;
    const TWalk w = tw_get(W, c);
    if (tw_is_host(w)) host_phase = true;
    const u32 ka = w_common(w, W.S, a, pos, n);
    const bool full = ka == w.npages;
    if (ka == 0) break;
    if (!full) t_split(D, L, c, ka);
    if (host_phase) {
      hm += ka;
    } else {
      N[c].last_access = now;
      matched += ka;
    }
    pos += ka;
    node = c;
    fc = w.first_child;
    if (!full) break;
  }
  L.hit_m += static_cast<double>(static_cast<u64>(matched) * L.ps);
  L.hit_r += static_cast<double>(len);
  *host_matched = static_cast<u64>(hm) * L.ps;
  return static_cast<u64>(matched) * L.ps;
}

// count_missing_slots, cache_tree.cpp:144-168 (pages).
__device__ __noinline__ u64 t_missing(const SimDev& D, const Lead& L, u32 a, u64 n64) {
  const TWc W = tw_ctx(D, L);
  const u32 n = static_cast<u32>(n64);
  u32 node = 0, fc = tw_get(W, 0).first_child;
  u32 pos = 0, m = 0;
  while (pos < n) {
    const u32 c = w_find_child(D, W, node, fc, a, pos, n);
    if (c == 0) return m + (n - pos);
    const TWalk w = tw_get(W, c);
    const u32 ka = w_common(w, W.S, a, pos, n);
    const bool full = ka == w.npages;
    if (ka == 0) return m;
    if (tw_is_host(w)) m += ka;
    pos += ka;
    node = c;
    fc = w.first_child;
    if (!full) return m + (n - pos);
  }
  return m;
}

// pin / unpin, cache_tree.cpp:370-402: every node covering [0, len); the walk
// can start mid-path at (node, pp) (the fused walks below continue one).
__device__ void t_pin_walk(const SimDev& D, Lead& L, const TWc& W, u32 a, u32 node, u32 pp, u64 len,
                           int delta) {
  // the reference's token position pp * ps stays page aligned: pp * ps < len
  // <=> pp < ceil(len / ps); (pp + np) * ps > len <=> pp + np > floor(len / ps)
  const u32 nf = static_cast<u32>((len + L.ps - 1) / L.ps);
  const u32 lf = static_cast<u32>(len / L.ps);
  u32 fc = tw_get(W, node).first_child;
  while (pp < nf) {
    const u32 c = w_find_child(D, W, node, fc, a, pp, nf);
    if (c == 0) {
      fail(L, E_PIN_MISSING);
      return;
    }
    const TWalk w = tw_get(W, c);
    if (pp + w.npages > lf) {
      fail(L, E_PIN_MISSING);
      return;
    }
    const int pc = tw_pin(W, c);
    if (delta < 0 && pc == 0) {
      fail(L, E_UNPIN_UNDERFLOW);
      return;
    }
    tw_set_pin(W, c, pc + delta);
    pp += w.npages;
    node = c;
    fc = w.first_child;
  }
}
__device__ __noinline__ void t_pin(const SimDev& D, Lead& L, u32 a, u64 len, int delta) {
  t_pin_walk(D, L, tw_ctx(D, L), a, 0, 0, len, delta);
}

// Pin moves fused into a path walk: the node [s, e) (pages) of a path that
// gains a pin over [0, new) and loses one over [0, old) changes by +1 when
// s >= old, by 0 when e <= old, and a node straddling old is the unpin's
// E_PIN_MISSING. Same final pin counts as pin(+1, new) then unpin(-1, old).
__device__ __forceinline__ bool pin_move(const SimDev& D, Lead& L, const TWc& W, u32 c, u32 s,
                                         u32 e, u32 old_p) {
  if (e <= old_p) return true;
  if (s < old_p) {
    fail(L, E_PIN_MISSING);
    return false;
  }
  tw_set_pin(W, c, tw_pin(W, c) + 1);
  return true;
}

// pin(+1, new_len) then unpin(-1, old_len), both whole pages, in one walk.
__device__ __noinline__ void t_pin_move(const SimDev& D, Lead& L, u32 a, u64 new_len, u64 old_len) {
  const TWc W = tw_ctx(D, L);
  const u32 nf = static_cast<u32>(new_len / L.ps), old_p = static_cast<u32>(old_len / L.ps);
  u32 node = 0, fc = tw_get(W, 0).first_child, pp = 0;
  while (pp < nf) {
    const u32 c = w_find_child(D, W, node, fc, a, pp, nf);
    if (c == 0) {
      fail(L, E_PIN_MISSING);
      return;
    }
    const TWalk w = tw_get(W, c);
    if (pp + w.npages > nf) {
      fail(L, E_PIN_MISSING);
      return;
    }
    if (!pin_move(D, L, W, c, pp, pp + w.npages, old_p)) return;
    pp += w.npages;
    node = c;
    fc = w.first_child;
  }
  if (old_p > nf) t_pin_walk(D, L, W, a, node, nf, old_len, -1);
}

// match_prefix (cache_tree.cpp:114-142), then pin(+1, matched) and
// unpin(-1, old_len) (engine.cpp:337-346) in one walk. Returns matched tokens.
__device__ __noinline__ u64 t_match_pin(const SimDev& D, Lead& L, u32 a, u64 len, u64 old_len,
                                        u64* host_matched) {
  const u64 now = ++L.cclock;
  const u32 n = static_cast<u32>(len / L.ps);
  const u32 old_p = static_cast<u32>(old_len / L.ps);  // pinned lengths are whole pages
  TNodeDev* N = D.tnodes;
  const TWc W = tw_ctx(D, L);
  u32 node = 0, fc = tw_get(W, 0).first_child, dnode = 0;
  u32 pos = 0, matched = 0, hm = 0;
  bool host_phase = false, ok = true;
  while (pos < n) {
    const u32 c = w_find_child(D, W, node, fc, a, pos, n);
    if (c == 0) break;
    const TWalk w = tw_get(W, c);
    if (tw_is_host(w)) host_phase = true;
    const u32 ka = w_common(w, W.S, a, pos, n);
    const bool full = ka == w.npages;
    if (ka == 0) break;
    if (!full) t_split(D, L, c, ka);
    if (host_phase) {
      hm += ka;
    } else {
      N[c].last_access = now;
      if (ok) ok = pin_move(D, L, W, c, pos, pos + ka, old_p);
      matched += ka;
      dnode = c;
    }
    pos += ka;
    node = c;
    fc = w.first_child;
    if (!full) break;
  }
  // the unpin reaching past the match continues from the match's last node
  if (ok && old_p > matched) t_pin_walk(D, L, W, a, dnode, matched, old_len, -1);
  L.hit_m += static_cast<double>(static_cast<u64>(matched) * L.ps);
  L.hit_r += static_cast<double>(len);
  *host_matched = static_cast<u64>(hm) * L.ps;
  return static_cast<u64>(matched) * L.ps;
}

// insert after the eviction loop (cache_tree.cpp:188-227): the clock bump,
// the path walk (promoting host nodes) and the new leaf. Returns new device
// slots.
__device__ __noinline__ u64 t_insert_commit(const SimDev& D, Lead& L, u32 a, u64 n,
                                            u32 old_p = 0, bool pins = false) {
  const u64 now = ++L.cclock;
  TNodeDev* N = D.tnodes;
  const TWc W = tw_ctx(D, L);
  u32 node = 0, fc = tw_get(W, 0).first_child;
  u64 pos = 0, inserted = 0;
  while (pos < n) {
    const u32 c = w_find_child(D, W, node, fc, a, static_cast<u32>(pos), static_cast<u32>(n));
    if (c == 0) {
      const u32 l = t_alloc(D, L);
      if (l == 0) return inserted;
      TNodeDev ln;
      ln.start = static_cast<u32>(pos);
      ln.npages = static_cast<u32>(n - pos);
      ln.tail = a + 1;
      ln.parent = node;
      ln.first_child = ln.next_sib = ln.prev_sib = 0;
      ln.last_access = now;
      ln.ordinal = L.t_next_ord++;
      ln.device_slots = static_cast<u32>(n - pos);
      ln.pin_count = 0;
      ln.cwd = 0;
      ln.host = 0;
      ln.alive = 1;
      N[l] = ln;
      tw_put(W, l, ln);
      L.used += n - pos;
      inserted += n - pos;
      t_add_child(D, L, node, l);
      h_insert(D, t_key(L, a, pos), l);
      t_gain(D, L, l);
      if (pins) pin_move(D, L, W, l, static_cast<u32>(pos), static_cast<u32>(n), old_p);
      pos = n;
      node = l;
      break;
    }
    const TWalk w = tw_get(W, c);
    const u64 ka = w_common(w, W.S, a, static_cast<u32>(pos), static_cast<u32>(n));
    const bool full = ka == w.npages;
    if (ka == 0) break;
    if (!full) t_split(D, L, c, ka);
    fc = full ? w.first_child : tw_get(W, c).first_child;  // a split re-parented c's children
    if (tw_is_host(w)) {
      const u32 pages = tw_get(W, c).npages;
      N[c].host = 0;
      tw_host(W, c, 0);
      tm_slots(W, c, pages);
      L.used += pages;
      inserted += pages;
      t_gain(D, L, c);
    }
    N[c].last_access = now;
    if (pins && !pin_move(D, L, W, c, static_cast<u32>(pos), static_cast<u32>(pos + ka), old_p))
      return inserted;
    pos += ka;
    node = c;
  }
  if (pins && old_p > pos) t_pin_walk(D, L, W, a, node, static_cast<u32>(pos),
                                      static_cast<u64>(old_p) * L.ps, -1);
  return inserted;
}

// discard_suffix, cache_tree.cpp:404-437. Returns device slots freed; adds the
// dropped tokens (device and host) to L.discarded.
__device__ __noinline__ u64 t_discard(const SimDev& D, Lead& L, u32 a, u64 len, u64 from) {
  TNodeDev* N = D.tnodes;
  const u64 fp = (from + L.ps - 1) / L.ps;  // from, rounded up, in pages
  if (fp * L.ps >= len) return 0;
  const u64 n = len / L.ps;
  const TWc W = tw_ctx(D, L);
  u32 node = 0, fc = tw_get(W, 0).first_child;
  u64 pp = 0;  // pages
  while (pp < fp) {
    const u32 c = w_find_child(D, W, node, fc, a, static_cast<u32>(pp), static_cast<u32>(n));
    if (c == 0) return 0;
    const TWalk w = tw_get(W, c);
    const u64 kp = w_common(w, W.S, a, static_cast<u32>(pp), static_cast<u32>(n));
    if (kp < w.npages && pp + kp < fp) return 0;
    if (w.npages > fp - pp) t_split(D, L, c, fp - pp);
    const TWalk w2 = tw_get(W, c);
    pp += w2.npages;
    node = c;
    fc = w2.first_child;
  }
  const u32 b = w_find_child(D, W, node, fc, a, static_cast<u32>(fp), static_cast<u32>(n));
  if (b == 0) return 0;
  u64 slots = 0, toks = 0;
  long long pins = 0;
  u32 sp = 0;
  D.tstack[sp++] = b;
  while (sp > 0) {
    const u32 x = D.tstack[--sp];
    slots += N[x].device_slots;
    toks += static_cast<u64>(N[x].npages) * L.ps;
    pins += N[x].pin_count;
    for (u32 c = N[x].first_child; c != 0; c = N[c].next_sib) D.tstack[sp++] = c;
  }
  if (pins > 0) {
    fail(L, E_DISCARD_PINNED);
    return 0;
  }
  if (t_subdev(N[b])) t_loss(D, L, b);
  L.used -= slots;
  L.discarded += toks;
  t_remove_child(D, L, node, b);
  // free the subtree: its head keys leave the hash, its nodes the pool
  sp = 0;
  D.tstack[sp++] = b;
  while (sp > 0) {
    const u32 x = D.tstack[--sp];
    for (u32 c = N[x].first_child; c != 0; c = N[c].next_sib) D.tstack[sp++] = c;
    h_erase(D, t_nkey(L, N[x], N[x].start));
    tm_alive(tw_ctx(D, L), x, 0);
    D.tfree[L.t_free_n++] = x;
  }
  return slots;
}

// ------------------------------------------------------------ eviction

__device__ __forceinline__ bool fr_less(const FrEnt& x, const FrEnt& y) {
  return x.la < y.la || (x.la == y.la && x.ord < y.ord);
}
__device__ void fr_sift_down(FrEnt* h, u32 n, u32 i) {
  const FrEnt e = h[i];
  for (;;) {
    u32 c = 2 * i + 1;
    if (c >= n) break;
    if (c + 1 < n && fr_less(h[c + 1], h[c])) ++c;
    if (!fr_less(h[c], e)) break;
    h[i] = h[c];
    i = c;
  }
  h[i] = e;
}
__device__ void fr_push(FrEnt* h, u32& n, const FrEnt& e) {
  u32 i = n++;
  while (i > 0) {
    const u32 p = (i - 1) >> 1;
    if (!fr_less(e, h[p])) break;
    h[i] = h[p];
    i = p;
  }
  h[i] = e;
}

// evict (cache_tree.cpp:270-319) after OP_FRONTIER compacted the initial
// frontier into D.fr[0, nf): heap pops by (last_access, ordinal), tail splits,
// offload to the host tier, parents pushed as they become frontier. Returns
// reclaimed slots; offloaded tokens accumulate into *offl.
__device__ __noinline__ u64 t_evict_pop(const SimDev& D, Lead& L, u32 nf, u64 needed, u64* offl) {
  TNodeDev* N = D.tnodes;
  FrEnt* h = D.fr;
  for (u32 i = nf / 2; i-- > 0;) fr_sift_down(h, nf, i);
  u64 reclaimed = 0;
  const unsigned long long log0 = L.n_log;
  log_rec(D, L, KVG_LOG_EVICT, L.m_id, needed, 0);
  while (reclaimed < needed && nf > 0) {
    const FrEnt e = h[0];
    h[0] = h[--nf];
    if (nf > 0) fr_sift_down(h, nf, 0);
    const u32 id = e.id;
    if (!t_frontier(N[id]) || N[id].last_access != e.la || N[id].ordinal != e.ord) continue;
    const u64 slots = N[id].device_slots;
    const u64 take = slots < needed - reclaimed ? slots : needed - reclaimed;
    u32 v = id;
    if (take < slots) v = t_split(D, L, id, N[id].npages - take);
    const TNodeDev vn = N[v];
    if (D.log != nullptr)
      for (u64 k = static_cast<u64>(vn.start) + vn.npages; k-- > vn.start;)
        log_rec(D, L, KVG_LOG_VICTIM, L.m_id, t_nkey(L, vn, k), vn.last_access);
    L.used -= vn.device_slots;
    reclaimed += vn.device_slots;
    const u64 toks = static_cast<u64>(vn.npages) * L.ps;
    L.offloaded += toks;
    *offl += toks;
    tm_slots(tw_ctx(D, L), v, 0);
    N[v].host = 1;
    tw_host(tw_ctx(D, L), v, 1);
    t_loss(D, L, v);
    const u32 parent = vn.parent;
    if (parent != 0 && t_frontier(N[parent]))
      fr_push(h, nf, FrEnt{N[parent].last_access, N[parent].ordinal, parent, 0});
  }
  if (D.log != nullptr && log0 < D.log_cap) D.log[log0].b = reclaimed;
  ++L.evict_calls;
  L.evicted += reclaimed;
  return reclaimed;
}

// ------------------------------------------------------------ link queue

// transfers_in_flight, engine.cpp:156-160. Transfer ends never decrease
// (each starts at max(clock, pcie_busy_until) with a non-negative duration),
// so the reference's multiset is a FIFO ring here.
__device__ __forceinline__ u32 x_in_flight(const SimDev& D, Lead& L, double clock) {
  while (L.x_size > 0 && D.xring[L.x_head] <= clock) {
    L.x_head = L.x_head + 1 == D.xcap ? 0 : L.x_head + 1;
    --L.x_size;
  }
  return L.x_size;
}

// enqueue_transfer, engine.cpp:164-174; transfer_time, cost_model.cpp:43-47.
__device__ double x_enqueue(const SimDev& D, Lead& L, double bytes) {
  const u32 depth = x_in_flight(D, L, L.clock) + 1;
  const double dur = D.cost.transfer_sync_overhead +
                     bytes * static_cast<double>(depth) / D.cost.pcie_bandwidth;
  const double start = L.clock < L.pcie_busy ? L.pcie_busy : L.clock;
  const double end = start + dur;
  L.pcie_busy = end;
  L.ledger.transfer += dur;
  L.link_busy += dur;
  if (L.x_size >= D.xcap) {
    fail(L, E_TABLE_FULL);
    return end;
  }
  u32 tail = L.x_head + L.x_size;
  if (tail >= D.xcap) tail -= D.xcap;
  D.xring[tail] = end;
  ++L.x_size;
  return end;
}

// account_evictions, engine.cpp:178-182
__device__ __forceinline__ void x_account(const SimDev& D, Lead& L, u64 offl_tokens) {
  if (offl_tokens > 0)
    x_enqueue(D, L, static_cast<double>(offl_tokens) * D.cost.bytes_per_token);
}

__device__ void tree_init(const SimDev& D, Lead& L) {
  TNodeDev r;
  r.last_access = r.ordinal = 0;
  r.parent = r.first_child = r.next_sib = r.prev_sib = 0;
  r.start = r.npages = r.tail = r.device_slots = 0;
  r.pin_count = r.cwd = 0;
  r.host = 0;
  r.alive = 0;  // the root is never a frontier candidate
  D.tnodes[0] = r;
  tw_put(tw_ctx(D, L), 0, r);
  L.t_alloc = 1;
  L.t_free_n = 0;
  L.t_next_ord = 0;
  L.x_head = L.x_size = 0;
  L.pcie_busy = L.link_busy = 0.0;
  L.offloaded = L.reloaded = 0;
}

}  // namespace kvg
