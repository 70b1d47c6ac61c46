// Cache-op executor: the CacheTree seam (cache_tree.hpp:96-167) on the device.
// One CTA executes a batch of ops in order with the same cooperative ops as the
// engine, but with EXPLICIT per-page pin counts (arbitrary pin/unpin order is
// allowed here, unlike the engine's one-pin-per-agent discipline).
#pragma once

namespace kvg {

// Cache-op executor (CacheTree seam). One CTA executes ops in order.

enum CPhase : int {
  C_NEXT = 0, C_MATCH_DONE, C_INS_COUNT, C_INS_COUNTED, C_INS_EVICTED, C_INS_COMMIT,
  C_INS_DONE, C_EVICT_DONE, C_PIN_DONE, C_DISC_PROBED, C_DISC_DONE, C_END
};

struct CLead {
  int phase;
  u32 i;
  u64 used, clock, pinned, discarded, n0_victims;
  double hit_m, hit_r;
  u64 n, k, e, fp, head_owner;
  int rebuilt;
};

__device__ void cache_result(const CacheDev& C, CLead& L, Op& op, int status, u64 r0, u64 r1) {
  kvg_cache_op_result& r = C.results[L.i];
  r.status = status;
  r.r0 = r0;
  r.r1 = r1;
  r.clock = L.clock;
  r.used = L.used;
  r.victims_begin = L.n0_victims;
  r.victims_end = __ldcg(op.vic_n);
  ++L.i;
  L.phase = C_NEXT;
}

__device__ void cache_leader(const CacheDev& C, CLead& L, Op& op) {
  op.kind = OP_NONE;
  for (;;) {
    const kvg_cache_op* o = &C.ops[L.i < C.n_ops ? L.i : 0];
    switch (L.phase) {
      case C_NEXT: {
        if (L.i >= C.n_ops) {
          L.phase = C_END;
          continue;
        }
        L.n0_victims = __ldcg(op.vic_n);
        L.rebuilt = 0;
        const u64 ps = C.page_size;
        switch (o->kind) {
          case KVG_OP_MATCH:  // cache_tree.cpp:114-142
            L.n = o->len / ps;
            ++L.clock;
            post_range(op, o->agent, 0, L.n, RF_STAMP, 0, L.clock);
            L.phase = C_MATCH_DONE;
            if (L.n == 0) { op.kind = OP_NONE; continue; }
            return;
          case KVG_OP_INSERT:  // cache_tree.cpp:170-228
            L.n = o->len / ps;
            if (L.n == 0) { cache_result(C, L, op, KVG_OK, 1, 0); continue; }
            L.phase = C_INS_COUNT;
            continue;
          case KVG_OP_EVICT:
            L.k = o->arg;
            L.e = L.used - L.pinned;
            if (L.k == 0 || L.e == 0) { cache_result(C, L, op, KVG_OK, 0, 0); continue; }
            op.kind = OP_EVICT; op.k = L.k; op.evictable = L.e; op.clock = L.clock;
            op.agent = 0; op.err = E_NONE;
            L.phase = C_EVICT_DONE;
            return;
          case KVG_OP_PIN:
          case KVG_OP_UNPIN:
            if (o->arg % ps != 0 || o->arg > o->len) {
              cache_result(C, L, op, KVG_ERR_CONFIG, 0, 0);
              continue;
            }
            post_range(op, o->agent, 0, o->arg / ps, RF_PIN | RF_STRICT, o->kind == KVG_OP_PIN ? 1 : -1, 0);
            L.phase = C_PIN_DONE;
            if (o->arg == 0) { op.kind = OP_NONE; continue; }
            return;
          case KVG_OP_DISCARD: {  // cache_tree.cpp:404-437
            L.fp = (o->arg + ps - 1) / ps;
            if (L.fp * ps >= o->len || L.fp >= o->len / ps) {
              cache_result(C, L, op, KVG_OK, 0, 0);
              continue;
            }
            post_range(op, o->agent, 0, L.fp + 1, 0, 0, 0);  // path + branch head present?
            L.phase = C_DISC_PROBED;
            return;
          }
          default:
            cache_result(C, L, op, KVG_ERR_CONFIG, 0, 0);
            continue;
        }
      }
      case C_MATCH_DONE: {
        const u64 f = op.first_miss < L.n ? op.first_miss : L.n;
        const u64 matched = f * C.page_size;
        L.hit_m += static_cast<double>(matched);
        L.hit_r += static_cast<double>(o->len);
        cache_result(C, L, op, op.resident == f ? KVG_OK : KVG_ERR_STATE, matched, 0);
        continue;
      }
      case C_INS_COUNT:  // count_missing_slots (cache_tree.cpp:144-168)
        post_range(op, o->agent, 0, L.n, 0, 0, 0);
        L.phase = C_INS_COUNTED;
        return;
      case C_INS_COUNTED: {
        const u64 f = op.first_miss < L.n ? op.first_miss : L.n;
        L.fp = f;
        const u64 need = L.n - f;
        const u64 free_slots = C.capacity - L.used;
        if (need <= free_slots) { L.phase = C_INS_COMMIT; continue; }
        L.k = need - free_slots;
        L.e = L.used - L.pinned;
        if (L.e == 0) { cache_result(C, L, op, KVG_OK, 0, 0); continue; }
        op.kind = OP_EVICT; op.k = L.k; op.evictable = L.e; op.clock = L.clock;
        op.agent = o->agent; op.err = E_NONE;
        L.phase = C_INS_EVICTED;
        return;
      }
      case C_INS_EVICTED: {
        const u64 r = op.freed;
        L.used -= r;
        L.discarded += r * C.page_size;
        L.phase = C_INS_COUNT;  // eviction may strip the unpinned path: recount
        continue;
      }
      case C_INS_COMMIT: {
        if (static_cast<u64>(op.occ_n) + range_chunks(0, L.n) > (static_cast<u64>(op.mask) + 1) / 2) {
          if (L.rebuilt) { cache_result(C, L, op, KVG_ERR_STATE, 0, 0); continue; }
          L.rebuilt = 1;
          op.kind = OP_REBUILD;
          return;
        }
        ++L.clock;
        post_range(op, o->agent, 0, L.n, RF_STAMP | RF_CREATE, 0, L.clock);
        L.phase = C_INS_DONE;
        return;
      }
      case C_INS_DONE:
        L.used += op.created;
        cache_result(C, L, op, KVG_OK, 1, op.created);
        continue;
      case C_EVICT_DONE: {
        const u64 r = op.freed;
        L.used -= r;
        L.discarded += r * C.page_size;
        cache_result(C, L, op, KVG_OK, r, 0);
        continue;
      }
      case C_PIN_DONE:
        L.pinned += op.pin_up;
        L.pinned -= op.pin_down;
        cache_result(C, L, op, op.err ? KVG_ERR_STATE : KVG_OK, 0, 0);
        continue;
      case C_DISC_PROBED: {
        if (op.first_miss <= L.fp) { cache_result(C, L, op, KVG_OK, 0, 0); continue; }
        const u64 head_owner = L.fp < C.shared_pages ? 0 : static_cast<u64>(o->agent) + 1;
        op.kind = OP_SCANFREE;
        op.p0 = L.fp;
        op.owner_filter = head_owner == 0 ? ~0ull : head_owner;
        op.freed = 0;
        op.err = E_NONE;
        L.phase = C_DISC_DONE;
        return;
      }
      case C_DISC_DONE:
        L.used -= op.freed;
        L.discarded += static_cast<u64>(op.freed) * C.page_size;
        // discard_suffix returns nothing (cache_tree.hpp:138); the pool
        // usage in the op result shows what it dropped
        cache_result(C, L, op, op.err ? KVG_ERR_STATE : KVG_OK, 0, 0);
        continue;
      default:
        op.kind = OP_EXIT;
        return;
    }
  }
}

__global__ void __launch_bounds__(1024) cache_kernel(const CacheDev* __restrict__ cd) {
  __shared__ CLead L;
  __shared__ Op op;
  const CacheDev& C = *cd;
  __shared__ unsigned int shist[2 * kBins];  // radix-select bins in shared memory
  Hist h{shist, shist + kBins, true};
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  CacheState* st = reinterpret_cast<CacheState*>(C.state);
  if (tid == 0) {
    L.phase = C_NEXT;
    L.i = 0;
    L.used = st->used;
    L.clock = st->clock;
    L.pinned = st->pinned_pages;
    L.discarded = st->discarded;
    L.hit_m = st->hit_m;
    L.hit_r = st->hit_r;
    const bool sw = st->swapped & 1;
    op.table = sw ? C.alt : C.table;
    op.alt = sw ? C.table : C.alt;
    op.occ = sw ? C.alt_occ : C.occ;
    op.alt_occ = sw ? C.occ : C.alt_occ;
    op.summ = sw ? C.alt_summ : C.summ;
    op.alt_summ = sw ? C.summ : C.alt_summ;
    op.mask = C.bucket_mask;
    op.occ_n = static_cast<unsigned int>(st->occ_n);
    op.shared_pages = C.shared_pages;
    op.log = nullptr;
    op.log_cap = 0;
    op.log_n = nullptr;
    op.vic = C.victims;
    op.vic_cap = C.victim_cap;
    op.vic_n = reinterpret_cast<unsigned long long*>(&st->n_victims);
    op.log_victims = 1;
    op.log_clock = 0;
    op.implicit_pins = 0;
    op.pin_max = 0;
    op.agents = nullptr;
  }
  __syncthreads();
  for (;;) {
    if (tid == 0) cache_leader(C, L, op);
    __syncthreads();
    if (op.kind == OP_EXIT) break;
    run_op<8>(op, h, tid, warp, lane, nw);
    __syncthreads();
    if (tid == 0 && op.kind == OP_REBUILD) st->swapped ^= 1;
  }
  if (tid == 0) {
    st->used = L.used;
    st->clock = L.clock;
    st->pinned_pages = L.pinned;
    st->discarded = L.discarded;
    st->hit_m = L.hit_m;
    st->hit_r = L.hit_r;
    st->occ_n = op.occ_n;
  }
}

}  // namespace kvg

// ==========================================================================
// Offload-mode CacheTree seam: the same node-level tree the engine runs
// (tree.cuh), driven op by op. Leader-serial (one thread), the frontier scan
// included: this is the parity / integration surface, not a throughput path.
// ==========================================================================

namespace kvg {

struct TreeCacheDev {
  SimDev sim;  // tree pointers; log = per-op victim scratch
  Lead lead;   // persistent scalars between exec calls
};

__device__ u64 tc_evict(const SimDev& D, Lead& L, u64 needed, u64* offl) {
  if (needed == 0) return 0;  // cache_tree.cpp:272
  u32 nf = 0;
  for (u32 i = 1; i < L.t_alloc; ++i)
    if (t_frontier(D.tnodes[i]))
      D.fr[nf++] = FrEnt{D.tnodes[i].last_access, D.tnodes[i].ordinal, i, 0};
  return t_evict_pop(D, L, nf, needed, offl);
}

// reload, cache_tree.cpp:321-368 (mirrors the engine's reload phases)
__device__ u64 tc_reload(const SimDev& D, Lead& L, u32 a, u64 len, u64 from, u64 maxt, u64* offl) {
  if (from >= len || maxt == 0) return 0;
  TNodeDev* N = D.tnodes;
  const u64 n = len / L.ps;
  u32 node = 0;
  u64 pos = 0;
  while (pos < from) {
    const u32 c = (pos % L.ps == 0) ? t_find_child(D, L, node, a, pos / L.ps, n) : 0;
    if (c == 0 || pos + static_cast<u64>(N[c].npages) * L.ps > from) {
      fail(L, E_OFFLOAD);
      return 0;
    }
    pos += static_cast<u64>(N[c].npages) * L.ps;
    node = c;
  }
  const u64 now = ++L.cclock;
  u64 promoted = 0;
  while (pos < len && promoted < maxt) {
    const u32 c = t_find_child(D, L, node, a, pos / L.ps, n);
    if (c == 0 || !N[c].host) break;
    u64 ka = t_common(D, L, c, a, pos / L.ps, n);
    bool full = ka == N[c].npages;
    const u64 want = (maxt - promoted) / L.ps;
    if (ka > want) {
      ka = want;
      full = false;
    }
    if (ka == 0) break;
    if (ka < N[c].npages) t_split(D, L, c, ka);
    if (L.capacity - L.used < ka) {
      tc_evict(D, L, ka - (L.capacity - L.used), offl);
      if (L.capacity - L.used < ka) break;
    }
    N[c].host = 0;
    tw_host(tw_ctx(D, L), c, 0);
    tm_slots(tw_ctx(D, L), c, static_cast<u32>(ka));
    N[c].last_access = now;
    L.used += ka;
    t_gain(D, L, c);
    promoted += ka * L.ps;
    pos += ka * L.ps;
    node = c;
    if (!full) break;
  }
  return promoted;
}

__global__ void cache_tree_kernel(TreeCacheDev* T, const kvg_cache_op* ops, u32 n_ops,
                                  kvg_cache_op_result* res, kvg_victim* vic, u64 vic_cap,
                                  u64* n_vic) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const SimDev& D = T->sim;
  Lead& L = T->lead;
  for (u32 i = 0; i < n_ops; ++i) {
    const kvg_cache_op& o = ops[i];
    kvg_cache_op_result r;
    r.status = KVG_OK;
    r._pad = 0;
    r.r0 = r.r1 = 0;
    r.victims_begin = *n_vic;
    L.err = E_NONE;
    L.status = KVG_OK;
    L.n_log = 0;
    L.m_id = o.agent;
    u64 offl = 0;
    switch (o.kind) {
      case KVG_OP_MATCH: {
        u64 hm = 0;
        r.r0 = t_match(D, L, o.agent, o.len, &hm);
        r.r1 = hm;
        break;
      }
      case KVG_OP_INSERT: {  // cache_tree.cpp:170-228
        const u64 n = o.len / L.ps;
        if (n == 0) {
          r.r0 = 1;
          break;
        }
        bool ok = true;
        for (;;) {
          const u64 need = t_missing(D, L, o.agent, n);
          const u64 free_slots = L.capacity - L.used;
          if (need <= free_slots) break;
          if (tc_evict(D, L, need - free_slots, &offl) == 0) {
            ok = false;
            break;
          }
        }
        if (ok) {
          r.r1 = t_insert_commit(D, L, o.agent, n);
          r.r0 = 1;
        }
        break;
      }
      case KVG_OP_RELOAD:
        r.r0 = tc_reload(D, L, o.agent, o.len, o.arg, o.arg2, &offl);
        r.r1 = offl;
        break;
      case KVG_OP_EVICT: r.r0 = tc_evict(D, L, o.arg, &offl); break;
      case KVG_OP_PIN:
      case KVG_OP_UNPIN:
        if (o.arg > o.len) fail(L, E_PIN_MISSING);
        else t_pin(D, L, o.agent, o.arg, o.kind == KVG_OP_PIN ? 1 : -1);
        break;
      case KVG_OP_DISCARD: t_discard(D, L, o.agent, o.len, o.arg); break;
      default: fail(L, E_PIN_MISSING); break;
    }
    if (L.err != E_NONE) r.status = KVG_ERR_STATE;
    // victims of this op, in the order the tree evicted them
    const u64 nl = L.n_log < D.log_cap ? L.n_log : D.log_cap;
    for (u64 k = 0; k < nl; ++k) {
      const kvg_log_record& lr = D.log[k];
      if (lr.kind != KVG_LOG_VICTIM) continue;
      if (*n_vic < vic_cap) vic[*n_vic] = kvg_victim{lr.a, lr.b};
      ++*n_vic;
    }
    r.victims_end = *n_vic;
    r.clock = L.cclock;
    r.used = L.used;
    res[i] = r;
  }
}

__global__ void cache_tree_init(TreeCacheDev* T) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  tree_init(T->sim, T->lead);
}

}  // namespace kvg
