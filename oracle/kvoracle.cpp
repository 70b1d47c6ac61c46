/* kvoracle — CPU restatement of the reference hot path. TEST INFRASTRUCTURE.
 *
 * Parity status: PINNED. Checked against the unmodified reference
 * (oracle/_ref/libkvref.so) per event (state digests through the paranoid
 * hooks), per result field (bit-exact doubles) and per eviction victim list;
 * see tests/test_oracle_vs_reference.py and tests/golden/.
 *
 * What it restates (every function cites the reference lines it follows):
 *  - the radix prefix cache as a FLAT PER-PAGE table. Every page of an
 *    agent's context is named by (owner, page index): owner 0 for a page
 *    wholly inside a shared prompt, agent+1 otherwise. This is exact for the
 *    population token scheme (workload.cpp:139-142, 167-171) and is the
 *    per-page reduction of CacheTree that SURVEY.md fact 0.3-2 / probe P4
 *    established: discard-mode eviction = the `needed` smallest
 *    (stamp asc, page index desc) unpinned resident pages.
 *  - the event loop with one outstanding event per agent plus one tick and at
 *    most one admission check, popped by (time, rank, ordinal) — equivalent
 *    to the reference heap.
 *  - controller (controller.cpp), cost model (cost_model.cpp), dispatch
 *    (engine.cpp:305-396) and completion handlers (engine.cpp:184-291).
 * Eviction-mode offload is not restated here.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py may load this library,
 * and only as the checker. The product never links it.
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <limits>
#include <map>
#include <queue>
#include <set>
#include <stdexcept>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "../include/kvgpu.h"
#include "digest.h"

#define KVO_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string t_err = "no error";

struct Horizon : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StateError : std::logic_error {
  using std::logic_error::logic_error;
};

/* ======================= flat page cache (cache_tree.cpp) =================== */

/* One page of the radix tree, named by (owner, page index). `host` is the
 * node tier (cache_tree.hpp:37-61, Tier::kHost in offload mode); `bnd` marks
 * a page that STARTS a radix node. Node boundaries are invisible to discard
 * mode, but offload-mode reload promotes host nodes one node-chunk at a time
 * (cache_tree.cpp:337-366), so the restatement tracks exactly where the
 * reference splits or creates nodes. */
struct Page {
  std::uint64_t stamp = 0;
  std::int64_t pins = 0;
  bool host = false;
  bool bnd = false;
};

struct FlatCache {
  std::uint64_t capacity = 0, ps = 1, prompt = 0, shared_pages = 0;
  bool shared = false, offload = false;
  std::unordered_map<std::uint64_t, Page> pages;  // every page in the tree (device or host)
  std::set<std::uint64_t> order;  // offload mode: page keys in (owner, index) order
  std::uint64_t used = 0, clock = 0, discarded = 0, offloaded = 0;
  double hit_m = 0, hit_r = 0;
  std::uint64_t evict_calls = 0, evicted = 0;
  std::uint64_t pinned = 0;  // DEVICE pages with pins > 0 (evictable = used - pinned)
  std::uint64_t dsum = 0;    // running sum of kvdigest::page_term over all pages
  /* owner (agent+1) whose page at index shared_pages still belongs to the node
   * holding the last shared page (the first agent to insert past the shared
   * prompt creates one leaf spanning both), 0 if none. */
  std::uint64_t glued = 0;
  std::vector<std::pair<std::uint64_t, std::uint64_t>>* victims = nullptr;
  std::vector<kvg_log_record>* log = nullptr;  // EVICT + VICTIM records
  std::uint32_t log_agent = 0;

  void init(std::uint64_t cap, std::uint64_t page, std::uint64_t p, bool sh, bool off) {
    if (cap == 0 || page == 0) throw std::invalid_argument("capacity and page size must be > 0");
    capacity = cap;
    ps = page;
    prompt = p;
    shared = sh;
    offload = off;
    shared_pages = sh ? p / page : 0;  // pages wholly inside the shared prompt
  }
  std::uint64_t key(std::uint32_t a, std::uint64_t k) const {
    std::uint64_t owner = k < shared_pages ? 0 : std::uint64_t(a) + 1;
    return (owner << 32) | k;
  }
  static std::uint64_t term(std::uint64_t key, const Page& p) {
    return kvdigest::page_term(key >> 32, key & 0xffffffffULL, p.stamp,
                               static_cast<std::uint64_t>(p.pins), p.host ? 1 : 0);
  }
  Page* find(std::uint32_t a, std::uint64_t k) {
    auto it = pages.find(key(a, k));
    return it == pages.end() ? nullptr : &it->second;
  }
  Page* find_key(std::uint64_t kk) {
    auto it = pages.find(kk);
    return it == pages.end() ? nullptr : &it->second;
  }
  /* Applies f to a page while keeping the digest sum and counters exact. */
  template <typename F>
  void modify(std::uint64_t kk, Page* p, F&& f) {
    dsum -= term(kk, *p);
    const bool was_dev = !p->host, was_pin = p->pins > 0;
    f(*p);
    if (was_dev && was_pin) --pinned;
    if (!p->host && p->pins > 0) ++pinned;
    if (was_dev && p->host) --used;
    if (!was_dev && !p->host) ++used;
    dsum += term(kk, *p);
  }
  void add_page(std::uint64_t kk, std::uint64_t stamp, bool bnd) {
    Page pg;
    pg.stamp = stamp;
    pg.bnd = bnd;
    pages.emplace(kk, pg);
    if (offload) order.insert(kk);
    dsum += term(kk, pg);
    ++used;
    if (!bnd && shared_pages > 0 && (kk & 0xffffffffULL) == shared_pages && (kk >> 32) != 0)
      glued = kk >> 32;
  }
  void drop_page(std::unordered_map<std::uint64_t, Page>::iterator it) {
    dsum -= term(it->first, it->second);
    if (!it->second.host) {
      if (it->second.pins > 0) --pinned;
      --used;
    }
    if (glued != 0 && it->first == ((glued << 32) | shared_pages)) glued = 0;
    if (offload) order.erase(it->first);
    pages.erase(it);
  }
  void set_bnd(std::uint64_t kk, Page* p) {
    if (p->bnd) return;
    p->bnd = true;
    if (glued != 0 && kk == ((glued << 32) | shared_pages)) glued = 0;
  }
  /* First page index in [0, n) absent from agent a's path (the tree is
   * prefix-closed along every path). */
  std::uint64_t walk(std::uint32_t a, std::uint64_t n) {
    std::uint64_t k = 0;
    while (k < n && find(a, k) != nullptr) ++k;
    return k;
  }
  /* split_node at the end of a walk over [0, f) that stopped at f (n = the
   * walk's limit): the node holding page f-1 is split where it leaves the
   * path (cache_tree.cpp:128, 212, 350, 415). Two ways a node continues past
   * the walked pages: the shared prompt's node glued to another agent's
   * private pages (whenever a walk covers the whole shared prompt), or the
   * agent's own next page when the walk stopped at its length limit. */
  void split_walk_end(std::uint32_t a, std::uint64_t f, std::uint64_t n) {
    if (shared_pages > 0 && glued != 0 && glued != std::uint64_t(a) + 1 && f >= shared_pages) {
      const std::uint64_t kk = (glued << 32) | shared_pages;
      set_bnd(kk, find_key(kk));
    }
    if (f == n && f > 0) {
      const std::uint64_t kk = key(a, f);
      if (Page* p = find_key(kk)) set_bnd(kk, p);
    }
  }
  /* split_node so a node boundary falls before page q of a's path (whatever
   * page continues the node holding page q-1 starts a new node). */
  void split_before(std::uint32_t a, std::uint64_t q) {
    if (q == 0) return;
    const std::uint64_t kk = key(a, q);
    if (Page* p = find_key(kk)) {
      if (!p->bnd) {
        set_bnd(kk, p);
        return;
      }
    }
    if (shared_pages > 0 && q == shared_pages && glued != 0) {
      const std::uint64_t gk = (glued << 32) | shared_pages;
      set_bnd(gk, find_key(gk));
    }
  }
  /* Does the node holding page q-1 of a's path continue past it? */
  bool continues(std::uint32_t a, std::uint64_t q) {
    if (q == 0) return false;
    if (Page* p = find(a, q))
      if (!p->bnd) return true;
    return shared_pages > 0 && q == shared_pages && glued != 0 && glued != std::uint64_t(a) + 1;
  }

  /* match_prefix, cache_tree.cpp:114-142: device pages until the first host
   * page are matched (and refreshed); every later page on the path counts as
   * host_matched (Q4: device pages below a host node are not refreshed). */
  std::uint64_t match(std::uint32_t a, std::uint64_t len, std::uint64_t* host_matched) {
    const std::uint64_t now = ++clock;
    const std::uint64_t n = len / ps;
    const std::uint64_t f = walk(a, n);
    split_walk_end(a, f, n);
    std::uint64_t d = 0;
    for (; d < f; ++d) {
      const std::uint64_t kk = key(a, d);
      Page* p = find_key(kk);
      if (p->host) break;
      modify(kk, p, [&](Page& q) { q.stamp = now; });
    }
    if (host_matched) *host_matched = (f - d) * ps;
    hit_m += static_cast<double>(d * ps);
    hit_r += static_cast<double>(len);
    return d * ps;
  }

  /* Eviction key: (M asc, page index desc) with M the newest device stamp in
   * the page's subtree. In discard mode stamps never increase
   * from root to leaf, so M is the page's own stamp; offload-mode reloads
   * stamp promoted chunks newer than their parents, and a node can only be
   * taken once its device subtree is gone, which M expresses per page. */
  struct Cand {
    std::uint64_t m, idx, kk;
    Page* p;
  };
  static bool lru_before(const Cand& x, const Cand& y) {
    if (x.m != y.m) return x.m < y.m;
    if (x.idx != y.idx) return x.idx > y.idx;
    return x.kk < y.kk;
  }
  /* Candidates with their keys. Offload: one descending pass over the
   * ordered page keys computes M as a suffix max along every private chain;
   * the shared chain's pages also cover every private chain below it. */
  void candidates(std::vector<Cand>& cand) {
    if (!offload) {
      for (auto& kv : pages)
        if (kv.second.pins == 0)
          cand.push_back(Cand{kv.second.stamp, kv.first & 0xffffffffULL, kv.first, &kv.second});
      return;
    }
    std::uint64_t run = 0, cur = ~0ULL, below_shared = 0;
    for (auto it = order.rbegin(); it != order.rend(); ++it) {
      const std::uint64_t kk = *it, owner = kk >> 32;
      if (owner != cur) {
        if (cur != ~0ULL && cur != 0) below_shared = std::max(below_shared, run);
        cur = owner;
        run = owner == 0 ? below_shared : 0;
      }
      Page& p = pages.find(kk)->second;
      if (!p.host) run = std::max(run, p.stamp);
      if (!p.host && p.pins == 0) cand.push_back(Cand{run, kk & 0xffffffffULL, kk, &p});
    }
  }

  /* evict, cache_tree.cpp:270-319 in its per-page form. Offload victims move
   * to the host tier (their pages stay in the tree); discard victims leave. */
  std::uint64_t evict(std::uint64_t needed, std::uint64_t* offl_tokens = nullptr) {
    if (needed == 0) return 0;
    ++evict_calls;
    if (used == pinned) {  // nothing evictable: the common stall-storm case
      if (log) log->push_back(kvg_log_record{KVG_LOG_EVICT, log_agent, clock, needed, 0});
      return 0;
    }
    std::vector<Cand> cand;
    candidates(cand);
    std::uint64_t take = std::min<std::uint64_t>(needed, cand.size());
    if (log) log->push_back(kvg_log_record{KVG_LOG_EVICT, log_agent, clock, needed, take});
    if (take == 0) return 0;
    std::partial_sort(cand.begin(), cand.begin() + take, cand.end(), lru_before);
    for (std::uint64_t i = 0; i < take; ++i) {
      const Cand& c = cand[i];
      if (victims) victims->emplace_back(c.kk, c.p->stamp);
      if (log)
        log->push_back(kvg_log_record{KVG_LOG_VICTIM, log_agent, clock, c.kk, c.p->stamp});
    }
    // the last node popped is split when only its tail was taken
    // (cache_tree.cpp:287-290): its first victim page starts a new node
    set_bnd(cand[take - 1].kk, cand[take - 1].p);
    for (std::uint64_t i = 0; i < take; ++i) {
      const Cand& c = cand[i];
      if (offload) modify(c.kk, c.p, [](Page& q) { q.host = true; });
      else drop_page(pages.find(c.kk));
    }
    evicted += take;
    if (offload) {
      offloaded += take * ps;
      if (offl_tokens) *offl_tokens += take * ps;
    } else {
      discarded += take * ps;
    }
    return take;
  }

  /* count_missing_slots, cache_tree.cpp:144-168: absent pages plus host
   * pages on the path. */
  std::uint64_t missing(std::uint32_t a, std::uint64_t n) {
    const std::uint64_t f = walk(a, n);
    std::uint64_t m = n - f;
    if (offload)
      for (std::uint64_t k = 0; k < f; ++k)
        if (find(a, k)->host) ++m;
    return m;
  }

  /* insert, cache_tree.cpp:170-228. Returns ok; *inserted = new device slots
   * (created + promoted from host). */
  bool insert(std::uint32_t a, std::uint64_t len, std::uint64_t* inserted,
              std::uint64_t* evicted_pages, std::uint64_t* offl_tokens = nullptr) {
    const std::uint64_t n = len / ps;
    if (inserted) *inserted = 0;
    if (n == 0) return true;
    for (;;) {
      std::uint64_t need = missing(a, n);
      std::uint64_t free_slots = capacity - used;
      if (need <= free_slots) break;
      std::uint64_t ev = evict(need - free_slots, offl_tokens);
      if (evicted_pages) *evicted_pages += ev;
      if (ev == 0) return false;  // evictions so far persist (Q3)
    }
    const std::uint64_t now = ++clock;
    const std::uint64_t f = walk(a, n);
    split_walk_end(a, f, n);
    for (std::uint64_t k = 0; k < f; ++k) {
      const std::uint64_t kk = key(a, k);
      Page* p = find_key(kk);
      if (p->host && inserted) ++*inserted;
      modify(kk, p, [&](Page& q) {
        q.host = false;
        q.stamp = now;
      });
    }
    for (std::uint64_t k = f; k < n; ++k) {
      add_page(key(a, k), now, k == f);
      if (inserted) ++*inserted;
    }
    return true;
  }

  /* reload, cache_tree.cpp:321-368: promote host nodes from `from`, one
   * node-chunk at a time, evicting per chunk; a chunk that still does not fit
   * stops the reload. Promoted chunks can be evicted again by later chunks'
   * evictions (quirk Q1). Returns promoted tokens. */
  std::uint64_t reload(std::uint32_t a, std::uint64_t len, std::uint64_t from,
                       std::uint64_t max_tokens, std::uint64_t* offl_tokens) {
    if (from >= len || max_tokens == 0) return 0;
    // walk to `from` (cache_tree.cpp:326-334): it must lie on the cached
    // path, on a node boundary
    if (from % ps != 0) throw StateError("reload offset is not a node boundary");
    for (std::uint64_t k = 0; k < from / ps; ++k)
      if (find(a, k) == nullptr) throw StateError("reload offset is not on a cached path");
    if (continues(a, from / ps)) throw StateError("reload offset is not a node boundary");
    const std::uint64_t now = ++clock;
    const std::uint64_t n = len / ps;
    std::uint64_t p = from / ps, promoted = 0;
    while (p < n && promoted < max_tokens) {
      Page* head = find(a, p);
      if (head == nullptr || !head->host) break;
      std::uint64_t j = p + 1;
      while (j < n) {
        Page* q = find(a, j);
        if (q == nullptr || q->bnd) break;
        ++j;
      }
      bool full = !continues(a, j);
      std::uint64_t ka = j - p;
      const std::uint64_t want = (max_tokens - promoted) / ps;
      if (ka > want) {
        ka = want;
        full = false;
      }
      if (ka == 0) break;
      if (!full) split_before(a, p + ka);
      if (capacity - used < ka) {
        evict(ka - (capacity - used), offl_tokens);
        if (capacity - used < ka) break;
      }
      for (std::uint64_t k = p; k < p + ka; ++k) {
        const std::uint64_t kk = key(a, k);
        modify(kk, find_key(kk), [&](Page& q) {
          q.host = false;
          q.stamp = now;
        });
      }
      promoted += ka * ps;
      p += ka;
      if (!full) break;
    }
    return promoted;
  }

  /* pin / unpin, cache_tree.cpp:370-402: every node covering [0, len). */
  void pin(std::uint32_t a, std::uint64_t len, int delta) {
    if (len % ps != 0) throw std::invalid_argument("pin length not on a node boundary");
    const std::uint64_t n = len / ps;
    for (std::uint64_t k = 0; k < n; ++k) {
      Page* p = find(a, k);
      if (p == nullptr) throw StateError("pin path missing from tree");
      if (delta < 0 && p->pins == 0) throw StateError("unpin on a node with zero pin count");
    }
    if (continues(a, n)) throw std::invalid_argument("pin length not on a node boundary");
    for (std::uint64_t k = 0; k < n; ++k) {
      const std::uint64_t kk = key(a, k);
      modify(kk, find_key(kk), [&](Page& q) { q.pins += delta; });
    }
  }

  /* discard_suffix, cache_tree.cpp:404-437. */
  void discard_suffix(std::uint32_t a, std::uint64_t len, std::uint64_t from) {
    from = (from + ps - 1) / ps * ps;  // page_ceil (Q2: straddling page survives)
    if (from >= len) return;
    const std::uint64_t fp = from / ps;
    for (std::uint64_t k = 0; k < fp; ++k)  // path to `from`
      if (find(a, k) == nullptr) return;
    split_before(a, fp);  // the node straddling `from` is split there (:415)
    if (fp >= len / ps) return;  // no full page at `from`: no branch
    if (find(a, fp) == nullptr) return;
    // the branch subtree: pages on any path through page fp
    std::vector<std::uint64_t> doomed;
    const std::uint64_t head_owner = key(a, fp) >> 32;
    if (head_owner != 0) {
      // private head: this agent's chain from fp (present pages of a chain
      // are a contiguous prefix: walk until the first miss)
      for (std::uint64_t k = fp;; ++k) {
        auto it = pages.find((head_owner << 32) | k);
        if (it == pages.end()) break;
        if (it->second.pins > 0) throw StateError("discard_suffix would drop pinned nodes");
        doomed.push_back(it->first);
      }
    } else {
      // shared head: every page deeper than it, shared or private
      for (auto& kv : pages) {
        if ((kv.first & 0xffffffffULL) < fp) continue;
        if (kv.second.pins > 0) throw StateError("discard_suffix would drop pinned nodes");
        doomed.push_back(kv.first);
      }
    }
    for (std::uint64_t k : doomed) drop_page(pages.find(k));
    discarded += doomed.size() * ps;
  }

  std::uint64_t digest() const {  // O(1): dsum is maintained incrementally
    std::uint64_t h = kvdigest::fold(0x1234, dsum);
    h = kvdigest::fold(h, used);
    h = kvdigest::fold(h, clock);
    h = kvdigest::fold(h, kvdigest::dbits(hit_m));
    h = kvdigest::fold(h, kvdigest::dbits(hit_r));
    h = kvdigest::fold(h, discarded);
    h = kvdigest::fold(h, offloaded);
    return h;
  }
};

/* ================== node-level tree cache (offload mode) ==================== */

/* Offload-mode restatement at NODE granularity. Every reference algorithm
 * (cache_tree.cpp) is followed step for step, including the node
 * bookkeeping that decides eviction order: splits, ordinals, pin counts and
 * children_with_device. That last counter is not self-consistent in offload
 * mode: a reload (or insert) that promotes a host node whose subtree already
 * holds a device node (quirk Q1) calls propagate_gain again and double-counts
 * it in the parent (cache_tree.cpp:94-102, 357-361), after which the parent
 * can never become an eviction frontier. A per-page model cannot see that,
 * so offload mode keeps nodes. Segments are (first page, page count) along
 * the population's token scheme: pages below the shared prompt belong to
 * owner 0, the rest to the node's `tail` owner. */
struct TNode {
  std::uint32_t parent = 0;
  std::uint64_t start = 0, npages = 0;
  std::uint64_t tail = 0;  // owner (agent+1) of the pages at or past the shared prompt
  std::map<std::uint64_t, std::uint32_t> children;  // child head page key -> node
  std::uint64_t last_access = 0, ordinal = 0, device_slots = 0;
  int pin_count = 0, cwd = 0;  // cwd = children_with_device
  bool host = false, alive = true;
  bool subtree_has_device() const { return device_slots > 0 || cwd > 0; }
};

struct TreeCache {
  std::uint64_t capacity = 0, ps = 1, shared_pages = 0;
  bool offload = true;
  std::vector<TNode> nodes;  // nodes[0] = root
  std::vector<std::uint32_t> free_ids;
  std::uint64_t used = 0, clock = 0, discarded = 0, offloaded = 0, next_ordinal = 0;
  double hit_m = 0, hit_r = 0;
  std::uint64_t evict_calls = 0, evicted = 0;
  std::uint64_t dsum = 0;
  std::vector<std::pair<std::uint64_t, std::uint64_t>>* victims = nullptr;
  std::vector<kvg_log_record>* log = nullptr;
  std::uint32_t log_agent = 0;

  void init(std::uint64_t cap, std::uint64_t page, std::uint64_t p, bool sh, bool off) {
    if (cap == 0 || page == 0) throw std::invalid_argument("capacity and page size must be > 0");
    capacity = cap;
    ps = page;
    shared_pages = sh ? p / page : 0;
    offload = off;
    nodes.assign(1, TNode{});
  }
  std::uint64_t key(std::uint32_t a, std::uint64_t k) const {
    std::uint64_t owner = k < shared_pages ? 0 : std::uint64_t(a) + 1;
    return (owner << 32) | k;
  }
  std::uint64_t nkey(const TNode& n, std::uint64_t k) const {
    return ((k < shared_pages ? 0 : n.tail) << 32) | k;
  }
  std::uint64_t terms(const TNode& n) const {
    std::uint64_t s = 0;
    for (std::uint64_t k = n.start; k < n.start + n.npages; ++k) {
      const std::uint64_t kk = nkey(n, k);
      s += kvdigest::page_term(kk >> 32, k, n.last_access, static_cast<std::uint64_t>(n.pin_count),
                               n.host ? 1 : 0);
    }
    return s;
  }
  template <typename F>
  void modify(std::uint32_t id, F&& f) {
    dsum -= terms(nodes[id]);
    f(nodes[id]);
    dsum += terms(nodes[id]);
  }
  std::uint32_t new_node() {
    if (!free_ids.empty()) {
      std::uint32_t id = free_ids.back();
      free_ids.pop_back();
      nodes[id] = TNode{};
      return id;
    }
    nodes.emplace_back();
    return static_cast<std::uint32_t>(nodes.size() - 1);
  }
  /* find_child (cache_tree.cpp:56-66): needs a full page of the sequence. */
  std::uint32_t find_child(std::uint32_t node, std::uint32_t a, std::uint64_t p,
                           std::uint64_t n_full) const {
    if (p >= n_full) return 0;
    auto it = nodes[node].children.find(key(a, p));
    return it == nodes[node].children.end() ? 0 : it->second;
  }
  /* common_len in whole pages (a partial trailing page never counts). */
  std::uint64_t common(std::uint32_t c, std::uint32_t a, std::uint64_t p, std::uint64_t n_full) const {
    const TNode& n = nodes[c];
    std::uint64_t k = std::min(n.npages, n_full - p);
    if (n.tail != std::uint64_t(a) + 1) {
      const std::uint64_t sh = shared_pages > p ? shared_pages - p : 0;
      k = std::min(k, sh);
    }
    return k;
  }
  /* split_node, cache_tree.cpp:68-92 (offset in pages). */
  std::uint32_t split(std::uint32_t id, std::uint64_t off) {
    const std::uint32_t sid = new_node();
    TNode& node = nodes[id];
    TNode& s = nodes[sid];
    s.start = node.start + off;
    s.npages = node.npages - off;
    s.tail = node.tail;
    s.children = std::move(node.children);
    for (auto& kv : s.children) nodes[kv.second].parent = sid;
    s.parent = id;
    s.last_access = node.last_access;
    s.ordinal = next_ordinal++;
    s.host = node.host;
    s.pin_count = node.pin_count;
    s.cwd = node.cwd;
    if (!node.host) {
      s.device_slots = node.device_slots - off;
      node.device_slots = off;
    }
    node.npages = off;
    node.children.clear();
    node.cwd = s.subtree_has_device() ? 1 : 0;
    node.children.emplace(nkey(s, s.start), sid);
    return sid;  // page attributes unchanged: the digest sum is unchanged
  }
  void propagate_gain(std::uint32_t id) {  // cache_tree.cpp:94-102
    std::uint32_t p = nodes[id].parent;
    for (;;) {
      TNode& pn = nodes[p];
      const bool had = pn.subtree_has_device();
      pn.cwd += 1;
      if (had || p == 0) break;  // the root has no parent
      p = pn.parent;
    }
  }
  void propagate_loss(std::uint32_t id) {  // cache_tree.cpp:104-112
    std::uint32_t p = nodes[id].parent;
    for (;;) {
      TNode& pn = nodes[p];
      pn.cwd -= 1;
      if (pn.subtree_has_device() || p == 0) break;
      p = pn.parent;
    }
  }

  /* match_prefix, cache_tree.cpp:114-142 */
  std::uint64_t match(std::uint32_t a, std::uint64_t len, std::uint64_t* host_matched) {
    const std::uint64_t now = ++clock;
    const std::uint64_t n = len / ps;
    std::uint32_t node = 0;
    std::uint64_t pos = 0, matched = 0, hm = 0;
    bool host_phase = false;
    while (pos < n) {
      const std::uint32_t c = find_child(node, a, pos, n);
      if (c == 0) break;
      if (nodes[c].host) host_phase = true;
      const std::uint64_t ka = common(c, a, pos, n);
      const bool full = ka == nodes[c].npages;
      if (ka == 0) break;
      if (!full) split(c, ka);
      if (host_phase) {
        hm += ka;
      } else {
        modify(c, [&](TNode& x) { x.last_access = now; });
        matched += ka;
      }
      pos += ka;
      node = c;
      if (!full) break;
    }
    hit_m += static_cast<double>(matched * ps);
    hit_r += static_cast<double>(len);
    if (host_matched) *host_matched = hm * ps;
    return matched * ps;
  }

  std::uint64_t missing(std::uint32_t a, std::uint64_t n) const {  // cache_tree.cpp:144-168
    std::uint32_t node = 0;
    std::uint64_t pos = 0, m = 0;
    while (pos < n) {
      const std::uint32_t c = find_child(node, a, pos, n);
      if (c == 0) return m + (n - pos);
      const std::uint64_t ka = common(c, a, pos, n);
      const bool full = ka == nodes[c].npages;
      if (ka == 0) return m;
      if (nodes[c].host) m += ka;
      pos += ka;
      node = c;
      if (!full) return m + (n - pos);
    }
    return m;
  }

  bool is_frontier(std::uint32_t id) const {  // cache_tree.cpp:230-234
    const TNode& n = nodes[id];
    return id != 0 && !n.host && n.device_slots > 0 && n.pin_count == 0 && n.cwd == 0;
  }
  using Ent = std::pair<std::pair<std::uint64_t, std::uint64_t>, std::uint32_t>;
  void collect_frontier(std::uint32_t id, std::vector<Ent>& out) const {  // :236-249
    for (const auto& kv : nodes[id].children) {
      const std::uint32_t c = kv.second;
      if (!nodes[c].subtree_has_device()) continue;
      if (is_frontier(c)) {
        out.push_back({{nodes[c].last_access, nodes[c].ordinal}, c});
        continue;
      }
      collect_frontier(c, out);
    }
  }
  void free_subtree(std::uint32_t id, std::uint64_t* toks) {
    for (auto& kv : nodes[id].children) free_subtree(kv.second, toks);
    if (toks) *toks += nodes[id].npages * ps;
    dsum -= terms(nodes[id]);
    nodes[id].alive = false;
    nodes[id].children.clear();
    free_ids.push_back(id);
  }

  /* evict, cache_tree.cpp:270-319 */
  std::uint64_t evict(std::uint64_t needed, std::uint64_t* offl_tokens = nullptr) {
    if (needed == 0) return 0;
    ++evict_calls;
    std::vector<Ent> init;
    collect_frontier(0, init);
#ifdef KVO_CHECK_FLAT_FRONTIER
    {  // the DFS frontier equals the flat set of frontier nodes (no counter
       // under-count hides a frontier node below a device-less ancestor)
      std::vector<Ent> flat;
      for (std::uint32_t i = 1; i < nodes.size(); ++i)
        if (nodes[i].alive && is_frontier(i))
          flat.push_back({{nodes[i].last_access, nodes[i].ordinal}, i});
      std::vector<Ent> a = init;
      std::sort(a.begin(), a.end());
      std::sort(flat.begin(), flat.end());
      if (a != flat) throw StateError("flat frontier differs from the DFS frontier");
    }
#endif
    std::priority_queue<Ent, std::vector<Ent>, std::greater<Ent>> heap(std::greater<Ent>(),
                                                                       std::move(init));
    std::uint64_t reclaimed = 0;
    const std::size_t log0 = log ? log->size() : 0;
    if (log) log->push_back(kvg_log_record{KVG_LOG_EVICT, log_agent, clock, needed, 0});
    while (reclaimed < needed && !heap.empty()) {
      auto [stamp, id] = heap.top();
      heap.pop();
      if (!is_frontier(id) || nodes[id].last_access != stamp.first ||
          nodes[id].ordinal != stamp.second)
        continue;
      const std::uint64_t take = std::min(nodes[id].device_slots, needed - reclaimed);
      std::uint32_t v = id;
      if (take < nodes[id].device_slots) v = split(id, nodes[id].npages - take);
      const TNode& vn = nodes[v];
      for (std::uint64_t k = vn.start + vn.npages; k-- > vn.start;) {  // record_victims
        const std::uint64_t kk = nkey(vn, k);
        if (victims) victims->emplace_back(kk, vn.last_access);
        if (log) log->push_back(kvg_log_record{KVG_LOG_VICTIM, log_agent, clock, kk, vn.last_access});
      }
      used -= vn.device_slots;
      reclaimed += vn.device_slots;
      const std::uint32_t parent = vn.parent;
      if (offload) {
        const std::uint64_t toks = vn.npages * ps;
        offloaded += toks;
        if (offl_tokens) *offl_tokens += toks;
        modify(v, [](TNode& x) {
          x.device_slots = 0;
          x.host = true;
        });
        propagate_loss(v);
      } else {
        std::uint64_t dropped = 0;
        propagate_loss(v);
        const std::uint64_t head = nkey(nodes[v], nodes[v].start);
        free_subtree(v, &dropped);
        discarded += dropped;
        nodes[parent].children.erase(head);
      }
      if (is_frontier(parent))
        heap.push({{nodes[parent].last_access, nodes[parent].ordinal}, parent});
    }
    if (log) (*log)[log0].b = reclaimed;
    evicted += reclaimed;
    return reclaimed;
  }

  /* insert, cache_tree.cpp:170-228 */
  bool insert(std::uint32_t a, std::uint64_t len, std::uint64_t* inserted,
              std::uint64_t* evicted_pages, std::uint64_t* offl_tokens = nullptr) {
    const std::uint64_t n = len / ps;
    if (inserted) *inserted = 0;
    if (n == 0) return true;
    for (;;) {
      const std::uint64_t need = missing(a, n);
      const std::uint64_t free_slots = capacity - used;
      if (need <= free_slots) break;
      const std::uint64_t ev = evict(need - free_slots, offl_tokens);
      if (evicted_pages) *evicted_pages += ev;
      if (ev == 0) return false;
    }
    const std::uint64_t now = ++clock;
    std::uint32_t node = 0;
    std::uint64_t pos = 0;
    while (pos < n) {
      const std::uint32_t c = find_child(node, a, pos, n);
      if (c == 0) {
        const std::uint32_t l = new_node();
        TNode& ln = nodes[l];
        ln.start = pos;
        ln.npages = n - pos;
        ln.tail = std::uint64_t(a) + 1;
        ln.parent = node;
        ln.last_access = now;
        ln.ordinal = next_ordinal++;
        ln.device_slots = n - pos;
        dsum += terms(ln);
        used += ln.device_slots;
        if (inserted) *inserted += ln.device_slots;
        nodes[node].children.emplace(key(a, pos), l);
        propagate_gain(l);
        pos = n;
        break;
      }
      const std::uint64_t ka = common(c, a, pos, n);
      const bool full = ka == nodes[c].npages;
      if (ka == 0) break;
      if (!full) split(c, ka);
      if (nodes[c].host) {
        const std::uint64_t pages = nodes[c].npages;
        modify(c, [&](TNode& x) {
          x.host = false;
          x.device_slots = pages;
        });
        used += pages;
        if (inserted) *inserted += pages;
        propagate_gain(c);
      }
      modify(c, [&](TNode& x) { x.last_access = now; });
      pos += ka;
      node = c;
    }
    return true;
  }

  /* reload, cache_tree.cpp:321-368 */
  std::uint64_t reload(std::uint32_t a, std::uint64_t len, std::uint64_t from,
                       std::uint64_t max_tokens, std::uint64_t* offl_tokens) {
    if (from >= len || max_tokens == 0) return 0;
    const std::uint64_t n = len / ps;
    std::uint32_t node = 0;
    std::uint64_t pos = 0;  // tokens
    while (pos < from) {
      const std::uint32_t c = (pos % ps == 0) ? find_child(node, a, pos / ps, n) : 0;
      if (c == 0) throw StateError("reload offset is not on a cached path");
      if (nodes[c].npages * ps > from - pos) throw StateError("reload offset is not a node boundary");
      pos += nodes[c].npages * ps;
      node = c;
    }
    const std::uint64_t now = ++clock;
    std::uint64_t promoted = 0;
    while (pos < len && promoted < max_tokens) {
      const std::uint32_t c = find_child(node, a, pos / ps, n);
      if (c == 0) break;
      if (!nodes[c].host) break;
      std::uint64_t ka = common(c, a, pos / ps, n);
      bool full = ka == nodes[c].npages;
      const std::uint64_t want = (max_tokens - promoted) / ps;
      if (ka > want) {
        ka = want;
        full = false;
      }
      if (ka == 0) break;
      if (ka < nodes[c].npages) split(c, ka);
      const std::uint64_t pages = ka;
      if (capacity - used < pages) {
        evict(pages - (capacity - used), offl_tokens);
        if (capacity - used < pages) break;
      }
      modify(c, [&](TNode& x) {
        x.host = false;
        x.device_slots = pages;
        x.last_access = now;
      });
      used += pages;
      propagate_gain(c);
      promoted += ka * ps;
      pos += ka * ps;
      node = c;
      if (!full) break;
    }
    return promoted;
  }

  /* pin / unpin, cache_tree.cpp:370-402 */
  void pin(std::uint32_t a, std::uint64_t len, int delta) {
    const std::uint64_t n = len / ps;
    std::uint32_t node = 0;
    std::uint64_t pos = 0;  // tokens
    std::vector<std::uint32_t> path;
    while (pos < len) {
      const std::uint32_t c = (pos % ps == 0) ? find_child(node, a, pos / ps, (len + ps - 1) / ps) : 0;
      if (c == 0) throw StateError(delta > 0 ? "pin path missing from tree" : "unpin path missing from tree");
      if (pos + nodes[c].npages * ps > len)
        throw std::invalid_argument("pin length not on a node boundary");
      if (delta < 0 && nodes[c].pin_count == 0)
        throw StateError("unpin on a node with zero pin count");
      path.push_back(c);
      pos += nodes[c].npages * ps;
      node = c;
    }
    (void)n;
    for (std::uint32_t c : path) modify(c, [&](TNode& x) { x.pin_count += delta; });
  }

  /* discard_suffix, cache_tree.cpp:404-437 */
  void discard_suffix(std::uint32_t a, std::uint64_t len, std::uint64_t from) {
    from = (from + ps - 1) / ps * ps;
    if (from >= len) return;
    const std::uint64_t n = len / ps;
    std::uint32_t node = 0;
    std::uint64_t pos = 0;  // tokens
    while (pos < from) {
      const std::uint32_t c = find_child(node, a, pos / ps, n);
      if (c == 0) return;
      const std::uint64_t kp = common(c, a, pos / ps, n);
      if (kp < nodes[c].npages && pos + kp * ps < from) return;
      if (nodes[c].npages * ps > from - pos) split(c, (from - pos) / ps);
      pos += nodes[c].npages * ps;
      node = c;
    }
    const std::uint32_t b = find_child(node, a, from / ps, n);
    if (b == 0) return;
    std::uint64_t slots = 0, toks = 0;
    int pins = 0;
    std::vector<std::uint32_t> st{b};
    while (!st.empty()) {
      const std::uint32_t x = st.back();
      st.pop_back();
      slots += nodes[x].device_slots;
      toks += nodes[x].npages * ps;
      pins += nodes[x].pin_count;
      for (auto& kv : nodes[x].children) st.push_back(kv.second);
    }
    if (pins > 0) throw StateError("discard_suffix would drop pinned nodes");
    if (nodes[b].subtree_has_device()) propagate_loss(b);
    used -= slots;
    discarded += toks;
    const std::uint64_t head = nkey(nodes[b], nodes[b].start);
    free_subtree(b, nullptr);
    nodes[node].children.erase(head);
  }

  std::uint64_t digest() const {
    std::uint64_t h = kvdigest::fold(0x1234, dsum);
    h = kvdigest::fold(h, used);
    h = kvdigest::fold(h, clock);
    h = kvdigest::fold(h, kvdigest::dbits(hit_m));
    h = kvdigest::fold(h, kvdigest::dbits(hit_r));
    h = kvdigest::fold(h, discarded);
    h = kvdigest::fold(h, offloaded);
    return h;
  }
};

/* ======================= controller (controller.cpp) ======================== */

struct Ctl {
  std::uint32_t kind = KVG_POLICY_UNCONTROLLED, cap = 1, total = 0;
  kvg_controller_config cfg{};
  double window = 1.0, su = 0, sh = 0;
  bool have_smoothed = false;
  std::vector<std::uint32_t> active;
  std::deque<std::uint32_t> pending, paused;
  std::uint64_t ticks = 0;

  void init(const kvg_policy& p, std::uint32_t n) {  // controller.cpp:55-65
    kind = p.kind;
    cap = p.cap;
    cfg = p.aimd;
    total = n;
    if (kind == KVG_POLICY_AIMD) {
      if (cfg.w_max == 0) cfg.w_max = std::max(cfg.w_min, static_cast<double>(n));
      if (cfg.initial_window == 0) cfg.initial_window = cfg.w_min;
      window = cfg.initial_window;
    }
  }
  bool agent_gated() const { return kind == KVG_POLICY_AGENT_CAP || kind == KVG_POLICY_AIMD; }
  /* update_window, controller.cpp:67-91 */
  void update(double usage, double hit) {
    ++ticks;
    if (kind != KVG_POLICY_AIMD) return;
    double u = usage, h = hit;
    if (cfg.signal_smoothing > 0) {
      if (have_smoothed) {
        u = cfg.signal_smoothing * su + (1 - cfg.signal_smoothing) * usage;
        h = cfg.signal_smoothing * sh + (1 - cfg.signal_smoothing) * hit;
      }
      su = u;
      sh = h;
      have_smoothed = true;
    }
    double w = window;
    if (u < cfg.u_low)
      w = w + cfg.alpha;
    else if (u > cfg.u_high && h < cfg.h_thresh)
      w = w * cfg.beta;
    window = w < cfg.w_min ? cfg.w_min : (cfg.w_max < w ? cfg.w_max : w);
  }
  std::uint64_t limit() const {  // controller.cpp:93-104
    switch (kind) {
      case KVG_POLICY_UNCONTROLLED: return std::numeric_limits<std::uint64_t>::max();
      case KVG_POLICY_AIMD: return static_cast<std::uint64_t>(std::floor(window));
      default: return cap;
    }
  }
  double display() const {  // controller.cpp:106-117
    switch (kind) {
      case KVG_POLICY_UNCONTROLLED: return static_cast<double>(total);
      case KVG_POLICY_AIMD: return window;
      default: return static_cast<double>(cap);
    }
  }
  void remove_active(std::uint32_t id, const char* what) {
    auto it = std::find(active.begin(), active.end(), id);
    if (it == active.end()) throw StateError(what);
    active.erase(it);
  }
  std::uint64_t digest() const {
    std::uint64_t h = 0x5678;
    for (auto id : active) h = kvdigest::fold(h, id);
    h = kvdigest::fold(h, 0xAAAA);
    for (auto id : pending) h = kvdigest::fold(h, id);
    h = kvdigest::fold(h, 0xBBBB);
    for (auto id : paused) h = kvdigest::fold(h, id);
    h = kvdigest::fold(h, kvdigest::dbits(window));
    h = kvdigest::fold(h, ticks);
    return h;
  }
};

/* ======================= engine (engine.cpp) ================================ */

enum : std::uint8_t { S_PENDING, S_AWAIT, S_GEN, S_TOOL, S_PAUSED, S_DONE };
enum : std::uint8_t { EV_GEN = 0, EV_TOOL = 1, EV_XFER = 2 };

/* lifecycle_edge, workload.cpp:110-128 */
bool legal(std::uint8_t from, std::uint8_t to) {
  switch (from) {
    case S_PENDING: return to == S_AWAIT;
    case S_AWAIT: return to == S_GEN || to == S_PAUSED;
    case S_GEN: return to == S_TOOL || to == S_DONE || to == S_AWAIT;
    case S_TOOL: return to == S_AWAIT;
    case S_PAUSED: return to == S_AWAIT;
    default: return false;
  }
}

struct AgentRec {
  std::uint8_t state = S_PENDING;
  std::uint32_t step = 0;
  std::uint64_t ctx = 0, high_water = 0, pinned = 0;
  double ready_since = 0;
  std::uint64_t f_gen = 0, f_rec = 0, f_obs = 0;
  double f_tool = 0;
  bool f_has_tool = false;
  kvg_agent_stats st{};
};

template <typename CacheT>
struct Sim {
  const kvg_sim_desc* d;
  const kvg_step_plan* plans;
  std::uint32_t n = 0, steps = 0;
  CacheT cache;
  Ctl ctl;
  std::vector<AgentRec> ag;
  std::set<std::tuple<double, std::uint64_t, std::uint32_t>> agent_q;  // rank 0
  std::vector<std::uint8_t> ev_kind;
  std::uint64_t ord = 0;
  bool tick_on = false, adm_on = false;
  double tick_t = 0, adm_t = 0;
  std::uint64_t tick_o = 0, adm_o = 0;
  double clock = 0, gpu_busy = 0, makespan = 0;
  std::uint32_t finished = 0;
  std::uint64_t decoded_cum = 0, rec_cum = 0, lookups = 0, agent_steps = 0;
  std::uint64_t events = 0;
  kvg_ledger ledger{};
  double device_busy = 0;
  // link queue (engine.cpp:156-182)
  std::multiset<double> xfer_ends;
  double pcie_busy = 0, link_busy = 0;
  std::uint64_t reloaded = 0;
  std::vector<kvg_trace_row> trace;
  std::vector<std::uint64_t>* digests = nullptr;
  std::vector<kvg_log_record>* log = nullptr;

  void logrec(std::uint32_t kind, std::uint32_t agent, std::uint64_t a, std::uint64_t b) {
    if (log) log->push_back(kvg_log_record{kind, agent, cache.clock, a, b});
  }
  void set_state(std::uint32_t id, std::uint8_t s) {  // workload.cpp:130-137
    if (!legal(ag[id].state, s)) throw StateError("illegal lifecycle transition");
    ag[id].state = s;
  }
  double interval() const { return d->policy.aimd.control_interval; }
  /* cost_model.cpp:28-41 */
  double prefill(std::uint64_t nt, std::uint64_t c) const {
    double x = static_cast<double>(nt), y = static_cast<double>(c);
    return d->cost.prefill_linear * x + d->cost.prefill_quadratic * x * y;
  }
  double decode(std::uint64_t nt, std::uint64_t c) const {
    double x = static_cast<double>(nt), y = static_cast<double>(c);
    return d->cost.decode_base * x + d->cost.decode_context * (x * y + x * (x - 1.0) / 2.0);
  }
  void schedule_agent(double t, std::uint8_t kind, std::uint32_t id) {  // engine.cpp:143-145
    agent_q.emplace(t, ord++, id);
    ev_kind[id] = kind;
  }
  /* transfers_in_flight, engine.cpp:156-160 */
  std::size_t in_flight() {
    while (!xfer_ends.empty() && *xfer_ends.begin() <= clock) xfer_ends.erase(xfer_ends.begin());
    return xfer_ends.size();
  }
  /* enqueue_transfer, engine.cpp:164-174; transfer_time, cost_model.cpp:43-47 */
  double enqueue_transfer(double bytes) {
    const std::size_t depth = in_flight() + 1;
    const double dur = d->cost.transfer_sync_overhead +
                       bytes * static_cast<double>(depth) / d->cost.pcie_bandwidth;
    const double start = clock < pcie_busy ? pcie_busy : clock;
    const double end = start + dur;
    pcie_busy = end;
    ledger.transfer += dur;
    link_busy += dur;
    xfer_ends.insert(end);
    return end;
  }
  /* account_evictions, engine.cpp:178-182 */
  void account(std::uint64_t offl_tokens) {
    if (offl_tokens > 0)
      enqueue_transfer(static_cast<double>(offl_tokens) * d->cost.bytes_per_token);
  }
  void schedule_admission() {  // engine.cpp:149-154
    if (adm_on && adm_t == clock) return;
    if (adm_on) throw StateError("two admission checks outstanding");
    adm_on = true;
    adm_t = clock;
    adm_o = ord++;
  }

  void init(const kvg_sim_desc* desc) {
    d = desc;
    const kvg_population* pop = d->population;
    n = pop->agents;
    steps = pop->steps;
    plans = pop->plans;
    cache.init(d->engine.capacity, d->engine.page_size, pop->prompt_tokens,
               pop->shared_prompt != 0, d->engine.eviction == KVG_EVICT_OFFLOAD);
    ctl.init(d->policy, n);
    ag.assign(n, AgentRec{});
    ev_kind.assign(n, 0);
    for (std::uint32_t i = 0; i < n; ++i) {
      ag[i].ctx = pop->prompt_tokens;
      ctl.pending.push_back(i);  // engine.cpp:89-93
      ag[i].st.finish_time = -1.0;
    }
  }

  /* engine.cpp:337-396 */
  bool dispatch_member(std::uint32_t id, double* t_out, double* ft, double* rt, double* dt) {
    AgentRec& a = ag[id];
    const std::uint64_t ctx = a.ctx;
    std::uint64_t host_matched = 0;
    const std::uint64_t matched = cache.match(id, ctx, &host_matched);
    {
      std::uint64_t r = (matched + host_matched) / cache.ps;
      lookups += r + (r < ctx / cache.ps ? 1 : 0);
    }
    logrec(KVG_LOG_MATCH, id, matched, host_matched);
    cache.pin(id, matched, +1);
    if (a.pinned > 0) cache.pin(id, a.pinned, -1);
    a.pinned = matched;
    if (cache.offload && host_matched > 0) {  // engine.cpp:343-360
      std::uint64_t offl = 0;
      cache.log = log;
      cache.log_agent = id;
      const std::uint64_t promoted = cache.reload(id, ctx, matched, host_matched, &offl);
      cache.log = nullptr;
      account(offl);
      logrec(KVG_LOG_RELOAD, id, promoted, offl);
      if (promoted > 0) {
        cache.pin(id, matched + promoted, +1);
        cache.pin(id, matched, -1);
        a.pinned = matched + promoted;
        reloaded += promoted;
        const double end = enqueue_transfer(static_cast<double>(promoted) * d->cost.bytes_per_token);
        a.st.wait_time += clock - a.ready_since;
        set_state(id, S_GEN);
        schedule_agent(end, EV_XFER, id);
        return false;
      }
    }
    const kvg_step_plan& plan = plans[std::size_t(id) * steps + a.step];
    a.ctx += plan.gen_tokens;  // append_tokens
    std::uint64_t inserted = 0, offl = 0;
    cache.log = log;
    cache.log_agent = id;
    bool ok = cache.insert(id, a.ctx, &inserted, nullptr, &offl);
    cache.log = nullptr;
    account(offl);
    logrec(KVG_LOG_INSERT, id, ok ? 1 : 0, ok ? a.ctx / cache.ps * cache.ps : 0);
    if (!ok) {
      a.ctx = ctx;
      cache.pin(id, matched, -1);
      a.pinned = 0;
      ++a.st.stall_events;
      return false;
    }
    const std::uint64_t stored = a.ctx - a.ctx % cache.ps;
    cache.pin(id, stored, +1);
    cache.pin(id, matched, -1);
    a.pinned = stored;
    const std::uint64_t missing = ctx - matched;
    const std::uint64_t rec = a.high_water > matched ? a.high_water - matched : 0;
    const std::uint64_t fresh = missing - rec;
    a.high_water = stored;
    *ft = prefill(fresh, ctx);
    *rt = prefill(rec, ctx);
    *dt = decode(plan.gen_tokens, ctx);
    *t_out = *ft + *rt + *dt;
    a.f_gen = plan.gen_tokens;
    a.f_rec = rec;
    a.f_has_tool = plan.has_tool != 0;
    a.f_obs = plan.obs_tokens;
    a.f_tool = plan.tool_latency;
    a.st.wait_time += clock - a.ready_since;
    set_state(id, S_GEN);
    ++agent_steps;
    return true;
  }

  /* engine.cpp:305-333 */
  void dispatch_batch() {
    std::vector<std::uint32_t> ready;
    for (std::uint32_t id : ctl.active)
      if (ag[id].state == S_AWAIT) ready.push_back(id);
    std::sort(ready.begin(), ready.end());
    struct M { std::uint32_t id; double t, f, r, dd; };
    std::vector<M> batch;
    for (std::uint32_t id : ready) {
      M m{id, 0, 0, 0, 0};
      if (dispatch_member(id, &m.t, &m.f, &m.r, &m.dd)) batch.push_back(m);
    }
    if (batch.empty()) return;
    double wall = 0.0, total = 0.0;
    for (const M& m : batch) {
      wall = wall < m.t ? m.t : wall;
      total += m.t;
    }
    double start = clock < gpu_busy ? gpu_busy : clock;
    gpu_busy = start + wall;
    device_busy += wall;
    double share = total > 0 ? wall / total : 0.0;
    for (const M& m : batch) {
      ledger.prefill_fresh += share * m.f;
      ledger.prefill_recompute += share * m.r;
      ledger.decode += share * m.dd;
      schedule_agent(start + wall, EV_GEN, m.id);
    }
  }

  /* controller.cpp:124-160 + engine.cpp:268-291 */
  void on_admission() {
    adm_on = false;
    std::uint64_t lim = ctl.limit();
    struct Cmd { int kind; std::uint32_t id; };  // 0 admit 1 pause 2 resume
    std::vector<Cmd> cmds;
    if (ctl.agent_gated()) {
      while (ctl.active.size() > lim) {
        long victim = -1;
        for (long i = long(ctl.active.size()) - 1; i >= 0; --i)
          if (ag[ctl.active[i]].state == S_AWAIT) { victim = i; break; }
        if (victim < 0) break;
        std::uint32_t id = ctl.active[victim];
        ctl.active.erase(ctl.active.begin() + victim);
        ctl.paused.push_back(id);
        cmds.push_back({1, id});
      }
    }
    while (ctl.active.size() < lim) {
      if (ctl.agent_gated() && !ctl.paused.empty()) {
        std::uint32_t id = ctl.paused.front();
        ctl.paused.pop_front();
        ctl.active.push_back(id);
        cmds.push_back({2, id});
      } else if (!ctl.pending.empty()) {
        std::uint32_t id = ctl.pending.front();
        ctl.pending.pop_front();
        ctl.active.push_back(id);
        cmds.push_back({0, id});
      } else {
        break;
      }
    }
    for (const Cmd& c : cmds) {
      if (c.kind == 1) {
        set_state(c.id, S_PAUSED);
        ++ag[c.id].st.pause_events;
      } else if (c.kind == 0) {
        if (ag[c.id].state == S_PENDING) set_state(c.id, S_AWAIT);
      } else {
        set_state(c.id, S_AWAIT);
      }
    }
    dispatch_batch();
  }

  /* engine.cpp:184-222 */
  void on_generation_complete(std::uint32_t id) {
    AgentRec& a = ag[id];
    makespan = makespan < clock ? clock : makespan;
    if (a.pinned > 0) {
      cache.pin(id, a.pinned, -1);
      a.pinned = 0;
    }
    decoded_cum += a.f_gen;
    rec_cum += a.f_rec;
    a.st.generated_tokens += a.f_gen;
    a.st.recompute_tokens += a.f_rec;
    if (a.f_rec > 0) ++a.st.recompute_events;
    ++a.step;
    const bool req = ctl.kind == KVG_POLICY_REQUEST_CAP;
    if (a.step >= steps) {
      set_state(id, S_DONE);
      const std::uint64_t before = cache.used;
      cache.discard_suffix(id, a.ctx, d->population->shared_prompt_tokens);
      logrec(KVG_LOG_DISCARD, id, 0, before - cache.used);
      if (req)
        ctl.remove_active(id, "request completion for inactive agent");
      else
        ctl.remove_active(id, "finished agent is not active");
      ++finished;
      a.st.finish_time = clock;
      a.st.finish_ordinal = events;
      std::uint64_t tb;
      std::memcpy(&tb, &clock, 8);
      logrec(KVG_LOG_FINISH, id, tb, events);
    } else if (a.f_has_tool) {
      set_state(id, S_TOOL);
      ledger.tool_wait += a.f_tool;
      if (req) ctl.remove_active(id, "request completion for inactive agent");
      schedule_agent(clock + a.f_tool, EV_TOOL, id);
    } else {
      set_state(id, S_AWAIT);
      a.ready_since = clock;
      if (req) {
        ctl.remove_active(id, "request completion for inactive agent");
        ctl.pending.push_back(id);
      }
    }
    schedule_admission();
  }

  /* engine.cpp:224-235 */
  void on_tool_complete(std::uint32_t id) {
    AgentRec& a = ag[id];
    makespan = makespan < clock ? clock : makespan;
    a.ctx += a.f_obs;
    a.f_obs = 0;
    a.f_has_tool = false;
    set_state(id, S_AWAIT);
    a.ready_since = clock;
    if (ctl.kind == KVG_POLICY_REQUEST_CAP) {
      ctl.pending.push_back(id);
    } else if (std::find(ctl.active.begin(), ctl.active.end(), id) == ctl.active.end()) {
      throw StateError("tool return for inactive agent");
    }
    schedule_admission();
  }

  /* engine.cpp:237-243 */
  void on_transfer_complete(std::uint32_t id) {
    AgentRec& a = ag[id];
    makespan = makespan < clock ? clock : makespan;
    set_state(id, S_AWAIT);
    a.ready_since = clock;
    schedule_admission();
  }

  /* engine.cpp:245-266 */
  void on_tick() {
    const double usage = static_cast<double>(cache.used) / static_cast<double>(cache.capacity);
    const double m = cache.hit_m, r = cache.hit_r;
    const double hit = r > 0 ? m / r : 1.0;
    ctl.update(usage, hit);
    kvg_trace_row row{clock, usage, hit, ctl.display(),
                      ctl.active.size(), ctl.pending.size() + ctl.paused.size(),
                      decoded_cum, rec_cum, in_flight(), m, r};
    trace.push_back(row);
    cache.hit_m *= d->engine.hit_window_decay;
    cache.hit_r *= d->engine.hit_window_decay;
    tick_on = true;
    tick_t = clock + interval();
    tick_o = ord++;
    schedule_admission();
  }

  /* engine.cpp:98-136 */
  int run() {
    adm_on = true;  // schedule(0.0, admission): ordinal 0
    adm_t = 0.0;
    adm_o = ord++;
    tick_on = true;  // schedule(interval, tick): ordinal 1
    tick_t = interval();
    tick_o = ord++;
    for (;;) {
      // pop the minimum (time, rank, ordinal)
      int which = -1;  // 0 agent, 1 tick, 2 admission
      double bt = 0;
      std::uint64_t bo = 0;
      if (!agent_q.empty()) {
        which = 0;
        bt = std::get<0>(*agent_q.begin());
        bo = std::get<1>(*agent_q.begin());
      }
      auto better = [&](double t, int rank, std::uint64_t o) {
        if (which < 0) return true;
        if (t != bt) return t < bt;
        if (rank != which) return rank < which;
        return o < bo;
      };
      if (tick_on && better(tick_t, 1, tick_o)) { which = 1; bt = tick_t; bo = tick_o; }
      if (adm_on && better(adm_t, 2, adm_o)) { which = 2; bt = adm_t; bo = adm_o; }
      if (which < 0) break;
      std::uint32_t agent = 0;
      if (which == 0) {
        agent = std::get<2>(*agent_q.begin());
        agent_q.erase(agent_q.begin());
      } else if (which == 1) {
        tick_on = false;
      } else {
        adm_on = false;
      }
      if (which != 0 && finished == n) continue;  // housekeeping after the end
      if (bt > d->engine.horizon) return KVG_ERR_HORIZON;
      clock = bt;
      if (which == 0) {
        switch (ev_kind[agent]) {
          case EV_GEN: on_generation_complete(agent); break;
          case EV_TOOL: on_tool_complete(agent); break;
          default: on_transfer_complete(agent); break;
        }
      } else if (which == 1) {
        on_tick();
      } else {
        on_admission();
      }
      ++events;
      if (digests) digests->push_back(kvdigest::fold(cache.digest(), ctl.digest()));
    }
    if (finished != n) throw StateError("event queue drained with unfinished agents");
    return KVG_OK;
  }

  void fill(kvg_sim_result* res, int status) const {  // engine.cpp:398-415
    std::memset(res, 0, sizeof *res);
    res->status = status;
    res->ledger = ledger;
    res->makespan = makespan < pcie_busy ? pcie_busy : makespan;  // engine.cpp:400
    res->device_busy = device_busy;
    res->link_busy = link_busy;
    res->reloaded_tokens = reloaded;
    res->decoded_tokens = decoded_cum;
    res->recompute_tokens = rec_cum;
    double wait = 0;
    for (const AgentRec& a : ag) {
      res->recompute_events += a.st.recompute_events;
      res->stall_events += a.st.stall_events;
      wait += a.st.wait_time;
    }
    res->total_wait_time = wait;
    res->discarded_tokens = cache.discarded;
    res->offloaded_tokens = cache.offloaded;
    res->ticks = trace.size();
    res->workload_hash = d->population->stream_hash;
    res->agent_steps = agent_steps;
    res->lookups = lookups;
    res->events = events;
    res->evict_calls = cache.evict_calls;
    res->evicted_pages = cache.evicted;
    res->cache_clock = cache.clock;
    res->pool_used = cache.used;
    res->hit_matched = cache.hit_m;
    res->hit_requested = cache.hit_r;
    classify(res);
  }

  /* classify_phases, metrics.cpp:41-81 (called from finish_result, engine.cpp:413) */
  void classify(kvg_sim_result* res) const {
    const kvg_phase_params& pp = d->engine.phases;
    const double mk = res->makespan;
    res->n_phases = 0;
    if (mk <= 0) return;
    auto hot = [&](const kvg_trace_row& r) {
      return r.usage >= pp.sat_threshold && r.hit_rate < pp.hit_threshold;
    };
    auto push = [&](std::uint32_t ph, double a, double b) {
      res->phases[res->n_phases++] = kvg_phase_label{ph, 0, a, b};
    };
    std::size_t enter = trace.size();
    for (std::size_t i = 0; i < trace.size(); ++i)
      if (hot(trace[i])) { enter = i; break; }
    if (enter == trace.size()) {
      push(KVG_PHASE_WARMUP, 0.0, mk);
      return;
    }
    const double ms = trace[enter].time;
    double me = mk;
    int bad = 0;
    for (std::size_t i = enter + 1; i < trace.size(); ++i) {
      if (hot(trace[i])) { bad = 0; continue; }
      if (++bad >= pp.hysteresis) {
        me = trace[i + 1 - static_cast<std::size_t>(pp.hysteresis)].time;
        break;
      }
    }
    if (ms > 0) push(KVG_PHASE_WARMUP, 0.0, ms);
    push(KVG_PHASE_MIDDLE, ms, me);
    if (me < mk) push(KVG_PHASE_COOLDOWN, me, mk);
  }
};

}  // namespace

KVO_API const char* kvo_last_error(void) { return t_err.c_str(); }

namespace {
template <typename CacheT>
int run_one(const kvg_sim_desc* d, kvg_sim_result* res, kvg_trace_row* trace,
                    size_t trace_cap, size_t* n_trace, kvg_agent_stats* agents,
                    size_t agents_cap, uint64_t* digests, size_t digest_cap,
                    size_t* n_digests, kvg_log_record* log, size_t log_cap,
                    size_t* n_log) {
  Sim<CacheT> sim;
  std::vector<std::uint64_t> dig;
  std::vector<kvg_log_record> lg;
  if (digests) sim.digests = &dig;
  if (log) sim.log = &lg;
  int status;
  try {
    sim.init(d);
    status = sim.run();
  } catch (const std::exception& e) {
    t_err = e.what();
    return KVG_ERR_STATE;
  }
  sim.fill(res, status);
  if (n_trace) *n_trace = sim.trace.size();
  if (trace)
    std::memcpy(trace, sim.trace.data(),
                std::min(trace_cap, sim.trace.size()) * sizeof(kvg_trace_row));
  if (agents)
    for (std::size_t i = 0; i < sim.n && i < agents_cap; ++i) agents[i] = sim.ag[i].st;
  if (n_digests) *n_digests = dig.size();
  if (digests)
    std::memcpy(digests, dig.data(), std::min(digest_cap, dig.size()) * sizeof(std::uint64_t));
  if (n_log) *n_log = lg.size();
  if (log)
    std::memcpy(log, lg.data(), std::min(log_cap, lg.size()) * sizeof(kvg_log_record));
  return status;
}
}  // namespace

/* Runs one simulation on the CPU. Buffers may be NULL; counts are always
 * reported so a caller can size and retry. Discard mode uses the flat page
 * table, offload mode the node-level tree (see TreeCache). */
KVO_API int kvo_run(const kvg_sim_desc* d, kvg_sim_result* res, kvg_trace_row* trace,
                    size_t trace_cap, size_t* n_trace, kvg_agent_stats* agents,
                    size_t agents_cap, uint64_t* digests, size_t digest_cap,
                    size_t* n_digests, kvg_log_record* log, size_t log_cap,
                    size_t* n_log) {
  if (d->engine.eviction == KVG_EVICT_OFFLOAD)
    return run_one<TreeCache>(d, res, trace, trace_cap, n_trace, agents, agents_cap, digests,
                              digest_cap, n_digests, log, log_cap, n_log);
  return run_one<FlatCache>(d, res, trace, trace_cap, n_trace, agents, agents_cap, digests,
                            digest_cap, n_digests, log, log_cap, n_log);
}

/* ----------------------- cache-level differential surface ------------------- */

/* Cache handle: the flat page table (discard) or the node-level tree
 * (offload; or discard when `eviction` has bit 8 set, to cross-check the two
 * restatements against each other). */
struct AnyCache {
  FlatCache* f = nullptr;
  TreeCache* t = nullptr;
  ~AnyCache() {
    delete f;
    delete t;
  }
};

KVO_API void* kvo_cache_new(uint64_t capacity, uint64_t page_size, uint32_t eviction,
                            uint64_t prompt_tokens, uint32_t shared) {
  try {
    auto* c = new AnyCache();
    const bool off = (eviction & 0xff) == KVG_EVICT_OFFLOAD;
    if (off || (eviction & 0x100)) {
      c->t = new TreeCache();
      c->t->init(capacity, page_size, prompt_tokens, shared != 0, off);
    } else {
      c->f = new FlatCache();
      c->f->init(capacity, page_size, prompt_tokens, shared != 0, false);
    }
    return c;
  } catch (const std::exception& e) {
    t_err = e.what();
    return nullptr;
  }
}

KVO_API void kvo_cache_free(void* h) { delete static_cast<AnyCache*>(h); }

namespace {
template <typename CacheT>
int cache_op(CacheT* c, const kvg_cache_op* op, kvg_cache_op_result* r, kvg_victim* victims,
             size_t cap, size_t* n_victims) {
  std::vector<std::pair<std::uint64_t, std::uint64_t>> v;
  c->victims = &v;
  std::memset(r, 0, sizeof *r);
  int rc = KVG_OK;
  try {
    switch (op->kind) {
      case KVG_OP_MATCH: r->r0 = c->match(op->agent, op->len, &r->r1); break;
      case KVG_OP_INSERT: {
        std::uint64_t ins = 0;
        r->r0 = c->insert(op->agent, op->len, &ins, nullptr) ? 1 : 0;
        r->r1 = ins;
        break;
      }
      case KVG_OP_RELOAD: {
        std::uint64_t offl = 0;
        r->r0 = c->reload(op->agent, op->len, op->arg, op->arg2, &offl);
        r->r1 = offl;
        break;
      }
      case KVG_OP_EVICT: r->r0 = c->evict(op->arg); break;
      case KVG_OP_PIN: c->pin(op->agent, op->arg, +1); break;
      case KVG_OP_UNPIN: c->pin(op->agent, op->arg, -1); break;
      case KVG_OP_DISCARD: c->discard_suffix(op->agent, op->len, op->arg); break;
      default: throw std::invalid_argument("unknown op");
    }
  } catch (const std::exception& e) {
    t_err = e.what();
    rc = KVG_ERR_STATE;
  }
  c->victims = nullptr;
  r->status = rc;
  r->clock = c->clock;
  r->used = c->used;
  if (n_victims) *n_victims = v.size();
  for (std::size_t i = 0; i < v.size() && i < cap && victims; ++i)
    victims[i] = kvg_victim{v[i].first, v[i].second};
  return rc;
}
}  // namespace

KVO_API int kvo_cache_op(void* h, const kvg_cache_op* op, kvg_cache_op_result* r,
                         kvg_victim* victims, size_t cap, size_t* n_victims) {
  AnyCache* c = static_cast<AnyCache*>(h);
  return c->t ? cache_op(c->t, op, r, victims, cap, n_victims)
              : cache_op(c->f, op, r, victims, cap, n_victims);
}

KVO_API void kvo_cache_stats(void* h, double* m, double* r, uint64_t* discarded) {
  AnyCache* c = static_cast<AnyCache*>(h);
  if (m) *m = c->t ? c->t->hit_m : c->f->hit_m;
  if (r) *r = c->t ? c->t->hit_r : c->f->hit_r;
  if (discarded) *discarded = c->t ? c->t->discarded : c->f->discarded;
}

KVO_API uint64_t kvo_cache_digest(void* h) {
  AnyCache* c = static_cast<AnyCache*>(h);
  return c->t ? c->t->digest() : c->f->digest();
}
