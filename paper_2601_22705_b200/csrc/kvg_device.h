// Device-side data layout of the B200 engine (shared by engine.cu and capi.cu).
//
// One simulation = one CTA (NW warps). Everything a simulation owns lives in
// one HBM workspace carved by the host (capi.cu: plan_workspace):
//
//   table / alt   paged prefix cache: open-addressing hash of 32-page CHUNKS.
//                 A bucket is 32 x 16 B slots = 512 B; lane l of a warp owns
//                 slot l, so one bucket is one fully coalesced 128-bit-per-lane
//                 probe. Slot = {u64 key = owner<<32 | page, u64 meta}.
//   occ           dense list of claimed bucket indices (eviction scans this,
//                 not the whole table).
//   agents        AgentDev records (hot agent state + its single pending event).
//   pend / paus   controller FIFO rings; active set is a linked list in AgentDev.
//   ready/batch   dispatch scratch.
//   trace / log   outputs (trace rows per control tick; optional event log).
#pragma once
#include <stdint.h>

#include "../../include/kvgpu.h"

namespace kvg {

typedef unsigned long long u64;
typedef unsigned int u32;

constexpr int kChunk = 32;                   // pages per bucket
constexpr u64 kEmptyKey = ~0ull;             // unclaimed bucket marker
constexpr u64 kResident = 1ull << 63;        // meta: page is device resident
constexpr int kPinShift = 40;                // meta: pins in bits 40..61
constexpr u64 kPinMask = (1ull << 22) - 1;
constexpr u64 kStampMask = (1ull << 40) - 1; // meta: stamp in bits 0..39

struct Slot {
  u64 key;
  u64 meta;
};

// Dense 32 B summary of one claimed bucket, kept parallel to the table and
// rewritten by whichever warp last modified the bucket. The eviction select
// reads summaries (one lane per bucket) instead of whole 512 B buckets: in
// the engine every resident page of a chunk carries the same stamp (an
// agent's path is always refreshed as a whole prefix), so a bucket's
// candidates are (dev mask, one stamp). Buckets that break that shape
// (explicit pins, mixed stamps) are flagged kMixed and handled per page.
struct Summ {
  u64 tag;   // owner << 32 | first page of the chunk
  u64 sf;    // bits 0..39: stamp of every resident page; kMixed
  u32 dev;   // device-resident slots (bit l = slot l)
  u32 host;  // host-tier slots (offload)
  u32 bnd;   // node-start slots (offload: reload chunk boundaries)
  u32 pad;
};
constexpr u64 kMixed = 1ull << 63;
static_assert(sizeof(Summ) == 32, "Summ must stay 32 B");

enum AgentState : uint8_t { S_PENDING, S_AWAIT, S_GEN, S_TOOL, S_PAUSED, S_DONE };
enum EventKind : uint8_t { EV_NONE = 0, EV_GEN = 1, EV_TOOL = 2, EV_XFER = 3 };

struct AgentDev {     // 64 B: two agents per 128 B line
  u32 ctx;            // context length in tokens (< 2^32: checked at batch create)
  u32 high_water;
  u64 lazy;           // discard mode: stamp of this agent's latest path refresh
                      // (match or insert); every resident page of its private
                      // chain carries it
  double ready_since;
  double f_tool;      // InFlight (engine.cpp:71-77)
  u32 pinned_pg;      // pinned_len / page_size: pages [0, pinned_pg) of this
                      // agent's path carry its pin (implicit per-page pins)
  u32 f_gen, f_rec, f_obs;
  u32 act_seq;        // admission order: active_ is insertion ordered
                      // (controller.hpp:122); larger = newer
  u32 priv;           // discard mode: resident private pages [S, S+priv) of its path
  uint16_t step;
  uint8_t state, ev_kind, f_has_tool, in_active;
  uint8_t ready;      // mirror of this agent's bit in the ready bitmap
  uint8_t stalled;    // last dispatch attempt stalled
};
static_assert(sizeof(AgentDev) == 64, "AgentDev must stay 64 B");

// Offload mode (EvictionMode::kOffload) keeps the reference's radix tree at
// NODE granularity: reload promotes host nodes one node-chunk at a time and
// the reference's children_with_device bookkeeping (including its quirk-Q1
// over-count) decides which nodes can ever become eviction frontiers, so a
// per-page model cannot reproduce it. One 64 B record per
// node in a per-simulation pool; a node is found by the key of its first
// page through an open-addressing head-key hash.
struct TNodeDev {
  u64 last_access, ordinal;
  u32 parent, first_child, next_sib, prev_sib;  // 0 = none (node 0 is the root)
  u32 start, npages;   // first page index, segment length in pages
  u32 tail;            // owner (agent+1) of pages at or past the shared prompt
  u32 device_slots;
  int pin_count, cwd;  // cwd = children_with_device
  u32 host, alive;
};
static_assert(sizeof(TNodeDev) == 64, "TNodeDev must stay 64 B");

// Mirror of the node fields the path walks read (find_child / common_len /
// host): one 16 B record per node, so a walk level is one 128-bit load that
// also yields the next level's first child. The low node ids (the pool reuses
// freed ids first) live in shared memory together with a pin-count mirror;
// higher ids use this HBM array (and TNodeDev.pin_count). TNodeDev stays
// authoritative; every write of a mirrored field writes both (tree.cuh).
struct TWalk {
  u32 first_child, start, npages;
  u32 tailh;  // tail | host << 31
};
static_assert(sizeof(TWalk) == 16, "TWalk must stay 16 B");
// Shared-memory twin of the frontier fields (node ids below the mirror bound):
// the eviction sweep decides frontier membership from shared memory alone.
struct TMeta {
  u32 device_slots;
  int pin_count, cwd;
  u32 alive;
};
static_assert(sizeof(TMeta) == 16, "TMeta must stay 16 B");
constexpr unsigned kTWalkSmemBytes = sizeof(TWalk) + sizeof(TMeta);

struct FrEnt {  // eviction frontier heap entry: (last_access, ordinal) order
  u64 la, ord;
  u32 id, pad;
};
constexpr u64 kTombKey = ~0ull - 1;  // head-hash tombstone

// Event heap entry: (time, ordinal) lexicographic; key = ordinal << 20 | agent.
struct HeapEnt {
  double t;
  u64 k;
};
constexpr int kAgentBits = 20;  // <= 1,048,575 agents per simulation
// key = ordinal << kKeyShift | group flag | (agent id, or member count of a
// completion group: its members wait at the group ring's head, FIFO)
constexpr int kKeyShift = kAgentBits + 1;
constexpr u64 kGroupFlag = 1ull << kAgentBits;

struct Member {       // one dispatched batch member (engine.cpp:293-299)
  u32 id, pad;
  double t, f, r, d;
};

// Per-simulation device descriptor (inputs, workspace pointers, outputs).
struct SimDev {
  // ---- inputs
  const kvg_step_plan* plans;
  u32 n_agents, n_steps;
  u64 prompt_tokens;
  u64 shared_len;     // Population::shared_prompt_tokens
  u64 shared_pages;   // pages wholly inside a shared prompt (owner 0)
  u64 workload_hash;
  kvg_policy policy;
  kvg_cost_params cost;
  kvg_engine_params engine;
  // ---- workspace
  Slot* table;
  Slot* alt;
  u32* occ;
  u32* alt_occ;
  Summ* summ;
  Summ* alt_summ;
  u32 bucket_mask;    // buckets - 1 (power of two)
  u32 verify;         // 1: re-derive every match by a block-hash probe and check it
  AgentDev* agents;
  u32* pend;
  u32* paus;
  unsigned long long* pack_cursor;  // pack_mode: batch-wide cursor of the dense row region
  Member* batch;
  HeapEnt* heap;      // agent events (leader-only binary heap)
  u32* rbits;         // ready bitmap: in_active && AwaitingAdmission
  u32* rl1;           // second level: non-empty words of rbits
  u32* lru;           // [2 * n_agents] chain LRU links {prev, next} (leader.cuh)
  u32* gring;         // [n_agents] completion-group member ring (FIFO of batches)
  u32 group_min;      // dispatch batches of >= group_min members complete as a group
  u32 storm_on;       // stall runs advance on the warp (coop_storm); 0: per member
  u32* pin_hist;      // [shared_pages+1]: agents per shared-pin depth
  u32* pin_lvl;       // bitmap of non-empty pin_hist levels
  u32* hist;          // [2 * 512]: eviction radix-select histogram scratch
  // ---- offload-mode tree (unused, 1-element regions, in discard mode)
  TNodeDev* tnodes;   // [tcap] node pool, node 0 = root
  TWalk* twalk;       // [tcap] walk mirror for ids past the shared-memory part
  u32* tfree;         // [tcap] free-node stack
  u32* tstack;        // [tcap] DFS stack (subtree walks)
  FrEnt* fr;          // [tcap] frontier heap
  u64* hkeys;         // [hmask+1] head-key hash: page key of a node's first page
  u32* hvals;         //           -> node id
  double* xring;      // [xcap] link transfer end times (FIFO: ends never decrease)
  u32 tcap, hmask, xcap;
  u32 pack_mode;      // 1: at its end the simulation copies its rows densely to trace_out
                      // at a base taken from *pack_cursor (counts[3]); no streaming
  // ---- outputs
  kvg_agent_stats* stats;
  kvg_trace_row* trace;
  u64 trace_cap;
  kvg_log_record* log;
  u64 log_cap;
  kvg_sim_result* result;
  u64* counts;        // [0] = trace rows produced, [1] = log records produced, [2] = error
  // host delivery (host_outputs): the simulation streams its trace rows into
  // its slice of a mapped pinned host array while it runs (in chunks after
  // control-tick rounds, the rest at its end), so the PCIe transfer overlaps
  // the run instead of following it (nullptr: rows stay in HBM). With
  // pack_mode it is the batch's dense device row region instead.
  kvg_trace_row* trace_out;
};

// Cache-op (CacheTree seam) executor descriptor.
struct CacheDev {
  u64 capacity, page_size, shared_pages;
  Slot* table;
  Slot* alt;
  u32* occ;
  u32* alt_occ;
  Summ* summ;
  Summ* alt_summ;
  u32 bucket_mask;
  u32 n_ops;
  const kvg_cache_op* ops;
  kvg_cache_op_result* results;
  kvg_victim* victims;  // appended per op (unordered within an op; host sorts)
  u64 victim_cap;
  u64* state;           // persistent scalars across exec calls (see CacheState)
  u32* hist;            // [2 * 512] eviction histogram scratch
};

// Persistent cache scalars for the cache-op executor.
struct CacheState {
  u64 used, clock, pinned_pages, occ_n, discarded, n_victims;
  double hit_m, hit_r;
  u64 swapped;  // table/alt swapped by a rebuild (parity of rebuilds)
};

// Grid-wide seam kernels (grid.cuh): launch arguments.
#ifndef KVG_GRID_ITEM_CHUNKS
#define KVG_GRID_ITEM_CHUNKS 8
#endif
constexpr int kGridItemChunks = KVG_GRID_ITEM_CHUNKS;  // private chunks per match work item (8: 4 KB of slots)
constexpr int kGridSumDepth = 8;    // bucket summaries in flight per lane (grid evict)

struct GridMatchArgs {
  Slot* table;
  Summ* summ;
  u32 mask;
  u32 n;             // queries
  u64 S;             // shared-prompt pages (owner 0)
  u64 ps;            // page size, tokens
  u64 clock0;        // cache clock before the batch
  const u32* agents; // [n]
  const u64* lens;   // [n] sequence lengths, tokens
  u32 max_groups;    // most private chunk groups of any query
  u32 pad;
  ulonglong2* items; // continuation work items {query << 32 | group, pages}: the groups
                     // past the first of queries whose first group was fully resident
  unsigned int* n_items;
  u32* fm;           // [n] first missing private page (NIL32 = none), atomicMin
  u32* res;          // [n] resident private pages, atomicAdd
  u32* smask;        // [S/32 + 1] resident pages of each shared chunk
  u32* best;         // [S] shared winners: max(i+1) of queries whose shared range ends at page p+1
};

constexpr int kGridDigit = 11;
constexpr u32 kGridBins = 1u << kGridDigit;

struct GridEvictArgs {
  Slot* table;
  Summ* summ;
  u32* occ;
  u32 occ_n, mask;
  u64 S;
  u64 k, evictable, clock;
  kvg_victim* vic;
  u64 vic_cap;
  unsigned long long* vic_n;
  u32* ghist;           // [3][2][kGridBins], zeroed by the host
  unsigned int* freed;  // pages freed (zeroed by the host)
  int* err;
};

}  // namespace kvg
