/* Per-event state digest shared by the reference harness (ref_harness.cpp)
 * and the oracle restatement (kvoracle.cpp). TEST INFRASTRUCTURE ONLY.
 *
 * After every processed event the reference engine, in paranoid mode, calls
 * CacheTree::check_invariants() then Controller::check_invariants()
 * (/root/reference/proj/src/engine.cpp:128-131). The harness intercepts both
 * calls and folds the complete cache + controller state into one 64-bit
 * digest; the oracle computes the same fold from its own flat page table.
 * Equal digest sequences mean equal state after every single event. */
#ifndef KVG_ORACLE_DIGEST_H_
#define KVG_ORACLE_DIGEST_H_

#include <cstdint>
#include <cstring>

namespace kvdigest {

inline std::uint64_t mix(std::uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

inline std::uint64_t dbits(double d) {
  std::uint64_t b;
  std::memcpy(&b, &d, sizeof b);
  return b;
}

/* One resident (or host-tier) page: order-independent contribution. */
inline std::uint64_t page_term(std::uint64_t owner, std::uint64_t page,
                               std::uint64_t stamp, std::uint64_t pins,
                               std::uint64_t host) {
  std::uint64_t h = mix(owner * 0x9e3779b97f4a7c15ULL + page);
  h = mix(h ^ (stamp * 0x632be59bd9b4e019ULL));
  h = mix(h ^ (pins << 1) ^ host);
  return h;
}

/* Ordered fold for sequences (controller lists, scalars). */
inline std::uint64_t fold(std::uint64_t h, std::uint64_t v) {
  return mix(h ^ (v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2)));
}

}  // namespace kvdigest

#endif
