// ws_aref.cuh — the device-side asynchronous reference (aref).
//
// An aref is a depth-D ring of shared-memory slots, each guarded by a pair of mbarriers
// (full[s], empty[s]). It is the hardware realisation of the reference's channel:
//   ArefSlot / ArefChannel      ref proj/include/warpspec/aref.hpp:16-104
//   slot = k mod D               ref aref.hpp:72-75, expand.hpp:91-92
//   parity p = floor(k / D) mod 2  ref expand.hpp:84-97
//   put      = wait(empty_s, p); expect_tx(full_s, sum of member bytes); TMA x members
//   get      = wait(full_s, p)
//   consumed = arrive(empty_s)          (ref proj/include/warpspec/lower.hpp:210-283)
// Barrier rule (ref proj/include/warpspec/sim.hpp:284-302): a wait on parity p passes once the
// phase with that parity has completed; a phase completes when arrivals reach the init count
// AND the transaction bytes reach the expected count.
//
// The reference primes every empty barrier with one completed phase (sim.hpp:86-92). A fresh
// hardware mbarrier sits in phase 0, so the producer waits on parity (p ^ 1) instead: the first
// lap passes immediately and later laps wait for the consumer's release, which is the same
// credit sequence.
//
// On the MMA side `consumed` is not a thread arrive: tcgen05.commit arrives on empty[s] when the
// tensor core has finished reading the slot, so the release happens exactly when the operands
// are dead (the fine-grained pipeline with P = D, ref proj/include/warpspec/pipeline.hpp:44-142).
#pragma once

#include "ws_ptx.cuh"

namespace ws {

static __device__ WatchdogRecord ws_watchdog_record;
// host-mapped copy (pinned, zero-copy; set by the host launcher): readable after the trap has
// torn down the context, which is how ws_watchdog() reports the Deadlock verdict
static __device__ WatchdogRecord* ws_watchdog_host;
// suspend-time hint (ns) for blocked waits; 0 = the hardware default (set by the host launcher)
static __constant__ uint32_t ws_wait_hint_ns;  // constant bank: a cached LDC, not an L2 round trip per wait

// The watchdog's report, out of line and noreturn: no caller state survives a trap, so the call
// costs the wait sites nothing (an inline version that could fall back into the wait loop slowed
// the hdim-128 attention kernel by 14%). The first waiter to time out (elected in device memory)
// records where it waited — in the device record and in the host-mapped copy, which survives the
// trap — and the others hold their trap until it has (a trap ends every thread of the grid).
[[noreturn]] static __device__ __noinline__ void ws_watchdog_fire(uint32_t bar, uint32_t parity, uint32_t tag) {
  if (atomicCAS(&ws_watchdog_record.fired, 0u, 1u) == 0u) {
    const unsigned long long blk = blockIdx.x | (static_cast<unsigned long long>(blockIdx.y) << 32);
    ws_watchdog_record.block = blk;
    ws_watchdog_record.thread = threadIdx.x;
    ws_watchdog_record.bar_smem = bar;
    ws_watchdog_record.parity = parity;
    ws_watchdog_record.tag = tag;
    volatile WatchdogRecord* v = *reinterpret_cast<WatchdogRecord* volatile*>(&ws_watchdog_host);
    if (v != nullptr) {
      v->block = blk;
      v->thread = threadIdx.x;
      v->bar_smem = bar;
      v->parity = parity;
      v->tag = tag;
      __threadfence_system();
      v->fired = 1u;
    }
    __threadfence_system();
    atomicExch(&ws_watchdog_record.fired, 2u);
  } else {
    const uint64_t t1 = globaltimer();
    while (*reinterpret_cast<volatile unsigned int*>(&ws_watchdog_record.fired) != 2u &&
           globaltimer() - t1 < 100000000ull) {
    }
  }
  __threadfence_system();
  asm volatile("trap;");
  __builtin_unreachable();
}

static __device__ __forceinline__ void mbar_wait_slow(uint32_t bar, uint32_t parity, uint32_t tag) {
  uint64_t t0 = globaltimer();
  uint32_t spins = 0;
  // written only by the host (cudaMemcpyToSymbol) before the launch; a constant-bank read (the
  // volatile global load it replaces cost every slow-path wait an L2 round trip)
  const uint32_t hint = ws_wait_hint_ns;
  while (!(hint ? mbar_try_wait_hint(bar, parity, hint) : mbar_try_wait(bar, parity))) {
    if (((++spins) & 1023u) == 0 && globaltimer() - t0 > WS_WATCHDOG_NS) ws_watchdog_fire(bar, parity, tag);
  }
}

// Iteration cursor over a depth-D ring: slot = k mod D, phase = floor(k / D) mod 2.
struct ArefCursor {
  uint32_t slot = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void advance(uint32_t depth) {
    if (++slot == depth) {
      slot = 0;
      phase ^= 1u;
    }
  }
};

// The barrier pairs of one aref; the payload slots are carved separately so that each kernel
// can lay its tiles out with the alignment the swizzle needs.
template <int MAXD>
struct ArefBarriers {
  uint64_t full[MAXD];
  uint64_t empty[MAXD];

  // full: one arrival (the producer's expect_tx) + transaction bytes.
  // empty: `consumers` arrivals (1 for a tcgen05.commit release).
  __device__ __forceinline__ void init(uint32_t depth, uint32_t producers, uint32_t consumers) {
    for (uint32_t i = 0; i < depth; ++i) {
      mbar_init(&full[i], producers);
      mbar_init(&empty[i], consumers);
    }
  }

  // producer side of put: acquire the slot's empty credit
  __device__ __forceinline__ void put_acquire(const ArefCursor& c, uint32_t tag = 1) {
    mbar_wait(&empty[c.slot], c.phase ^ 1u, tag);
  }
  // producer side of put: announce the tuple bytes the TMA members will deliver
  __device__ __forceinline__ void put_expect(const ArefCursor& c, uint32_t bytes) {
    mbar_arrive_expect_tx(&full[c.slot], bytes);
  }
  // consumer get
  __device__ __forceinline__ void get(const ArefCursor& c, uint32_t tag = 2) {
    mbar_wait(&full[c.slot], c.phase, tag);
  }
  // thread-side consumed (softmax / epilogue consumers)
  __device__ __forceinline__ void consumed(const ArefCursor& c) { mbar_arrive(&empty[c.slot]); }
  // tensor-core-side consumed: released when all previously issued MMAs finish reading
  __device__ __forceinline__ void consumed_by_mma(const ArefCursor& c) { mma_commit(&empty[c.slot]); }
};

}  // namespace ws
