// lk_internal.h -- structures shared by the host runtime (lk_host.cu) and the
// sm_100a kernels (lk_kernels.cu).  Not part of the public ABI.
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>
#include "../../include/lk.h"

// One device trace record (16 B): a value-changing from_gpu write.
struct lk_dev_trace {
  uint32_t word;
  uint32_t hseq;   // host write index (per worker) last observed by the worker
  uint64_t t_ns;   // %globaltimer
};

// Kernel arguments of the persistent kernel.  Mailbox cells live in pinned
// mapped host memory (to_gpu, status, hseq, err, smid); everything else is
// device-resident.
struct lk_dev_args {
  const unsigned long long* to_gpu;  // host-mapped; worker i replica k at to_gpu[(i*replicas + k)*cell_u64]:
                                     // word | seq<<32 (seq = host write index, monotone per worker)
  unsigned long long* status;      // host-mapped, cell i at status[i*status_u64]: word | phase<<32
  unsigned long long* err;         // host-mapped, err[i] = code | word<<32
  uint32_t* err_any;               // host-mapped, set to 1 after any err[i] is written
  uint32_t* smid;                  // host-mapped, smid[i]
  const lk_desc* desc;             // device, num_slots entries
  const unsigned long long* slot_mask;  // device, num_slots * nwords
  uint32_t* reduce_ctr;            // device, num_slots
  unsigned long long* spans;       // device, LK_TIMELINE_WORDS per worker: the last dispatch's
                                   // timeline (lk_last_timeline)
  const unsigned long long* ring;  // host-mapped event ring (GATEWAY): replica k, entry e at
                                   // ring[(k*ring_entries + e)*8], 8 u64 per entry
  unsigned long long* gw_tail;     // host-mapped: events the gateway has consumed
  unsigned long long* dmb;         // device mailboxes (GATEWAY), worker i at dmb[i*dmb_u64]
  uint32_t* exited;                // device: workers that left their loop
  uint32_t* sink;                  // device (own line): busy_loop results of the fast path land here
  uint32_t ring_entries;           // entries per event-ring replica
  uint32_t dmb_u64;
  uint32_t nw;                     // workers
  uint32_t wthreads;               // worker threads per CTA (the gateway warp comes after)
  uint32_t poll_mode;              // LK_POLL_*
  uint32_t use_tma;                // payload tiles through the TMA bulk ring in dynamic smem
  uint32_t ring_stages;            // TMA ring depth (16-KiB stages)
  uint32_t ack_delay_cyc;          // DIRECT, 1 replica: SM cycles between FINISHED and the first ack poll
  uint32_t idle_delay_cyc;         // ... and between the handshake's closing NOP and the next poll
  uint32_t tma_min_workers;        // payload dispatches to fewer workers take the LSU path
  lk_dev_trace* trace;             // device, num_workers * trace_cap
  uint32_t* trace_cnt;             // device, num_workers
  uint32_t* fast_cnt;              // device, num_workers: values settled by the kernel's fast path
  uint32_t cell_u64;               // to_gpu cell stride in u64 (DIRECT cells and replicas)
  uint32_t status_u64;             // from_gpu status cell stride in u64
  uint32_t replicas;               // to_gpu replicas per worker: 1, 2, 4 or 8
  uint32_t spacing_ns;             // stagger between replica loads
  uint32_t num_slots;
  uint32_t nwords;
  uint32_t trace_cap;
  uint32_t record_trace;
  uint32_t backoff_ns;
  uint32_t flags;                  // LK_CF_*
  uint32_t red_share8;             // block_reduce: static share of a fair share, in eighths (8: static only)
  uint32_t red_claim;              // block_reduce: blocks per pool claim
};

// Launch wrappers (lk_kernels.cu).
cudaError_t lk_launch_persistent(const lk_dev_args& a, uint32_t grid, uint32_t threads,
                                 size_t smem, cudaStream_t st);
cudaError_t lk_persistent_configure(size_t smem);
cudaError_t lk_preload_kernels();
cudaError_t lk_launch_clocksync(const uint32_t* flag, unsigned long long* echo, uint32_t rounds,
                                cudaStream_t st);
#define LK_TIMELINE_WORDS 16
cudaError_t lk_launch_topo(uint32_t* smids, uint32_t grid, uint32_t cluster, size_t smem, cudaStream_t st);
cudaError_t lk_persistent_occupancy(uint32_t threads, size_t smem, int* blocks_per_sm);
cudaError_t lk_launch_work(const lk_desc& d, uint32_t grid, uint32_t threads,
                           uint32_t* reduce_ctr, cudaStream_t st, int use_tma);
size_t lk_ring_bytes(uint32_t stages);
cudaError_t lk_launch_empty(cudaStream_t st);
uint32_t lk_ring_max_stages();
cudaError_t lk_launch_pingpong(volatile uint32_t* flag, volatile uint32_t* echo,
                               uint64_t rounds, cudaStream_t st);
