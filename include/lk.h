/*
 * lk.h -- C ABI of the B200 LightKernel (LK) persistent-worker runtime.
 *
 * This is the drop-in boundary for the reference's `native` executor
 * (persistkern.native.NativeSession, /root/reference/pkg/src/persistkern/native.py).
 * Every entry point is extern "C", never throws, takes plain pointers and
 * sizes, and returns an int status (LK_OK or a negative LK_E_* code).
 * Worker = one CTA of one persistent sm_100a kernel, pinned to its own SM.
 *
 * Each function names the reference interface it replaces (file:line, paths
 * relative to /root/reference/pkg/src/persistkern/).
 */
#ifndef LK_H_
#define LK_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: 1:1 with persistkern.errors (errors.py:5-59) ---------- */
#define LK_OK               0
#define LK_E_USAGE         -1  /* UsageError            errors.py:58-59 */
#define LK_E_BUSY          -2  /* BusyTriggerError      errors.py:31-32 */
#define LK_E_DISPOSE_BUSY  -3  /* DisposeWhileBusyError errors.py:35-36 */
#define LK_E_HANG          -4  /* HangDetected          errors.py:43-55 */
#define LK_E_INIT          -5  /* InitError             errors.py:39-40 */
#define LK_E_WORKER_DIED   -6  /* UsageError("worker i died") native.py:128-131 */
#define LK_E_CUDA          -7  /* CUDA runtime failure (no reference analogue) */
#define LK_E_CONFIG        -8  /* ConfigError           errors.py:23-24 */
#define LK_E_PROTOCOL      -9  /* ProtocolViolation     errors.py:9-20 */
#define LK_E_TRACE_LOST   -10  /* device trace ring overflowed */

/* ---- wire words: protocol.py:31-45 ---------------------------------------- */
#define LK_INIT       0u
#define LK_FINISHED   1u
#define LK_WORKING    2u
#define LK_NOP        4u
#define LK_EXIT       8u
#define LK_WORK_BASE 16u

/* ---- worker phases: protocol.py:104-109 ----------------------------------- */
#define LK_PHASE_BOOTING   0u
#define LK_PHASE_IDLE      1u
#define LK_PHASE_WORKING   2u
#define LK_PHASE_FINISHED  3u   /* FINISHED_PENDING_ACK */
#define LK_PHASE_EXITED    4u

/* ---- device-side error codes (lk_worker_error) ---------------------------- */
#define LK_WERR_NONE          0u
#define LK_WERR_ILLEGAL_WORD  1u  /* decode_to_gpu rejects: protocol.py:83-91 */
#define LK_WERR_BUSY_SLOT     2u  /* other slot while WORKING: protocol.py:182-186 */
#define LK_WERR_UNACKED_SLOT  3u  /* other slot while awaiting ack: protocol.py:192-197 */
#define LK_WERR_AFTER_EXIT    4u  /* stepped after exit: protocol.py:163-164 */
#define LK_WERR_BAD_SLOT      5u  /* slot outside the device descriptor table */
#define LK_WERR_BAD_KIND      6u  /* UnsupportedWorkloadError analogue (device.py:114-118) */
#define LK_WERR_BAD_COMPLETE  7u  /* completion outside WORKING: protocol.py:203-204 */

/* ---- work kinds (device.py:16 has only "busy_loop") ------------------------ */
#define LK_KIND_EMPTY             0u  /* iterations ignored: the 0-iteration task */
#define LK_KIND_BUSY_LOOP         1u  /* native.py:63-67 */
#define LK_KIND_VECTOR_ADD_I32    2u  /* out[i] = in0[i] + in1[i] mod 2^32 */
#define LK_KIND_SAXPY_F32         3u  /* out[i] = fl(fl(alpha*in0[i]) + in1[i]) */
#define LK_KIND_BLOCK_REDUCE_F32  4u  /* ((double*)out)[b] = fp64 sum of 4096-element block b (ceil(n/4096)
                                          entries); *(double*)aux = their fp64 combine.  Fixed order of
                                          operations (oracle/work.py): the same bits for any mask/schedule */
#define LK_KIND_HBM_STREAM        5u  /* out[i] = in0[i], `iterations` passes (>=1) */
#define LK_KIND_COUNT             6u

/* to_gpu hint bits (top byte of a cell; set by the host from the staged
 * descriptor of the slot a WORK word names) */
#define LK_HINT_EMPTY  1u   /* the slot holds no work (EMPTY, or busy_loop of 0 iterations): no descriptor fetch */
#define LK_HINT_CACHED 2u   /* every masked worker last fetched this slot at its current stage version:
                               reuse the cached descriptor (and trigger mask), no fetch */
#define LK_HINT_SYSMEM 4u   /* the slot's payload touches host-mapped memory: the worker makes the poll
                               that saw the value an acquire at system scope (fence.acq_rel.sys) */

/* descriptor flags */
#define LK_DF_SCALAR   1u   /* pointers not 16-B aligned: scalar path */
#define LK_DF_HOSTMEM  2u   /* set by the runtime at staging (cudaPointerGetAttributes), never by the
                               caller: a payload pointer is host-mapped pinned memory (lk_host_alloc,
                               cudaHostAlloc).  The worker reads it with sys-scope LSU loads (no TMA,
                               no stale L2 line) and publishes FINISHED with st.release.sys, so the
                               outputs are in host memory before the host can see FINISHED.
                               block_reduce_f32's partials (out) must be device memory. */

/*
 * Work descriptor, 64 B POD, device-resident per slot.
 * Replaces WorkDescriptor (device.py:48-66) + the `descriptors` dict
 * (native.py:91, written 223, read 180).  Multi-worker kinds shard [0, n)
 * over the workers of the trigger mask: worker of rank r (popcount of mask
 * bits below it) takes the r-th 128-B-aligned chunk.
 */
typedef struct lk_desc {
  uint32_t kind;
  uint32_t flags;
  uint64_t iterations;
  uint64_t n;          /* elements */
  uint64_t in0;        /* device pointers */
  uint64_t in1;
  uint64_t out;
  uint64_t aux;        /* BLOCK_REDUCE: double* total (0 = block partials only) */
  float    alpha;
  uint32_t reserved;
} lk_desc;

/* Session configuration; replaces NativeConfig (native.py:44-60). */
typedef struct lk_config {
  uint32_t num_workers;          /* 0 = one per SM (148 on B200) */
  uint32_t threads_per_worker;   /* 0 = 512 */
  int32_t  device;               /* CUDA ordinal */
  uint32_t spin_strategy;        /* 0 pure_spin, 1 spin_then_yield (native.py:40-41) */
  uint32_t spin_yield_threshold; /* host spins before sched_yield */
  uint32_t record_trace;         /* native.py:51 */
  uint32_t trace_capacity;       /* device records per worker; 0 = 65536 */
  uint32_t poll_backoff_ns;      /* device __nanosleep between idle polls (0 = none) */
  uint32_t cell_stride;          /* bytes between to_gpu cells: 8..128 (power of 2); 0 = 128 */
  uint32_t num_slots;            /* descriptor table entries; 0 = 1024 */
  uint64_t wait_timeout_ns;      /* wait_timeout_s (native.py:52) */
  uint32_t flags;                /* LK_CF_* */
  uint32_t poll_replicas;        /* 0 or 1 (one to_gpu cell / event ring; replicas were measured slower
                                    and removed) */
  uint32_t poll_spacing_ns;      /* unused since replicas were removed (kept for the ABI) */
  uint32_t poll_mode;            /* LK_POLL_DIRECT (0, default), LK_POLL_GATEWAY or LK_POLL_HYBRID */
  uint32_t status_stride;        /* bytes between from_gpu status cells: 16..128 (power of 2); 0 = 32 */
  uint32_t ring_stages;          /* TMA payload ring depth in 16-KiB stages, 2..12; 0 = 6 */
  uint32_t sm_partition;         /* 0: the persistent kernel spans the GPU.  N: it runs in a green
                                    context of >= N SMs (driver granularity: multiples of 8), one
                                    worker per partition SM; the remaining SMs form a second green
                                    context for ordinary kernels (lk_baseline_create_in) */
  uint32_t ack_delay_ns;         /* DIRECT, 1 replica: after publishing FINISHED a worker waits this
                                    long before it polls for the host's NOP ack.  A poll issued at
                                    once is ordered behind FINISHED on the link, reaches host memory
                                    before the host can have answered, and costs a wasted round
                                    trip.  The starting value: each worker adapts it to the host's
                                    answer time, within 1/4..4x (LK_CF_ACK_FIXED: no adaptation);
                                    0 = 300 (LK_CF_NO_ACK_DELAY: poll at once) */
  uint32_t idle_delay_ns;        /* the same after publishing the NOP that ends a handshake, for a
                                    host that re-triggers the same worker at once (~300 ns from a C
                                    loop, ~600 ns through Python).  The starting value: each worker
                                    grows it while its WORK keeps arriving one load late, and leaves
                                    it at 0 when other workers are triggered in between (round
                                    robin); LK_CF_ACK_FIXED keeps it fixed.  0 = start at none */
  uint32_t tma_min_workers;      /* payload dispatches to fewer workers use 128-bit LSU loads even
                                    with the TMA ring on: a lone SM streams ~30% faster that way,
                                    the whole GPU faster through the ring (tools/tma_vs_lsu_count.py);
                                    0 = 49, 1 = always the ring */
} lk_config;

/* How to_gpu words reach the workers.  DIRECT: every worker polls its own
 * host cell over PCIe (lowest single-worker latency).  GATEWAY: one warp
 * polls an event ring in host memory (one 64-B event per logical write,
 * carrying the worker mask) and forwards new values to per-worker mailboxes
 * in device memory: one host store per wide dispatch, one extra L2 hop per
 * worker. */
#define LK_POLL_DIRECT  0u
#define LK_POLL_GATEWAY 1u
/* HYBRID: writes to at most LK_HYBRID_DIRECT_MAX workers go to their direct
 * cells, wider ones (full-mask triggers, EXIT) as one ring event, and every
 * ack to the direct cells as each FINISHED is seen; each
 * CTA runs a host-cell poller warp and a mailbox poller warp that forward into
 * shared memory, where the protocol thread watches both. */
#define LK_POLL_HYBRID  2u
#define LK_HYBRID_DIRECT_MAX 8u

#define LK_CF_ACQUIRE_POLL   1u  /* (the default; kept for ABI compatibility) DIRECT polls of a to_gpu
                                    cell are ld.acquire.sys.  The gateway's ring and the mailboxes are
                                    polled relaxed (acquire loads there cost 1.2 us per wide dispatch);
                                    host-mapped payloads get explicit fences on that path */
#define LK_CF_RELAXED_POLL 2048u /* polls with ld.relaxed.sys / .gpu instead; a host-mapped payload
                                    (LK_HINT_SYSMEM) then costs a fence.acq_rel.sys (~1.5 us) */
#define LK_CF_FENCE_ALWAYS   2u  /* release fence before every FINISHED, even for no-write kinds */
#define LK_CF_LSU_PAYLOAD    4u  /* payload items with 128-bit LSU loads instead of the TMA bulk ring */
#define LK_CF_TIMELINE       8u  /* GATEWAY: stamp forward times into the device timeline (+1 L2 load per value) */
#define LK_CF_ACK_WINDOW    32u  /* removed (measured neutral): refused by lk_create */
#define LK_CF_DYNAMIC_TILES 64u  /* removed (measured neutral at 64 MiB, -11% at 16 MiB): refused */
#define LK_CF_NO_ACK_DELAY 128u  /* DIRECT, 1 replica: poll for the ack right after FINISHED
                                    (lk_config.ack_delay_ns) */
#define LK_CF_ACK_FIXED    256u  /* keep ack_delay_ns as configured (no per-worker adaptation) */
#define LK_CF_HOST_DESC    512u  /* DIRECT only: the descriptor table and slot masks live in the pinned
                                    mapped host block (workers fetch them with sys-scope loads after an
                                    acquire poll), so register/trigger/wait make no CUDA call at all: a
                                    session stays usable while a profiler that serialises launches (ncu)
                                    holds the runtime inside the persistent kernel's launch */
#define LK_CF_FULL_BOARD  1024u  /* DIRECT: every to_gpu write also re-stores every other worker's cell
                                    unchanged, shipping the whole mailbox board (the paper's workaround
                                    for deferred small transfers; measured, not needed) */
#define LK_CF_LAZY_ACK      16u  /* lk_wait returns once the NOP ack is written; the next trigger or
                                    dispose touching that worker waits for its republished NOP */

/* One linearized protocol write; replaces TraceRecord (protocol.py:253-261). */
typedef struct lk_trace_rec {
  uint64_t step;     /* global order, consistent with per-worker causality */
  uint32_t side;     /* 'H' or 'D' */
  uint32_t worker;
  uint32_t word;
  uint32_t hseq;     /* host write index this record follows (per worker) */
  uint64_t t_ns;     /* host: CLOCK_MONOTONIC; device: %globaltimer */
} lk_trace_rec;

typedef struct lk_session lk_session;
typedef struct lk_baseline lk_baseline;

/* ---- session lifecycle ---------------------------------------------------- */

/* NativeSession.start (native.py:104-122): context, pinned mapped mailboxes,
 * device descriptor table, cooperative launch of the persistent kernel, wait
 * until every worker published INIT then NOP.  *init_ns = wall time. */
int lk_create(const lk_config* cfg, lk_session** out, uint64_t* init_ns);

/* NativeSession.dispose (native.py:277-295): EXIT to every worker, wait for the
 * kernel to retire (timeout -> LK_E_HANG). */
int lk_dispose(lk_session* s, uint64_t* elapsed_ns);

/* Teardown ignoring the host rules (no reference analogue: the reference
 * leaves dead sessions' daemon threads behind): EXIT to every worker, wait up
 * to timeout_ns (0 = wait_timeout) for the kernel to retire. */
int lk_abort(lk_session* s, uint64_t timeout_ns);

/* Free host/device resources (after dispose, or to abandon a session). */
int lk_destroy(lk_session* s);

/* descriptors[slot] = work (native.py:223), staged device-resident ahead of
 * the WORK word.  mask (nwords u64, little-endian bit i = worker i) is the
 * worker set that will shard the payload.  Fails LK_E_USAGE while the slot is
 * referenced by an un-waited dispatch (native.py:215-217). */
int lk_register_desc(lk_session* s, uint32_t slot, const lk_desc* d,
                     const uint64_t* mask, uint32_t nwords);

/* NativeSession.trigger (native.py:208-231): validate (mask, busy workers,
 * slot lock, idle cells -- in the reference's order), stage `d` into the slot
 * when given and different from the staged copy (descriptors[slot] = work,
 * "in place before the word lands"; NULL = use the registered descriptor),
 * then write 16+slot to each masked worker in ascending order.
 * *elapsed_ns = staging + word writes. */
int lk_trigger(lk_session* s, const uint64_t* mask, uint32_t nwords,
               uint32_t slot, const lk_desc* d, uint64_t* elapsed_ns);

/* NativeSession.wait (native.py:250-275): spin until every masked worker
 * published FINISHED (*finished_ns = call start -> that observation), write
 * NOP acks ascending, spin until every masked worker republished NOP (with
 * LK_CF_LAZY_ACK that last spin moves to the next trigger of the worker). */
int lk_wait(lk_session* s, const uint64_t* mask, uint32_t nwords,
            uint64_t* finished_ns);

/* ---- introspection -------------------------------------------------------- */

/* to_gpu / from_gpu cells and worker_phase (native.py:88-94), n entries. */
int lk_read_cells(lk_session* s, uint32_t* to_gpu, uint32_t* from_gpu,
                  uint32_t* phase, uint32_t n);
/* worker_error (native.py:93, 196-199): device-side code + offending word. */
int lk_worker_error(lk_session* s, uint32_t worker, uint32_t* code, uint32_t* word);
/* %smid of each worker (check_block_mapping idea, device.py:102-111). */
int lk_smid_map(lk_session* s, uint32_t* smid, uint32_t n);
int lk_num_workers(lk_session* s, uint32_t* n);
/* pending_mask (native.py:95); mask out, nwords u64. */
int lk_pending(lk_session* s, uint64_t* mask, uint32_t nwords);
/* 1 while the persistent kernel is resident (Thread.is_alive analogue). */
int lk_kernel_alive(lk_session* s, uint32_t* alive);

/* Fault injection: store a raw word into worker's to_gpu cell, bypassing every
 * host rule (the reference tests inject illegal words into traces,
 * T/test_acceptance.py:168-176; this injects them into the live device). */
int lk_debug_poke(lk_session* s, uint32_t worker, uint32_t word);

/* ---- tracing (native.py:135-147, 297-299) ---------------------------------- */
/* Number of linearized records available (host + device). */
int lk_trace_count(lk_session* s, uint64_t* n);
/* Merge the host log and the per-worker device rings into one linearization
 * (per-worker causal order; cross-worker order by host time). */
int lk_trace_read(lk_session* s, lk_trace_rec* out, uint64_t cap, uint64_t* n);

/* ---- protocol: shared host/device state machine ---------------------------- */
/* worker_step (protocol.py:151-198) as compiled into the kernel, run on the
 * host: phase/slot in-out, publish = word or 0xFFFFFFFF (none), action =
 * 0 none, 1 begin work, 2 exit.  Returns LK_OK or LK_E_PROTOCOL (*werr set). */
int lk_protocol_step(uint32_t* phase, uint32_t* slot, uint32_t observed,
                     uint32_t* publish, uint32_t* action, uint32_t* werr);
/* complete_work (protocol.py:201-206). */
int lk_protocol_complete(uint32_t* phase, uint32_t* slot, uint32_t* publish,
                         uint32_t* werr);
/* replay_trace / validate_trace (protocol.py:372-398) over n writes given as
 * parallel arrays (side 'H'/'D').  *bad_index = -1 when valid; reason gets a
 * NUL-terminated message.  counts (optional, 3*max_workers u64: sm id, host
 * work writes, begins) mirror ReplayState.dispatch_counts (protocol.py:287-295). */
int lk_validate_trace(const uint32_t* side, const int64_t* sm_id, const uint32_t* word,
                      uint64_t n, int64_t* bad_index, char* reason, uint32_t reason_cap,
                      uint64_t* counts, uint32_t max_workers, uint32_t* n_workers);

/* ---- measurement ------------------------------------------------------------ */
/* Closed-loop trigger+wait rounds entirely in C (GIL-free).  Round k uses
 * masks[k % nmasks] (nwords u64 each) and `slot`.  Per round (arrays may be
 * NULL): trig_ns = trigger call, done_ns = trigger start -> last FINISHED
 * observed, cycle_ns = trigger start -> ack consumed. */
int lk_bench_roundtrip(lk_session* s, const uint64_t* masks, uint32_t nmasks,
                       uint32_t nwords, uint32_t slot, uint64_t rounds,
                       uint64_t* trig_ns, uint64_t* done_ns, uint64_t* cycle_ns);
/* The same loop, plus gap_ns[k] = the largest gap between consecutive TSC
 * reads of the calling thread within round k's spins: microseconds there
 * mean the host thread was not running (interrupt, tick, vCPU preemption),
 * which attributes a slow round to the host rather than the link or GPU. */
int lk_bench_roundtrip_gaps(lk_session* s, const uint64_t* masks, uint32_t nmasks,
                            uint32_t nwords, uint32_t slot, uint64_t rounds,
                            uint64_t* trig_ns, uint64_t* done_ns, uint64_t* cycle_ns,
                            uint64_t* gap_ns);
/* A profiling run of the persistent kernel itself: boots a DIRECT session
 * whose handshakes come from a host thread started before the kernel launch
 * and tears it down.  The thread runs `rounds` dispatches, then EXIT: with
 * ndesc == 0 round-robin empty tasks on single workers; else full-mask
 * dispatches of descs[r % ndesc] (staged in slots 1..ndesc before the
 * launch), each acked before the next.  Under a profiler that returns from
 * the launch only once the kernel has exited (ncu; use --replay-mode
 * application), this is a complete run rather than a deadlock.  The thread
 * makes no CUDA calls.  *elapsed_ns: the rounds' host wall time. */
int lk_profile_run(const lk_config* cfg, const lk_desc* descs, uint32_t ndesc, uint64_t rounds,
                   uint64_t* elapsed_ns);
/* Device-side spans of the last dispatch per worker (globaltimer ns):
 * begin (WORK observed) and end (work done, before FINISHED). */
int lk_last_spans(lk_session* s, uint64_t* begin_ns, uint64_t* end_ns, uint32_t n);
/* Device timeline of the last dispatch per worker, 16 words each (t[16*i+k]):
 * globaltimer ns at k=0 to_gpu value seen, 1 work begin, 2 work end,
 * 3 FINISHED issued, 4 gateway forward (LK_CF_TIMELINE, else 0); clock64 at
 * 5 value seen, 6 work begin, 7 FINISHED issued.  The ack phase of an empty
 * task on a DIRECT session with LK_CF_TIMELINE (else 0): 8 globaltimer at
 * FINISHED issued, 9 globaltimer when the NOP ack was seen, 10 cell loads
 * issued in between, 11 clock64 when the NOP ack was seen.  The phases of a
 * block_reduce_f32 dispatch on the TMA ring with LK_CF_TIMELINE (else 0):
 * globaltimer at 12 first bulk copy issued, 13 last bulk copy issued, 14
 * first block's data in shared memory, 15 arrival counted (before the
 * last worker's combine). */
int lk_last_timeline(lk_session* s, uint64_t* t, uint32_t n);
/* Launch+sync floor: the cheapest conventional per-task flow, an empty
 * <<<1,32,0>>> kernel joined by stream sync (LK_FLOOR_SYNC), by a host spin
 * on cudaStreamQuery (LK_FLOOR_QUERY), or launched as a one-node CUDA graph
 * (LK_FLOOR_GRAPH); spin_sched != 0 sets cudaDeviceScheduleSpin first.
 * total_ns[k]: launch call start -> completion observed; launch_ns[k]: the
 * launch call.  Replaces ThreadSpawnBaseline.launch/wait (native.py:304-331). */
#define LK_FLOOR_SYNC  0u
#define LK_FLOOR_QUERY 1u
#define LK_FLOOR_GRAPH 2u
int lk_launch_floor_bench(int device, uint32_t mode, uint32_t spin_sched, uint64_t rounds, uint64_t* total_ns,
                          uint64_t* launch_ns);
/* Per-worker count of to_gpu values the kernel's fast path settled in place
 * (IDLE x WORK of an empty / cached single-thread item, IDLE x WORK begin of
 * a payload item, FINISHED x NOP) since boot -- the path configs[1] times.
 * With record_trace on, those steps append the same trace records as the
 * general path.  Replaces no reference call: test/bench evidence only. */
int lk_fast_count(lk_session* s, uint32_t* counts, uint32_t n);
/* Host side of the same dispatches (CLOCK_MONOTONIC ns, t[3*i+k]): k=0
 * trigger call start, 1 WORK word written, 2 FINISHED observed by wait. */
int lk_last_host_times(lk_session* s, uint64_t* t, uint32_t n);
/* globaltimer - CLOCK_MONOTONIC offset (ns) from `rounds` host<->GPU echoes,
 * taken from the echo with the shortest round trip (*best_rtt_ns). */
int lk_clock_offset(int device, uint32_t rounds, int64_t* offset_ns, uint64_t* best_rtt_ns);
/* GPC membership of each SM (the placement side of check_block_mapping,
 * device.py:102-111): clustered launches of a probe kernel -- a cluster's
 * CTAs share a GPC -- with the SM ids of each cluster unioned.  Needs every
 * SM (no session live).  gpc[smid] = dense group id, -1 if never observed. */
int lk_sm_topology(int device, int32_t* gpc, uint32_t n, uint32_t* ngroups);

/* Raw host<->GPU ping-pong floor: one thread polls a mapped host word and
 * echoes it back; rounds samples of the round trip. */
int lk_pingpong(int device, uint64_t rounds, uint64_t* rt_ns);

/* ---- conventional baseline: cudaLaunchKernel + cudaStreamSynchronize --------
 * Replaces ThreadSpawnBaseline (native.py:304-331).  The same device work
 * functions as the persistent kernel, one CTA per worker of `grid`. */
int lk_baseline_create(int device, uint32_t threads, lk_baseline** out);
int lk_baseline_launch(lk_baseline* b, const lk_desc* d, uint32_t grid, uint64_t* launch_ns);
int lk_baseline_wait(lk_baseline* b, uint64_t* wait_ns);
/* rounds of launch+sync; launch_ns / total_ns per round (may be NULL). */
int lk_baseline_bench(lk_baseline* b, const lk_desc* d, uint32_t grid, uint64_t rounds,
                      uint64_t* launch_ns, uint64_t* total_ns);
/* Device time of one launch via CUDA events on the launching stream: reps
 * launches, avg ms per launch. */
int lk_baseline_time_kernel(lk_baseline* b, const lk_desc* d, uint32_t grid,
                            uint32_t reps, float* avg_ms);
/* 1 (default): payload work functions stream through the same TMA bulk ring
 * as the persistent kernel (96 KiB dynamic shared memory per CTA); 0: LSU
 * path, which also fits beside a resident LK session. */
int lk_baseline_set_tma(lk_baseline* b, int on);
int lk_baseline_destroy(lk_baseline* b);
/* The baseline's launches go to the SMs a partitioned session left free
 * (lk_config.sm_partition), so they run beside the resident LK kernel.
 * Replaces nothing in the reference: its workers are host threads. */
int lk_baseline_create_in(lk_session* s, uint32_t threads, lk_baseline** out);
/* SMs of the session's partition and of the rest (0, 0 when unpartitioned). */
int lk_partition_info(lk_session* s, uint32_t* lk_sms, uint32_t* rest_sms);

/* ---- host helpers ----------------------------------------------------------- */
/* Pin the calling thread to the CPU cores local to the GPU's NUMA node
 * (/sys/bus/pci/devices/<bdf>/local_cpulist).  *ncores = cores in the set. */
int lk_pin_thread_near(int device, uint32_t* ncores);
int lk_device_count(int* n);
int lk_sm_count(int device, int* n);
/* device memory helpers (payload buffers when the caller has no allocator) */
int lk_dev_alloc(int device, uint64_t bytes, uint64_t* ptr);
int lk_dev_free(uint64_t ptr);
/* Mapped pinned host memory (cudaHostAlloc Mapped|Portable) for zero-copy
 * payloads: pass the returned address as an lk_desc pointer and the workers
 * read/write it over the link (LK_DF_HOSTMEM).  Replaces the reference's
 * Copyin/Copyout phases (P/host.py:212-224) for small transfers.  Allocate and
 * free it outside a live session's hot loop: cudaHostAlloc/cudaFreeHost are
 * driver calls of ~10-100 us. */
int lk_host_alloc(int device, uint64_t bytes, void** host);
int lk_host_free(void* host);
int lk_memcpy_h2d(uint64_t dst, const void* src, uint64_t bytes);
int lk_memcpy_d2h(void* dst, uint64_t src, uint64_t bytes);
const char* lk_strerror(int code);
/* message of the last failing call on this thread (may be empty) */
const char* lk_last_error(void);
uint32_t lk_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LK_H_ */
