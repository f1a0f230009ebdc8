// lk_protocol.cuh -- the dual-mailbox handshake as one __host__ __device__
// state machine, compiled both into the persistent kernel (each CTA's
// elected thread runs it on every changed to_gpu word) and into the host
// library (lk_protocol_step, used by the parity tests).
//
// Semantics follow persistkern.protocol.worker_step / complete_work
// (/root/reference/pkg/src/persistkern/protocol.py:151-206); the word
// values are Table I of the paper (protocol.py:31-45).
#pragma once
#include <stdint.h>
#include "../../include/lk.h"

#if defined(__CUDACC__)
#define LK_HD __host__ __device__ __forceinline__
#else
#define LK_HD inline
#endif

#define LK_NO_PUBLISH 0xFFFFFFFFu
#define LK_ACT_NONE  0u
#define LK_ACT_BEGIN 1u
#define LK_ACT_EXIT  2u

struct lk_wstate {
  uint32_t phase;  // LK_PHASE_*
  uint32_t slot;   // valid while WORKING / FINISHED
};

struct lk_step_out {
  uint32_t publish;  // from_gpu word, or LK_NO_PUBLISH
  uint32_t action;   // LK_ACT_*
  uint32_t werr;     // LK_WERR_* (0 = legal step)
};

// One poll: the worker observed `word` in its to_gpu cell.
// protocol.py:151-198.  On a violation the state is left unchanged and
// werr names the rule; the caller (device) records it and leaves its loop.
LK_HD lk_step_out lk_worker_step(lk_wstate& st, uint32_t word) {
  lk_step_out o{LK_NO_PUBLISH, LK_ACT_NONE, LK_WERR_NONE};
  if (st.phase == LK_PHASE_EXITED) { o.werr = LK_WERR_AFTER_EXIT; return o; }
  // decode_to_gpu (protocol.py:83-91): NOP, EXIT, or 16+slot; 0..15 else illegal
  const bool is_work = word >= LK_WORK_BASE;
  if (!is_work && word != LK_NOP && word != LK_EXIT) { o.werr = LK_WERR_ILLEGAL_WORD; return o; }
  const uint32_t slot = word - LK_WORK_BASE;

  // EXIT ends the loop from every phase but WORKING, without a publish.
  if (word == LK_EXIT && st.phase != LK_PHASE_WORKING) {
    st.phase = LK_PHASE_EXITED;
    o.action = LK_ACT_EXIT;
    return o;
  }
  switch (st.phase) {
    case LK_PHASE_BOOTING:  // announce INIT once; the command stays in the cell
      st.phase = LK_PHASE_IDLE;
      o.publish = LK_INIT;
      return o;
    case LK_PHASE_IDLE:
      if (!is_work) { o.publish = LK_NOP; return o; }
      st.phase = LK_PHASE_WORKING;
      st.slot = slot;
      o.publish = LK_WORKING;
      o.action = LK_ACT_BEGIN;
      return o;
    case LK_PHASE_WORKING:  // stale own word, early NOP or EXIT: keep working
      if (is_work && slot != st.slot) { o.werr = LK_WERR_BUSY_SLOT; return o; }
      o.publish = LK_WORKING;
      return o;
    default:  // LK_PHASE_FINISHED (awaiting the ack)
      if (!is_work) {  // NOP (EXIT handled above)
        st.phase = LK_PHASE_IDLE;
        o.publish = LK_NOP;
        return o;
      }
      if (slot != st.slot) { o.werr = LK_WERR_UNACKED_SLOT; return o; }
      o.publish = LK_FINISHED;
      return o;
  }
}

// Executor-signalled completion (protocol.py:201-206).
LK_HD lk_step_out lk_complete_work(lk_wstate& st) {
  lk_step_out o{LK_NO_PUBLISH, LK_ACT_NONE, LK_WERR_NONE};
  if (st.phase != LK_PHASE_WORKING) { o.werr = LK_WERR_BAD_COMPLETE; return o; }
  st.phase = LK_PHASE_FINISHED;
  o.publish = LK_FINISHED;
  return o;
}
