// lk_validate.cpp -- native replay of a recorded mailbox trace against the
// handshake rules, used to validate GPU traces at criterion-8 scale (millions
// of records) without Python overhead.
//
// Rules restate persistkern.protocol._host_write / _device_write / replay_trace
// (/root/reference/pkg/src/persistkern/protocol.py:298-398): each worker is
// replayed independently; a leading device INIT marks a recorded boot,
// otherwise the worker is taken as already idle.  The first illegal write is
// reported with its index and a message in the reference's wording.
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/lk.h"

namespace {

enum RPhase : uint8_t { kUnset, kIdle, kWorking, kAwaitAck };

struct Replay {
  RPhase phase = kUnset;
  uint32_t slot = 0;
  uint32_t to_gpu = LK_NOP;
  uint32_t from_gpu = LK_NOP;
  bool work_pending = false;
  uint64_t work_writes = 0;
  uint64_t begins = 0;
};

inline bool is_work(uint32_t w) { return w >= LK_WORK_BASE; }
inline bool from_gpu_word(uint32_t w) {
  return w == LK_INIT || w == LK_FINISHED || w == LK_WORKING || w == LK_NOP;
}

// Returns an empty string when the host write is legal.
std::string host_write(Replay& r, uint32_t w) {
  if (r.to_gpu == LK_EXIT) return "host write after exit";
  if (w == LK_NOP) {
    if (r.from_gpu != LK_FINISHED)
      return "ack written while from_gpu=" + std::to_string(r.from_gpu) + ", not FINISHED";
    r.to_gpu = LK_NOP;
    return {};
  }
  if (w == LK_EXIT) {
    if (r.from_gpu == LK_WORKING) return "exit written to a working cluster";
    if (r.work_pending) return "exit would discard an undelivered work command";
    r.to_gpu = LK_EXIT;
    return {};
  }
  if (is_work(w)) {
    if (is_work(r.to_gpu)) return "trigger while busy: previous work command not consumed";
    if (r.from_gpu != LK_FINISHED && r.from_gpu != LK_NOP)
      return "work written while from_gpu=" + std::to_string(r.from_gpu);
    r.to_gpu = w;
    r.work_pending = true;
    ++r.work_writes;
    return {};
  }
  return "illegal to_gpu word " + std::to_string(w);
}

std::string device_write(Replay& r, uint32_t w) {
  if (!from_gpu_word(w)) return "illegal from_gpu word " + std::to_string(w);
  if (r.phase == kUnset) {
    r.phase = kIdle;
    if (w == LK_INIT) {  // recorded boot announcement
      r.from_gpu = LK_INIT;
      return {};
    }
    r.from_gpu = LK_NOP;  // trace starts post-boot
  }
  switch (r.phase) {
    case kIdle:
      if (w == LK_NOP && r.from_gpu == LK_INIT) {
        r.from_gpu = LK_NOP;
        return {};
      }
      if (w == LK_WORKING && is_work(r.to_gpu) && r.work_pending) {
        r.phase = kWorking;
        r.slot = r.to_gpu - LK_WORK_BASE;
        r.from_gpu = LK_WORKING;
        r.work_pending = false;
        ++r.begins;
        return {};
      }
      return "word " + std::to_string(w) + " not producible by an idle worker";
    case kWorking:
      if (w == LK_FINISHED) {
        r.phase = kAwaitAck;
        r.from_gpu = LK_FINISHED;
        return {};
      }
      return "word " + std::to_string(w) + " not producible by a working worker";
    default:
      if (w == LK_NOP && r.to_gpu == LK_NOP) {
        r.phase = kIdle;
        r.from_gpu = LK_NOP;
        return {};
      }
      return "word " + std::to_string(w) + " not producible while awaiting ack";
  }
}

}  // namespace

extern "C" int lk_validate_trace(const uint32_t* side, const int64_t* sm_id, const uint32_t* word, uint64_t n,
                                 int64_t* bad_index, char* reason, uint32_t reason_cap, uint64_t* counts,
                                 uint32_t max_workers, uint32_t* n_workers) {
  if ((n && (!side || !sm_id || !word)) || !bad_index) return LK_E_USAGE;
  std::unordered_map<int64_t, Replay> sms;
  std::vector<int64_t> order;  // first-seen order of sm ids
  *bad_index = -1;
  std::string why;
  for (uint64_t i = 0; i < n; ++i) {
    if (sm_id[i] < 0) {
      why = "negative sm_id " + std::to_string(sm_id[i]);
      *bad_index = int64_t(i);
      break;
    }
    auto it = sms.find(sm_id[i]);
    if (it == sms.end()) {
      it = sms.emplace(sm_id[i], Replay()).first;
      order.push_back(sm_id[i]);
    }
    if (side[i] == 'H') why = host_write(it->second, word[i]);
    else if (side[i] == 'D') why = device_write(it->second, word[i]);
    else {
      char c[2] = {char(side[i]), 0};
      why = std::string("unknown side '") + c + "'";
    }
    if (!why.empty()) {
      *bad_index = int64_t(i);
      break;
    }
  }
  if (reason && reason_cap) {
    snprintf(reason, reason_cap, "%s", why.c_str());
  }
  if (n_workers) *n_workers = uint32_t(order.size());
  if (counts) {
    for (size_t k = 0; k < order.size() && k < max_workers; ++k) {
      const Replay& r = sms[order[k]];
      counts[3 * k] = uint64_t(order[k]);
      counts[3 * k + 1] = r.work_writes;
      counts[3 * k + 2] = r.begins;
    }
  }
  return LK_OK;
}
