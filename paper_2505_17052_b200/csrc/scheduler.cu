// Pipeline-aware verification scheduler and draft-depth calibration (PAPER.md
// §4.3: "interleaving verification tasks across multiple requests processed on separate
// edge devices ... server verification time ~= edge drafting time + network round-trip time";
// worked depths P:516; SPEC.md S:311-383 for the interface).  Host code only: the decision point
// in front of specedge_verify_batch.  Readings in DESIGN.md §4 (R-sched).
//
// * admission: at most one outstanding request per session (protocol error otherwise);
// * plan: work-conserving — whenever the server is free and >= 1 request is queued, take the
//   oldest min(capacity, queued) requests (arrival time, then admission order);
// * depth: max(1, round-half-away((verify - rtt) / draft_pass)) over exponentially weighted
//   estimates (weight w; the first observation initialises an estimate without a prior).
#include "internal.h"

#include <cmath>
#include <map>
#include <unordered_map>
#include <utility>

struct specedge_scheduler {
  specedge_scheduler_config cfg;
  // queue ordered by (arrival, admission sequence) -> request
  std::map<std::pair<double, uint64_t>, specedge_sched_request> queue;
  std::unordered_map<uint64_t, int> outstanding;   // session -> 1 (queued or in service)
  uint64_t seq = 0;
  double est[3];
  bool have[3];
};

extern "C" {

int32_t specedge_calibrate_draft_depth(double verify_ms, double draft_pass_ms, double rtt_ms) {
  if (!(draft_pass_ms > 0.0) || !std::isfinite(verify_ms) || !std::isfinite(rtt_ms)) return 1;
  const double x = (verify_ms - rtt_ms) / draft_pass_ms;
  const double r = std::round(x);   // C99 round(): nearest, halfway cases away from zero
  return r < 1.0 ? 1 : (r > 1e6 ? 1000000 : (int32_t)r);
}

specedge_status specedge_scheduler_create(const specedge_scheduler_config* cfg, specedge_scheduler** out) {
  if (!cfg || !out || cfg->capacity < 1 || !(cfg->ewma_weight > 0.0 && cfg->ewma_weight <= 1.0) ||
      cfg->fixed_depth < 0)
    return SPECEDGE_E_INVALID;
  specedge_scheduler* s = new specedge_scheduler();
  s->cfg = *cfg;
  const double init[3] = {cfg->init_verify_ms, cfg->init_draft_pass_ms, cfg->init_rtt_ms};
  for (int k = 0; k < 3; ++k) {
    s->have[k] = init[k] > 0.0;
    s->est[k] = s->have[k] ? init[k] : 0.0;
  }
  *out = s;
  return SPECEDGE_OK;
}

specedge_status specedge_scheduler_destroy(specedge_scheduler* s) {
  if (!s) return SPECEDGE_E_INVALID;
  delete s;
  return SPECEDGE_OK;
}

specedge_status specedge_scheduler_admit(specedge_scheduler* s, const specedge_sched_request* req) {
  if (!s || !req) return SPECEDGE_E_INVALID;
  if (s->outstanding.count(req->session_id)) return SPECEDGE_E_PROTOCOL;
  s->outstanding.emplace(req->session_id, 1);
  s->queue.emplace(std::make_pair(req->arrival_ms, s->seq++), *req);
  return SPECEDGE_OK;
}

specedge_status specedge_scheduler_plan(specedge_scheduler* s, specedge_sched_request* members, int32_t max_members,
                                        int32_t* n_members, int32_t* padded_len) {
  if (!s || !n_members || (max_members > 0 && !members) || max_members < 0) return SPECEDGE_E_INVALID;
  const int32_t take = std::min<int32_t>(std::min<int32_t>(s->cfg.capacity, max_members), (int32_t)s->queue.size());
  int32_t longest = 0;
  auto it = s->queue.begin();
  for (int32_t i = 0; i < take; ++i) {
    members[i] = it->second;
    longest = std::max(longest, it->second.length);
    it = s->queue.erase(it);
  }
  *n_members = take;
  if (padded_len) *padded_len = longest;
  return SPECEDGE_OK;
}

specedge_status specedge_scheduler_complete(specedge_scheduler* s, const uint64_t* sessions, int32_t n,
                                            double verify_ms) {
  if (!s || n < 0 || (n > 0 && !sessions)) return SPECEDGE_E_INVALID;
  for (int32_t i = 0; i < n; ++i) s->outstanding.erase(sessions[i]);
  return specedge_scheduler_observe(s, SPECEDGE_TIMING_VERIFY, verify_ms);
}

specedge_status specedge_scheduler_observe(specedge_scheduler* s, int32_t kind, double ms) {
  if (!s || kind < 0 || kind > 2 || !(ms >= 0.0) || !std::isfinite(ms)) return SPECEDGE_E_INVALID;
  if (!s->have[kind]) {
    s->est[kind] = ms;
    s->have[kind] = true;
  } else {
    const double w = s->cfg.ewma_weight;
    s->est[kind] = (1.0 - w) * s->est[kind] + w * ms;
  }
  return SPECEDGE_OK;
}

specedge_status specedge_scheduler_state(const specedge_scheduler* s, int32_t* depth, int32_t* queued,
                                         int32_t* outstanding, double* estimates3) {
  if (!s) return SPECEDGE_E_INVALID;
  if (depth) {
    if (s->cfg.fixed_depth > 0) *depth = s->cfg.fixed_depth;
    else if (!(s->have[0] && s->have[1] && s->have[2])) *depth = 1;
    else *depth = specedge_calibrate_draft_depth(s->est[0], s->est[1], s->est[2]);
  }
  if (queued) *queued = (int32_t)s->queue.size();
  if (outstanding) *outstanding = (int32_t)s->outstanding.size();
  if (estimates3)
    for (int k = 0; k < 3; ++k) estimates3[k] = s->have[k] ? s->est[k] : -1.0;
  return SPECEDGE_OK;
}

}  // extern "C"
