// rlpipe_adapter.hpp — header-only adapter from the reference's C++ API
// (namespace rlpipe, /root/reference/proj/core/include/rlpipe/*.hpp) to the
// C ABI of liboppo.so.  Include the rlpipe headers first.  This is the
// binding a maintainer of the reference adds to route its hot path through
// the B200 executor; tests/integration/shim_check.cpp
// compiles it against the real reference headers.
//
//   rlpipe::run_step(active, schedule, model, stop_after)   engine.hpp:91-93
//     -> oppo_rlpipe::run_step(engine, active, schedule, stop_after)  (GPU)
//     -> oppo_rlpipe::run_step_logical(active, schedule, stop_after) (CPU,
//        the lockstep logical clock the GPU executor obeys)
//   rlpipe::ConfigError / InputError / InternalError   errors.hpp:9-24
//     <- OPPO_ERR_CONFIG / OPPO_ERR_INPUT / OPPO_ERR_INTERNAL
#pragma once

#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "oppo/oppo.h"

namespace oppo_rlpipe {

inline void check(oppo_status st, const char* msg) {
    if (st == OPPO_OK) return;
    const std::string m = msg ? msg : "";
    switch (st) {
    case OPPO_ERR_CONFIG: throw rlpipe::ConfigError(m);
    case OPPO_ERR_INPUT: throw rlpipe::InputError(m);
    case OPPO_ERR_INTERNAL: throw rlpipe::InternalError(m);
    default: throw std::runtime_error("oppo: " + m);
    }
}

inline oppo_seq_state to_c(const rlpipe::SequenceState& s) {
    oppo_seq_state c{};
    c.id = s.prompt.id;
    c.prompt_len = s.prompt.prompt_len;
    c.arrival_step = s.prompt.arrival_step;
    c.target_len = s.target_len;
    c.generated = s.generated;
    c.prefilled_tokens = s.prefilled_tokens;
    c.chunks_emitted = s.chunks_emitted;
    c.chunks_prefilled = s.chunks_prefilled;
    c.finished = s.finished;
    c.scored = s.scored;
    c.admitted_at = s.admitted_at;
    c.deferrals = s.deferrals;
    return c;
}

inline rlpipe::SequenceOutcome from_c(const oppo_seq_outcome& o) {
    rlpipe::SequenceOutcome r;
    r.seq_id = o.seq_id;
    if (o.score_ready >= 0) r.score_ready = o.score_ready;
    r.tokens_decoded = o.tokens_decoded;
    r.tokens_prefilled = o.tokens_prefilled;
    r.decode_chunks_completed = o.decode_chunks_completed;
    r.prefill_tasks_completed = o.prefill_tasks_completed;
    r.carry_prefill_completed = o.carry_prefill_completed != 0;
    return r;  // per-chunk tick vectors are not part of the C ABI
}

inline rlpipe::ResourceLedger from_c(const oppo_ledger& l) {
    rlpipe::ResourceLedger r;
    r.wall = l.wall;
    r.busy_generation = l.busy_generation;
    r.busy_scoring = l.busy_scoring;
    r.work_generation = l.work_generation;
    r.work_scoring = l.work_scoring;
    return r;
}

inline std::pair<rlpipe::StepTimeline, rlpipe::ResourceLedger> finish(
    const std::vector<oppo_seq_outcome>& out, const oppo_ledger& led) {
    rlpipe::StepTimeline tl;
    tl.wall = led.wall;
    for (const auto& o : out) tl.sequences.push_back(from_c(o));
    return {std::move(tl), from_c(led)};
}

inline std::vector<oppo_seq_state> to_c(const std::vector<rlpipe::SequenceState>& v) {
    std::vector<oppo_seq_state> c;
    c.reserve(v.size());
    for (const auto& s : v) c.push_back(to_c(s));
    return c;
}

inline int32_t mode_of(const rlpipe::StepSchedule& s) {
    return s.mode == rlpipe::ScheduleMode::Streamed ? OPPO_MODE_STREAMED : OPPO_MODE_SEQUENTIAL;
}

// run_step on the GPU executor (one engine per GPU; the sequences must have
// been admitted with oppo_admit).  stop_after defaults to "all" as in rlpipe.
inline std::pair<rlpipe::StepTimeline, rlpipe::ResourceLedger> run_step(
    oppo_engine* e, const std::vector<rlpipe::SequenceState>& active,
    const rlpipe::StepSchedule& schedule, std::optional<int> stop_after = std::nullopt) {
    const auto c = to_c(active);
    std::vector<oppo_seq_outcome> out(c.size());
    oppo_ledger led{};
    const int32_t stop = stop_after ? *stop_after : static_cast<int32_t>(c.size());
    // status first: argument evaluation order is unspecified, and the error
    // string must be read after the call that sets it
    const oppo_status st = oppo_run_step(e, c.data(), static_cast<int32_t>(c.size()),
                                         schedule.chunk_size, mode_of(schedule), stop, out.data(), &led);
    check(st, st == OPPO_OK ? nullptr : oppo_last_error(e));
    return finish(out, led);
}

// The same decisions without a GPU: the reference's run_step under the
// lockstep latency model {decode=1, prefill=0, residual=0, disaggregated}.
inline std::pair<rlpipe::StepTimeline, rlpipe::ResourceLedger> run_step_logical(
    const std::vector<rlpipe::SequenceState>& active, const rlpipe::StepSchedule& schedule,
    std::optional<int> stop_after = std::nullopt, int32_t carry = OPPO_CARRY_CHUNK) {
    const auto c = to_c(active);
    std::vector<oppo_seq_outcome> out(c.size());
    oppo_ledger led{};
    const int32_t stop = stop_after ? *stop_after : static_cast<int32_t>(c.size());
    const oppo_status st = oppo_plan_step(c.data(), static_cast<int32_t>(c.size()),
                                          schedule.chunk_size, mode_of(schedule), stop, carry,
                                          out.data(), &led);
    check(st, st == OPPO_OK ? nullptr : oppo_last_error_global());
    return finish(out, led);
}

}  // namespace oppo_rlpipe
