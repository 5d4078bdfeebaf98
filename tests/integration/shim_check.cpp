// shim_check.cpp — compiles include/oppo/rlpipe_adapter.hpp against the real
// reference headers and checks that the adapter's run_step (the drop-in a
// reference maintainer would call) makes the same decisions as
// rlpipe::run_step under the lockstep latency model, on random active sets
// (fresh and carried sequences, both schedule modes, random cuts).
// Built and run by tests/test_integration.py where /root/reference exists.
#include <string>
#include <cstdio>
#include <random>
#include <vector>

#include "rlpipe/chunking.hpp"
#include "rlpipe/engine.hpp"
#include "rlpipe/errors.hpp"
#include "rlpipe/model.hpp"

#include "oppo/rlpipe_adapter.hpp"

int main() {
    std::mt19937_64 g(20250925);
    rlpipe::LatencyModel lock;
    lock.decode_per_token = 1;
    lock.prefill_per_token = 0;
    lock.reward_residual = 0;
    lock.chunk_switch_cost = 0;
    lock.placement = rlpipe::Placement::Disaggregated;
    lock.transfer_per_chunk = 0;
    lock.count_prompt_in_prefill = false;
    int cases = 0, mismatches = 0;
    for (int t = 0; t < 400; ++t) {
        const int n = 1 + static_cast<int>(g() % 24);
        const int chunk = 1 + static_cast<int>(g() % 40);
        std::vector<rlpipe::SequenceState> act(n);
        for (int i = 0; i < n; ++i) {
            auto& s = act[i];
            s.prompt.id = 1000 * t + i;
            s.prompt.prompt_len = 1 + static_cast<int>(g() % 16);
            s.target_len = 1 + static_cast<int>(g() % 200);
            if (g() % 3 == 0) {  // carried: whole chunks of an earlier step decoded / prefilled
                s.generated = static_cast<int>(g() % s.target_len);
                s.prefilled_tokens = s.generated ? static_cast<int>(g() % (s.generated + 1)) : 0;
                s.chunks_emitted = s.generated ? 1 : 0;
                s.chunks_prefilled = s.prefilled_tokens ? 1 : 0;
                s.deferrals = 1;
            }
        }
        const auto mode = (g() % 2) ? rlpipe::ScheduleMode::Streamed : rlpipe::ScheduleMode::Sequential;
        const int stop = 1 + static_cast<int>(g() % n);
        const auto sched = rlpipe::build_schedule(act, chunk, mode);
        const auto ref = rlpipe::run_step(act, sched, lock, stop);
        const auto got = oppo_rlpipe::run_step_logical(act, sched, stop);
        ++cases;
        bool ok = ref.first.wall == got.first.wall && ref.second.wall == got.second.wall &&
                  ref.first.sequences.size() == got.first.sequences.size();
        for (size_t i = 0; ok && i < ref.first.sequences.size(); ++i) {
            const auto& a = ref.first.sequences[i];
            const auto& b = got.first.sequences[i];
            ok = a.seq_id == b.seq_id && a.score_ready == b.score_ready &&
                 a.tokens_decoded == b.tokens_decoded && a.tokens_prefilled == b.tokens_prefilled &&
                 a.decode_chunks_completed == b.decode_chunks_completed &&
                 a.prefill_tasks_completed == b.prefill_tasks_completed &&
                 a.carry_prefill_completed == b.carry_prefill_completed;
        }
        if (!ok) {
            ++mismatches;
            if (mismatches < 5)
                std::printf("mismatch case %d: n=%d chunk=%d stop=%d wall ref %lld got %lld\n", t, n, chunk,
                            stop, static_cast<long long>(ref.first.wall),
                            static_cast<long long>(got.first.wall));
        }
    }
    // error mapping: an invalid chunk size surfaces as the reference's exception type
    bool mapped = false;
    try {
        rlpipe::StepSchedule bad;
        bad.chunk_size = 0;
        std::vector<rlpipe::SequenceState> one(1);
        one[0].prompt.id = 1;
        one[0].target_len = 5;
        oppo_rlpipe::run_step_logical(one, bad, 1);
    } catch (const rlpipe::ConfigError& ex) {
        mapped = std::string(ex.what()).find("chunk") != std::string::npos;  // the call's own message
        if (!mapped) std::printf("error message: '%s'\n", ex.what());
    } catch (const rlpipe::InputError& ex) {
        mapped = std::string(ex.what()).find("chunk") != std::string::npos;
        if (!mapped) std::printf("error message: '%s'\n", ex.what());
    }
    std::printf("cases %d mismatches %d error_mapping %s\n", cases, mismatches, mapped ? "ok" : "BAD");
    return (mismatches == 0 && mapped) ? 0 : 1;
}
