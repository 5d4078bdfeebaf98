// driver.hpp — the OPPO step loop (driver.cpp:69-202), parameterised over
// the executor so the same loop drives the logical clock (CPU-only) and the
// GPU engine.
#pragma once

#include <cstring>
#include <string>
#include <vector>

#include "sched.hpp"

namespace oppo {

struct LoopHooks {
    virtual ~LoopHooks() = default;
    // refill side effects for newly admitted entries (slots, prompts)
    virtual void admit(const std::vector<oppo_seq_state>& fresh) = 0;
    // run_step replacement; fills outcomes (input order) and the ledger
    virtual void execute(const std::vector<oppo_seq_state>& active, int chunk_size, int mode,
                         int stop_after, std::vector<oppo_seq_outcome>& out,
                         oppo_ledger& ledger) = 0;
    // fill_values + toy_rlhf_step replacement; returns the batch mean reward.
    // `train` is false in simulate/tune modes, where the reward proxy is used.
    virtual double update(const std::vector<oppo_seq_state>& batch, bool train,
                          oppo_step_record& rec) = 0;
    // selected sequences leave the buffer for good
    virtual void release(const std::vector<oppo_seq_state>& batch) = 0;
};

// Returns the number of records; throws oppo::Error on configuration errors.
// Runtime failures are caught like run_seed does (driver.cpp:196-199): the
// partial log is kept and *error receives the message.
inline int run_seed_loop(const oppo_run_config& cfg, uint64_t seed, LoopHooks& hooks,
                         oppo_step_record* records, int64_t* sel_ids, std::string* error) {
    validate(cfg);
    Stream lengths = Stream::derive(seed, "lengths");
    PromptStream source{cfg.prompt_len, cfg.prompt_count};
    Buffer buffer;
    buffer.batch_size = cfg.batch_size;
    buffer.delta = cfg.delta_init;
    DeltaCtl ctl;
    ctl.mode = cfg.controller;
    ctl.window = cfg.window;
    ctl.dmin = cfg.delta_min;
    ctl.dmax = cfg.delta_max;
    ctl.inc = cfg.delta_inc;
    ctl.dec = cfg.delta_dec;
    const bool training = cfg.mode == OPPO_RUN_TRAIN;
    const bool tuning = cfg.mode == OPPO_RUN_TUNE || cfg.tune_chunks;
    Tuner tuner;
    if (tuning)
        tuner = Tuner::make(std::vector<int>(cfg.chunk_candidates,
                                             cfg.chunk_candidates + cfg.n_candidates),
                            cfg.retune_period);
    int delta = cfg.delta_init;
    int max_deferrals = 0;
    int n = 0;
    try {
        for (int step = 0; step < cfg.steps; ++step) {
            if (cfg.fail_after_step >= 0 && step >= cfg.fail_after_step)
                throw std::runtime_error("injected failure (debug.fail_after_step)");
            buffer.delta = delta;  // capacity change takes effect at refill
            const size_t before = buffer.entries.size();
            refill(buffer, source, step, cfg.lengths, lengths);
            if (buffer.entries.empty()) break;  // source exhausted
            hooks.admit(std::vector<oppo_seq_state>(buffer.entries.begin() + before,
                                                    buffer.entries.end()));
            int chunk = cfg.chunk_size;
            std::optional<int> explored;
            if (tuning) {
                explored = tuner.explore(step % cfg.retune_period);
                chunk = explored ? *explored : tuner.current;
            }
            std::vector<oppo_seq_state> active;
            int pre_scored = 0;
            for (const auto& e : buffer.entries) {
                if (e.scored) ++pre_scored;
                else active.push_back(e);
            }
            std::vector<oppo_seq_outcome> outcomes;
            oppo_ledger ledger{};
            const int still_needed = cfg.batch_size - pre_scored;
            if (!active.empty() && still_needed > 0)
                hooks.execute(active, chunk, cfg.schedule_mode, still_needed, outcomes, ledger);
            Selection sel = select_finished(buffer, outcomes, cfg.batch_size);
            for (const auto& e : buffer.entries) max_deferrals = std::max(max_deferrals, e.deferrals);

            oppo_step_record& rec = records[n];
            std::memset(&rec, 0, sizeof(rec));
            double reward = 0.0;
            if (training) {
                if (!sel.batch.empty()) reward = hooks.update(sel.batch, true, rec);
            } else {
                hooks.update(sel.batch, false, rec);
                reward = proxy_reward(cfg, step);
            }
            hooks.release(sel.batch);
            ctl.history.push_back(reward);
            const auto up = ctl.update(delta);

            rec.step = step;
            rec.wall_ticks = ledger.wall;
            rec.finished = static_cast<int>(sel.batch.size());
            rec.deferred = sel.deferred;
            rec.delta = delta;
            rec.has_controller_stat = up.stat.has_value();
            rec.controller_stat = up.stat.value_or(0.0);
            rec.mean_reward = reward;
            if (ledger.wall > 0) {  // utilization (engine.cpp:225-233)
                rec.util_generation = double(ledger.busy_generation) / double(ledger.wall);
                rec.util_scoring = double(ledger.busy_scoring) / double(ledger.wall);
            }
            rec.max_deferrals = max_deferrals;
            rec.chunk_size = chunk;
            rec.pre_scored = pre_scored;
            rec.step_us = ledger.step_us;
            if (sel_ids)
                for (int i = 0; i < cfg.batch_size; ++i)
                    sel_ids[static_cast<size_t>(n) * cfg.batch_size + i] =
                        i < static_cast<int>(sel.batch.size()) ? sel.batch[i].id : -1;
            ++n;
            if (tuning && explored) {
                // the tuner's measurement: the reference's tick wall (driver.cpp:187-192);
                // on the GPU the measured step time in us replaces it
                const double m = ledger.step_us > 0.0 ? ledger.step_us : double(ledger.wall);
                tuner.fold(*explored, m);
            }
            delta = up.delta;
        }
    } catch (const Error& e) {
        if (e.code == OPPO_ERR_CONFIG) throw;
        if (error) *error = e.what();
    } catch (const std::exception& e) {
        if (error) *error = e.what();
    }
    return n;
}

}  // namespace oppo
