// driver.hpp — the OPPO step loop (driver.cpp:69-202), parameterised over
// the executor so the same loop drives the logical clock (CPU-only) and the
// GPU engine.
#pragma once

#include <algorithm>
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

    // ---- data parallelism and admission control; the defaults
    // are the single-rank, unbounded-memory reference behaviour
    virtual int rank() const { return 0; }
    virtual int world() const { return 1; }
    // in-place sum over the ranks (host doubles)
    virtual void allreduce_sum(double* v, int n) { (void)v; (void)n; }
    // true when update() already returns the mean reward over all ranks
    virtual bool reward_is_global() const { return true; }
    // simulate / tune modes: the reward fed to the controller (the reference's
    // proxy, driver.cpp:21-32, unless a hook supplies one from the batch)
    virtual double sim_reward(const oppo_run_config& cfg, int step, const std::vector<oppo_seq_state>& batch,
                              bool& is_local) {
        (void)batch;
        is_local = false;
        return proxy_reward(cfg, step);
    }
    // KV admission control: called before each refill, then once per
    // candidate in admission order; false defers the candidate
    virtual void begin_refill() {}
    virtual bool fits(const oppo_seq_state& s) { (void)s; return true; }
};

// Optional per-run host callbacks of the loop (C ABI: oppo_loop_hooks).
struct LoopExtras {
    oppo_step_fn on_step = nullptr;
    void* step_ctx = nullptr;
    oppo_ledger* ledgers = nullptr;  // [cfg.steps] each step's ledger
};

// Returns the number of records; throws oppo::Error on configuration errors.
// Runtime failures are caught like run_seed does (driver.cpp:196-199): the
// partial log is kept and *error receives the message.
inline int run_seed_loop(const oppo_run_config& cfg, uint64_t seed, LoopHooks& hooks,
                         oppo_step_record* records, int64_t* sel_ids, std::string* error,
                         const LoopExtras& extras = LoopExtras{}) {
    validate(cfg);
    const int rank = hooks.rank(), world = hooks.world();
    if (world < 1 || rank < 0 || rank >= world) config_error("rank / world out of range");
    // rank r draws its own lengths; rank 0 of 1 is the reference stream
    Stream lengths = Stream::derive(seed ^ static_cast<uint64_t>(rank), "lengths");
    PromptStream source{cfg.prompt_len, cfg.prompt_count};
    source.rank = rank;
    source.world = world;
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
            hooks.begin_refill();
            refill_fit(buffer, source, step, cfg.lengths, lengths,
                       [&](const oppo_seq_state& s) { return hooks.fits(s); });
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
            bool local = false;
            if (training) {
                if (!sel.batch.empty()) reward = hooks.update(sel.batch, true, rec);
                local = !hooks.reward_is_global();
            } else {
                hooks.update(sel.batch, false, rec);
                reward = hooks.sim_reward(cfg, step, sel.batch, local);
            }
            if (world > 1 && local) {  // the controller sees the global mean
                double v[2] = {reward * static_cast<double>(sel.batch.size()), static_cast<double>(sel.batch.size())};
                hooks.allreduce_sum(v, 2);
                reward = v[1] > 0 ? v[0] / v[1] : 0.0;
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
            if (ledger.step_us > 0.0) {  // utilization (engine.cpp:225-233), measured on the GPU:
                // busy time of each SM partition over the step's device time
                rec.util_generation = ledger.decode_loop_us / ledger.step_us;
                rec.util_scoring = ledger.score_busy_us / ledger.step_us;
            } else if (ledger.wall > 0) {  // logical executor: the reference's tick ledger
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
                // on the GPU the measured step time in us replaces it,
                // the max over the ranks so every rank picks the same chunk size
                double m = ledger.step_us > 0.0 ? ledger.step_us : double(ledger.wall);
                if (world > 1) {
                    std::vector<double> v(world, 0.0);
                    v[rank] = m;
                    hooks.allreduce_sum(v.data(), world);
                    m = *std::max_element(v.begin(), v.end());
                }
                tuner.fold(*explored, m);
            }
            delta = up.delta;
            if (extras.ledgers) extras.ledgers[n - 1] = ledger;
            if (extras.on_step && extras.on_step(extras.step_ctx, &rec) != 0) break;
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
