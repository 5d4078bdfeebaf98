// capi_host.cpp — extern "C" host-scheduler entry points of liboppo.so.
#include <cstring>
#include <string>

#include "driver.hpp"
#include "oppo/oppo.h"
#include "sched.hpp"

namespace {
thread_local std::string g_error;

template <class F>
oppo_status guarded(F&& f) {
    try {
        f();
        return OPPO_OK;
    } catch (const oppo::Error& e) {
        g_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_error = e.what();
        return OPPO_ERR_INTERNAL;
    }
}

struct LogicalHooks final : oppo::LoopHooks {
    void admit(const std::vector<oppo_seq_state>&) override {}
    void execute(const std::vector<oppo_seq_state>& active, int chunk, int mode, int stop,
                 std::vector<oppo_seq_outcome>& out, oppo_ledger& ledger) override {
        auto plan = oppo::plan_step(active, chunk, mode, stop, carry);
        out = std::move(plan.outcomes);
        ledger = plan.ledger;
    }
    double update(const std::vector<oppo_seq_state>&, bool train, oppo_step_record&) override {
        if (train) oppo::config_error("train mode needs the GPU engine (oppo_run_seed)");
        return 0.0;
    }
    void release(const std::vector<oppo_seq_state>&) override {}
    int rank() const override { return rank_; }
    int world() const override { return world_; }
    void allreduce_sum(double* v, int n) override {
        if (world_ <= 1) return;
        if (!ar || ar(ar_ctx, v, n) != 0) oppo::internal_error("host allreduce failed");
    }
    double sim_reward(const oppo_run_config& cfg, int step, const std::vector<oppo_seq_state>& batch,
                      bool& is_local) override {
        if (!rw) {
            is_local = false;
            return oppo::proxy_reward(cfg, step);
        }
        std::vector<int64_t> ids;
        for (const auto& s : batch) ids.push_back(s.id);
        is_local = true;
        return rw(rw_ctx, ids.data(), static_cast<int32_t>(ids.size()));
    }
    int carry = OPPO_CARRY_CHUNK;
    int rank_ = 0, world_ = 1;
    oppo_host_allreduce_fn ar = nullptr;
    void* ar_ctx = nullptr;
    oppo_batch_reward_fn rw = nullptr;
    void* rw_ctx = nullptr;
};
}  // namespace

extern "C" {

const char* oppo_last_error_global(void) { return g_error.c_str(); }

void oppo_set_global_error(const char* msg) { g_error = msg ? msg : ""; }

void oppo_run_config_default(oppo_run_config* cfg) { oppo::config_defaults(*cfg); }

void oppo_run_config_baseline(const oppo_run_config* cfg, oppo_run_config* out) {
    *out = oppo::config_baseline(*cfg);
}

oppo_status oppo_run_config_validate(const oppo_run_config* cfg) {
    return guarded([&] { oppo::validate(*cfg); });
}

oppo_status oppo_rng_draws(uint64_t seed, const char* purpose, int32_t kind, int64_t n,
                           void* out) {
    return guarded([&] {
        auto s = oppo::Stream::derive(seed, purpose ? purpose : "");
        for (int64_t i = 0; i < n; ++i) {
            if (kind == 0) static_cast<uint64_t*>(out)[i] = s.u64();
            else if (kind == 1) static_cast<double*>(out)[i] = s.uniform();
            else if (kind == 2) static_cast<double*>(out)[i] = s.gauss();
            else oppo::input_error("unknown draw kind");
        }
    });
}

oppo_status oppo_sample_lengths(const oppo_length_dist* dist, uint64_t seed, int64_t n,
                                int32_t* out) {
    return guarded([&] {
        auto s = oppo::Stream::derive(seed, "lengths");
        for (int64_t i = 0; i < n; ++i) out[i] = oppo::draw_length(*dist, s);
    });
}

oppo_status oppo_build_schedule(const oppo_seq_state* seqs, int32_t n, int32_t chunk_size,
                                int32_t mode, oppo_chunk_task* tasks, int32_t cap,
                                int32_t* n_tasks) {
    return guarded([&] {
        if (chunk_size < 1) oppo::config_error("chunk size must be >= 1");
        (void)mode;  // the chunk list does not depend on the mode (chunking.cpp:20-48)
        int k = 0;
        for (int i = 0; i < n; ++i)
            for (const auto& c : oppo::chunks_for(seqs[i], chunk_size)) {
                if (k >= cap) oppo::input_error("task buffer too small");
                tasks[k++] = {seqs[i].id, c.first, c.last, c.index, c.needs_decode ? 1 : 0};
            }
        *n_tasks = k;
    });
}

oppo_status oppo_plan_step(const oppo_seq_state* active, int32_t n, int32_t chunk_size,
                           int32_t mode, int32_t stop_after, int32_t carry_granularity,
                           oppo_seq_outcome* out, oppo_ledger* ledger) {
    return guarded([&] {
        std::vector<oppo_seq_state> v(active, active + n);
        const auto p = oppo::plan_step(v, chunk_size, mode, stop_after, carry_granularity);
        std::memcpy(out, p.outcomes.data(), sizeof(oppo_seq_outcome) * p.outcomes.size());
        *ledger = p.ledger;
    });
}

oppo_status oppo_select_finished(oppo_seq_state* entries, int32_t n,
                                 const oppo_seq_outcome* outcomes, int32_t n_out_in,
                                 int32_t batch_size, oppo_seq_state* batch, int32_t* n_batch,
                                 int32_t* n_remaining, int32_t* short_batch) {
    return guarded([&] {
        oppo::Buffer b;
        b.batch_size = batch_size;
        b.entries.assign(entries, entries + n);
        const auto sel = oppo::select_finished(
            b, std::vector<oppo_seq_outcome>(outcomes, outcomes + n_out_in), batch_size);
        std::memcpy(batch, sel.batch.data(), sizeof(oppo_seq_state) * sel.batch.size());
        *n_batch = static_cast<int32_t>(sel.batch.size());
        std::memcpy(entries, b.entries.data(), sizeof(oppo_seq_state) * b.entries.size());
        *n_remaining = static_cast<int32_t>(b.entries.size());
        *short_batch = sel.short_batch;
    });
}

oppo_status oppo_delta_update(int32_t mode, int32_t window, int32_t dmin, int32_t dmax,
                              int32_t inc, int32_t dec, double* history, int32_t* n_hist,
                              int32_t delta, int32_t* new_delta, int32_t* has_stat,
                              double* stat) {
    return guarded([&] {
        oppo::DeltaCtl c;
        c.mode = mode;
        c.window = window;
        c.dmin = dmin;
        c.dmax = dmax;
        c.inc = inc;
        c.dec = dec;
        c.history.assign(history, history + *n_hist);
        const auto r = c.update(delta);
        *new_delta = r.delta;
        *has_stat = r.stat.has_value();
        *stat = r.stat.value_or(0.0);
        std::memcpy(history, c.history.data(), sizeof(double) * c.history.size());
        *n_hist = static_cast<int32_t>(c.history.size());
    });
}

oppo_status oppo_tuner_replay(const int32_t* candidates, int32_t n_cand, int32_t window,
                              const int32_t* meas_cand, const double* meas, int32_t n_meas,
                              int32_t* chosen) {
    return guarded([&] {
        auto t = oppo::Tuner::make(std::vector<int>(candidates, candidates + n_cand), window);
        for (int i = 0; i < n_meas; ++i) {
            t.fold(meas_cand[i], meas[i]);
            chosen[i] = t.current;
        }
    });
}

oppo_status oppo_run_seed_logical_dp(const oppo_run_config* cfg, uint64_t seed, int32_t rank, int32_t world,
                                     oppo_host_allreduce_fn allreduce, void* allreduce_ctx,
                                     oppo_batch_reward_fn batch_reward, void* reward_ctx,
                                     oppo_step_record* records, int32_t* n_records, int64_t* sel_ids) {
    std::string err;
    const oppo_status st = guarded([&] {
        LogicalHooks hooks;
        hooks.carry = cfg->carry_granularity;
        hooks.rank_ = rank;
        hooks.world_ = world;
        hooks.ar = allreduce;
        hooks.ar_ctx = allreduce_ctx;
        hooks.rw = batch_reward;
        hooks.rw_ctx = reward_ctx;
        *n_records = oppo::run_seed_loop(*cfg, seed, hooks, records, sel_ids, &err);
    });
    if (st != OPPO_OK) return st;
    if (!err.empty()) {
        g_error = err;
        return OPPO_ERR_INTERNAL;
    }
    return OPPO_OK;
}

oppo_status oppo_run_seed_logical(const oppo_run_config* cfg, uint64_t seed,
                                  oppo_step_record* records, int32_t* n_records,
                                  int64_t* sel_ids) {
    std::string err;
    const oppo_status st = guarded([&] {
        LogicalHooks hooks;
        hooks.carry = cfg->carry_granularity;
        *n_records = oppo::run_seed_loop(*cfg, seed, hooks, records, sel_ids, &err);
    });
    if (st != OPPO_OK) return st;
    if (!err.empty()) {
        g_error = err;
        return OPPO_ERR_INTERNAL;
    }
    return OPPO_OK;
}

// sizeof of every ABI struct, for the binding's layout check.
int32_t oppo_abi_sizes(int64_t* out, int32_t cap) {
    const int64_t s[] = {sizeof(oppo_seq_state), sizeof(oppo_chunk_task),
                         sizeof(oppo_seq_outcome), sizeof(oppo_ledger),
                         sizeof(oppo_latency), sizeof(oppo_length_dist),
                         sizeof(oppo_ppo_hparams), sizeof(oppo_run_config),
                         sizeof(oppo_step_record), sizeof(oppo_model_dims),
                         sizeof(oppo_engine_cfg), sizeof(oppo_ppo_stats)};
    const int32_t n = static_cast<int32_t>(sizeof(s) / sizeof(s[0]));
    for (int32_t i = 0; i < n && i < cap; ++i) out[i] = s[i];
    return n;
}

}  // extern "C"
