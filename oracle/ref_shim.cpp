// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// extern "C" wrappers over the UNMODIFIED reference library compiled from
// /root/reference/proj/core/src/*.cpp by oracle/Makefile into
// oracle/_ref/librlpipe_ref.so.  Python tests, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs call these through ctypes.
// Nothing under paper_2509_25762_b200/ links or loads this file.
//
// Every function forwards to the rlpipe function it names; the only logic
// here is struct conversion and one traced copy of the run_seed step loop
// (driver.cpp:103-195) that records selected ids, validated in the tests
// against rlpipe::run_seed's own StepRecords.
#include <algorithm>
#include <cstdio>
#include <filesystem>
#include <cstring>
#include <exception>
#include <string>
#include <unordered_map>
#include <vector>

#include "rlpipe/chunking.hpp"
#include "rlpipe/config.hpp"
#include "rlpipe/driver.hpp"
#include "rlpipe/engine.hpp"
#include "rlpipe/errors.hpp"
#include "rlpipe/model.hpp"
#include "rlpipe/overcommit.hpp"
#include "rlpipe/ppo.hpp"
#include "rlpipe/rng.hpp"

#include "oppo/oppo.h"

using namespace rlpipe;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const InputError& e) {
        g_err = e.what();
        return 2;
    } catch (const InternalError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

LengthDistribution to_ref(const oppo_length_dist& d) {
    LengthDistribution r;
    r.kind = static_cast<LengthDistribution::Kind>(d.kind);
    r.fast_len = d.fast_len;
    r.slow_len = d.slow_len;
    r.p_slow = d.p_slow;
    r.mu_log = d.mu_log;
    r.sigma_log = d.sigma_log;
    r.cap = d.cap;
    for (int i = 0; i < d.table_n; ++i) r.table.emplace_back(d.table_len[i], d.table_w[i]);
    return r;
}

LatencyModel to_ref(const oppo_latency& l) {
    LatencyModel m;
    m.decode_per_token = l.decode_per_token;
    m.prefill_per_token = l.prefill_per_token;
    m.reward_residual = l.reward_residual;
    m.chunk_switch_cost = l.chunk_switch_cost;
    m.transfer_per_chunk = l.transfer_per_chunk;
    m.placement = static_cast<Placement>(l.placement);
    m.count_prompt_in_prefill = l.count_prompt_in_prefill != 0;
    return m;
}

RunConfig to_ref(const oppo_run_config& c) {
    RunConfig r;
    r.mode = static_cast<RunMode>(c.mode);
    r.steps = c.steps;
    r.batch_size = c.batch_size;
    r.prompt_len = c.prompt_len;
    r.prompt_count = c.prompt_count;
    r.delta_init = c.delta_init;
    r.delta_min = c.delta_min;
    r.delta_max = c.delta_max;
    r.controller = static_cast<DeltaMode>(c.controller);
    r.window = c.window;
    r.delta_inc = c.delta_inc;
    r.delta_dec = c.delta_dec;
    r.chunk_size = c.chunk_size;
    r.schedule_mode = static_cast<ScheduleMode>(c.schedule_mode);
    r.tune_chunks = c.tune_chunks != 0;
    r.chunk_candidates.assign(c.chunk_candidates, c.chunk_candidates + c.n_candidates);
    r.retune_period = c.retune_period;
    r.latency = to_ref(c.latency);
    r.lengths = to_ref(c.lengths);
    r.ppo.gamma = c.ppo.gamma;
    r.ppo.lambda = c.ppo.lambda;
    r.ppo.clip_epsilon = c.ppo.clip_epsilon;
    r.ppo.learning_rate = c.ppo.learning_rate;
    r.ppo.value_learning_rate = c.ppo.value_learning_rate;
    r.vocab = c.vocab;
    r.target_token = c.target_token;
    r.reward_scale = c.reward_scale;
    r.reward_bias = c.reward_bias;
    r.reward_proxy.kind = static_cast<RewardProxy::Kind>(c.proxy_kind);
    r.reward_proxy.value = c.proxy_value;
    r.reward_proxy.ramp_scale = c.proxy_ramp_scale;
    r.reward_proxy.ramp_steps = c.proxy_ramp_steps;
    r.fail_after_step = c.fail_after_step;
    r.seeds = {1};
    return r;
}

oppo_length_dist from_ref(const LengthDistribution& d) {
    oppo_length_dist r{};
    r.kind = static_cast<int32_t>(d.kind);
    r.fast_len = d.fast_len;
    r.slow_len = d.slow_len;
    r.p_slow = d.p_slow;
    r.mu_log = d.mu_log;
    r.sigma_log = d.sigma_log;
    r.cap = d.cap;
    r.table_n = 0;
    for (const auto& [len, w] : d.table) {
        if (r.table_n >= static_cast<int>(sizeof(r.table_len) / sizeof(r.table_len[0]))) break;
        r.table_len[r.table_n] = len;
        r.table_w[r.table_n] = w;
        ++r.table_n;
    }
    return r;
}

oppo_latency from_ref(const LatencyModel& m) {
    oppo_latency l{};
    l.decode_per_token = m.decode_per_token;
    l.prefill_per_token = m.prefill_per_token;
    l.reward_residual = m.reward_residual;
    l.chunk_switch_cost = m.chunk_switch_cost;
    l.transfer_per_chunk = m.transfer_per_chunk;
    l.placement = static_cast<int32_t>(m.placement);
    l.count_prompt_in_prefill = m.count_prompt_in_prefill ? 1 : 0;
    return l;
}

// rlpipe::RunConfig as the C struct (inverse of to_ref), so the reference arm
// of bench.py builds its configs from the reference alone.
void from_ref(const RunConfig& r, oppo_run_config& c) {
    std::memset(&c, 0, sizeof(c));
    c.mode = static_cast<int32_t>(r.mode);
    c.steps = r.steps;
    c.batch_size = r.batch_size;
    c.prompt_len = r.prompt_len;
    c.prompt_count = r.prompt_count;
    c.delta_init = r.delta_init;
    c.delta_min = r.delta_min;
    c.delta_max = r.delta_max;
    c.controller = static_cast<int32_t>(r.controller);
    c.window = r.window;
    c.delta_inc = r.delta_inc;
    c.delta_dec = r.delta_dec;
    c.chunk_size = r.chunk_size;
    c.schedule_mode = static_cast<int32_t>(r.schedule_mode);
    c.tune_chunks = r.tune_chunks ? 1 : 0;
    c.n_candidates = 0;
    for (int x : r.chunk_candidates) {
        if (c.n_candidates >= static_cast<int>(sizeof(c.chunk_candidates) / sizeof(c.chunk_candidates[0]))) break;
        c.chunk_candidates[c.n_candidates++] = x;
    }
    c.retune_period = r.retune_period;
    c.latency = from_ref(r.latency);
    c.lengths = from_ref(r.lengths);
    c.ppo.gamma = r.ppo.gamma;
    c.ppo.lambda = r.ppo.lambda;
    c.ppo.clip_epsilon = r.ppo.clip_epsilon;
    c.ppo.learning_rate = r.ppo.learning_rate;
    c.ppo.value_learning_rate = r.ppo.value_learning_rate;
    c.vocab = r.vocab;
    c.target_token = r.target_token;
    c.reward_scale = r.reward_scale;
    c.reward_bias = r.reward_bias;
    c.proxy_kind = static_cast<int32_t>(r.reward_proxy.kind);
    c.proxy_value = r.reward_proxy.value;
    c.proxy_ramp_scale = r.reward_proxy.ramp_scale;
    c.proxy_ramp_steps = r.reward_proxy.ramp_steps;
    c.fail_after_step = r.fail_after_step;
}

SequenceState to_ref(const oppo_seq_state& s) {
    SequenceState r;
    r.prompt.id = s.id;
    r.prompt.prompt_len = s.prompt_len;
    r.prompt.arrival_step = s.arrival_step;
    r.target_len = s.target_len;
    r.generated = s.generated;
    r.prefilled_tokens = s.prefilled_tokens;
    r.chunks_emitted = s.chunks_emitted;
    r.chunks_prefilled = s.chunks_prefilled;
    r.finished = s.finished != 0;
    r.scored = s.scored != 0;
    r.admitted_at = s.admitted_at;
    r.deferrals = s.deferrals;
    return r;
}

oppo_seq_state from_ref(const SequenceState& s) {
    oppo_seq_state r{};
    r.id = s.prompt.id;
    r.prompt_len = s.prompt.prompt_len;
    r.arrival_step = s.prompt.arrival_step;
    r.target_len = s.target_len;
    r.generated = s.generated;
    r.prefilled_tokens = s.prefilled_tokens;
    r.chunks_emitted = s.chunks_emitted;
    r.chunks_prefilled = s.chunks_prefilled;
    r.finished = s.finished;
    r.scored = s.scored;
    r.admitted_at = s.admitted_at;
    r.deferrals = s.deferrals;
    return r;
}

void fill_record(oppo_step_record& o, const StepRecord& r) {
    std::memset(&o, 0, sizeof(o));
    o.step = r.step;
    o.wall_ticks = r.wall_ticks;
    o.finished = r.finished;
    o.deferred = r.deferred;
    o.delta = r.delta;
    o.has_controller_stat = r.controller_stat.has_value();
    o.controller_stat = r.controller_stat.value_or(0.0);
    o.mean_reward = r.mean_reward;
    o.util_generation = r.util_generation;
    o.util_scoring = r.util_scoring;
    o.max_deferrals = r.max_deferrals;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Rng::derive(seed, purpose) then n draws: kind 0 next_u64, 1 uniform01, 2 normal.
int ref_rng_draws(uint64_t seed, const char* purpose, int kind, int64_t n, void* out) {
    return guard([&] {
        Rng rng = Rng::derive(seed, purpose);
        for (int64_t i = 0; i < n; ++i) {
            if (kind == 0) static_cast<uint64_t*>(out)[i] = rng.next_u64();
            else if (kind == 1) static_cast<double*>(out)[i] = rng.uniform01();
            else static_cast<double*>(out)[i] = rng.normal();
        }
    });
}

int ref_sample_lengths(const oppo_length_dist* d, uint64_t seed, int64_t n, int32_t* out) {
    return guard([&] {
        const auto dist = to_ref(*d);
        Rng rng = Rng::derive(seed, "lengths");
        for (int64_t i = 0; i < n; ++i) out[i] = sample_response_length(dist, rng);
    });
}

int ref_build_schedule(const oppo_seq_state* seqs, int n, int chunk, int mode,
                       oppo_chunk_task* tasks, int cap, int* n_tasks) {
    return guard([&] {
        std::vector<SequenceState> v;
        for (int i = 0; i < n; ++i) v.push_back(to_ref(seqs[i]));
        const auto sch = build_schedule(v, chunk, static_cast<ScheduleMode>(mode));
        int k = 0;
        for (const auto& p : sch.sequences)
            for (const auto& c : p.chunks) {
                if (k >= cap) throw InputError("task buffer too small");
                tasks[k++] = {p.seq_id, c.range.first, c.range.last, c.index,
                              c.needs_decode ? 1 : 0};
            }
        *n_tasks = k;
    });
}

// run_step over build_schedule(active, chunk, mode); stop_after <= 0 = none.
int ref_run_step(const oppo_seq_state* seqs, int n, int chunk, int mode,
                 const oppo_latency* lat, int stop_after, oppo_seq_outcome* out,
                 oppo_ledger* ledger) {
    return guard([&] {
        std::vector<SequenceState> v;
        for (int i = 0; i < n; ++i) v.push_back(to_ref(seqs[i]));
        const auto sch = build_schedule(v, chunk, static_cast<ScheduleMode>(mode));
        std::optional<int> stop;
        if (stop_after > 0) stop = stop_after;
        const auto [tl, led] = run_step(v, sch, to_ref(*lat), stop);
        for (size_t i = 0; i < tl.sequences.size(); ++i) {
            const auto& o = tl.sequences[i];
            out[i] = {o.seq_id, o.score_ready ? *o.score_ready : -1, o.tokens_decoded,
                      o.tokens_prefilled, o.decode_chunks_completed,
                      o.prefill_tasks_completed, o.carry_prefill_completed ? 1 : 0, 0};
        }
        std::memset(ledger, 0, sizeof(*ledger));
        ledger->wall = led.wall;
        ledger->busy_generation = led.busy_generation;
        ledger->busy_scoring = led.busy_scoring;
        ledger->work_generation = led.work_generation;
        ledger->work_scoring = led.work_scoring;
    });
}

int ref_select_finished(oppo_seq_state* entries, int n, const oppo_seq_outcome* outs,
                        int n_out, int batch, oppo_seq_state* sel, int* n_sel, int* n_rem,
                        int* short_batch) {
    return guard([&] {
        OvercommitBuffer buf;
        buf.batch_size = batch;
        for (int i = 0; i < n; ++i) buf.entries.push_back(to_ref(entries[i]));
        StepTimeline tl;
        for (int i = 0; i < n_out; ++i) {
            SequenceOutcome o;
            o.seq_id = outs[i].seq_id;
            if (outs[i].score_ready >= 0) o.score_ready = outs[i].score_ready;
            o.tokens_decoded = outs[i].tokens_decoded;
            o.tokens_prefilled = outs[i].tokens_prefilled;
            o.decode_chunks_completed = outs[i].decode_chunks_completed;
            o.prefill_tasks_completed = outs[i].prefill_tasks_completed;
            o.carry_prefill_completed = outs[i].carry_prefill_completed != 0;
            tl.sequences.push_back(o);
        }
        const auto r = select_finished(buf, tl, batch);
        for (size_t i = 0; i < r.ppo_batch.size(); ++i) sel[i] = from_ref(r.ppo_batch[i]);
        *n_sel = static_cast<int>(r.ppo_batch.size());
        for (size_t i = 0; i < buf.entries.size(); ++i) entries[i] = from_ref(buf.entries[i]);
        *n_rem = static_cast<int>(buf.entries.size());
        *short_batch = r.short_batch;
    });
}

int ref_delta_update(int mode, int window, int dmin, int dmax, int inc, int dec,
                     double* hist, int* n_hist, int delta, int* new_delta, int* has_stat,
                     double* stat) {
    return guard([&] {
        DeltaController c;
        c.mode = static_cast<DeltaMode>(mode);
        c.window = window;
        c.delta_min = dmin;
        c.delta_max = dmax;
        c.inc = inc;
        c.dec = dec;
        c.reward_history.assign(hist, hist + *n_hist);
        const auto u = c.update(delta);
        *new_delta = u.delta;
        *has_stat = u.stat.has_value();
        *stat = u.stat.value_or(0.0);
        std::copy(c.reward_history.begin(), c.reward_history.end(), hist);
        *n_hist = static_cast<int>(c.reward_history.size());
    });
}

// retune_chunk_size replay: feeds (candidate, ticks) pairs in order, writes the
// chosen `current` after each.
int ref_tuner_replay(const int* candidates, int n_cand, int window, const int* meas_cand,
                     const double* meas_ticks, int n_meas, int* chosen) {
    return guard([&] {
        TunerState t = make_tuner(std::vector<int>(candidates, candidates + n_cand), window);
        for (int i = 0; i < n_meas; ++i) {
            t = retune_chunk_size(t, meas_cand[i], meas_ticks[i]);
            chosen[i] = t.current;
        }
    });
}

// rlpipe::run_seed itself (driver.cpp:69-202).  Returns n_records; complete in *complete.
int ref_run_seed(const oppo_run_config* cfg, uint64_t seed, oppo_step_record* recs,
                 int* n_recs, int* complete) {
    return guard([&] {
        const auto run = run_seed(to_ref(*cfg), seed);
        for (size_t i = 0; i < run.steps.size(); ++i) fill_record(recs[i], run.steps[i]);
        *n_recs = static_cast<int>(run.steps.size());
        *complete = run.complete;
    });
}

// rlpipe::load_config_text + config_echo + RunConfig::task_fingerprint
// (config.cpp:75-250, :306-409), and the echo of RunConfig::baseline()
// (config.cpp:411-420): the JSON config schema parity tests.
// Returns 0 (ok: echo / baseline echo / fingerprint filled), 1 (ConfigError:
// message in err), 2 (other error).
int ref_load_config(const char* text, char* echo, char* base_echo, int cap, char* fp, char* err,
                    int err_cap) {
    try {
        const RunConfig c = load_config_text(text);
        const std::string e = config_echo(c), b = config_echo(c.baseline()), f = c.task_fingerprint();
        std::snprintf(echo, cap, "%s", e.c_str());
        std::snprintf(base_echo, cap, "%s", b.c_str());
        std::snprintf(fp, 17, "%s", f.c_str());
        return 0;
    } catch (const ConfigError& x) {
        std::snprintf(err, err_cap, "%s", x.what());
        return 1;
    } catch (const std::exception& x) {
        std::snprintf(err, err_cap, "%s", x.what());
        return 2;
    }
}

// rlpipe::run_experiment_in_memory + write_outputs (driver.cpp:228-350):
// steps_<seed>.csv, tuner_<seed>.csv and summary.json of the reference, for
// the run-output compatibility tests.
int ref_write_outputs(const oppo_run_config* cfg, const uint64_t* seeds, int n_seeds, const char* dir) {
    return guard([&] {
        RunConfig config = to_ref(*cfg);
        config.seeds.assign(seeds, seeds + n_seeds);
        const auto exp = run_experiment_in_memory(config);
        write_outputs(exp, std::filesystem::path(dir));
    });
}

// RunConfig{} defaults (config.hpp:28-77); with base != 0, of RunConfig::baseline()
// applied to *cfg (config.cpp:411-420).
int ref_run_config_default(oppo_run_config* out) {
    return guard([&] { from_ref(RunConfig{}, *out); });
}
int ref_run_config_baseline(const oppo_run_config* cfg, oppo_run_config* out) {
    return guard([&] {
        const RunConfig b = to_ref(*cfg).baseline();
        oppo_run_config c{};
        from_ref(b, c);
        c.carry_granularity = cfg->carry_granularity;  // engine-side field, not in rlpipe
        *out = c;
    });
}

// Runs rlpipe::run_seed for each seed on its own std::thread (the reference
// is single-threaded per seed); returns total finished samples.
int ref_run_seeds_parallel(const oppo_run_config* cfg, const uint64_t* seeds, int n_seeds,
                           int64_t* total_finished);

// Traced copy of the run_seed step loop (driver.cpp:103-195) built only from
// reference functions; records selected ids (batch slots per step, -1 pad)
// and the buffer state after selection (entries, up to buf_cap per step).
int ref_trace_seed(const oppo_run_config* c, uint64_t seed, oppo_step_record* recs,
                   int* n_recs, int64_t* sel_ids, oppo_seq_state* buf_states, int buf_cap,
                   int* buf_counts) {
    return guard([&] {
        const RunConfig config = to_ref(*c);
        config.validate();
        Rng length_rng = Rng::derive(seed, "lengths");
        StreamPromptSource source(config.prompt_len, config.prompt_count);
        OvercommitBuffer buffer;
        buffer.batch_size = config.batch_size;
        buffer.delta = config.delta_init;
        DeltaController controller;
        controller.mode = config.controller;
        controller.window = config.window;
        controller.delta_min = config.delta_min;
        controller.delta_max = config.delta_max;
        controller.inc = config.delta_inc;
        controller.dec = config.delta_dec;
        const bool tuning = config.mode == RunMode::Tune || config.tune_chunks;
        TunerState tuner;
        if (tuning) tuner = make_tuner(config.chunk_candidates, config.retune_period);
        int delta = config.delta_init;
        int max_def = 0;
        int n = 0;
        for (int step = 0; step < config.steps; ++step) {
            buffer.delta = delta;
            refill(buffer, source, step, config.lengths, length_rng);
            if (buffer.entries.empty()) break;
            int chunk = config.chunk_size;
            std::optional<int> explored;
            if (tuning) {
                explored = tuner_exploration_candidate(tuner, step % config.retune_period);
                chunk = explored ? *explored : tuner.current;
            }
            std::vector<SequenceState> active;
            int pre = 0;
            for (const auto& e : buffer.entries) {
                if (e.scored) ++pre;
                else active.push_back(e);
            }
            StepTimeline tl;
            ResourceLedger led;
            const int need = config.batch_size - pre;
            if (!active.empty() && need > 0) {
                const auto sch = build_schedule(active, chunk, config.schedule_mode);
                std::tie(tl, led) = run_step(active, sch, config.latency, need);
            }
            const auto sel = select_finished(buffer, tl, config.batch_size);
            for (const auto& e : buffer.entries) max_def = std::max(max_def, e.deferrals);
            double reward = 0.0;
            {
                const auto& p = config.reward_proxy;
                reward = p.value;
                if (p.kind == RewardProxy::Kind::Ramp)
                    reward = p.value + p.ramp_scale * std::min(step, p.ramp_steps) /
                                           static_cast<double>(std::max(1, p.ramp_steps));
            }
            controller.observe(reward);
            const auto up = controller.update(delta);
            StepRecord r;
            r.step = step;
            r.wall_ticks = tl.wall;
            r.finished = static_cast<int>(sel.ppo_batch.size());
            r.deferred = sel.deferred;
            r.delta = delta;
            r.controller_stat = up.stat;
            r.mean_reward = reward;
            if (tl.wall > 0) {
                const auto u = utilization(led);
                r.util_generation = u.generation;
                r.util_scoring = u.scoring;
            }
            r.max_deferrals = max_def;
            fill_record(recs[n], r);
            recs[n].chunk_size = chunk;
            recs[n].pre_scored = pre;
            for (int i = 0; i < config.batch_size; ++i)
                sel_ids[static_cast<size_t>(n) * config.batch_size + i] =
                    i < static_cast<int>(sel.ppo_batch.size()) ? sel.ppo_batch[i].prompt.id
                                                                : -1;
            if (buf_states) {
                const int k = std::min<int>(buf_cap, static_cast<int>(buffer.entries.size()));
                for (int i = 0; i < k; ++i)
                    buf_states[static_cast<size_t>(n) * buf_cap + i] = from_ref(buffer.entries[i]);
                buf_counts[n] = k;
            }
            if (tuning && explored) tuner = retune_chunk_size(tuner, *explored, tl.wall);
            delta = up.delta;
            ++n;
        }
        *n_recs = n;
    });
}

// ------------------------------------------------------------------ ppo-core
// Ragged batch: n samples, offsets[n+1] token prefix; values at offsets[i]+i
// (len+1 each); prefix_ends unused (final prefix = whole response).
static TrajectoryBatch make_batch(int n, const int32_t* offsets, const int32_t* tokens,
                                  const double* old_lp, const double* values,
                                  const double* rewards) {
    TrajectoryBatch b;
    for (int i = 0; i < n; ++i) {
        TrajectorySample s;
        s.prompt = {i, 1, 0};
        const int len = offsets[i + 1] - offsets[i];
        s.response.assign(tokens + offsets[i], tokens + offsets[i + 1]);
        s.old_logprobs.assign(old_lp + offsets[i], old_lp + offsets[i + 1]);
        if (values) s.values.assign(values + offsets[i] + i, values + offsets[i] + i + len + 1);
        s.reward = rewards[i];
        s.prefix_ends = {len};
        b.samples.push_back(std::move(s));
    }
    return b;
}

static PpoHyperparams hp_of(double g, double l, double eps) {
    PpoHyperparams hp;
    hp.gamma = g;
    hp.lambda = l;
    hp.clip_epsilon = eps;
    return hp;
}

int ref_compute_gae(const double* rewards, const double* values, int t, double gamma,
                    double lambda, double* out) {
    return guard([&] {
        const auto a = compute_gae(std::vector<double>(rewards, rewards + t),
                                   std::vector<double>(values, values + t + 1), gamma, lambda);
        std::copy(a.begin(), a.end(), out);
    });
}

// Tabular policy: theta (V+1)*V, value V+1.
static PolicyParams policy_of(int vocab, const double* theta, const double* value) {
    PolicyParams p = PolicyParams::uniform(vocab);
    if (theta) std::copy(theta, theta + p.theta.size(), p.theta.begin());
    if (value) std::copy(value, value + p.value.size(), p.value.begin());
    return p;
}

int ref_clipped_objective(int vocab, const double* theta, int n, const int32_t* offsets,
                          const int32_t* tokens, const double* old_lp, const double* values,
                          const double* rewards, double gamma, double lambda, double eps,
                          double* obj, double* grad) {
    return guard([&] {
        const auto b = make_batch(n, offsets, tokens, old_lp, values, rewards);
        const auto p = policy_of(vocab, theta, nullptr);
        const auto hp = hp_of(gamma, lambda, eps);
        *obj = clipped_objective(b, p, hp);
        if (grad) {
            const auto g = clipped_objective_grad(b, p, hp);
            std::copy(g.begin(), g.end(), grad);
        }
    });
}

int ref_policy_logprobs(int vocab, const double* theta, int state, double* out) {
    return guard([&] {
        const auto lp = policy_logprobs(policy_of(vocab, theta, nullptr), state);
        std::copy(lp.begin(), lp.end(), out);
    });
}

// rollout (ppo.cpp:241-272) from Rng::derive(seed, "ppo"); lengths[n] in order.
int ref_rollouts(int vocab, const double* theta, int target_token, double scale, double bias,
                 uint64_t seed, int n, const int32_t* lengths, int32_t* tokens, double* old_lp,
                 double* rewards) {
    return guard([&] {
        ToyEnv env{vocab, target_token, scale, bias};
        const auto p = policy_of(vocab, theta, nullptr);
        Rng rng = Rng::derive(seed, "ppo");
        int64_t off = 0;
        for (int i = 0; i < n; ++i) {
            const auto s = rollout(env, p, {i, 1, 0}, lengths[i], {}, rng);
            std::copy(s.response.begin(), s.response.end(), tokens + off);
            std::copy(s.old_logprobs.begin(), s.old_logprobs.end(), old_lp + off);
            rewards[i] = s.reward;
            off += lengths[i];
        }
    });
}

// toy_rlhf_step (ppo.cpp:281-317) on a batch; theta/value updated in place.
int ref_toy_rlhf_step(int vocab, int target_token, double scale, double bias, double* theta,
                      double* value, int n, const int32_t* offsets, const int32_t* tokens,
                      const double* old_lp, const double* rewards, double gamma, double lambda,
                      double eps, double lr, double vlr, double* mean_reward) {
    return guard([&] {
        ToyEnv env{vocab, target_token, scale, bias};
        PolicyParams p = policy_of(vocab, theta, value);
        auto b = make_batch(n, offsets, tokens, old_lp, nullptr, rewards);
        for (auto& s : b.samples) fill_values(s, p);
        PpoHyperparams hp = hp_of(gamma, lambda, eps);
        hp.learning_rate = lr;
        hp.value_learning_rate = vlr;
        *mean_reward = toy_rlhf_step(env, p, b, hp);
        std::copy(p.theta.begin(), p.theta.end(), theta);
        std::copy(p.value.begin(), p.value.end(), value);
    });
}

} // extern "C"

#include <thread>
extern "C" int ref_run_seeds_parallel(const oppo_run_config* cfg, const uint64_t* seeds,
                                      int n_seeds, int64_t* total_finished) {
    return guard([&] {
        const RunConfig c = to_ref(*cfg);
        std::vector<int64_t> fin(static_cast<size_t>(n_seeds), 0);
        std::vector<std::thread> th;
        for (int i = 0; i < n_seeds; ++i)
            th.emplace_back([&, i] {
                const auto run = run_seed(c, seeds[i]);
                int64_t f = 0;
                for (const auto& r : run.steps) f += r.finished;
                fin[static_cast<size_t>(i)] = f;
            });
        for (auto& t : th) t.join();
        int64_t tot = 0;
        for (auto f : fin) tot += f;
        *total_finished = tot;
    });
}
