// sched.cpp — host-side OPPO scheduler.  See sched.hpp; reference citations
// are file:line under /root/reference/proj/core.
#include "sched.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <unordered_map>

namespace oppo {

// ------------------------------------------------------------------ streams

uint64_t splitmix64(uint64_t x) {  // rng.hpp:57-62
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

uint64_t fnv1a(std::string_view s, uint64_t h) {
    for (unsigned char c : s) h = (h ^ c) * 0x100000001b3ull;
    return h;
}

Stream Stream::derive(uint64_t root, std::string_view purpose) {  // rng.hpp:20-27
    return Stream(splitmix64(root ^ fnv1a(purpose)));
}

double Stream::gauss() {  // rng.hpp:41-54
    if (cached_) {
        cached_ = false;
        return spare_;
    }
    double a = uniform();
    const double b = uniform();
    while (a <= 0.0) a = uniform();
    const double radius = std::sqrt(-2.0 * std::log(a));
    const double angle = 2.0 * 3.141592653589793238462643383279502884 * b;
    spare_ = radius * std::sin(angle);
    cached_ = true;
    return radius * std::cos(angle);
}

// ------------------------------------------------------------------ lengths

void check_lengths(const oppo_length_dist& d) {  // model.cpp:10-45
    if (d.cap < 1) config_error("length distribution: cap must be >= 1");
    switch (d.kind) {
    case OPPO_LEN_TWO_POINT:
        if (d.fast_len < 1 || d.slow_len < 1) config_error("two-point lengths must be >= 1");
        if (d.fast_len > d.cap || d.slow_len > d.cap)
            config_error("two-point lengths must be <= cap");
        if (d.p_slow < 0.0 || d.p_slow > 1.0) config_error("two-point p_slow must be in [0,1]");
        break;
    case OPPO_LEN_LOGNORMAL:
        if (d.sigma_log < 0.0) config_error("lognormal sigma must be >= 0");
        break;
    case OPPO_LEN_EMPIRICAL: {
        if (d.table_n < 1 || d.table_n > OPPO_MAX_TABLE)
            config_error("empirical table must be non-empty");
        double total = 0.0;
        for (int i = 0; i < d.table_n; ++i) {
            if (d.table_len[i] < 1 || d.table_len[i] > d.cap)
                config_error("empirical table lengths must be in [1, cap]");
            if (d.table_w[i] < 0.0) config_error("empirical table weights must be >= 0");
            total += d.table_w[i];
        }
        if (total <= 0.0) config_error("empirical table needs positive total weight");
        break;
    }
    default:
        config_error("unknown length distribution kind");
    }
}

int draw_length(const oppo_length_dist& d, Stream& rng) {  // model.cpp:50-72
    check_lengths(d);
    if (d.kind == OPPO_LEN_TWO_POINT) return rng.uniform() < d.p_slow ? d.slow_len : d.fast_len;
    if (d.kind == OPPO_LEN_LOGNORMAL) {
        const long long n = std::llround(std::exp(d.mu_log + d.sigma_log * rng.gauss()));
        return static_cast<int>(std::min<long long>(std::max<long long>(n, 1), d.cap));
    }
    double total = 0.0;
    for (int i = 0; i < d.table_n; ++i) total += d.table_w[i];
    double u = rng.uniform() * total;
    for (int i = 0; i < d.table_n; ++i) {
        u -= d.table_w[i];
        if (u < 0.0) return d.table_len[i];
    }
    return d.table_len[d.table_n - 1];
}

// --------------------------------------------------------------- schedules

std::vector<Chunk> chunks_for(const oppo_seq_state& s, int chunk_size) {
    if (chunk_size < 1) config_error("chunk size must be >= 1");
    std::vector<Chunk> out;
    int index = 0;
    // decoded-but-unprefilled tokens leave first, as one ready chunk (chunking.cpp:32-37)
    if (s.prefilled_tokens < s.generated)
        out.push_back({s.prefilled_tokens + 1, s.generated, index++, false});
    if (s.generated < s.target_len) {  // undone work, partitioned from `generated` (:38-44)
        for (int first = s.generated + 1; first <= s.target_len; first += chunk_size)
            out.push_back({first, std::min(first + chunk_size - 1, s.target_len), index++, true});
    }
    return out;
}

// The logical clock.  Under {decode=1/token, prefill=0, residual=0,
// transfer=0, disaggregated} the reference's serial scoring queue
// (engine.cpp:109-142) never delays a task (every head is available no
// earlier than the queue clock), so each task completes at its availability:
//   - a carried chunk at tick 0;
//   - a new chunk at its decode completion (streamed) or at the sequence's
//     last decode (sequential) (engine.cpp:77-82);
//   - the residual at the last task's completion (engine.cpp:93-105).
// Score-ready of an active sequence is therefore its remaining decode length
// (0 if nothing is left to decode), and the cut (engine.cpp:161-172) is the
// stop_after-th smallest (time, id).
StepPlan plan_step(const std::vector<oppo_seq_state>& active, int chunk_size, int mode,
                   int stop_after, int carry_granularity) {
    if (active.empty()) input_error("run_step requires a non-empty active set");
    if (chunk_size < 1) config_error("chunk size must be >= 1");
    const size_t n = active.size();
    StepPlan plan;
    plan.finish_iter.resize(n);
    std::vector<std::pair<int64_t, int64_t>> scores;  // (tick, id)
    scores.reserve(n);
    int64_t t_full = 0;
    for (size_t i = 0; i < n; ++i) {
        const auto& s = active[i];
        if (s.generated > s.target_len) internal_error("sequence decoded past its target length");
        const int64_t rem = s.target_len - s.generated;
        plan.finish_iter[i] = rem;
        t_full = std::max(t_full, rem);
        scores.emplace_back(rem, s.id);
    }
    std::sort(scores.begin(), scores.end());
    const bool cut = stop_after >= 1 && stop_after <= static_cast<int>(n);
    plan.t_end = cut ? scores[static_cast<size_t>(stop_after) - 1].first : t_full;
    const int64_t t_end = plan.t_end;
    const bool streamed = mode == OPPO_MODE_STREAMED;

    plan.outcomes.resize(n);
    int64_t last_decode = 0, work_gen = 0;
    for (size_t i = 0; i < n; ++i) {
        const auto& s = active[i];
        auto& o = plan.outcomes[i];
        o = {};
        o.seq_id = s.id;
        o.score_ready = -1;
        const int64_t rem = plan.finish_iter[i];
        if (s.prefilled_tokens < s.generated) {  // carry chunk: ready at tick 0
            o.tokens_prefilled += s.generated - s.prefilled_tokens;
            o.prefill_tasks_completed += 1;
            o.carry_prefill_completed = 1;
        }
        if (rem > 0) {
            const bool done = rem <= t_end;
            const int64_t whole = done ? rem : (t_end / chunk_size) * chunk_size;
            const int n_chunks = static_cast<int>(done ? (rem + chunk_size - 1) / chunk_size
                                                       : t_end / chunk_size);
            int64_t kept = whole;
            if (carry_granularity == OPPO_CARRY_TOKEN) kept = std::min(rem, t_end);
            o.tokens_decoded = static_cast<int32_t>(kept);
            o.decode_chunks_completed = n_chunks;
            work_gen += kept;
            if (whole > 0) last_decode = std::max(last_decode, done ? rem : whole);
            if (carry_granularity == OPPO_CARRY_TOKEN && kept > 0)
                last_decode = std::max(last_decode, kept);
            if (streamed || done) {  // prefill follows decode (streamed) or the last decode
                o.tokens_prefilled += static_cast<int32_t>(whole);
                o.prefill_tasks_completed += n_chunks;
            }
        }
        if (rem <= t_end) o.score_ready = rem;
    }
    plan.ledger.wall = t_end;
    plan.ledger.work_generation = work_gen;
    plan.ledger.busy_generation = std::min(last_decode, t_end);
    return plan;
}

// --------------------------------------------------------------- overcommit

bool PromptStream::next(int step, oppo_seq_state& out) {
    if (total >= 0 && issued >= total) return false;
    out = {};
    out.id = issued * world + rank;
    ++issued;
    out.prompt_len = prompt_len;
    out.arrival_step = step;
    return true;
}

int refill(Buffer& b, PromptStream& src, int step, const oppo_length_dist& d, Stream& rng) {
    if (b.batch_size < 1) config_error("batch size must be >= 1");
    if (static_cast<int>(b.entries.size()) > b.capacity())
        internal_error("buffer over capacity at refill");
    int added = 0;
    oppo_seq_state s;
    while (static_cast<int>(b.entries.size()) < b.capacity() && src.next(step, s)) {
        s.target_len = draw_length(d, rng);  // length drawn at admission (overcommit.cpp:22)
        s.admitted_at = step;
        b.entries.push_back(s);
        ++added;
    }
    return added;
}

Selection select_finished(Buffer& b, const std::vector<oppo_seq_outcome>& outcomes,
                          int batch_size) {
    std::unordered_map<int64_t, const oppo_seq_outcome*> by_id;
    by_id.reserve(outcomes.size());
    for (const auto& o : outcomes) by_id.emplace(o.seq_id, &o);

    struct Ready {
        int64_t tick, id;
        size_t pos;
    };
    std::vector<Ready> ready;
    for (size_t pos = 0; pos < b.entries.size(); ++pos) {
        auto& s = b.entries[pos];
        const bool was_scored = s.scored != 0;
        const auto it = by_id.find(s.id);
        if (it == by_id.end()) {
            if (was_scored) ready.push_back({-1, s.id, pos});
            continue;
        }
        const auto& o = *it->second;
        const int emitted_before = s.chunks_emitted;
        s.generated += o.tokens_decoded;
        s.chunks_emitted += o.decode_chunks_completed;
        s.prefilled_tokens += o.tokens_prefilled;
        // a completed carry task covers every chunk emitted before this step (overcommit.cpp:53-57)
        const int base = o.carry_prefill_completed ? emitted_before : s.chunks_prefilled;
        s.chunks_prefilled = base + o.prefill_tasks_completed - (o.carry_prefill_completed ? 1 : 0);
        if (s.generated > s.target_len) internal_error("sequence decoded past its target length");
        s.finished = s.generated == s.target_len;
        if (o.score_ready >= 0) s.scored = 1;
        if (s.chunks_prefilled > s.chunks_emitted)
            internal_error("prefilled chunk count exceeds emitted count");
        if (o.score_ready >= 0 || was_scored)
            ready.push_back({was_scored ? -1 : o.score_ready, s.id, pos});
    }
    std::sort(ready.begin(), ready.end(), [](const Ready& a, const Ready& c) {
        return a.tick != c.tick ? a.tick < c.tick : a.id < c.id;
    });
    Selection sel;
    const size_t take = std::min(ready.size(), static_cast<size_t>(batch_size));
    std::vector<char> taken(b.entries.size(), 0);
    for (size_t i = 0; i < take; ++i) {
        sel.batch.push_back(b.entries[ready[i].pos]);
        taken[ready[i].pos] = 1;
    }
    sel.short_batch = take < static_cast<size_t>(batch_size);
    std::vector<oppo_seq_state> left;
    left.reserve(b.entries.size() - take);
    for (size_t pos = 0; pos < b.entries.size(); ++pos) {
        if (taken[pos]) continue;
        b.entries[pos].deferrals += 1;  // every entry left behind, new ones included
        left.push_back(b.entries[pos]);
    }
    b.entries = std::move(left);
    sel.deferred = static_cast<int>(b.entries.size());
    return sel;
}

// --------------------------------------------------------------- controller

void DeltaCtl::check() const {
    if (window < 1) config_error("controller window must be >= 1");
    if (dmin > dmax) config_error("delta_min must be <= delta_max");
    if (dmin < 0) config_error("delta_min must be >= 0");
    if (inc < 1 || dec < 1) config_error("delta momenta must be >= 1");
}

DeltaCtl::Result DeltaCtl::update(int delta) {
    if (mode == OPPO_DELTA_FIXED) return {delta, std::nullopt};
    check();
    const size_t w = static_cast<size_t>(window);
    const size_t n = history.size();
    auto mean = [&](size_t a, size_t b) {
        return std::accumulate(history.begin() + static_cast<std::ptrdiff_t>(a),
                               history.begin() + static_cast<std::ptrdiff_t>(b), 0.0) /
               static_cast<double>(b - a);
    };
    if (mode == OPPO_DELTA_ALG1) {  // windowed difference, overcommit.cpp:112-125
        if (n < 2 * w) return {delta, std::nullopt};
        const double d = mean(n - w, n) - mean(n - 2 * w, n - w);
        const int sign = (d > 0.0) - (d < 0.0);
        const int step = std::max(1, delta / 4);
        const int next = std::clamp(delta - sign * step, dmin, dmax);
        history.erase(history.begin(), history.end() - static_cast<std::ptrdiff_t>(w));
        return {next, d};
    }
    if (mode == OPPO_DELTA_EQ4) {  // telescoped slope, overcommit.cpp:140-152, :127-132
        if (n < w + 1) return {delta, std::nullopt};
        const double slope = (history[n - 1] - history[n - 1 - w]) / static_cast<double>(w);
        if (n > w + 1)
            history.erase(history.begin(), history.end() - static_cast<std::ptrdiff_t>(w + 1));
        const int next = slope > 0.0 ? std::min(dmax, delta + inc) : std::max(dmin, delta - dec);
        return {next, slope};
    }
    internal_error("unreachable controller mode");
}

// -------------------------------------------------------------------- tuner

Tuner Tuner::make(std::vector<int> c, int window) {
    std::sort(c.begin(), c.end());
    c.erase(std::unique(c.begin(), c.end()), c.end());
    if (c.empty()) config_error("tuner needs at least one candidate");
    if (window < 1) config_error("tuner window must be >= 1");
    for (int x : c)
        if (x < 1) config_error("tuner candidates must be >= 1");
    Tuner t;
    t.candidates = std::move(c);
    t.window = window;
    t.current = t.candidates.front();
    return t;
}

void Tuner::fold(int candidate, double mean_step) {  // chunking.cpp:73-100
    if (std::find(candidates.begin(), candidates.end(), candidate) == candidates.end())
        input_error("measurement for a chunk size that is not a candidate");
    auto& [sum, count] = trials[candidate];
    sum += mean_step;
    count += 1;
    if (trials.size() != candidates.size()) return;
    int best = candidates.front();
    double best_mean = 0.0;
    bool first = true;
    for (int c : candidates) {  // ascending: ties keep the smaller C
        const auto& [s, k] = trials.at(c);
        const double m = s / k;
        if (first || m < best_mean) {
            best = c;
            best_mean = m;
            first = false;
        }
    }
    current = best;
    trials.clear();
}

std::optional<int> Tuner::explore(int step_in_period) const {  // chunking.cpp:102-107
    if (step_in_period < 0 || step_in_period >= static_cast<int>(candidates.size()))
        return std::nullopt;
    return candidates[static_cast<size_t>(step_in_period)];
}

// ------------------------------------------------------------------- config

void config_defaults(oppo_run_config& c) {  // RunConfig{} (config.hpp:28-77)
    c = {};
    c.mode = OPPO_RUN_SIMULATE;
    c.steps = 100;
    c.batch_size = 8;
    c.prompt_len = 8;
    c.prompt_count = -1;
    c.delta_init = 0;
    c.delta_min = 0;
    c.delta_max = 8;
    c.controller = OPPO_DELTA_FIXED;
    c.window = 8;
    c.delta_inc = 1;
    c.delta_dec = 1;
    c.chunk_size = 256;
    c.schedule_mode = OPPO_MODE_STREAMED;
    c.tune_chunks = 0;
    c.n_candidates = 3;
    c.chunk_candidates[0] = 128;
    c.chunk_candidates[1] = 256;
    c.chunk_candidates[2] = 512;
    c.retune_period = 50;
    c.vocab = 4;
    c.target_token = 0;
    c.reward_scale = 1.0;
    c.reward_bias = 0.0;
    c.proxy_kind = 0;
    c.proxy_value = 1.0;
    c.proxy_ramp_scale = 1.0;
    c.proxy_ramp_steps = 100;
    c.fail_after_step = -1;
    c.carry_granularity = OPPO_CARRY_CHUNK;
    c.latency = {1, 1, 0, 0, 0, OPPO_PLACE_DISAGGREGATED, 1};
    c.lengths.kind = OPPO_LEN_TWO_POINT;
    c.lengths.fast_len = 100;
    c.lengths.slow_len = 600;
    c.lengths.p_slow = 0.0;
    c.lengths.mu_log = 5.0;
    c.lengths.sigma_log = 0.8;
    c.lengths.cap = 4096;
    c.ppo = {1.0, 1.0, 0.2, 0.1, 0.2, 0.0, 0, 0};
}

oppo_run_config config_baseline(const oppo_run_config& c) {  // config.cpp:411-420
    oppo_run_config b = c;
    b.delta_init = b.delta_min = b.delta_max = 0;
    b.controller = OPPO_DELTA_FIXED;
    b.schedule_mode = OPPO_MODE_SEQUENTIAL;
    b.tune_chunks = 0;
    return b;
}

void validate(const oppo_run_config& c) {  // config.cpp:253-289 (all violations listed)
    std::vector<std::string> e;
    if (c.steps < 1) e.push_back("steps must be >= 1");
    if (c.batch_size < 1) e.push_back("batch.size must be >= 1");
    if (c.prompt_len < 1) e.push_back("batch.prompt_len must be >= 1");
    if (c.delta_min > c.delta_max) e.push_back("delta.min must be <= delta.max");
    if (c.delta_min < 0) e.push_back("delta.min must be >= 0");
    if (c.delta_init < c.delta_min || c.delta_init > c.delta_max)
        e.push_back("delta.init must lie within [delta.min, delta.max]");
    if (c.window < 1) e.push_back("delta.window must be >= 1");
    if (c.delta_inc < 1 || c.delta_dec < 1) e.push_back("delta momenta must be >= 1");
    if (c.chunk_size < 1) e.push_back("chunk.size must be >= 1");
    if (c.retune_period < 1) e.push_back("chunk.retune_period must be >= 1");
    if (c.tune_chunks) {
        if (c.n_candidates < 1 || c.n_candidates > OPPO_MAX_CANDIDATES)
            e.push_back("chunk.candidates must be non-empty when tuning");
        for (int i = 0; i < c.n_candidates && i < OPPO_MAX_CANDIDATES; ++i)
            if (c.chunk_candidates[i] < 1) e.push_back("chunk.candidates must all be >= 1");
        if (c.retune_period < c.n_candidates)
            e.push_back("chunk.retune_period must cover one step per candidate");
    }
    if (c.vocab < 2 || c.vocab > 16) e.push_back("ppo.vocab must be in [2,16]");
    if (c.target_token < 0 || c.target_token >= c.vocab)
        e.push_back("ppo.target_token must be a vocabulary token");
    const auto& l = c.latency;
    if (l.decode_per_token < 0 || l.prefill_per_token < 0 || l.reward_residual < 0 ||
        l.chunk_switch_cost < 0 || l.transfer_per_chunk < 0)
        e.push_back("latency model: all tick costs must be >= 0");
    try {
        check_lengths(c.lengths);
    } catch (const Error& x) {
        e.push_back(x.what());
    }
    const auto& p = c.ppo;
    if (p.gamma < 0.0 || p.gamma > 1.0) e.push_back("gamma must be in [0,1]");
    if (p.lambda < 0.0 || p.lambda > 1.0) e.push_back("lambda must be in [0,1]");
    if (!(p.clip_epsilon > 0.0)) e.push_back("clip epsilon must be > 0");
    if (!(p.learning_rate > 0.0)) e.push_back("learning rate must be > 0");
    if (!(p.value_learning_rate > 0.0)) e.push_back("value learning rate must be > 0");
    if (c.carry_granularity != OPPO_CARRY_CHUNK && c.carry_granularity != OPPO_CARRY_TOKEN)
        e.push_back("carry_granularity must be chunk|token");
    if (!e.empty()) {
        std::string all = "config rejected:";
        for (const auto& s : e) all += "\n  - " + s;
        config_error(all);
    }
}

double proxy_reward(const oppo_run_config& c, int step) {  // driver.cpp:21-32
    if (c.proxy_kind == 1) {
        const double f = std::min(step, c.proxy_ramp_steps) /
                         static_cast<double>(std::max(1, c.proxy_ramp_steps));
        return c.proxy_value + c.proxy_ramp_scale * f;
    }
    return c.proxy_value;
}

}  // namespace oppo
