// sched.hpp — host-side OPPO scheduler (C++20, namespace oppo).
//
// Restates, field for field, the scheduling semantics of the reference
// (`/root/reference/proj/core`): deterministic RNG streams, response-length
// draws, chunk schedules, overcommit refill/selection, Delta controllers and
// the chunk-size tuner.  The step executor itself is NOT here: it is the GPU
// engine (engine.cu), whose decisions follow the logical lockstep clock that
// plan_step() computes.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "oppo/oppo.h"

namespace oppo {

// Error taxonomy mapped 1:1 onto rlpipe's (errors.hpp:9-24) and onto oppo_status.
struct Error : std::runtime_error {
    oppo_status code;
    Error(oppo_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void config_error(const std::string& m) { throw Error(OPPO_ERR_CONFIG, m); }
[[noreturn]] inline void input_error(const std::string& m) { throw Error(OPPO_ERR_INPUT, m); }
[[noreturn]] inline void internal_error(const std::string& m) {
    throw Error(OPPO_ERR_INTERNAL, m);
}

// Purpose-keyed splittable stream (rng.hpp:15-67): mt19937_64 seeded with
// splitmix64(root ^ FNV-1a(purpose)).
class Stream {
public:
    static Stream derive(uint64_t root, std::string_view purpose);
    explicit Stream(uint64_t seed) : mt_(seed) {}
    uint64_t u64() { return mt_(); }
    double uniform() { return double(mt_() >> 11) * 0x1.0p-53; }
    double gauss();  // Box-Muller; cosine branch first, sine cached

private:
    std::mt19937_64 mt_;
    bool cached_ = false;
    double spare_ = 0.0;
};

uint64_t splitmix64(uint64_t x);
uint64_t fnv1a(std::string_view s, uint64_t h = 0xcbf29ce484222325ull);

// Length distribution draw (model.cpp:50-72).
void check_lengths(const oppo_length_dist& d);
int draw_length(const oppo_length_dist& d, Stream& rng);

// Chunked work list of one sequence (chunking.cpp:20-48).
struct Chunk {
    int first, last, index;
    bool needs_decode;
};
std::vector<Chunk> chunks_for(const oppo_seq_state& s, int chunk_size);

// Logical lockstep executor: outcomes of one step when each decode iteration
// is one tick and scoring is free (what the GPU realises).
struct StepPlan {
    int64_t t_end = 0;                       // decode iterations to run
    std::vector<oppo_seq_outcome> outcomes;  // input order
    oppo_ledger ledger{};
    std::vector<int64_t> finish_iter;        // per seq: iteration its decode ends (0 = none)
};
StepPlan plan_step(const std::vector<oppo_seq_state>& active, int chunk_size, int mode,
                   int stop_after, int carry_granularity);

// Overcommit buffer (overcommit.hpp:39-44) and its two mutators.
struct Buffer {
    std::vector<oppo_seq_state> entries;  // FIFO: carried first, then new
    int batch_size = 1;
    int delta = 0;
    int capacity() const { return batch_size + delta; }
};
struct PromptStream {  // StreamPromptSource (overcommit.hpp:23-37)
    int prompt_len;
    int64_t total;
    int64_t issued = 0;
    // data parallel: rank r of N serves prompt ids = r (mod N)
    int rank = 0, world = 1;
    // KV admission control: a prompt drawn (with its length) that did not fit
    // waits here and is admitted first at the next refill
    bool has_pending = false;
    oppo_seq_state pending{};
    bool next(int step, oppo_seq_state& out);
};
int refill(Buffer& b, PromptStream& src, int step, const oppo_length_dist& d, Stream& rng);
// refill with admission control: a candidate (length already drawn) enters
// only if fits(candidate) — the engine has a slot and KV pages for it; else
// it is held in src.pending and refill stops (the reference's refill is this
// with fits == always true, overcommit.cpp:11-28)
template <class Fits>
int refill_fit(Buffer& b, PromptStream& src, int step, const oppo_length_dist& d, Stream& rng, Fits&& fits);

struct Selection {
    std::vector<oppo_seq_state> batch;  // earliest score-ready first
    int deferred = 0;
    bool short_batch = false;
};
Selection select_finished(Buffer& b, const std::vector<oppo_seq_outcome>& outcomes,
                          int batch_size);

// Reward-driven overcommit controller (overcommit.cpp:97-155).
struct DeltaCtl {
    int mode = OPPO_DELTA_ALG1;
    int window = 8, dmin = 0, dmax = 8, inc = 1, dec = 1;
    std::vector<double> history;
    struct Result {
        int delta;
        std::optional<double> stat;
    };
    void check() const;
    Result update(int delta);
};

// Periodic chunk-size tuner (chunking.cpp:61-107).
struct Tuner {
    std::vector<int> candidates;
    int window = 50;
    int current = 0;
    std::map<int, std::pair<double, int>> trials;
    static Tuner make(std::vector<int> candidates, int window);
    void fold(int candidate, double mean_step);
    std::optional<int> explore(int step_in_period) const;
};

void config_defaults(oppo_run_config& c);
oppo_run_config config_baseline(const oppo_run_config& c);
void validate(const oppo_run_config& c);
int draw_length(const oppo_length_dist& d, Stream& rng);

template <class Fits>
int refill_fit(Buffer& b, PromptStream& src, int step, const oppo_length_dist& d, Stream& rng, Fits&& fits) {
    if (b.batch_size < 1) config_error("batch size must be >= 1");
    if (static_cast<int>(b.entries.size()) > b.capacity()) internal_error("buffer over capacity at refill");
    int added = 0;
    while (static_cast<int>(b.entries.size()) < b.capacity()) {
        oppo_seq_state s;
        if (src.has_pending) {
            s = src.pending;
            src.has_pending = false;
        } else {
            if (!src.next(step, s)) break;
            s.target_len = draw_length(d, rng);  // length drawn at admission (overcommit.cpp:22)
            s.admitted_at = step;
        }
        if (!fits(s)) {
            if (b.entries.empty()) input_error("a single sequence needs more KV pages / slots than the engine has");
            src.pending = s;
            src.has_pending = true;
            break;
        }
        b.entries.push_back(s);
        ++added;
    }
    return added;
}

double proxy_reward(const oppo_run_config& c, int step);

}  // namespace oppo
