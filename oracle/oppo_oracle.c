/*
 * oppo_oracle.c — TEST INFRASTRUCTURE ONLY: a plain-C CPU restatement of the
 * reference's hot path, used as the checker by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg.  The product (liboppo.so) never links it.
 *
 * Pinned against the compiled reference (oracle/_ref) and its golden vectors
 * (tests/golden/reference_vectors.json) by tests/test_oracle.py:
 *   - Rng (rng.hpp:15-67): mt19937_64 seeded by splitmix64(root ^ FNV-1a(purpose))
 *   - sample_response_length (model.cpp:50-72)
 *   - build_schedule (chunking.cpp:20-48), run_step (engine.cpp:24-223)
 *   - select_finished / refill (overcommit.cpp:11-95), DeltaController (:97-155)
 *   - tuner (chunking.cpp:61-107), run_seed loop (driver.cpp:103-195)
 *   - compute_gae / clipped_objective / clipped_objective_grad (ppo.cpp:71-177)
 * Extensions with NO reference counterpart ("parity unpinned" by the
 * reference; pinned only by this restatement and its own tests):
 *   - run_step's credit_partial rule (north_star token-granular carry): tokens
 *     of the chunk in flight at the cut are kept instead of discarded
 *     (engine.cpp:190 otherwise).
 *   - oracle_gpt_forward: fp64 Qwen2-style decoder (RMSNorm, RoPE theta 1e6,
 *     GQA, SwiGLU with interleaved gate/up rows, q/k/v bias) on the weights the
 *     engine exports; the counter-based sampling noise of the engine.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oppo/oppo.h"

/* ------------------------------------------------------------ mt19937_64 */
typedef struct {
    uint64_t mt[312];
    int idx;
    int have_spare;
    double spare;
} orng;

static void mt_seed(orng* r, uint64_t s) {
    r->mt[0] = s;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
    r->have_spare = 0;
    r->spare = 0.0;
}
static uint64_t mt_next(orng* r) {
    const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
            r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t x = r->mt[r->idx++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    return x;
}
static uint64_t o_splitmix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
static void rng_derive(orng* r, uint64_t root, const char* purpose) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (const unsigned char* p = (const unsigned char*)purpose; *p; ++p) h = (h ^ *p) * 0x100000001b3ull;
    mt_seed(r, o_splitmix(root ^ h));
}
static double rng_u01(orng* r) { return (double)(mt_next(r) >> 11) * 0x1.0p-53; }
static double rng_normal(orng* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    double u1 = rng_u01(r), u2 = rng_u01(r);
    while (u1 <= 0.0) u1 = rng_u01(r);
    const double rad = sqrt(-2.0 * log(u1)), a = 2.0 * 3.141592653589793238462643383279502884 * u2;
    r->spare = rad * sin(a);
    r->have_spare = 1;
    return rad * cos(a);
}

int oracle_rng_draws(uint64_t seed, const char* purpose, int kind, int64_t n, void* out) {
    orng r;
    rng_derive(&r, seed, purpose);
    for (int64_t i = 0; i < n; ++i) {
        if (kind == 0) ((uint64_t*)out)[i] = mt_next(&r);
        else if (kind == 1) ((double*)out)[i] = rng_u01(&r);
        else ((double*)out)[i] = rng_normal(&r);
    }
    return 0;
}

static int draw_length(const oppo_length_dist* d, orng* r) {
    if (d->kind == OPPO_LEN_TWO_POINT) return rng_u01(r) < d->p_slow ? d->slow_len : d->fast_len;
    if (d->kind == OPPO_LEN_LOGNORMAL) {
        long long n = llround(exp(d->mu_log + d->sigma_log * rng_normal(r)));
        if (n < 1) n = 1;
        if (n > d->cap) n = d->cap;
        return (int)n;
    }
    double tot = 0;
    for (int i = 0; i < d->table_n; ++i) tot += d->table_w[i];
    double u = rng_u01(r) * tot;
    for (int i = 0; i < d->table_n; ++i) {
        u -= d->table_w[i];
        if (u < 0.0) return d->table_len[i];
    }
    return d->table_len[d->table_n - 1];
}

int oracle_sample_lengths(const oppo_length_dist* d, uint64_t seed, int64_t n, int32_t* out) {
    orng r;
    rng_derive(&r, seed, "lengths");
    for (int64_t i = 0; i < n; ++i) out[i] = draw_length(d, &r);
    return 0;
}

/* --------------------------------------------------------------- run_step */
typedef struct {
    int first, last, needs_decode;
    int64_t done;  /* decode completion (0 for carried chunks) */
} ochunk;
typedef struct {
    int seq, chunk_index, is_residual, is_carry, size;
    int64_t avail, dur, done;
} otask;

/* Restates run_step (engine.cpp:24-223) for one step.  credit_partial = 1 keeps
 * the decoded tokens of each sequence's in-flight chunk at the cut. */
int oracle_run_step(const oppo_seq_state* seqs, int n, int C, int mode, const oppo_latency* lat,
                    int stop_after, int credit_partial, oppo_seq_outcome* out, oppo_ledger* led) {
    if (n <= 0 || C < 1) return 2;
    const int streamed = mode == OPPO_MODE_STREAMED;
    const int coloc = lat->placement == OPPO_PLACE_COLOCATED;
    int max_chunks = 0;
    for (int i = 0; i < n; ++i) max_chunks += (seqs[i].target_len - seqs[i].generated) / C + 3;
    ochunk* ch = calloc((size_t)max_chunks, sizeof(ochunk));
    otask* tk = calloc((size_t)max_chunks + n, sizeof(otask));
    int* c_off = calloc((size_t)n + 1, sizeof(int));
    int* t_off = calloc((size_t)n + 1, sizeof(int));
    int64_t* last_dec = calloc((size_t)n, sizeof(int64_t));
    int nc = 0, nt = 0;
    for (int s = 0; s < n; ++s) {
        const oppo_seq_state* q = &seqs[s];
        c_off[s] = nc;
        if (q->prefilled_tokens < q->generated) ch[nc++] = (ochunk){q->prefilled_tokens + 1, q->generated, 0, 0};
        if (q->generated < q->target_len)
            for (int f = q->generated + 1; f <= q->target_len; f += C)
                ch[nc++] = (ochunk){f, f + C - 1 < q->target_len ? f + C - 1 : q->target_len, 1, 0};
        int64_t clock = 0;
        for (int c = c_off[s]; c < nc; ++c)
            if (ch[c].needs_decode) {
                clock += (int64_t)(ch[c].last - ch[c].first + 1) * lat->decode_per_token;
                ch[c].done = clock;
            }
        last_dec[s] = clock;
        t_off[s] = nt;
        int prompt_pending = lat->count_prompt_in_prefill && q->chunks_prefilled == 0 && q->prefilled_tokens == 0;
        int first = 1;
        for (int c = c_off[s]; c < nc; ++c) {
            otask t = {s, c - c_off[s], 0, !ch[c].needs_decode, ch[c].last - ch[c].first + 1, 0, 0, -1};
            if (ch[c].needs_decode) {
                t.avail = streamed ? ch[c].done : clock;
                if (!coloc) t.avail += lat->transfer_per_chunk;
            }
            t.dur = (int64_t)t.size * lat->prefill_per_token;
            if (prompt_pending) {
                t.dur += (int64_t)q->prompt_len * lat->prefill_per_token;
                prompt_pending = 0;
            }
            if (coloc && (streamed || first)) t.dur += lat->chunk_switch_cost;
            first = 0;
            tk[nt++] = t;
        }
        const int reaches = (nc > c_off[s] && ch[nc - 1].last == q->target_len) ||
                            (nc == c_off[s] && q->prefilled_tokens >= q->target_len && !q->scored);
        if (reaches) tk[nt++] = (otask){s, nc - c_off[s], 1, 0, 0, 0, lat->reward_residual, -1};
    }
    c_off[n] = nc;
    t_off[n] = nt;
    /* serial queue (engine.cpp:109-142) */
    int* next = calloc((size_t)n, sizeof(int));
    int64_t qclock = 0;
    for (;;) {
        int best = -1;
        for (int s = 0; s < n; ++s) {
            const int k = t_off[s] + next[s];
            if (k >= t_off[s + 1]) continue;
            if (next[s] > 0 && tk[k - 1].done > tk[k].avail) tk[k].avail = tk[k - 1].done;
            if (best < 0 || tk[k].avail < tk[best].avail ||
                (tk[k].avail == tk[best].avail &&
                 (seqs[s].id < seqs[tk[best].seq].id ||
                  (seqs[s].id == seqs[tk[best].seq].id && tk[k].chunk_index < tk[best].chunk_index))))
                best = k;
        }
        if (best < 0) break;
        const int64_t start = qclock > tk[best].avail ? qclock : tk[best].avail;
        tk[best].done = start + tk[best].dur;
        qclock = tk[best].done;
        next[tk[best].seq] += 1;
    }
    /* cut: stop_after-th score-ready (ties by id), else full completion */
    int64_t* sc_t = calloc((size_t)n, sizeof(int64_t));
    int64_t* sc_id = calloc((size_t)n, sizeof(int64_t));
    int ns = 0;
    for (int k = 0; k < nt; ++k)
        if (tk[k].is_residual) {
            sc_t[ns] = tk[k].done;
            sc_id[ns++] = seqs[tk[k].seq].id;
        }
    for (int a = 1; a < ns; ++a)  /* insertion sort by (time, id) */
        for (int b = a; b > 0 && (sc_t[b] < sc_t[b - 1] || (sc_t[b] == sc_t[b - 1] && sc_id[b] < sc_id[b - 1])); --b) {
            int64_t x = sc_t[b]; sc_t[b] = sc_t[b - 1]; sc_t[b - 1] = x;
            x = sc_id[b]; sc_id[b] = sc_id[b - 1]; sc_id[b - 1] = x;
        }
    int64_t t_end = 0;
    if (stop_after >= 1 && stop_after <= ns) t_end = sc_t[stop_after - 1];
    else
        for (int s = 0; s < n; ++s) {
            if (last_dec[s] > t_end) t_end = last_dec[s];
            if (t_off[s + 1] > t_off[s] && tk[t_off[s + 1] - 1].done > t_end) t_end = tk[t_off[s + 1] - 1].done;
        }
    memset(led, 0, sizeof(*led));
    led->wall = t_end;
    int64_t last_any = 0;
    for (int s = 0; s < n; ++s) {
        oppo_seq_outcome* o = &out[s];
        memset(o, 0, sizeof(*o));
        o->seq_id = seqs[s].id;
        o->score_ready = -1;
        int64_t prev_done = 0;
        int partial_done = 0;
        for (int c = c_off[s]; c < c_off[s + 1]; ++c) {
            if (!ch[c].needs_decode) continue;
            const int size = ch[c].last - ch[c].first + 1;
            if (ch[c].done <= t_end) {
                o->tokens_decoded += size;
                o->decode_chunks_completed += 1;
                led->work_generation += (int64_t)size * lat->decode_per_token;
                if (ch[c].done > last_any) last_any = ch[c].done;
                prev_done = ch[c].done;
            } else if (credit_partial && !partial_done && lat->decode_per_token > 0) {
                partial_done = 1;
                int64_t k = (t_end - prev_done) / lat->decode_per_token;
                if (k > size) k = size;
                if (k > 0) {
                    o->tokens_decoded += (int)k;
                    led->work_generation += k * lat->decode_per_token;
                    const int64_t tdone = prev_done + k * lat->decode_per_token;
                    if (tdone > last_any) last_any = tdone;
                }
            }
        }
        for (int k = t_off[s]; k < t_off[s + 1]; ++k) {
            if (tk[k].done < 0 || tk[k].done > t_end) continue;
            if (tk[k].is_residual) o->score_ready = tk[k].done;
            else {
                o->tokens_prefilled += tk[k].size;
                o->prefill_tasks_completed += 1;
                if (tk[k].is_carry) o->carry_prefill_completed = 1;
            }
            led->work_scoring += tk[k].dur;
        }
    }
    led->busy_scoring = led->work_scoring;
    led->busy_generation = last_any < t_end ? last_any : t_end;
    free(ch); free(tk); free(c_off); free(t_off); free(last_dec); free(next); free(sc_t); free(sc_id);
    return 0;
}

/* --------------------------------------------------- select_finished etc. */
static int select_finished(oppo_seq_state* e, int n, const oppo_seq_outcome* o, int no, int B,
                           int64_t* sel_ids, int* n_sel) {
    int64_t* rt = malloc(sizeof(int64_t) * (size_t)(n + 1));
    int64_t* rid = malloc(sizeof(int64_t) * (size_t)(n + 1));
    int* rpos = malloc(sizeof(int) * (size_t)(n + 1));
    int nr = 0;
    for (int p = 0; p < n; ++p) {
        oppo_seq_state* s = &e[p];
        const int was = s->scored;
        const oppo_seq_outcome* oc = NULL;
        for (int k = 0; k < no; ++k)
            if (o[k].seq_id == s->id) { oc = &o[k]; break; }
        if (!oc) {
            if (was) { rt[nr] = -1; rid[nr] = s->id; rpos[nr++] = p; }
            continue;
        }
        const int emitted = s->chunks_emitted;
        s->generated += oc->tokens_decoded;
        s->chunks_emitted += oc->decode_chunks_completed;
        s->prefilled_tokens += oc->tokens_prefilled;
        s->chunks_prefilled = (oc->carry_prefill_completed ? emitted : s->chunks_prefilled) +
                              oc->prefill_tasks_completed - (oc->carry_prefill_completed ? 1 : 0);
        s->finished = s->generated == s->target_len;
        if (oc->score_ready >= 0) s->scored = 1;
        if (oc->score_ready >= 0 || was) { rt[nr] = was ? -1 : oc->score_ready; rid[nr] = s->id; rpos[nr++] = p; }
    }
    for (int a = 1; a < nr; ++a)
        for (int b = a; b > 0 && (rt[b] < rt[b - 1] || (rt[b] == rt[b - 1] && rid[b] < rid[b - 1])); --b) {
            int64_t x = rt[b]; rt[b] = rt[b - 1]; rt[b - 1] = x;
            x = rid[b]; rid[b] = rid[b - 1]; rid[b - 1] = x;
            int y = rpos[b]; rpos[b] = rpos[b - 1]; rpos[b - 1] = y;
        }
    const int take = nr < B ? nr : B;
    char* taken = calloc((size_t)n + 1, 1);
    for (int i = 0; i < take; ++i) { sel_ids[i] = e[rpos[i]].id; taken[rpos[i]] = 1; }
    int w = 0;
    for (int p = 0; p < n; ++p) {
        if (taken[p]) continue;
        oppo_seq_state s = e[p];
        s.deferrals += 1;
        e[w++] = s;
    }
    *n_sel = take;
    free(rt); free(rid); free(rpos); free(taken);
    return w;
}

/* run_seed step loop (driver.cpp:103-195), simulate/tune mode, with the
 * engine's lockstep latency model or any other.  carry = 1 credits partial
 * chunks (token granularity).  Records: wall, finished, deferred, delta. */
int oracle_run_seed(const oppo_run_config* cfg, uint64_t seed, int64_t* rec4, int64_t* sel_ids,
                    int* n_rec) {
    orng lr;
    rng_derive(&lr, seed, "lengths");
    const int cap_max = cfg->batch_size + cfg->delta_max + 1;
    oppo_seq_state* buf = calloc((size_t)cap_max * 2 + 8, sizeof(oppo_seq_state));
    oppo_seq_state* act = calloc((size_t)cap_max * 2 + 8, sizeof(oppo_seq_state));
    oppo_seq_outcome* outc = calloc((size_t)cap_max * 2 + 8, sizeof(oppo_seq_outcome));
    double* hist = calloc((size_t)cfg->steps + 8, sizeof(double));
    int nh = 0, nb = 0, delta = cfg->delta_init, n = 0;
    int64_t issued = 0;
    /* tuner */
    int cands[OPPO_MAX_CANDIDATES], ncand = 0, current = 0;
    double tsum[OPPO_MAX_CANDIDATES];
    int tcnt[OPPO_MAX_CANDIDATES];
    const int tuning = cfg->mode == OPPO_RUN_TUNE || cfg->tune_chunks;
    if (tuning) {
        for (int i = 0; i < cfg->n_candidates; ++i) {
            int v = cfg->chunk_candidates[i], dup = 0;
            for (int j = 0; j < ncand; ++j) dup |= cands[j] == v;
            if (!dup) cands[ncand++] = v;
        }
        for (int a = 1; a < ncand; ++a)
            for (int b = a; b > 0 && cands[b] < cands[b - 1]; --b) { int x = cands[b]; cands[b] = cands[b - 1]; cands[b - 1] = x; }
        current = cands[0];
        for (int i = 0; i < ncand; ++i) { tsum[i] = 0; tcnt[i] = 0; }
    }
    for (int step = 0; step < cfg->steps; ++step) {
        while (nb < cfg->batch_size + delta && (cfg->prompt_count < 0 || issued < cfg->prompt_count)) {
            oppo_seq_state s;
            memset(&s, 0, sizeof(s));
            s.id = issued++;
            s.prompt_len = cfg->prompt_len;
            s.arrival_step = step;
            s.target_len = draw_length(&cfg->lengths, &lr);
            s.admitted_at = step;
            buf[nb++] = s;
        }
        if (nb == 0) break;
        int chunk = cfg->chunk_size, explored = -1;
        if (tuning) {
            const int in_p = step % cfg->retune_period;
            if (in_p < ncand) explored = cands[in_p];
            chunk = explored >= 0 ? explored : current;
        }
        int na = 0, pre = 0;
        for (int i = 0; i < nb; ++i) {
            if (buf[i].scored) ++pre;
            else act[na++] = buf[i];
        }
        oppo_ledger led;
        memset(&led, 0, sizeof(led));
        int no = 0;
        const int need = cfg->batch_size - pre;
        if (na > 0 && need > 0) {
            oracle_run_step(act, na, chunk, cfg->schedule_mode, &cfg->latency, need,
                            cfg->carry_granularity == OPPO_CARRY_TOKEN, outc, &led);
            no = na;
        }
        int nsel = 0;
        nb = select_finished(buf, nb, outc, no, cfg->batch_size,
                             sel_ids + (size_t)n * cfg->batch_size, &nsel);
        for (int i = nsel; i < cfg->batch_size; ++i) sel_ids[(size_t)n * cfg->batch_size + i] = -1;
        double reward = cfg->proxy_value;
        if (cfg->proxy_kind == 1) {
            const int rs = cfg->proxy_ramp_steps < 1 ? 1 : cfg->proxy_ramp_steps;
            reward = cfg->proxy_value + cfg->proxy_ramp_scale * (step < cfg->proxy_ramp_steps ? step : cfg->proxy_ramp_steps) / (double)rs;
        }
        hist[nh++] = reward;
        int nd = delta;
        const int W = cfg->window;
        if (cfg->controller == OPPO_DELTA_ALG1 && nh >= 2 * W) {
            double a = 0, b = 0;
            for (int i = nh - W; i < nh; ++i) a += hist[i];
            for (int i = nh - 2 * W; i < nh - W; ++i) b += hist[i];
            const double d = a / W - b / W;
            const int sg = (d > 0) - (d < 0);
            int ch = delta / 4;
            if (ch < 1) ch = 1;
            nd = delta - sg * ch;
            if (nd < cfg->delta_min) nd = cfg->delta_min;
            if (nd > cfg->delta_max) nd = cfg->delta_max;
            memmove(hist, hist + nh - W, sizeof(double) * W);
            nh = W;
        } else if (cfg->controller == OPPO_DELTA_EQ4 && nh >= W + 1) {
            const double slope = (hist[nh - 1] - hist[nh - 1 - W]) / W;
            if (nh > W + 1) { memmove(hist, hist + nh - (W + 1), sizeof(double) * (W + 1)); nh = W + 1; }
            nd = slope > 0 ? (delta + cfg->delta_inc < cfg->delta_max ? delta + cfg->delta_inc : cfg->delta_max)
                           : (delta - cfg->delta_dec > cfg->delta_min ? delta - cfg->delta_dec : cfg->delta_min);
        }
        rec4[n * 4 + 0] = led.wall;
        rec4[n * 4 + 1] = nsel;
        rec4[n * 4 + 2] = nb;
        rec4[n * 4 + 3] = delta;
        ++n;
        if (tuning && explored >= 0) {
            int ci = 0;
            while (cands[ci] != explored) ++ci;
            tsum[ci] += (double)led.wall;
            tcnt[ci] += 1;
            int all = 1;
            for (int i = 0; i < ncand; ++i) all &= tcnt[i] > 0;
            if (all) {
                double bm = 0;
                for (int i = 0; i < ncand; ++i) {
                    const double m = tsum[i] / tcnt[i];
                    if (i == 0 || m < bm) { bm = m; current = cands[i]; }
                }
                for (int i = 0; i < ncand; ++i) { tsum[i] = 0; tcnt[i] = 0; }
            }
        }
        delta = nd;
    }
    *n_rec = n;
    free(buf); free(act); free(outc); free(hist);
    return 0;
}

/* ------------------------------------------------------------- PPO math */
/* compute_gae (ppo.cpp:71-85) */
void oracle_gae(const double* r, const double* v, int T, double g, double l, double* adv) {
    double run = 0.0;
    for (int i = T; i-- > 0;) {
        const double d = r[i] + g * v[i + 1] - v[i];
        run = d + g * l * run;
        adv[i] = run;
    }
}

/* Per-token clipped objective and dObj/dlogp (ppo.cpp:101-177); returns the token mean. */
double oracle_ppo_clip(int n, const double* new_lp, const double* old_lp, const double* adv,
                       double eps, double* dobj) {
    double tot = 0.0;
    for (int i = 0; i < n; ++i) {
        const double ratio = exp(new_lp[i] - old_lp[i]);
        const double c = ratio < 1 - eps ? 1 - eps : (ratio > 1 + eps ? 1 + eps : ratio);
        const double un = ratio * adv[i], cl = c * adv[i];
        tot += un < cl ? un : cl;
        double dt;
        if (un <= cl) dt = adv[i];
        else dt = (ratio > 1 - eps && ratio < 1 + eps) ? adv[i] : 0.0;
        if (dobj) dobj[i] = dt * ratio / n;
    }
    return n ? tot / n : 0.0;
}

/* --------------------------------------------------------- GPT forward */
typedef struct {
    int n_layers, d, H, KV, hd, dff, V;
    const float* embed;
    const float* lm_head;
    const float* final_norm;
    const float* const* ln1;
    const float* const* wqkv;
    const float* const* bqkv;
    const float* const* wo;
    const float* const* ln2;
    const float* const* wgu;
    const float* const* wdown;
} oracle_gpt;

static void rms(const double* x, const float* w, int d, double* out) {
    double ss = 0;
    for (int i = 0; i < d; ++i) ss += x[i] * x[i];
    const double inv = 1.0 / sqrt(ss / d + 1e-6);
    for (int i = 0; i < d; ++i) out[i] = x[i] * inv * w[i];
}
static void matvec(const float* W, const double* x, int rows, int cols, double* y) {
    for (int r = 0; r < rows; ++r) {
        const float* w = W + (size_t)r * cols;
        double s = 0;
        for (int c = 0; c < cols; ++c) s += w[c] * x[c];
        y[r] = s;
    }
}

/* Full-sequence causal forward of T tokens at positions 0..T-1.
 * hidden_out [T, d] = final normed hidden; logits_out [T, V] (optional). */
int oracle_gpt_forward(const oracle_gpt* m, const int32_t* tok, int T, double* hidden_out,
                       double* logits_out) {
    const int d = m->d, H = m->H, KV = m->KV, hd = m->hd, F = m->dff, G = H / KV;
    const int qkvw = (H + 2 * KV) * hd;
    double* x = calloc((size_t)T * d, sizeof(double));
    double* h = calloc((size_t)d, sizeof(double));
    double* qkv = calloc((size_t)T * qkvw, sizeof(double));
    double* att = calloc((size_t)H * hd, sizeof(double));
    double* o = calloc((size_t)d, sizeof(double));
    double* gu = calloc((size_t)2 * F, sizeof(double));
    double* a = calloc((size_t)F, sizeof(double));
    double* sc = calloc((size_t)T, sizeof(double));
    for (int t = 0; t < T; ++t)
        for (int i = 0; i < d; ++i) x[(size_t)t * d + i] = m->embed[(size_t)tok[t] * d + i];
    for (int l = 0; l < m->n_layers; ++l) {
        for (int t = 0; t < T; ++t) {
            rms(x + (size_t)t * d, m->ln1[l], d, h);
            double* q = qkv + (size_t)t * qkvw;
            matvec(m->wqkv[l], h, qkvw, d, q);
            for (int i = 0; i < qkvw; ++i) q[i] += m->bqkv[l][i];
            for (int hh = 0; hh < H + KV; ++hh)  /* RoPE on q and k heads (rotate-half) */
                for (int i = 0; i < hd / 2; ++i) {
                    const double inv = pow(1e6, -2.0 * i / hd);
                    const double ang = t * inv, cs = cos(ang), sn = sin(ang);
                    double* p = q + hh * hd;
                    const double x1 = p[i], x2 = p[i + hd / 2];
                    p[i] = x1 * cs - x2 * sn;
                    p[i + hd / 2] = x2 * cs + x1 * sn;
                }
        }
        for (int t = 0; t < T; ++t) {
            for (int hh = 0; hh < H; ++hh) {
                const int kvh = hh / G;
                const double* q = qkv + (size_t)t * qkvw + hh * hd;
                double mx = -1e300;
                for (int s = 0; s <= t; ++s) {
                    const double* k = qkv + (size_t)s * qkvw + (H + kvh) * hd;
                    double dot = 0;
                    for (int i = 0; i < hd; ++i) dot += q[i] * k[i];
                    sc[s] = dot / sqrt((double)hd);
                    if (sc[s] > mx) mx = sc[s];
                }
                double z = 0;
                for (int s = 0; s <= t; ++s) { sc[s] = exp(sc[s] - mx); z += sc[s]; }
                for (int i = 0; i < hd; ++i) {
                    double acc = 0;
                    for (int s = 0; s <= t; ++s) acc += sc[s] * qkv[(size_t)s * qkvw + (H + KV + kvh) * hd + i];
                    att[hh * hd + i] = acc / z;
                }
            }
            matvec(m->wo[l], att, d, H * hd, o);
            for (int i = 0; i < d; ++i) x[(size_t)t * d + i] += o[i];
            rms(x + (size_t)t * d, m->ln2[l], d, h);
            matvec(m->wgu[l], h, 2 * F, d, gu);
            for (int i = 0; i < F; ++i) {
                const double g = gu[2 * i], u = gu[2 * i + 1];
                a[i] = g / (1.0 + exp(-g)) * u;
            }
            matvec(m->wdown[l], a, d, F, o);
            for (int i = 0; i < d; ++i) x[(size_t)t * d + i] += o[i];
        }
    }
    for (int t = 0; t < T; ++t) {
        rms(x + (size_t)t * d, m->final_norm, d, hidden_out + (size_t)t * d);
        if (logits_out) matvec(m->lm_head, hidden_out + (size_t)t * d, m->V, d, logits_out + (size_t)t * m->V);
    }
    free(x); free(h); free(qkv); free(att); free(o); free(gu); free(a); free(sc);
    return 0;
}

/* The engine's sampling stream (kernels/common.cuh): key per (seed, seq, pos),
 * uniform per vocab entry, Gumbel noise -log(-log(u)) in single precision. */
static uint64_t mix64(uint64_t x) { return o_splitmix(x); }
static uint32_t lowbias32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}
uint64_t oracle_token_key(uint64_t seed, int64_t seq, int32_t pos) {
    return mix64(seed ^ mix64((uint64_t)seq * 0x100000001b3ull + (uint64_t)(uint32_t)pos));
}
float oracle_gumbel(uint64_t key, uint32_t v) {
    uint32_t x = (uint32_t)key ^ (v * 0x9e3779b9u);
    x = lowbias32(x) ^ (uint32_t)(key >> 32);
    x = lowbias32(x);
    const float u = ((float)(x >> 9) + 0.5f) * (1.0f / 8388608.0f);
    return -logf(-logf(u));
}
int32_t oracle_prompt_token(uint64_t seed, int64_t id, int32_t q, int32_t vocab) {
    const uint64_t h = mix64(seed ^ 0x70726f6d7074ull ^ mix64((uint64_t)id * 0x100000001b3ull + (uint64_t)q));
    return (int32_t)(h % (uint64_t)vocab);
}

/* The engine's two-level categorical draw (kernels/gemm.cuh logits_tile +
 * kernels/model.cuh logits_combine) on fp64 logits:
 *   block b* = argmax_b (lse_b + Gumbel(key ^ kBlockKey, b)), blocks of 256 ids;
 *   inside b*: first id whose running sum of exp(x - max_b) exceeds
 *   U(key ^ kInBlockKey, b*) * sum_b (fallback: the block's last id).
 * margins: gap between the two best block scores, and the relative distance
 * of the in-block threshold from the nearest cumulative-sum boundary. */
static float key_uniform_o(uint64_t key, uint32_t v) {
    uint32_t x = (uint32_t)key ^ (v * 0x9e3779b9u);
    x = lowbias32(x) ^ (uint32_t)(key >> 32);
    x = lowbias32(x);
    return ((float)(x >> 9) + 0.5f) * (1.0f / 8388608.0f);
}
int oracle_sample_token(const double* x, int V, uint64_t key, double* lp_out,
                        double* margin_block, double* margin_inblock) {
    const uint64_t kIn = 0x696e626c6f636bull, kBlk = 0x626c6f636b6e7a65ull;
    const int SB = 256, nb = (V + SB - 1) / SB;
    double best = -INFINITY, second = -INFINITY, tot_m = -INFINITY;
    int bb = 0;
    for (int b = 0; b < nb; ++b)
        for (int i = b * SB; i < V && i < (b + 1) * SB; ++i) if (x[i] > tot_m) tot_m = x[i];
    double tot = 0.0;
    for (int i = 0; i < V; ++i) tot += exp(x[i] - tot_m);
    for (int b = 0; b < nb; ++b) {
        const int a = b * SB, e = (b + 1) * SB < V ? (b + 1) * SB : V;
        double m = -INFINITY, se = 0.0;
        for (int i = a; i < e; ++i) if (x[i] > m) m = x[i];
        for (int i = a; i < e; ++i) se += exp(x[i] - m);
        const double sc = m + log(se) + (double)oracle_gumbel(key ^ kBlk, (uint32_t)b);
        if (sc > best) { second = best; best = sc; bb = b; }
        else if (sc > second) second = sc;
    }
    *margin_block = best - second;
    const int a = bb * SB, e = (bb + 1) * SB < V ? (bb + 1) * SB : V;
    double m = -INFINITY, se = 0.0;
    for (int i = a; i < e; ++i) if (x[i] > m) m = x[i];
    for (int i = a; i < e; ++i) se += exp(x[i] - m);
    const double thr = (double)key_uniform_o(key ^ kIn, (uint32_t)bb) * se;
    double run = 0.0, gap = INFINITY;
    int pick = e - 1;
    for (int i = a; i < e; ++i) {
        run += exp(x[i] - m);
        const double d = fabs(run - thr);
        if (d < gap) gap = d;
        if (run > thr) { pick = i; break; }
    }
    *margin_inblock = gap / se;
    *lp_out = x[pick] - tot_m - log(tot);
    return pick;
}
