// report.cpp — reporting on the decode path, host C++:
// the two-lane schedule model (schedule.cpp:92-217), per-token reports from
// measured events (executor.cpp:361-382) and the routing metrics
// (metrics.cpp:9-28).  Pure CPU code behind the C ABI, so it is tested on
// GPU-less hosts against the reference library itself (tests/test_report.py).
#include "../../include/smoe.h"

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

namespace smoe {
namespace report {

enum Lane { kCompute = 0, kCopy = 1 };
enum Kind { kAttn = 0, kGate = 1, kExpert = 2, kCopyK = 3, kIdle = 4 };

struct Ev {
    int lane, kind, layer;
    double start, end;
};

struct Report {
    std::vector<Ev> events;
    double tpot = 0.0;
};

struct Timing {
    std::vector<double> attn, gate, expert, copy;
    double cold = -1.0;
    int layers() const { return static_cast<int>(attn.size()); }
    double compute(int l) const { return attn[l] + gate[l] + expert[l]; }
    double cold_copy() const { return cold < 0.0 ? copy[0] : cold; }
    void validate() const {  // schedule.cpp:14-32
        const size_t L = attn.size();
        if (L == 0) throw std::invalid_argument("timing model: no layers");
        if (gate.size() != L || expert.size() != L || copy.size() != L)
            throw std::invalid_argument("timing model: ragged duration arrays");
        auto check = [](const std::vector<double>& v, const char* n) {
            for (double x : v)
                if (!(x >= 0.0) || !std::isfinite(x))
                    throw std::invalid_argument(std::string("timing model: negative ") + n);
        };
        check(attn, "t_attn");
        check(gate, "t_gate_topk");
        check(expert, "t_expert");
        check(copy, "t_copy");
        if (cold >= 0.0 && !std::isfinite(cold))
            throw std::invalid_argument("timing model: bad cold_start_copy");
    }
};

// simulate_on_demand (schedule.cpp:92-109): fully serial.
Report on_demand(const Timing& tm) {
    tm.validate();
    Report r;
    double t = 0.0;
    for (int l = 0; l < tm.layers(); ++l) {
        r.events.push_back({kCompute, kAttn, l, t, t + tm.attn[l]});
        t += tm.attn[l];
        r.events.push_back({kCompute, kGate, l, t, t + tm.gate[l]});
        t += tm.gate[l];
        const double c = l == 0 ? tm.cold_copy() : tm.copy[l];
        r.events.push_back({kCopy, kCopyK, l, t, t + c});
        t += c;
        r.events.push_back({kCompute, kExpert, l, t, t + tm.expert[l]});
        t += tm.expert[l];
    }
    r.tpot = t;
    return r;
}

// simulate_prefetch (schedule.cpp:111-148): layer-0 blocking copy after
// gating, copy of l+1 issued after gating l on a FIFO copy lane.
Report prefetch(const Timing& tm) {
    tm.validate();
    const int L = tm.layers();
    Report r;
    std::vector<double> cs(L), ce(L);
    double cursor = 0.0, gate_end = 0.0;
    for (int l = 0; l < L; ++l) {
        r.events.push_back({kCompute, kAttn, l, cursor, cursor + tm.attn[l]});
        cursor += tm.attn[l];
        r.events.push_back({kCompute, kGate, l, cursor, cursor + tm.gate[l]});
        cursor += tm.gate[l];
        gate_end = cursor;
        if (l == 0) {
            cs[0] = gate_end;
            ce[0] = cs[0] + tm.cold_copy();
        }
        if (l + 1 < L) {
            cs[l + 1] = std::max(ce[l], gate_end);
            ce[l + 1] = cs[l + 1] + tm.copy[l + 1];
        }
        const double es = std::max(gate_end, ce[l]);
        r.events.push_back({kCompute, kExpert, l, es, es + tm.expert[l]});
        cursor = es + tm.expert[l];
    }
    for (int l = 0; l < L; ++l) r.events.push_back({kCopy, kCopyK, l, cs[l], ce[l]});
    r.tpot = cursor;
    return r;
}

// analytic_improvement (schedule.cpp:150-155): Eq. 1.
double analytic(const Timing& tm) {
    tm.validate();
    double s = 0.0;
    for (int l = 0; l < tm.layers(); ++l) s += std::min(tm.copy[l], tm.compute(l));
    return s;
}

struct Iv {
    double a, b;
};

std::vector<Iv> busy(const std::vector<Ev>& ev, int lane) {  // schedule.cpp:160-180
    std::vector<Iv> v;
    for (const Ev& e : ev)
        if (e.lane == lane && e.end > e.start) v.push_back({e.start, e.end});
    std::sort(v.begin(), v.end(), [](const Iv& x, const Iv& y) { return x.a < y.a; });
    std::vector<Iv> m;
    for (const Iv& i : v) {
        if (!m.empty() && i.a <= m.back().b)
            m.back().b = std::max(m.back().b, i.b);
        else
            m.push_back(i);
    }
    return m;
}

double total(const std::vector<Iv>& v) {
    double s = 0.0;
    for (const Iv& i : v) s += i.b - i.a;
    return s;
}

double overlap(const std::vector<Iv>& a, const std::vector<Iv>& b) {
    double s = 0.0;
    size_t i = 0, j = 0;
    while (i < a.size() && j < b.size()) {
        const double lo = std::max(a[i].a, b[j].a), hi = std::min(a[i].b, b[j].b);
        if (hi > lo) s += hi - lo;
        if (a[i].b < b[j].b)
            ++i;
        else
            ++j;
    }
    return s;
}

// breakdown (schedule.cpp:205-217): compute / critical-path copy / idle.
void breakdown(const Report& r, double* f) {
    f[0] = f[1] = f[2] = 0.0;
    if (r.tpot <= 0.0) return;
    const auto c = busy(r.events, kCompute), k = busy(r.events, kCopy);
    const double cb = total(c), ov = overlap(c, k);
    f[0] = cb / r.tpot;
    f[1] = (total(k) - ov) / r.tpot;
    f[2] = 1.0 - f[0] - f[1];
}

// ---- trace-driven two-lane schedule with a per-layer slot cache ----------
// (SURVEY §8f row 4.)  simulate_prefetch / simulate_on_demand
// (schedule.cpp:92-148) assume every layer copies its experts; here each
// layer holds `capacity` expert slots (LRU or LFU), a copy moves one expert,
// and requests come from a decode trace: the executed experts of layer l are
// copied on demand after layer-l gating when absent; predictions for layer
// l+1 (lookahead 1, Algorithm 1) — and, with lookahead 2, for layer l+2 —
// are copied after layer-l gating into slots not needed by layer l's own
// executed set.  One copy lane, FIFO.  When every request misses and the
// predictions are exact this reduces to the reference's simulators with
// t_copy[l] = k * t_copy_expert (pinned in tests/test_report.py).
struct CacheSim {
    struct Slot {
        int e = -1;
        double ready = 0.0;
        long long last = -1, uses = 0;
        bool prefetched = false;
    };
    int L, C, policy;
    std::vector<std::vector<Slot>> slots;  // [L][C]
    CacheSim(int l, int c, int pol) : L(l), C(c), policy(pol), slots(l, std::vector<Slot>(c)) {}
    Slot* find(int l, int e) {
        for (Slot& s : slots[l])
            if (s.e == e) return &s;
        return nullptr;
    }
    // victim slot of layer l avoiding the experts in `keep`; null if none
    Slot* victim(int l, const std::vector<int>& keep) {
        Slot* best = nullptr;
        for (Slot& s : slots[l]) {
            if (s.e >= 0 && std::find(keep.begin(), keep.end(), s.e) != keep.end()) continue;
            if (s.e < 0) return &s;
            if (!best) {
                best = &s;
                continue;
            }
            const bool better = policy == 1 ? (s.uses < best->uses || (s.uses == best->uses && s.last < best->last))
                                            : s.last < best->last;
            if (better) best = &s;
        }
        return best;
    }
};

struct CacheSimOut {
    double tpot = 0.0, stall_copies = 0.0, prefetch_copies = 0.0, useful_prefetch = 0.0;
};

CacheSimOut simulate_cache(int T, int L, int K, int C, int policy, int lookahead, int warm, const int* exec,
                           const int* pred, const int* pred2, const double* ta, const double* tg, const double* te,
                           double tc) {
    CacheSim cs(L, C, policy);
    CacheSimOut o;
    double clock = 0.0, copy_free = 0.0;
    long long seq = 0;
    int measured = 0;
    for (int t = 0; t < T; ++t) {
        const double t0 = clock;
        double cursor = clock;
        long long stall = 0, pf = 0, useful = 0;
        copy_free = std::max(copy_free, clock);
        for (int l = 0; l < L; ++l) {
            cursor += ta[l] + tg[l];
            const double gate_end = cursor;
            const int* ex = exec + (static_cast<long long>(t) * L + l) * K;
            const std::vector<int> need(ex, ex + K);
            // executed experts: hits wait for their copy, misses copy on demand
            double ready = gate_end;
            for (int i = 0; i < K; ++i) {
                CacheSim::Slot* s = cs.find(l, ex[i]);
                if (s) {
                    if (s->prefetched) {
                        ++useful;
                        s->prefetched = false;
                    }
                } else {
                    s = cs.victim(l, need);
                    const double st = std::max(copy_free, gate_end);
                    copy_free = st + tc;
                    ++stall;
                    if (s) {
                        *s = CacheSim::Slot{ex[i], copy_free, seq, 0, false};
                    } else {  // capacity below k: streamed through without caching
                        ready = std::max(ready, copy_free);
                        continue;
                    }
                }
                s->last = seq;
                ++s->uses;
                ready = std::max(ready, s->ready);
            }
            ++seq;
            // speculative copies issued after layer-l gating
            for (int ahead = 1; ahead <= lookahead && ahead <= 2; ++ahead) {
                const int* pr = ahead == 1 ? pred : pred2;
                const int tl = l + ahead;
                if (!pr || tl >= L) continue;
                const int* pi = pr + (static_cast<long long>(t) * L + tl) * K;
                const std::vector<int> keep(pi, pi + K);
                for (int i = 0; i < K; ++i) {
                    if (cs.find(tl, pi[i])) continue;
                    CacheSim::Slot* s = cs.victim(tl, keep);
                    if (!s) continue;
                    const double st = std::max(copy_free, gate_end);
                    copy_free = st + tc;
                    ++pf;
                    *s = CacheSim::Slot{pi[i], copy_free, seq, 0, true};
                }
            }
            cursor = std::max(cursor, ready) + te[l];
        }
        clock = cursor;
        if (t >= warm) {
            o.tpot += cursor - t0;
            o.stall_copies += static_cast<double>(stall);
            o.prefetch_copies += static_cast<double>(pf);
            o.useful_prefetch += static_cast<double>(useful);
            ++measured;
        }
    }
    if (measured) {
        o.tpot /= measured;
        o.stall_copies /= measured;
        o.prefetch_copies /= measured;
        o.useful_prefetch /= measured;
    }
    return o;
}

}  // namespace report
}  // namespace smoe

void smoe_set_last_error(const std::string& msg);  // capi.cpp

namespace {
template <typename F>
int guard_r(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        smoe_set_last_error(e.what());
        return 1;
    } catch (const std::exception& e) {
        smoe_set_last_error(e.what());
        return 2;
    }
}

smoe::report::Timing timing(int L, const double* a, const double* g, const double* e,
                            const double* c, double cold) {
    if (L < 1 || !a || !g || !e || !c) throw std::invalid_argument("timing model: no layers");
    smoe::report::Timing tm;
    tm.attn.assign(a, a + L);
    tm.gate.assign(g, g + L);
    tm.expert.assign(e, e + L);
    tm.copy.assign(c, c + L);
    tm.cold = cold;
    return tm;
}
}  // namespace

extern "C" {

int smoe_simulate(int32_t layers, const double* t_attn, const double* t_gate,
                  const double* t_expert, const double* t_copy, double cold_start_copy,
                  int32_t mode, double* tpot, double* fractions3, double* analytic) {
    return guard_r([&] {
        const auto tm = timing(layers, t_attn, t_gate, t_expert, t_copy, cold_start_copy);
        const auto r = mode == SMOE_PREFETCH ? smoe::report::prefetch(tm)
                                             : smoe::report::on_demand(tm);
        if (tpot) *tpot = r.tpot;
        if (fractions3) smoe::report::breakdown(r, fractions3);
        if (analytic) *analytic = smoe::report::analytic(tm);
    });
}

// per_token_reports (executor.cpp:361-382) + breakdown, averaged over tokens.
int smoe_breakdown(const smoe_event* events, int32_t n, double* mean_fractions3,
                   double* mean_tpot) {
    return guard_r([&] {
        int max_token = -1;
        for (int i = 0; i < n; ++i) max_token = std::max(max_token, events[i].token);
        const int T = max_token + 1;
        std::vector<smoe::report::Report> reps(T);
        std::vector<double> begin(T, 1e300);
        for (int i = 0; i < n; ++i) {
            const smoe_event& e = events[i];
            if (e.token < 0) continue;
            reps[e.token].events.push_back({e.lane, e.kind, e.layer, e.start_ms, e.end_ms});
            begin[e.token] = std::min(begin[e.token], e.start_ms);
            reps[e.token].tpot = std::max(reps[e.token].tpot, e.end_ms);
        }
        double f[3], acc[3] = {0, 0, 0}, tp = 0.0;
        int cnt = 0;
        for (int t = 0; t < T; ++t) {
            if (reps[t].events.empty()) continue;
            for (auto& e : reps[t].events) {
                e.start -= begin[t];
                e.end -= begin[t];
            }
            reps[t].tpot -= begin[t];
            smoe::report::breakdown(reps[t], f);
            for (int k = 0; k < 3; ++k) acc[k] += f[k];
            tp += reps[t].tpot;
            ++cnt;
        }
        for (int k = 0; k < 3; ++k) mean_fractions3[k] = cnt ? acc[k] / cnt : 0.0;
        if (mean_tpot) *mean_tpot = cnt ? tp / cnt : 0.0;
    });
}

// recall_at_k (metrics.cpp:9-20) and rank_alignment (metrics.cpp:22-28).
int smoe_recall_at_k(const int32_t* pred, const int32_t* truth, int32_t k, double* recall,
                     int32_t* rank_match) {
    return guard_r([&] {
        if (k < 1 || !pred || !truth) throw std::invalid_argument("recall_at_k: k mismatch");
        int hits = 0;
        for (int i = 0; i < k; ++i)
            for (int j = 0; j < k; ++j)
                if (pred[i] == truth[j]) {
                    ++hits;
                    break;
                }
        if (recall) *recall = static_cast<double>(hits) / k;
        if (rank_match)
            for (int i = 0; i < k; ++i) rank_match[i] = pred[i] == truth[i];
    });
}

// Per-layer online hit rates of a decode: for every
// recorded step t and layer l >= 1, recall_at_k (metrics.cpp:9-20) of the
// executed decision (the one predicted at l-1) against the true router's
// decision at l on the actual stream.  rates[l-1] = mean over steps (the
// predictor for layer l is the one dispatched at l-1, speculation.cpp:243-252).
int smoe_layer_hit_rates(const int32_t* exec_ids, const int32_t* true_ids, int32_t steps, int32_t layers,
                         int32_t k, double* rates) {
    return guard_r([&] {
        if (!exec_ids || !true_ids || !rates || steps < 1 || layers < 2 || k < 1)
            throw std::invalid_argument("layer_hit_rates: bad arguments");
        for (int l = 1; l < layers; ++l) {
            double sum = 0.0;
            for (int t = 0; t < steps; ++t) {
                const int32_t* p = exec_ids + (static_cast<long long>(t) * layers + l) * k;
                const int32_t* q = true_ids + (static_cast<long long>(t) * layers + l) * k;
                int hits = 0;
                for (int i = 0; i < k; ++i)
                    for (int j = 0; j < k; ++j)
                        if (p[i] == q[j]) {
                            ++hits;
                            break;
                        }
                sum += static_cast<double>(hits) / k;
            }
            rates[l - 1] = sum / steps;
        }
    });
}

// Hybrid map selection ("applying the estimator only where
// prefetch hit rates were low"; the map format is load_hybrid_map's,
// speculation.cpp:145-165): rates [n_kinds][layers-1] per candidate kind
// (SMOE_PRED_* codes in `kinds`, no hybrid/oracle).  threshold > 0: the first
// candidate (the default, router-pf) unless its rate is below threshold, then
// the best of the others; threshold <= 0: the best rate per layer (ties: the
// earlier candidate).
int smoe_select_hybrid_map(const double* rates, const int32_t* kinds, int32_t n_kinds, int32_t layers,
                           double threshold, int32_t* map_out) {
    return guard_r([&] {
        if (!rates || !kinds || !map_out || n_kinds < 1 || layers < 2)
            throw std::invalid_argument("select_hybrid_map: bad arguments");
        for (int i = 0; i < n_kinds; ++i)
            if (kinds[i] < SMOE_PRED_BASELINE_S || kinds[i] > SMOE_PRED_EST_PF)
                throw std::invalid_argument("hybrid map: entries must be concrete predictors");
        const int n = layers - 1;
        for (int l = 0; l < n; ++l) {
            int best = 0;
            const int from = threshold > 0.0 ? 1 : 0;
            if (threshold > 0.0 && (n_kinds == 1 || rates[l] >= threshold)) {
                map_out[l] = kinds[0];
                continue;
            }
            best = from;
            for (int i = from + 1; i < n_kinds; ++i)
                if (rates[static_cast<long long>(i) * n + l] > rates[static_cast<long long>(best) * n + l]) best = i;
            map_out[l] = kinds[best];
        }
    });
}

// Trace-driven cache + lookahead schedule, see CacheSim.
int smoe_simulate_cache(const smoe_cache_sim* c, const int32_t* exec_ids, const int32_t* pred_ids,
                        const int32_t* pred2_ids, const double* t_attn, const double* t_gate,
                        const double* t_expert, double t_copy_expert, double* out4) {
    return guard_r([&] {
        if (!c || !exec_ids || !t_attn || !t_gate || !t_expert || !out4)
            throw std::invalid_argument("simulate_cache: null argument");
        if (c->tokens < 1 || c->layers < 1 || c->k < 1) throw std::invalid_argument("simulate_cache: empty trace");
        if (c->capacity < 0 || c->policy < 0 || c->policy > 1 || c->lookahead < 0 || c->lookahead > 2)
            throw std::invalid_argument("simulate_cache: bad capacity / policy / lookahead");
        if (c->lookahead >= 1 && !pred_ids) throw std::invalid_argument("simulate_cache: lookahead needs predictions");
        if (c->lookahead == 2 && !pred2_ids)
            throw std::invalid_argument("simulate_cache: lookahead 2 needs two-ahead predictions");
        if (c->warm_tokens < 0 || c->warm_tokens >= c->tokens)
            throw std::invalid_argument("simulate_cache: warm_tokens must leave measured tokens");
        const auto o = smoe::report::simulate_cache(c->tokens, c->layers, c->k, c->capacity, c->policy,
                                                    c->lookahead, c->warm_tokens, exec_ids, pred_ids, pred2_ids,
                                                    t_attn, t_gate, t_expert, t_copy_expert);
        out4[0] = o.tpot;
        out4[1] = o.stall_copies;
        out4[2] = o.prefetch_copies;
        out4[3] = o.useful_prefetch;
    });
}

}  // extern "C"
