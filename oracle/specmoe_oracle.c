/* specmoe_oracle.c — CPU restatement of the reference's speculative-decode
 * path.  TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg as the *checker*; the product path never
 * links or calls it.
 *
 * Every function restates one reference function with the same IEEE
 * operation order (compiled with -ffp-contract=off, like the reference's
 * x86-64 Release build which emits no FMA):
 *   f32 dot products accumulate sequentially (numerics.cpp:136-147),
 *   softmax / rms_norm / silu use f64 internally (numerics.cpp:37-89).
 * Pinned against the reference itself: tests/golden/ fixtures are produced by
 * oracle/_ref/libspecmoe_ref.so (the unmodified reference library) via
 * tests/golden/make_golden.py, and tests/test_oracle.py checks this file
 * bit-for-bit against them.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define G64 0x9E3779B97F4A7C15ull

/* ---- RNG: numerics.hpp:35-64, numerics.cpp:10-35 ------------------------ */

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* derive_seed: FNV-1a over the label, then two splitmix rounds (numerics.cpp:20-35). */
uint64_t orc_derive_seed(uint64_t seed, const char* label) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (const unsigned char* p = (const unsigned char*)label; *p; ++p) {
        h ^= *p;
        h *= 0x100000001b3ull;
    }
    uint64_t z = seed ^ h;
    for (int i = 0; i < 2; ++i) {
        z += G64;
        z = mix64(z);
    }
    return z;
}

/* splitmix64 is counter based: the n-th draw (1-based) of Rng(seed) is
 * mix64(seed + n*G).  Gaussian i consumes draws 12i+1 .. 12i+12
 * (next_gaussian, numerics.cpp:10-14: sum of 12 uniforms minus 6). */
static inline double gaussian_at(uint64_t seed, uint64_t i) {
    double s = 0.0;
    uint64_t st = seed + (12 * i) * G64;
    for (int j = 0; j < 12; ++j) {
        st += G64;
        s += (double)(mix64(st) >> 11) * 0x1.0p-53;
    }
    return s - 6.0;
}

typedef struct {
    float* out;
    uint64_t seed, begin, end;
    double stddev;
} fill_job;

static void* fill_worker(void* arg) {
    fill_job* j = (fill_job*)arg;
    for (uint64_t i = j->begin; i < j->end; ++i)
        j->out[i] = (float)(gaussian_at(j->seed, i) * j->stddev);
    return NULL;
}

static int g_threads = 8;
void orc_set_threads(int n) { g_threads = n < 1 ? 1 : n; }

/* Rng::fill_gaussian(out, stddev) with x = f32(next_gaussian() * f64(stddev)). */
void orc_fill_gaussian(uint64_t seed, double stddev, float* out, uint64_t n) {
    int nt = (n < (1u << 16)) ? 1 : g_threads;
    pthread_t th[64];
    fill_job jobs[64];
    int started[64] = {0};
    if (nt > 64) nt = 64;
    for (int t = 0; t < nt; ++t) {
        jobs[t].out = out;
        jobs[t].seed = seed;
        jobs[t].stddev = stddev;
        jobs[t].begin = n * t / nt;
        jobs[t].end = n * (t + 1) / nt;
        /* a thread that cannot be created (process / cgroup thread limits) runs inline */
        started[t] = nt > 1 && pthread_create(&th[t], NULL, fill_worker, &jobs[t]) == 0;
        if (!started[t]) fill_worker(&jobs[t]);
    }
    for (int t = 0; t < nt; ++t)
        if (started[t]) pthread_join(th[t], NULL);
}

/* Rng(seed).next_u64() stream, for random_token_stream (trace.cpp:205-211). */
void orc_token_stream(int64_t n, int vocab, uint64_t seed, int* out) {
    uint64_t st = orc_derive_seed(seed, "token-stream");
    for (int64_t i = 0; i < n; ++i) {
        st += G64;
        out[i] = (int)(mix64(st) % (uint64_t)vocab);
    }
}

float orc_round_bf16(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    u &= 0xFFFF0000u;
    float y;
    memcpy(&y, &u, 4);
    return y;
}

/* ---- numerics: numerics.cpp:37-162 --------------------------------------- */

static char g_err[256];
const char* orc_last_error(void) { return g_err; }
#define FAIL(code, ...)                                 \
    do {                                                \
        snprintf(g_err, sizeof g_err, __VA_ARGS__);     \
        return code;                                    \
    } while (0)

/* softmax (numerics.cpp:37-54): f64 exp of max-subtracted input, f32 out. */
int orc_softmax(const float* v, int n, float* out) {
    if (n < 1) FAIL(1, "softmax: empty input");
    float mx = v[0];
    for (int i = 0; i < n; ++i) {
        if (!isfinite(v[i])) FAIL(1, "softmax: non-finite input");
        mx = v[i] > mx ? v[i] : mx;
    }
    double* e = (double*)malloc(sizeof(double) * n);
    double z = 0.0;
    for (int i = 0; i < n; ++i) {
        e[i] = exp((double)v[i] - (double)mx);
        z += e[i];
    }
    for (int i = 0; i < n; ++i) out[i] = (float)(e[i] / z);
    free(e);
    return 0;
}

/* top_k (numerics.cpp:56-70): value desc, ties lower index first.  The
 * comparator is a strict total order, so selection by repeated max is the
 * same result as std::partial_sort. */
int orc_top_k(const float* v, int n, int k, int* idx, float* vals) {
    if (k < 1 || k > n) FAIL(1, "top_k: k out of range");
    for (int i = 0; i < k; ++i) {
        int best = -1;
        for (int j = 0; j < n; ++j) {
            int taken = 0;
            for (int t = 0; t < i; ++t)
                if (idx[t] == j) taken = 1;
            if (taken) continue;
            if (best < 0 || v[j] > v[best]) best = j; /* strict > keeps lower index on ties */
        }
        idx[i] = best;
        if (vals) vals[i] = v[best];
    }
    return 0;
}

/* rms_norm (numerics.cpp:72-84): f64 sum of squares, f32 scale, (v*scale)*gain. */
void orc_rms_norm(const float* v, const float* gain, int n, float eps, float* out) {
    double ss = 0.0;
    for (int i = 0; i < n; ++i) ss += (double)v[i] * (double)v[i];
    const float scale = (float)(1.0 / sqrt(ss / (double)n + (double)eps));
    for (int i = 0; i < n; ++i) out[i] = v[i] * scale * gain[i];
}

/* silu (numerics.cpp:86-89). */
float orc_silu(float x) {
    const double xd = (double)x;
    return (float)(xd / (1.0 + exp(-xd)));
}

/* linear (numerics.cpp:136-147): per-row sequential f32 dot. */
void orc_linear(const float* w, int rows, int cols, const float* x, float* out) {
    for (int r = 0; r < rows; ++r) {
        const float* wr = w + (size_t)r * cols;
        float acc = 0.0f;
        for (int c = 0; c < cols; ++c) acc += wr[c] * x[c];
        out[r] = acc;
    }
}

/* make_decision (model.cpp:258-274).  gating 0 = softmax-topk-renorm,
 * 1 = topk-softmax. */
int orc_make_decision(const float* logits, int E, int k, int gating, int* ids, float* gates) {
    float vals[1024];
    if (k > 1024) FAIL(1, "k too large");
    if (gating == 0) {
        float* probs = (float*)malloc(sizeof(float) * E);
        int rc = orc_softmax(logits, E, probs);
        if (rc) {
            free(probs);
            return rc;
        }
        rc = orc_top_k(probs, E, k, ids, vals);
        free(probs);
        if (rc) return rc;
        float total = 0.0f;
        for (int i = 0; i < k; ++i) total += vals[i];
        for (int i = 0; i < k; ++i) gates[i] = vals[i] / total;
    } else {
        int rc = orc_top_k(logits, E, k, ids, vals);
        if (rc) return rc;
        return orc_softmax(vals, k, gates);
    }
    return 0;
}

/* ---- model: model.hpp:28-91, model.cpp:112-396 --------------------------- */

typedef struct {
    int L, E, K, H, Hm, V, D;
    float eps;
    uint64_t seed;
    int gating;
} orc_config;

typedef struct {
    orc_config c;
    float *emb, *unemb, *final_gain;
    float **attn_gain, **moe_gain, **wq, **wk, **wv, **wo, **gate;
    float **wg, **wu, **wd; /* [l*E + e]; NULL until generated in a lazy model */
    int round;              /* bf16 rounding of generated tensors */
    float stddev;
} orc_model;

static float* alloc_f(size_t n) { return (float*)calloc(n, sizeof(float)); }

static void init_tensor(float* t, size_t n, uint64_t seed, const char* label, float stddev,
                        int round) {
    orc_fill_gaussian(orc_derive_seed(seed, label), (double)stddev, t, n);
    if (round)
        for (size_t i = 0; i < n; ++i) t[i] = orc_round_bf16(t[i]);
}

/* build_model (model.cpp:112-158): stddev = 0.4f / sqrt(f32 H), gains = 1,
 * every tensor from Rng(derive_seed(seed, label)).  `round` = 1 rounds every
 * matrix to bf16 (the values the GPU stores; SURVEY §8c parity recipe).
 * `layer_lo..layer_hi` allows depth-truncated construction: per-layer tensors
 * depend only on (seed, label, shape). */
/* One expert's three tensors (model.cpp:145-155 labels), generated on first
 * use in a lazy model: per-tensor streams depend only on (seed, label), so a
 * lazily generated expert equals the eagerly built one. */
static void gen_expert(orc_model* m, int l, int e) {
    const size_t n = (size_t)m->c.Hm * m->c.H, i = (size_t)l * m->c.E + e;
    char label[128];
    if (m->wg[i]) return;
    m->wg[i] = alloc_f(n);
    m->wu[i] = alloc_f(n);
    m->wd[i] = alloc_f(n);
    snprintf(label, sizeof label, "layer%d.expert%d.w_gate", l, e);
    init_tensor(m->wg[i], n, m->c.seed, label, m->stddev, m->round);
    snprintf(label, sizeof label, "layer%d.expert%d.w_up", l, e);
    init_tensor(m->wu[i], n, m->c.seed, label, m->stddev, m->round);
    snprintf(label, sizeof label, "layer%d.expert%d.w_down", l, e);
    init_tensor(m->wd[i], n, m->c.seed, label, m->stddev, m->round);
}

static orc_model* model_build(int L, int E, int K, int H, int Hm, int V, int D, float eps,
                              uint64_t seed, int gating, int round, int lazy);

orc_model* orc_model_build(int L, int E, int K, int H, int Hm, int V, int D, float eps,
                           uint64_t seed, int gating, int round) {
    return model_build(L, E, K, H, Hm, V, D, eps, seed, gating, round, 0);
}

/* The dense part only; experts are generated on first use (moe_block,
 * orc_model_tensor, orc_model_ensure_experts) and can be released again — the
 * streaming per-layer checker holds one layer's experts at a time, so a
 * 48-layer Q30 or a Q235 model fits in host memory. */
orc_model* orc_model_build_lazy(int L, int E, int K, int H, int Hm, int V, int D, float eps,
                                uint64_t seed, int gating, int round) {
    return model_build(L, E, K, H, Hm, V, D, eps, seed, gating, round, 1);
}

void orc_model_ensure_experts(orc_model* m, int l, const int* ids, int n) {
    for (int i = 0; i < n; ++i)
        if (l >= 0 && l < m->c.L && ids[i] >= 0 && ids[i] < m->c.E) gen_expert(m, l, ids[i]);
}

void orc_model_release_expert(orc_model* m, int l, int e) {
    const size_t i = (size_t)l * m->c.E + e;
    free(m->wg[i]); free(m->wu[i]); free(m->wd[i]);
    m->wg[i] = m->wu[i] = m->wd[i] = NULL;
}

static orc_model* model_build(int L, int E, int K, int H, int Hm, int V, int D, float eps,
                              uint64_t seed, int gating, int round, int lazy) {
    orc_model* m = (orc_model*)calloc(1, sizeof(orc_model));
    orc_config c = {L, E, K, H, Hm, V, D, eps, seed, gating};
    m->c = c;
    const float stddev = 0.4f / sqrtf((float)H);
    m->round = round;
    m->stddev = stddev;
    m->emb = alloc_f((size_t)V * H);
    init_tensor(m->emb, (size_t)V * H, seed, "embedding", stddev, round);
    m->unemb = alloc_f((size_t)V * H);
    init_tensor(m->unemb, (size_t)V * H, seed, "unembed", stddev, round);
    m->final_gain = alloc_f(H);
    for (int i = 0; i < H; ++i) m->final_gain[i] = 1.0f;
#define PL(name) m->name = (float**)calloc(L, sizeof(float*))
    PL(attn_gain); PL(moe_gain); PL(wq); PL(wk); PL(wv); PL(wo); PL(gate);
#undef PL
    m->wg = (float**)calloc((size_t)L * E, sizeof(float*));
    m->wu = (float**)calloc((size_t)L * E, sizeof(float*));
    m->wd = (float**)calloc((size_t)L * E, sizeof(float*));
    char label[128];
    for (int l = 0; l < L; ++l) {
        m->attn_gain[l] = alloc_f(H);
        m->moe_gain[l] = alloc_f(H);
        for (int i = 0; i < H; ++i) m->attn_gain[l][i] = m->moe_gain[l][i] = 1.0f;
        float** dst[4] = {&m->wq[l], &m->wk[l], &m->wv[l], &m->wo[l]};
        const char* nm[4] = {"wq", "wk", "wv", "wo"};
        for (int t = 0; t < 4; ++t) {
            *dst[t] = alloc_f((size_t)D * H);
            snprintf(label, sizeof label, "layer%d.%s", l, nm[t]);
            init_tensor(*dst[t], (size_t)D * H, seed, label, stddev, round);
        }
        m->gate[l] = alloc_f((size_t)E * H);
        snprintf(label, sizeof label, "layer%d.gate", l);
        init_tensor(m->gate[l], (size_t)E * H, seed, label, stddev, round);
        if (!lazy)
            for (int e = 0; e < E; ++e) gen_expert(m, l, e);
    }
    return m;
}

void orc_model_free(orc_model* m) {
    if (!m) return;
    const int L = m->c.L, E = m->c.E;
    for (int l = 0; l < L; ++l) {
        free(m->attn_gain[l]); free(m->moe_gain[l]); free(m->wq[l]); free(m->wk[l]);
        free(m->wv[l]); free(m->wo[l]); free(m->gate[l]);
        for (int e = 0; e < E; ++e) {
            free(m->wg[l * E + e]); free(m->wu[l * E + e]); free(m->wd[l * E + e]);
        }
    }
    free(m->attn_gain); free(m->moe_gain); free(m->wq); free(m->wk); free(m->wv); free(m->wo);
    free(m->gate); free(m->wg); free(m->wu); free(m->wd);
    free(m->emb); free(m->unemb); free(m->final_gain);
    free(m);
}

/* Pointer + element count of a named tensor (reference labels, model.cpp:132-155). */
float* orc_model_tensor(orc_model* m, const char* name, int64_t* count) {
    const orc_config* c = &m->c;
    int l = -1, e = -1;
    char rest[64];
    *count = 0;
    if (!strcmp(name, "embedding")) { *count = (int64_t)c->V * c->H; return m->emb; }
    if (!strcmp(name, "unembed")) { *count = (int64_t)c->V * c->H; return m->unemb; }
    if (!strcmp(name, "final_norm_gain")) { *count = c->H; return m->final_gain; }
    if (sscanf(name, "layer%d.expert%d.%63s", &l, &e, rest) == 3) {
        if (l < 0 || l >= c->L || e < 0 || e >= c->E) return NULL;
        *count = (int64_t)c->Hm * c->H;
        gen_expert(m, l, e);
        if (!strcmp(rest, "w_gate")) return m->wg[l * c->E + e];
        if (!strcmp(rest, "w_up")) return m->wu[l * c->E + e];
        if (!strcmp(rest, "w_down")) return m->wd[l * c->E + e];
        *count = 0;
        return NULL;
    }
    if (sscanf(name, "layer%d.%63s", &l, rest) == 2) {
        if (l < 0 || l >= c->L) return NULL;
        if (!strcmp(rest, "attn_norm_gain")) { *count = c->H; return m->attn_gain[l]; }
        if (!strcmp(rest, "moe_norm_gain")) { *count = c->H; return m->moe_gain[l]; }
        *count = (int64_t)c->D * c->H;
        if (!strcmp(rest, "wq")) return m->wq[l];
        if (!strcmp(rest, "wk")) return m->wk[l];
        if (!strcmp(rest, "wv")) return m->wv[l];
        if (!strcmp(rest, "wo")) return m->wo[l];
        *count = (int64_t)c->E * c->H;
        if (!strcmp(rest, "gate")) return m->gate[l];
    }
    *count = 0;
    return NULL;
}

/* expert_ffn (model.cpp:283-288). scratch >= 2*Hm floats. */
void orc_expert_ffn(const float* wg, const float* wu, const float* wd, int H, int Hm,
                    const float* x, float* y, float* scratch) {
    float* g = scratch;
    float* u = scratch + Hm;
    orc_linear(wg, Hm, H, x, g);
    orc_linear(wu, Hm, H, x, u);
    for (int i = 0; i < Hm; ++i) g[i] = orc_silu(g[i]) * u[i];
    orc_linear(wd, H, Hm, g, y);
}

/* expert_ffn of one generated expert of the model (y [H]). */
int orc_model_expert_ffn(const orc_model* m, int l, int e, const float* x, float* y) {
    const int H = m->c.H, Hm = m->c.Hm, E = m->c.E;
    if (l < 0 || l >= m->c.L || e < 0 || e >= E) FAIL(1, "expert_ffn: bad layer/expert");
    const size_t i = (size_t)l * E + e;
    if (!m->wg[i]) FAIL(1, "expert_ffn: expert not generated (orc_model_ensure_experts)");
    float* scratch = alloc_f(2 * (size_t)Hm);
    orc_expert_ffn(m->wg[i], m->wu[i], m->wd[i], H, Hm, x, y, scratch);
    free(scratch);
    return 0;
}

typedef struct {
    const orc_model* m;
    int l, e;
    const float* x;
    float* y;
} ffn_job;

static void* ffn_worker(void* a) {
    ffn_job* j = (ffn_job*)a;
    orc_model_expert_ffn(j->m, j->l, j->e, j->x, j->y);
    return NULL;
}

/* moe_block (model.cpp:290-304): out[j] += g_i * y_i[j] in decision order;
 * raw (nullable) receives the unweighted outputs [k][H].  The k expert_ffn
 * calls are independent and run on threads for large experts; the mixture
 * stays sequential in decision order. */
static void moe_block(const orc_model* m, int l, const float* s, const int* ids,
                      const float* gates, float* out, float* raw) {
    const int H = m->c.H, Hm = m->c.Hm, K = m->c.K;
    orc_model_ensure_experts((orc_model*)m, l, ids, K);
    float* ys = alloc_f((size_t)K * H);
    const int par = g_threads > 1 && (size_t)H * Hm >= (1u << 18) && K <= 64;
    pthread_t th[64];
    ffn_job jobs[64];
    int started[64] = {0};
    for (int i = 0; i < K; ++i) {
        ffn_job jb = {m, l, ids[i], s, ys + (size_t)i * H};
        jobs[i] = jb;
        /* a thread that cannot be created (process / cgroup thread limits) runs inline */
        started[i] = par && pthread_create(&th[i], NULL, ffn_worker, &jobs[i]) == 0;
        if (!started[i]) ffn_worker(&jobs[i]);
    }
    for (int i = 0; i < K; ++i)
        if (started[i]) pthread_join(th[i], NULL);
    for (int j = 0; j < H; ++j) out[j] = 0.0f;
    for (int i = 0; i < K; ++i) {
        const float g = gates[i];
        const float* y = ys + (size_t)i * H;
        for (int j = 0; j < H; ++j) out[j] += g * y[j];
        if (raw) memcpy(raw + (size_t)i * H, y, sizeof(float) * H);
    }
    free(ys);
}

/* DecodeState (model.hpp:82-91): per layer K/V history [cap][D]. */
typedef struct {
    int L, D, cap, position;
    float** keys;
    float** vals;
} orc_state;

orc_state* orc_state_new(int L, int D, int cap) {
    orc_state* s = (orc_state*)calloc(1, sizeof(orc_state));
    s->L = L; s->D = D; s->cap = cap; s->position = 0;
    s->keys = (float**)calloc(L, sizeof(float*));
    s->vals = (float**)calloc(L, sizeof(float*));
    for (int l = 0; l < L; ++l) {
        s->keys[l] = alloc_f((size_t)cap * D);
        s->vals[l] = alloc_f((size_t)cap * D);
    }
    return s;
}

void orc_state_free(orc_state* s) {
    if (!s) return;
    for (int l = 0; l < s->L; ++l) { free(s->keys[l]); free(s->vals[l]); }
    free(s->keys); free(s->vals); free(s);
}

/* apply_rope (model.cpp:309-321). */
static void apply_rope(float* v, int position, int D) {
    for (int i = 0; i < D / 2; ++i) {
        const double theta = pow(10000.0, -2.0 * (double)i / (double)D);
        const double angle = (double)position * theta;
        const float c = (float)cos(angle);
        const float s = (float)sin(angle);
        const float x0 = v[2 * i], x1 = v[2 * i + 1];
        v[2 * i] = x0 * c - x1 * s;
        v[2 * i + 1] = x0 * s + x1 * c;
    }
}

/* attention_step (model.cpp:325-353). */
static int attention_step(const orc_model* m, int l, orc_state* st, const float* x, float* out) {
    const int H = m->c.H, D = m->c.D, pos = st->position;
    if (pos >= st->cap) FAIL(2, "oracle: KV capacity exceeded");
    float* q = alloc_f(D);
    float* k = st->keys[l] + (size_t)pos * D;
    float* v = st->vals[l] + (size_t)pos * D;
    orc_linear(m->wq[l], D, H, x, q);
    orc_linear(m->wk[l], D, H, x, k);
    orc_linear(m->wv[l], D, H, x, v);
    apply_rope(q, pos, D);
    apply_rope(k, pos, D);
    const int n = pos + 1;
    const float inv_sqrt_d = 1.0f / sqrtf((float)D);
    float* scores = alloc_f(n);
    float* w = alloc_f(n);
    for (int j = 0; j < n; ++j) {
        const float* kj = st->keys[l] + (size_t)j * D;
        float acc = 0.0f;
        for (int i = 0; i < D; ++i) acc += q[i] * kj[i];
        scores[j] = acc * inv_sqrt_d;
    }
    orc_softmax(scores, n, w);
    float* ctx = alloc_f(D);
    for (int j = 0; j < n; ++j) {
        const float a = w[j];
        const float* vj = st->vals[l] + (size_t)j * D;
        for (int i = 0; i < D; ++i) ctx[i] += a * vj[i];
    }
    orc_linear(m->wo[l], H, D, ctx, out);
    free(q); free(scores); free(w); free(ctx);
    return 0;
}

/* Teacher-forced attention of one layer (model.cpp:376-380) over positions
 * 0..n-1 given each position's layer input x_j (X [n][H]): R_j = x_j +
 * attention_step(rms_norm(x_j, attn_gain_l)) with the K/V history built from
 * those same inputs — the per-layer check of a recorded decode. */
int orc_attn_layer(const orc_model* m, int l, const float* X, int n, float* R) {
    const int H = m->c.H;
    if (l < 0 || l >= m->c.L || n < 1) FAIL(1, "attn_layer: bad layer or length");
    orc_state* st = orc_state_new(m->c.L, m->c.D, n);
    float* a_in = alloc_f(H);
    float* a_out = alloc_f(H);
    int rc = 0;
    for (int j = 0; j < n && !rc; ++j) {
        st->position = j;
        orc_rms_norm(X + (size_t)j * H, m->attn_gain[l], H, m->c.eps, a_in);
        rc = attention_step(m, l, st, a_in, a_out);
        for (int i = 0; i < H; ++i) R[(size_t)j * H + i] = X[(size_t)j * H + i] + a_out[i];
    }
    free(a_in); free(a_out);
    orc_state_free(st);
    return rc;
}

/* ---- speculation: speculation.cpp:104-121, 167-399 ----------------------- */

typedef struct {
    int L, E, H;
    float* d;        /* [L][E][H] */
    int64_t* counts; /* [L][E] */
} orc_table;

orc_table* orc_table_new(int L, int E, int H) {
    orc_table* t = (orc_table*)calloc(1, sizeof(orc_table));
    t->L = L; t->E = E; t->H = H;
    t->d = alloc_f((size_t)L * E * H);
    t->counts = (int64_t*)calloc((size_t)L * E, sizeof(int64_t));
    return t;
}
void orc_table_free(orc_table* t) {
    if (!t) return;
    free(t->d); free(t->counts); free(t);
}
float* orc_table_data(orc_table* t) { return t->d; }
int64_t* orc_table_counts(orc_table* t) { return t->counts; }

/* layer_default (speculation.cpp:104-117). */
void orc_layer_default(const orc_table* t, const int* ids, const float* gates, int k, int l,
                       float* d) {
    const int H = t->H;
    for (int j = 0; j < H; ++j) d[j] = 0.0f;
    for (int i = 0; i < k; ++i) {
        const float* de = t->d + ((size_t)l * t->E + ids[i]) * H;
        const float g = gates[i];
        for (int j = 0; j < H; ++j) d[j] += g * de[j];
    }
}

/* quasi_hidden (speculation.cpp:119-121): rms_norm(r + d, gain_{l+1}). */
void orc_quasi_hidden(const float* r, const float* d, const float* gain, int H, float eps,
                      float* q) {
    float* t = alloc_f(H);
    for (int j = 0; j < H; ++j) t[j] = r[j] + d[j];
    orc_rms_norm(t, gain, H, eps, q);
    free(t);
}

/* ---- estimator: estimator.hpp:41-72, estimator.cpp:54-167 ---------------- */

typedef struct {
    int d, m, n, E, L;
    float eps;
    int64_t total;
    float* flat;
} orc_est;

static int64_t est_latent(const orc_est* p) { return p->d / p->m; }

orc_est* orc_est_new(int d, int mred, int nexp, int E, int L, float eps) {
    orc_est* p = (orc_est*)calloc(1, sizeof(orc_est));
    p->d = d; p->m = mred; p->n = nexp; p->E = E; p->L = L; p->eps = eps;
    const int64_t dm = d / mred, mlp = dm * nexp;
    p->total = dm * d + (int64_t)L * dm + mlp * dm + dm * mlp + 2 * dm + (int64_t)E * dm;
    p->flat = alloc_f((size_t)p->total);
    return p;
}
void orc_est_free(orc_est* p) {
    if (!p) return;
    free(p->flat); free(p);
}
float* orc_est_flat(orc_est* p, int64_t* total) {
    *total = p->total;
    return p->flat;
}

/* init_estimator_params (estimator.cpp:54-77). */
void orc_est_init(orc_est* p, uint64_t seed) {
    const int64_t dm = est_latent(p), mlp = dm * p->n;
    float* a = p->flat;
    float* pos = a + dm * p->d;
    float* b = pos + (int64_t)p->L * dm;
    float* c = b + mlp * dm;
    float* g = c + dm * mlp;
    float* bias = g + dm;
    float* wh = bias + dm;
    orc_fill_gaussian(orc_derive_seed(seed, "estimator.a"), 1.0 / sqrt((double)p->d), a, dm * p->d);
    orc_fill_gaussian(orc_derive_seed(seed, "estimator.pos"), 0.02, pos, (int64_t)p->L * dm);
    orc_fill_gaussian(orc_derive_seed(seed, "estimator.b"), 1.0 / sqrt((double)dm), b, mlp * dm);
    orc_fill_gaussian(orc_derive_seed(seed, "estimator.c"), 1.0 / sqrt((double)mlp), c, dm * mlp);
    orc_fill_gaussian(orc_derive_seed(seed, "estimator.w_head"), 1.0 / sqrt((double)dm), wh,
                      (int64_t)p->E * dm);
    for (int64_t i = 0; i < dm; ++i) { g[i] = 1.0f; bias[i] = 0.0f; }
}

/* estimator_forward<float> (estimator.cpp:94-161): logits only. */
int orc_est_logits(const orc_est* p, const float* q, int layer, float* logits) {
    if (layer < 0 || layer >= p->L) FAIL(1, "estimator: layer out of range");
    const int64_t dm = est_latent(p), mlp = dm * p->n;
    const float* A = p->flat;
    const float* pos = A + dm * p->d + (int64_t)layer * dm;
    const float* B = A + dm * p->d + (int64_t)p->L * dm;
    const float* C = B + mlp * dm;
    const float* gain = C + dm * mlp;
    const float* bias = gain + dm;
    const float* W = bias + dm;
    float* z = alloc_f(dm);
    float* act = alloc_f(mlp);
    float* h = alloc_f(dm);
    for (int64_t j = 0; j < dm; ++j) {
        const float* row = A + j * p->d;
        float acc = 0.0f;
        for (int i = 0; i < p->d; ++i) acc += row[i] * q[i];
        z[j] = acc + pos[j];
    }
    for (int64_t t = 0; t < mlp; ++t) {
        const float* row = B + t * dm;
        float acc = 0.0f;
        for (int64_t j = 0; j < dm; ++j) acc += row[j] * z[j];
        act[t] = acc / (1.0f + expf(-acc));
    }
    for (int64_t j = 0; j < dm; ++j) {
        const float* row = C + j * mlp;
        float acc = 0.0f;
        for (int64_t t = 0; t < mlp; ++t) acc += row[t] * act[t];
        h[j] = z[j] + acc;
    }
    float mean = 0.0f;
    for (int64_t j = 0; j < dm; ++j) mean += h[j];
    mean /= (float)dm;
    float var = 0.0f;
    for (int64_t j = 0; j < dm; ++j) {
        const float cc = h[j] - mean;
        var += cc * cc;
    }
    var /= (float)dm;
    const float inv_std = 1.0f / sqrtf(var + p->eps);
    for (int64_t j = 0; j < dm; ++j) h[j] = (h[j] - mean) * inv_std; /* xhat */
    for (int e = 0; e < p->E; ++e) {
        const float* row = W + (int64_t)e * dm;
        float acc = 0.0f;
        for (int64_t j = 0; j < dm; ++j) acc += row[j] * (gain[j] * h[j] + bias[j]);
        logits[e] = acc;
    }
    free(z); free(act); free(h);
    return 0;
}

/* ---- predictors + decode loops ------------------------------------------ */

enum { K_BASELINE = 0, K_ROUTER_PF = 1, K_EST_PF = 2, K_HYBRID = 3, K_ORACLE = 4 };

typedef struct {
    int kind;
    const orc_table* table;
    const orc_est* est;
    int* hybrid; /* L-1 entries */
    /* oracle shadow state + recorded true decisions of the current token */
    orc_state* shadow;
    int* sh_ids;
    float* sh_gates;
    float* sh_logits;
} orc_pred;

typedef struct {
    float *s, *r, *m, *logits, *gates, *outputs, *final_logits, *pred_logits, *pred_gates;
    int *ids, *pred_ids;
} orc_trace;

static int forward(const orc_model* m, orc_state* st, int token, orc_pred* pred, int spec,
                   const orc_trace* tr, int step, float* out_logits);

/* predict_next (speculation.cpp:174-306).  logits_out [E], ids/gates [K]. */
static int predict_next(const orc_model* m, orc_pred* p, int kind, int l, const float* s,
                        const float* r, const int* ex_ids, const float* ex_gates,
                        float* logits_out, int* ids, float* gates) {
    const orc_config* c = &m->c;
    if (l < 0 || l >= c->L - 1) FAIL(1, "predict_next: layer must be < L-1");
    if (kind == K_HYBRID) kind = p->hybrid ? p->hybrid[l] : K_ROUTER_PF;
    if (kind == K_BASELINE) {
        orc_linear(m->gate[l + 1], c->E, c->H, s, logits_out);
        return orc_make_decision(logits_out, c->E, c->K, c->gating, ids, gates);
    }
    if (kind == K_ORACLE) {
        memcpy(logits_out, p->sh_logits + (size_t)(l + 1) * c->E, sizeof(float) * c->E);
        memcpy(ids, p->sh_ids + (size_t)(l + 1) * c->K, sizeof(int) * c->K);
        memcpy(gates, p->sh_gates + (size_t)(l + 1) * c->K, sizeof(float) * c->K);
        return 0;
    }
    if (!p->table) FAIL(1, "router-pf: missing default-vector table");
    float* d = alloc_f(c->H);
    float* q = alloc_f(c->H);
    orc_layer_default(p->table, ex_ids, ex_gates, c->K, l, d);
    orc_quasi_hidden(r, d, m->moe_gain[l + 1], c->H, c->eps, q);
    int rc;
    if (kind == K_ROUTER_PF) {
        orc_linear(m->gate[l + 1], c->E, c->H, q, logits_out);
        rc = orc_make_decision(logits_out, c->E, c->K, c->gating, ids, gates);
    } else {
        if (!p->est) {
            free(d); free(q);
            FAIL(1, "est-pf: missing estimator");
        }
        rc = orc_est_logits(p->est, q, l, logits_out);
        if (!rc) rc = orc_make_decision(logits_out, c->E, c->K, c->gating, ids, gates);
    }
    free(d);
    free(q);
    return rc;
}

/* Oracle::begin_token / observe_prompt_token (speculation.cpp:266-280):
 * run the true path on the shadow state, capturing per-layer decisions. */
static int oracle_shadow(const orc_model* m, orc_pred* p, int token, int record) {
    const orc_config* c = &m->c;
    orc_trace tr;
    memset(&tr, 0, sizeof tr);
    if (record) {
        tr.logits = p->sh_logits;
        tr.ids = p->sh_ids;
        tr.gates = p->sh_gates;
    }
    float* lg = alloc_f(c->V);
    int rc = forward(m, p->shadow, token, NULL, 0, record ? &tr : NULL, 0, lg);
    free(lg);
    return rc;
}

/* forward_decode (model.cpp:355-389) when spec == 0, speculative_forward
 * (speculation.cpp:350-399) when spec == 1. */
static int forward(const orc_model* m, orc_state* st, int token, orc_pred* pred, int spec,
                   const orc_trace* tr, int step, float* out_logits) {
    const orc_config* c = &m->c;
    const int L = c->L, H = c->H, E = c->E, K = c->K;
    if (token < 0 || token >= c->V) FAIL(1, "forward: token out of vocab");
    int rc = 0;
    if (spec && pred->kind == K_ORACLE) {
        rc = oracle_shadow(m, pred, token, 1);
        if (rc) return rc;
    }
    float* x = alloc_f(H);
    float* a_in = alloc_f(H);
    float* a_out = alloc_f(H);
    float* r = alloc_f(H);
    float* s = alloc_f(H);
    float* mo = alloc_f(H);
    float* lg = alloc_f(E);
    float* plg = alloc_f(E);
    float* raw = alloc_f((size_t)K * H);
    int ex_ids[1024], pend_ids[1024], t_ids[1024];
    float ex_gates[1024], pend_gates[1024], t_gates[1024];
    memcpy(x, m->emb + (size_t)token * H, sizeof(float) * H);
    for (int l = 0; l < L && !rc; ++l) {
        orc_rms_norm(x, m->attn_gain[l], H, c->eps, a_in);
        rc = attention_step(m, l, st, a_in, a_out);
        if (rc) break;
        for (int j = 0; j < H; ++j) r[j] = x[j] + a_out[j];
        orc_rms_norm(r, m->moe_gain[l], H, c->eps, s);
        orc_linear(m->gate[l], E, H, s, lg);
        rc = orc_make_decision(lg, E, K, c->gating, t_ids, t_gates);
        if (rc) break;
        if (!spec || l == 0) {
            memcpy(ex_ids, t_ids, sizeof(int) * K);
            memcpy(ex_gates, t_gates, sizeof(float) * K);
        } else {
            memcpy(ex_ids, pend_ids, sizeof(int) * K);
            memcpy(ex_gates, pend_gates, sizeof(float) * K);
        }
        if (spec && l < L - 1) {
            rc = predict_next(m, pred, pred->kind, l, s, r, ex_ids, ex_gates, plg, pend_ids,
                              pend_gates);
            if (rc) break;
            if (tr && tr->pred_ids) {
                const size_t b = (size_t)step * (L - 1) + l;
                memcpy(tr->pred_logits + b * E, plg, sizeof(float) * E);
                memcpy(tr->pred_ids + b * K, pend_ids, sizeof(int) * K);
                memcpy(tr->pred_gates + b * K, pend_gates, sizeof(float) * K);
            }
        }
        for (int i = 0; i < K; ++i)
            if (ex_ids[i] < 0 || ex_ids[i] >= E) {
                rc = 1;
                snprintf(g_err, sizeof g_err, "moe_block: expert index out of range");
            }
        if (rc) break;
        moe_block(m, l, s, ex_ids, ex_gates, mo, raw);
        for (int j = 0; j < H; ++j) x[j] = r[j] + mo[j];
        if (tr) {
            const size_t b = (size_t)step * L + l;
            if (tr->s) memcpy(tr->s + b * H, s, sizeof(float) * H);
            if (tr->r) memcpy(tr->r + b * H, r, sizeof(float) * H);
            if (tr->m) memcpy(tr->m + b * H, mo, sizeof(float) * H);
            if (tr->logits) memcpy(tr->logits + b * E, lg, sizeof(float) * E);
            if (tr->ids) memcpy(tr->ids + b * K, ex_ids, sizeof(int) * K);
            if (tr->gates) memcpy(tr->gates + b * K, ex_gates, sizeof(float) * K);
            if (tr->outputs) memcpy(tr->outputs + b * K * H, raw, sizeof(float) * K * H);
        }
    }
    if (!rc) {
        st->position += 1;
        orc_rms_norm(x, m->final_gain, H, c->eps, a_in);
        orc_linear(m->unemb, c->V, H, a_in, out_logits);
    }
    free(x); free(a_in); free(a_out); free(r); free(s); free(mo); free(lg); free(plg); free(raw);
    return rc;
}

static int argmax_token(const float* v, int n) {
    int best = 0;
    for (int i = 1; i < n; ++i)
        if (v[i] > v[best]) best = i;
    return best;
}

orc_pred* orc_pred_new(int kind, const orc_table* table, const orc_est* est, const int* hybrid,
                       const orc_model* m) {
    orc_pred* p = (orc_pred*)calloc(1, sizeof(orc_pred));
    const orc_config* c = &m->c;
    p->kind = kind;
    p->table = table;
    p->est = est;
    if (hybrid) {
        p->hybrid = (int*)calloc(c->L, sizeof(int));
        memcpy(p->hybrid, hybrid, sizeof(int) * (c->L - 1));
    }
    if (kind == K_ORACLE) {
        p->shadow = NULL; /* created per generate() (capacity known there) */
        p->sh_ids = (int*)calloc((size_t)c->L * c->K, sizeof(int));
        p->sh_gates = alloc_f((size_t)c->L * c->K);
        p->sh_logits = alloc_f((size_t)c->L * c->E);
    }
    return p;
}

void orc_pred_free(orc_pred* p) {
    if (!p) return;
    free(p->hybrid); orc_state_free(p->shadow); free(p->sh_ids); free(p->sh_gates);
    free(p->sh_logits); free(p);
}

/* generate (speculation.cpp:401-421) with the same per-step trace layout as
 * oracle/ref_driver.cpp:ref_generate_trace (step s < P: prefill token s;
 * step P+i: decode step i; S = P + n_new - 1).  Any trace buffer may be NULL. */
/* `forced` (nullable, n_new-1 entries): teacher forcing — decode step i is fed
 * forced[i] instead of the previous argmax (the GPU's smoe_decode_stream). */
int orc_generate_trace_forced(const orc_model* m, const int* prompt, int P, int n_new,
                              orc_pred* pred, const int* forced, int* out_tokens, float* s,
                              float* r, float* mo, float* logits, int* ids, float* gates,
                              float* outputs, float* final_logits, float* pred_logits,
                              int* pred_ids, float* pred_gates) {
    const orc_config* c = &m->c;
    if (P < 1) FAIL(1, "generate: empty prompt");
    const int cap = P + n_new + 1;
    orc_state* st = orc_state_new(c->L, c->D, cap);
    if (pred && pred->kind == K_ORACLE) {
        orc_state_free(pred->shadow);
        pred->shadow = orc_state_new(c->L, c->D, cap);
    }
    orc_trace tr = {s, r, mo, logits, gates, outputs, NULL, pred_logits, pred_gates, ids, pred_ids};
    float* lg = alloc_f(c->V);
    int rc = 0, step = 0;
    for (int i = 0; i < P && !rc; ++i, ++step) {
        rc = forward(m, st, prompt[i], NULL, 0, &tr, step, lg);
        if (!rc && final_logits) memcpy(final_logits + (size_t)step * c->V, lg, sizeof(float) * c->V);
        if (!rc && pred && pred->kind == K_ORACLE) rc = oracle_shadow(m, pred, prompt[i], 0);
    }
    int next = argmax_token(lg, c->V);
    for (int i = 0; i < n_new && !rc; ++i) {
        out_tokens[i] = next;
        if (i + 1 == n_new) break;
        rc = forward(m, st, forced ? forced[i] : next, pred, pred != NULL, &tr, step, lg);
        if (rc) break;
        if (final_logits) memcpy(final_logits + (size_t)step * c->V, lg, sizeof(float) * c->V);
        next = argmax_token(lg, c->V);
        ++step;
    }
    free(lg);
    orc_state_free(st);
    return rc;
}

int orc_generate_trace(const orc_model* m, const int* prompt, int P, int n_new, orc_pred* pred,
                       int* out_tokens, float* s, float* r, float* mo, float* logits, int* ids,
                       float* gates, float* outputs, float* final_logits, float* pred_logits,
                       int* pred_ids, float* pred_gates) {
    return orc_generate_trace_forced(m, prompt, P, n_new, pred, NULL, out_tokens, s, r, mo, logits,
                                     ids, gates, outputs, final_logits, pred_logits, pred_ids,
                                     pred_gates);
}

/* accumulate_default_vectors over random_token_stream(ntok, vocab, seed) with
 * state resets every seq_len tokens (trace.cpp:187-211, speculation.cpp:23-58):
 * f64 sums of raw expert outputs per (layer, expert), frozen to f32. */
int orc_calibrate(const orc_model* m, int64_t ntok, uint64_t seed, int seq_len, orc_table* t) {
    const orc_config* c = &m->c;
    const int L = c->L, E = c->E, K = c->K, H = c->H;
    int* toks = (int*)malloc(sizeof(int) * ntok);
    orc_token_stream(ntok, c->V, seed, toks);
    double* sums = (double*)calloc((size_t)L * E * H, sizeof(double));
    int64_t* counts = (int64_t*)calloc((size_t)L * E, sizeof(int64_t));
    float* raw = alloc_f((size_t)L * K * H);
    int* ids = (int*)calloc((size_t)L * K, sizeof(int));
    float* lg = alloc_f(c->V);
    orc_state* st = NULL;
    orc_trace tr;
    memset(&tr, 0, sizeof tr);
    tr.outputs = raw;
    tr.ids = ids;
    int rc = 0;
    for (int64_t i = 0; i < ntok && !rc; ++i) {
        if (i % seq_len == 0) {
            orc_state_free(st);
            st = orc_state_new(L, c->D, seq_len + 1);
        }
        rc = forward(m, st, toks[i], NULL, 0, &tr, 0, lg);
        for (int l = 0; l < L && !rc; ++l)
            for (int k = 0; k < K; ++k) {
                const int e = ids[l * K + k];
                double* sum = sums + ((size_t)l * E + e) * H;
                const float* out = raw + ((size_t)l * K + k) * H;
                for (int j = 0; j < H; ++j) sum[j] += out[j];
                counts[l * E + e] += 1;
            }
    }
    for (size_t i = 0; i < (size_t)L * E && !rc; ++i) {
        t->counts[i] = counts[i];
        if (counts[i] == 0) continue;
        for (int j = 0; j < H; ++j)
            t->d[i * H + j] = (float)(sums[i * H + j] / (double)counts[i]);
    }
    orc_state_free(st);
    free(toks); free(sums); free(counts); free(raw); free(ids); free(lg);
    return rc;
}

/* ---- reporting: metrics.cpp:9-28, schedule.cpp:92-155 -------------------- */

double orc_recall_at_k(const int* pred, const int* truth, int k) {
    int hits = 0;
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j)
            if (pred[i] == truth[j]) {
                ++hits;
                break;
            }
    return (double)hits / (double)k;
}
