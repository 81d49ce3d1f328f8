// engine.cpp — host runtime (see engine.h).
#include "engine.h"
#include "train.h"

#include <cuda.h>
#include <immintrin.h>

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <unistd.h>
#include <sys/stat.h>
#include <cctype>
#include <sys/syscall.h>
#include <sys/mman.h>
#include <cerrno>
#include <set>
#include <string>

namespace smoe {

namespace {

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw std::runtime_error(std::string("CUDA error in ") + what + ": " +
                                 cudaGetErrorString(e));
}

// derive_seed (numerics.cpp:20-35): FNV-1a over the label, 2 splitmix rounds.
uint64_t derive_seed(uint64_t seed, const std::string& label) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (unsigned char c : label) {
        h ^= c;
        h *= 0x100000001b3ull;
    }
    uint64_t z = seed ^ h;
    for (int i = 0; i < 2; ++i) {
        z += 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z = z ^ (z >> 31);
    }
    return z;
}

uint16_t f2bf(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

// Scatter a row-major f32 [R][C] tensor into the 32-row tile layout
// (smoe_dev.h): virtual row vr = r*mul + add + row_off; tile [vr/32] of
// tile_cols columns; inside a tile, columns in groups of G (16 bytes):
// element (lane, c) at (c / G) * 32 * G + lane * G + c % G.
void tile_write_bf16(uint16_t* dst, const float* src, int R, int C, int tile_cols, int mul,
                     int add, int row_off) {
    for (int r = 0; r < R; ++r) {
        const long long vr = static_cast<long long>(r) * mul + add + row_off;
        uint16_t* base = dst + (vr / 32) * tile_cols * 32 + (vr % 32) * 8;
        for (int c = 0; c < C; ++c)
            base[static_cast<long long>(c / 8) * 256 + c % 8] = f2bf(src[static_cast<long long>(r) * C + c]);
    }
}

void tile_write_f32(float* dst, const float* src, int R, int C) {
    const int tc = round_up(C, 4);
    for (int r = 0; r < R; ++r) {
        float* base = dst + static_cast<long long>(r / 32) * tc * 32 + (r % 32) * 4;
        for (int c = 0; c < C; ++c)
            base[static_cast<long long>(c / 4) * 128 + c % 4] = src[static_cast<long long>(r) * C + c];
    }
}

// cuStreamWriteValue32 through the runtime's driver entry point, so the
// library does not link libcuda (it must load on GPU-less hosts too).
using WriteValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WriteValueFn write_value_fn() {
    static WriteValueFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p)
            throw std::runtime_error("cuStreamWriteValue32 entry point unavailable");
        return reinterpret_cast<WriteValueFn>(p);
    }();
    return fn;
}

// cuMemGetAddressRange: a cudaMalloc'd pointer may live inside a larger
// driver allocation; CUDA IPC handles name the allocation, and the peer's
// opened pointer is its base, so the offset must travel with the handle.
using AddrRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
AddrRangeFn addr_range_fn() {
    static AddrRangeFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p)
            throw std::runtime_error("cuMemGetAddressRange entry point unavailable");
        return reinterpret_cast<AddrRangeFn>(p);
    }();
    return fn;
}

// ncu / compute-sanitizer inject libraries into the process (and their
// launchers export NV_NSIGHT_INJECTION_* / NV_SANITIZER_INJECTION_*).  Both
// serialise kernels against the copy lane, so a device spin on a copy flag
// would never end under them.
bool profiler_attached() {
    for (const char* v : {"NV_NSIGHT_INJECTION_TRANSPORT_TYPE", "NV_SANITIZER_INJECTION_TRANSPORT_TYPE",
                          "NV_COMPUTE_PROFILER_PERFWORKS_DIR", "CUDA_INJECTION64_PATH"}) {
        const char* e = std::getenv(v);
        if (e && *e) return true;
    }
    FILE* f = std::fopen("/proc/self/maps", "r");
    if (!f) return false;
    char line[1024];
    bool hit = false;
    while (!hit && std::fgets(line, sizeof line, f))
        hit = std::strstr(line, "libcuda-injection") || std::strstr(line, "libsanitizer-collection");
    std::fclose(f);
    return hit;
}

bool parse_layer(const std::string& name, int* l, std::string* rest) {
    if (name.rfind("layer", 0) != 0) return false;
    const size_t dot = name.find('.');
    if (dot == std::string::npos) return false;
    *l = std::stoi(name.substr(5, dot - 5));
    *rest = name.substr(dot + 1);
    return true;
}

}  // namespace

// ------------------------------------------------------------------ config --

void ModelCfg::validate() const {
    if (L < 1) throw std::invalid_argument("config: L must be >= 1");
    if (E < 1) throw std::invalid_argument("config: E must be >= 1");
    if (K < 1 || K > E) throw std::invalid_argument("config: k must satisfy 1 <= k <= E");
    if (H < 1) throw std::invalid_argument("config: H must be >= 1");
    if (Hm < 1) throw std::invalid_argument("config: H_moe must be >= 1");
    if (V < 1) throw std::invalid_argument("config: vocab must be >= 1");
    if (D < 1) throw std::invalid_argument("config: head_dim must be >= 1");
    if (D % 2 != 0) throw std::invalid_argument("config: head_dim must be even for rotary pairs");
    if (!(eps > 0.0f)) throw std::invalid_argument("config: eps must be > 0");
    if (gating != 0 && gating != 1) throw std::invalid_argument("config: unknown gating order");
    if (K > kMaxK) throw std::invalid_argument("config: k > 16 not supported on this path");
    if (E > kMaxE) throw std::invalid_argument("config: E > 1024 not supported on this path");
    if (D > kMaxD) throw std::invalid_argument("config: head_dim > 256 not supported on this path");
    if (H > 16384) throw std::invalid_argument("config: hidden > 16384 not supported on this path");
    if (D % 8 != 0) throw std::invalid_argument("config: head_dim must be a multiple of 8 on this path");
    if (H % 8 != 0) throw std::invalid_argument("config: hidden must be a multiple of 8 on this path");
}

// ------------------------------------------------------------ ExpertStore --

namespace {
// NUMA node of a GPU's PCIe root (sysfs), -1 if unknown.
int gpu_numa_node(int device) {
    char bus[32] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) return -1;
    std::string id(bus);
    for (char& ch : id) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    FILE* f = std::fopen(("/sys/bus/pci/devices/" + id + "/numa_node").c_str(), "r");
    if (!f) return -1;
    int node = -1;
    if (std::fscanf(f, "%d", &node) != 1) node = -1;
    std::fclose(f);
    return node;
}
int numa_nodes() {
    int n = 0;
    for (int i = 0; i < 1024; ++i) {
        struct stat st;
        if (stat(("/sys/devices/system/node/node" + std::to_string(i)).c_str(), &st) != 0) break;
        ++n;
    }
    return n;
}
}  // namespace

// Pinned host memory for the expert shard.  On a multi-socket host the pages
// are bound to the NUMA node of the GPU's PCIe root (mmap + mbind, then
// cudaHostRegister pins them there), so each rank's H2D copies read local
// DRAM; otherwise cudaHostAlloc.
ExpertStore::ExpertStore(long long n, long long elems, int device) : n_(n), elems_(elems), packed_(n, 0) {
    const size_t bytes = static_cast<size_t>(n) * elems * 2;
    const int node = gpu_numa_node(device);
    if (node >= 0 && node < 64 && numa_nodes() > 1 && !std::getenv("SMOE_NO_NUMA_BIND")) {
        void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (p == MAP_FAILED) throw std::runtime_error("mmap(expert store) failed");
        unsigned long mask = 1ul << node;
        constexpr int kMpolBind = 2;
        if (syscall(SYS_mbind, p, bytes, kMpolBind, &mask, 64, 0) != 0) {
            munmap(p, bytes);
            throw std::runtime_error("mbind(expert store) to NUMA node " + std::to_string(node) + " failed");
        }
        const cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterPortable);
        if (e != cudaSuccess) {
            munmap(p, bytes);
            ck(e, "cudaHostRegister(expert store)");
        }
        base_ = static_cast<uint16_t*>(p);
        mapped_ = bytes;
        node_ = node;
        return;
    }
    ck(cudaHostAlloc(reinterpret_cast<void**>(&base_), bytes, cudaHostAllocPortable),
       "cudaHostAlloc(expert store)");
}

ExpertStore::~ExpertStore() {
    if (!base_) return;
    if (mapped_) {
        cudaHostUnregister(base_);
        munmap(base_, mapped_);
    } else {
        cudaFreeHost(base_);
    }
}

// Packs every raw block in place, on all host cores.  A block is packed into
// a scratch buffer first (the packed layout overlaps the raw one) and copied
// back over the block's head; blocks that do not pack stay raw.
long long ExpertStore::pack_all() {
    const int nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    std::atomic<long long> next{0}, done{0};
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&] {
            std::vector<uint8_t> buf(static_cast<size_t>(max_packed_bytes()));
            for (long long i; (i = next.fetch_add(1)) < n_;) {
                if (packed_[i]) continue;
                const long long b = xp_pack(expert(i), elems_, buf.data(), max_packed_bytes());
                if (!b) continue;
                std::memcpy(expert(i), buf.data(), static_cast<size_t>(b));
                packed_[i] = b;
                ++done;
            }
        });
    for (auto& t : th) t.join();
    return done.load();
}

void ExpertStore::unpack(long long i) {
    if (!packed_[i]) return;
    std::vector<uint8_t> buf(static_cast<size_t>(packed_[i]));
    std::memcpy(buf.data(), expert(i), buf.size());
    xp_unpack(buf.data(), expert(i));
    packed_[i] = 0;
}

// -------------------------------------------------------------- SlotCache --

SlotCache::SlotCache(int L, int E, int C)
    : L_(L), E_(E), C_(C), expert_slot_(L, std::vector<int>(E, -1)),
      slot_expert_(L, std::vector<int>(C, -1)), stamp_(L, std::vector<long long>(C, -1)),
      freq_(L, std::vector<long long>(E, 0)), hits_(L, 0), misses_(L, 0) {
    const char* p = std::getenv("SMOE_CACHE_POLICY");
    lfu_ = p && std::string(p) == "lfu";
}

void SlotCache::clear_stats() {
    std::fill(hits_.begin(), hits_.end(), 0);
    std::fill(misses_.begin(), misses_.end(), 0);
}

void SlotCache::invalidate() {
    for (int l = 0; l < L_; ++l) {
        std::fill(expert_slot_[l].begin(), expert_slot_[l].end(), -1);
        std::fill(slot_expert_[l].begin(), slot_expert_[l].end(), -1);
        std::fill(stamp_[l].begin(), stamp_[l].end(), -1);
    }
}

// LRU within the layer's pool; never evicts an expert of the same request.
std::vector<std::pair<int, int>> SlotCache::request(int layer, const int* ids, int n, int* hits,
                                                    int* misses) {
    if (layer < 0 || layer >= L_) throw std::runtime_error("copy request with bad layer");
    std::vector<std::pair<int, int>> out;
    *hits = *misses = 0;
    const long long now = ++clock_;
    auto& es = expert_slot_[layer];
    auto& se = slot_expert_[layer];
    auto& st = stamp_[layer];
    auto& fq = freq_[layer];
    for (int i = 0; i < n; ++i)
        if (ids[i] >= 0 && ids[i] < E_) ++fq[ids[i]];
    for (int i = 0; i < n; ++i) {
        const int e = ids[i];
        if (e < 0 || e >= E_) throw std::runtime_error("copy request with bad expert id");
        if (es[e] >= 0) {
            st[es[e]] = now;
            ++*hits;
            continue;
        }
        int victim = -1;
        for (int c = 0; c < C_; ++c) {
            if (st[c] == now) continue;  // holds an expert of this request
            if (victim < 0) {
                victim = c;
                continue;
            }
            if (lfu_ && se[c] >= 0 && se[victim] >= 0) {  // least requested, then least recent
                const long long fc = fq[se[c]], fv = fq[se[victim]];
                if (fc < fv || (fc == fv && st[c] < st[victim])) victim = c;
            } else if (st[c] < st[victim]) {
                victim = c;
            }
        }
        if (victim < 0) throw std::runtime_error("slot pool smaller than the request");
        if (se[victim] >= 0) es[se[victim]] = -1;
        se[victim] = e;
        es[e] = victim;
        st[victim] = now;
        out.emplace_back(victim, e);
        ++*misses;
    }
    hits_[layer] += *hits;
    misses_[layer] += *misses;
    return out;
}

// ---------------------------------------------------------- CopyScheduler --

// Copy threads still running at process exit (a session the host program
// never destroyed) must stop before the CUDA runtime tears itself down: the
// exit hook is registered after the runtime initialised (first scheduler
// start), so atexit's LIFO order runs it first.
namespace {
std::mutex g_live_mu;
std::set<CopyScheduler*>* g_live = nullptr;
void stop_live_schedulers() {
    std::set<CopyScheduler*> live;
    {
        std::lock_guard<std::mutex> g(g_live_mu);
        if (g_live) live = *g_live;
    }
    for (CopyScheduler* c : live) c->stop();
}
}  // namespace

CopyScheduler::CopyScheduler(Session* s) : s_(s) {}
CopyScheduler::~CopyScheduler() { stop(); }

void CopyScheduler::start() {
    {
        std::lock_guard<std::mutex> g(g_live_mu);
        if (!g_live) {
            g_live = new std::set<CopyScheduler*>();
            std::atexit(stop_live_schedulers);
        }
        g_live->insert(this);
    }
    stop_ = false;
    th_ = std::thread([this] { loop(); });
}

void CopyScheduler::stop() {
    stop_ = true;
    if (th_.joinable()) th_.join();
    std::lock_guard<std::mutex> g(g_live_mu);
    if (g_live) g_live->erase(this);
}

std::string CopyScheduler::error() {
    std::lock_guard<std::mutex> g(mu_);
    return err_;
}

std::vector<CopyRecord> CopyScheduler::records() {
    std::lock_guard<std::mutex> g(mu_);
    return recs_;
}

void CopyScheduler::clear_records() {
    std::lock_guard<std::mutex> g(mu_);
    recs_.clear();
    ev_next_ = 0;
}

void CopyScheduler::loop() {
    cudaSetDevice(s_->opts_.device);
    auto idle_since = std::chrono::steady_clock::now();
    while (!stop_.load(std::memory_order_relaxed)) {
        MailboxEntry* e = &s_->h_mailbox_[next_seq_ % kMailboxRing];
        const int seq = __atomic_load_n(const_cast<int*>(&e->seq), __ATOMIC_ACQUIRE);
        ++polls;
        if (seq != next_seq_) {
            _mm_pause();
            auto now = std::chrono::steady_clock::now();
            if (now - idle_since > std::chrono::milliseconds(200))
                std::this_thread::sleep_for(std::chrono::microseconds(50));
            continue;
        }
        MailboxEntry req;
        std::memcpy(&req, e, sizeof req);
        static const bool dbg = std::getenv("SMOE_DEBUG") != nullptr;
        if (dbg)
            std::fprintf(stderr, "[sched] t=%.3f ms seen seq %d layer %d\n",
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(),
                         req.seq, req.layer);
        try {
            handle(req);
        } catch (const std::exception& ex) {
            std::lock_guard<std::mutex> g(mu_);
            if (err_.empty()) err_ = ex.what();
            // unblock the device so it can observe the error instead of spinning
            write_value_fn()(reinterpret_cast<CUstream>(s_->s_copy_),
                                 reinterpret_cast<CUdeviceptr>(s_->ctl_.ready + req.layer),
                                 static_cast<cuuint32_t>(req.seq), 0);
        }
        ++next_seq_;
        idle_since = std::chrono::steady_clock::now();
    }
}

// Alg. 1 "WaitAndPrefetch": stage the requested experts of one layer into
// HBM slots (only cache misses move over PCIe), then publish the slot table
// row and the layer's ready value on the same copy stream (FIFO, like the
// reference's single copy worker, executor.cpp:138-198).
void CopyScheduler::handle(const MailboxEntry& e) {
    Session& s = *s_;
    if (e.nids < 1 || e.nids > kMaxK) throw std::runtime_error("copy request with bad id count");
    if (s.opts_.copy_latency_us > 0)
        std::this_thread::sleep_for(std::chrono::microseconds(s.opts_.copy_latency_us));
    int hits = 0, misses = 0;
    int local[kMaxK];
    int nloc = 0;
    for (int i = 0; i < e.nids; ++i)
        if (s.is_local(e.ids[i])) local[nloc++] = e.ids[i];  // EP: only this rank's shard
    auto copies = s.cache_->request(e.layer, local, nloc, &hits, &misses);
    if (e.flags & kMbAllHit) {
        // the device found every id resident and released the layer itself:
        // only the LRU order and the counters change here
        if (misses != 0)
            throw std::runtime_error("device hit path disagrees with the slot cache at layer " +
                                     std::to_string(e.layer));
        std::lock_guard<std::mutex> g(mu_);
        recs_.push_back({e.seq, e.layer, e.step, hits, 0, 0, -1});
        return;
    }
    const int npairs = static_cast<int>(s.ev_copy_.size() / 2);
    int ev = -1;
    {
        std::lock_guard<std::mutex> g(mu_);
        if (ev_next_ < npairs) ev = ev_next_++;
    }
    if (ev >= 0) ck(cudaEventRecord(s.ev_copy_[2 * ev], s.s_copy_), "event record");
    const int E = s.cfg_.E;
    long long wire = 0;
    for (auto& [slot, expert] : copies) {
        uint16_t* dst = s.d_slots_ + (static_cast<long long>(e.layer) * s.C_ + slot) * s.dm_.expert_elems;
        wire += s.copy_expert(e.layer, expert, dst, s.s_copy_, "H2D expert copy");
    }
    if (ev >= 0) ck(cudaEventRecord(s.ev_copy_[2 * ev + 1], s.s_copy_), "event record");  // link busy
    // The slot table and the ready flag follow every byte of the request.  A
    // packed store decodes on s_unpack_: the tail goes there (after this
    // request's H2Ds), so the copy stream starts the next request's H2D at
    // once instead of waiting for this request's last decode.  One tail
    // stream per session keeps the ready values of a layer in request order.
    cudaStream_t tail = s.s_copy_;
    if (s.store_packed_) {
        ck(cudaEventRecord(s.ev_h2d_tail_, s.s_copy_), "h2d tail");
        ck(cudaStreamWaitEvent(s.s_unpack_, s.ev_h2d_tail_, 0), "h2d tail");
        s.xp_pending_ = 0;  // the tail is ordered after every decode issued so far
        tail = s.s_unpack_;
    }
    if (!copies.empty()) {
        int* stage = s.h_stage_ + static_cast<long long>(stage_idx_ % 256) * E;
        // the copy that last used this staging row is >=256 requests old and
        // therefore complete: requests retire in FIFO order before the device
        // can post more than a few new ones.
        std::memcpy(stage, s.cache_->slot_row(e.layer).data(), sizeof(int) * E);
        ck(cudaMemcpyAsync(s.d_slot_of_ + static_cast<long long>(e.layer) * E, stage, sizeof(int) * E,
                           cudaMemcpyHostToDevice, tail),
           "slot table update");
        ++stage_idx_;
    }
    static const int ready_mode = std::getenv("SMOE_READY_MODE") ? std::atoi(std::getenv("SMOE_READY_MODE")) : 0;
    if (ready_mode == 2) {
        int* flag = s.h_stage_ + 256LL * E + (stage_idx_ % 256);
        *flag = e.seq;
        ++stage_idx_;
        ck(cudaMemcpyAsync(s.ctl_.ready + e.layer, flag, 4, cudaMemcpyHostToDevice, tail), "ready flag");
    } else {
        const CUresult r = write_value_fn()(reinterpret_cast<CUstream>(tail),
                                            reinterpret_cast<CUdeviceptr>(s.ctl_.ready + e.layer),
                                            static_cast<cuuint32_t>(e.seq),
                                            ready_mode == 1 ? CU_STREAM_WRITE_VALUE_NO_MEMORY_BARRIER : 0);
        if (r != CUDA_SUCCESS) throw std::runtime_error("cuStreamWriteValue32 failed");
    }
    std::lock_guard<std::mutex> g(mu_);
    recs_.push_back({e.seq, e.layer, e.step, hits, misses, wire, ev});
}

// ---------------------------------------------------------------- Session --

// Host<->device transfers and memsets outside the decode graph are ordered on
// the compute stream.  The streams are non-blocking, so a legacy-stream
// cudaMemcpy/cudaMemset is NOT ordered before their kernels: a pageable H2D
// cudaMemcpy may return before its DMA lands, and a kernel could read the old
// bytes (seen as wrong prompt tokens when another process time-sliced the GPU).
void Session::h2d(void* dst, const void* src, size_t n, const char* what) {
    ck(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, s_comp_), what);
    ck(cudaStreamSynchronize(s_comp_), what);  // the host buffer may be reused on return
}
void Session::d2h(void* dst, const void* src, size_t n, const char* what) {
    ck(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, s_comp_), what);
    ck(cudaStreamSynchronize(s_comp_), what);
}
void Session::dset(void* p, int v, size_t n, const char* what) {
    ck(cudaMemsetAsync(p, v, n, s_comp_), what);
}

long long Session::copy_expert(int layer, int expert, uint16_t* dst, cudaStream_t s, const char* what) {
    const long long b = store_index(layer, expert);
    const long long packed = store_->packed_bytes(b);
    if (!packed) {
        ck(cudaMemcpyAsync(dst, store_->expert(b), store_->bytes_per_expert(), cudaMemcpyHostToDevice, s), what);
        return store_->bytes_per_expert();
    }
    const int k = static_cast<int>(xp_next_.fetch_add(1) % kXpRing);
    unsigned char* stage = d_xp_stage_ + k * xp_stride_;
    ck(cudaStreamWaitEvent(s, ev_xp_[k], 0), "xp ring");  // the slot's previous decode is done
    ck(cudaMemcpyAsync(stage, store_->expert(b), static_cast<size_t>(packed), cudaMemcpyHostToDevice, s), what);
    ck(cudaEventRecord(ev_h2d_[k], s), "xp h2d");
    ck(cudaStreamWaitEvent(s_unpack_, ev_h2d_[k], 0), "xp h2d");
    ck(launch_xp_unpack(stage, dst, dm_.expert_elems, s_unpack_), "expert unpack");
    ck(cudaEventRecord(ev_xp_[k], s_unpack_), "xp decode");
    ++xp_pending_;
    return packed;
}

void Session::join_unpack(cudaStream_t s) {
    if (xp_pending_.exchange(0) == 0) return;
    ck(cudaEventRecord(ev_unp_join_, s_unpack_), "xp join");
    ck(cudaStreamWaitEvent(s, ev_unp_join_, 0), "xp join");
}

void* Session::dalloc(size_t bytes) {
    void* p = nullptr;
    ck(cudaMalloc(&p, bytes < 256 ? 256 : bytes), "cudaMalloc");
    dset(p, 0, bytes < 256 ? 256 : bytes, "cudaMemset");
    dev_allocs_.push_back(p);
    return p;
}

Session::Session(const ModelCfg& cfg, const SessionOpts& opts) : cfg_(cfg), opts_(opts) {
    cfg_.validate();
    if (!(opts_.cache_fraction > 0.0f && opts_.cache_fraction <= 1.0f))
        throw std::invalid_argument("cache_fraction must be in (0, 1]");
    if (opts_.max_positions < 2) throw std::invalid_argument("max_positions must be >= 2");
    if (opts_.ep_world < 1 || opts_.ep_world > kMaxEP)
        throw std::invalid_argument("ep_world must be in [1, 8]");
    if (opts_.ep_rank < 0 || opts_.ep_rank >= opts_.ep_world)
        throw std::invalid_argument("ep_rank must be in [0, ep_world)");
    ck(cudaSetDevice(opts_.device), "cudaSetDevice");
    write_value_fn();
    ck(preload_kernels(), "kernel preload");
    ck(pf_preload(), "prefill kernel preload");
    ck(tc_preload(), "tensor-core prefill kernel preload");
    try {
        alloc();
    } catch (...) {
        free_all();
        throw;
    }
    sched_ = std::make_unique<CopyScheduler>(this);
    sched_->start();
}

Session::~Session() {
    if (sched_) sched_->stop();
    free_all();
}

void Session::free_all() {
    drop_graphs();
    if (s_comp_) cudaStreamSynchronize(s_comp_);
    for (void* p : bd_allocs_) cudaFree(p);
    bd_allocs_.clear();
    bd_cap_ = 0;
    if (s_copy_) cudaStreamSynchronize(s_copy_);
    if (s_side_) cudaStreamSynchronize(s_side_);
    if (s_log_) cudaStreamSynchronize(s_log_);
    for (auto e : ev_fork_) cudaEventDestroy(e);
    for (auto e : ev_join_) cudaEventDestroy(e);
    if (ev_side_end_) cudaEventDestroy(ev_side_end_);
    if (ev_log_end_) cudaEventDestroy(ev_log_end_);
    ev_fork_.clear();
    ev_join_.clear();
    for (void* p : ipc_opened_) cudaIpcCloseMemHandle(p);
    ipc_opened_.clear();
    for (void* p : dev_allocs_) cudaFree(p);
    dev_allocs_.clear();
    for (auto e : ev_copy_) cudaEventDestroy(e);
    ev_copy_.clear();
    for (auto e : ev_step_) cudaEventDestroy(e);
    ev_step_.clear();
    if (ev_origin_) cudaEventDestroy(ev_origin_);
    ev_origin_ = nullptr;
    if (ev_hostord_) cudaEventDestroy(ev_hostord_);
    ev_hostord_ = nullptr;
    if (h_mailbox_) cudaFreeHost(h_mailbox_);
    if (h_stage_) cudaFreeHost(h_stage_);
    if (h_token_) cudaFreeHost(h_token_);
    if (h_logits_) cudaFreeHost(h_logits_);
    h_mailbox_ = nullptr;
    h_stage_ = nullptr;
    h_token_ = nullptr;
    h_logits_ = nullptr;
    store_.reset();
    if (s_comp_) cudaStreamDestroy(s_comp_);
    if (s_copy_) cudaStreamDestroy(s_copy_);
    if (s_side_) cudaStreamDestroy(s_side_);
    if (s_log_) cudaStreamDestroy(s_log_);
    if (s_unpack_) {
        cudaStreamSynchronize(s_unpack_);
        cudaStreamDestroy(s_unpack_);
    }
    for (int k = 0; k < kXpRing; ++k) {
        if (ev_h2d_[k]) cudaEventDestroy(ev_h2d_[k]);
        if (ev_xp_[k]) cudaEventDestroy(ev_xp_[k]);
        ev_h2d_[k] = ev_xp_[k] = nullptr;
    }
    if (ev_unp_join_) cudaEventDestroy(ev_unp_join_);
    if (ev_h2d_tail_) cudaEventDestroy(ev_h2d_tail_);
    if (ev_hostord2_) cudaEventDestroy(ev_hostord2_);
    ev_unp_join_ = ev_h2d_tail_ = ev_hostord2_ = nullptr;
    s_comp_ = s_copy_ = s_side_ = s_log_ = s_unpack_ = nullptr;
}

void Session::drop_graphs() {
    for (auto& [k, g] : graphs_) cudaGraphExecDestroy(g);
    graphs_.clear();
}

void Session::alloc() {
    const ModelCfg& c = cfg_;
    const int L = c.L, E = c.E, K = c.K, H = c.H, D = c.D, V = c.V;
    el_max_ = (E + opts_.ep_world - 1) / opts_.ep_world;
    DevModel& m = dm_;
    m.L = L; m.E = E; m.K = K; m.H = H; m.Hm = c.Hm; m.V = V; m.D = D;
    m.eps = c.eps;
    m.gating = c.gating;
    m.Hmp = round_up(c.Hm, 16);
    m.Hp = round_up(H, 32);
    m.Ep = round_up(E, 32);
    m.Vp = round_up(V, 32);
    m.QKVp = round_up(3 * D, 32);
    m.cap = opts_.max_positions;
    m.inv_sqrt_d = 1.0f / std::sqrt(static_cast<float>(D));  // model.cpp:336
    m.fast = 0;
    m.gu_elems = static_cast<long long>(m.Hmp) * H * 2;
    m.expert_elems = m.gu_elems + static_cast<long long>(m.Hp) * m.Hmp;
    C_ = slots_for(opts_.cache_fraction);
    m.C = C_;
    {
        const std::string v = kernel_limit_violation(m);
        if (!v.empty()) throw std::invalid_argument("config: " + v);
    }
    m.attn_grid = attn_grid_for(m, opts_.device);
    // the one-launch expert FFN (k_ffn) is opt-in, SMOE_FUSED_FFN=1: measured
    // slower on Q30 (29-30 us vs 12.5 + 8.3 us for k_ffn_gu + k_ffn_down: its
    // down phase streams each 96 KB pair of row blocks through the 48 KB
    // gate/up pipe in two round trips, and the L2 prefetch of the down blocks
    // during the gate/up phase did not turn those reads into L2 hits)
    m.ffn_fused = std::getenv("SMOE_FUSED_FFN") ? ffn_fused_ok(m, opts_.device) : 0;
    m.ffn_cs_fused = ffn_cs_fused_ok(m, opts_.device);
    // opt-in (SMOE_FFN_GUD=1): measured slower than k_ffn_gu_cs + k_ffn_down
    m.ffn_gud = std::getenv("SMOE_FFN_GUD") && std::string(std::getenv("SMOE_FFN_GUD")) == "1";
    // tolerance-mode down as one CTA per row block (k_ffn_down_rb; SMOE_DOWN_RB=0: k_ffn_down)
    m.down_rb = down_rb_ok(m) && !(std::getenv("SMOE_DOWN_RB") && std::string(std::getenv("SMOE_DOWN_RB")) == "0");

    ck(cudaStreamCreateWithFlags(&s_comp_, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&s_copy_, cudaStreamNonBlocking), "stream");
    {
        // the side stream (routers / predictor) gets the highest priority, so
        // its few CTAs are placed before pending expert-kernel CTAs
        int lo = 0, hi = 0;
        ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
        if (std::getenv("SMOE_NO_PRIO")) lo = hi = 0;  // diagnostics
        ck(cudaStreamCreateWithPriority(&s_side_, cudaStreamNonBlocking, hi), "stream");
        ck(cudaStreamCreateWithPriority(&s_log_, cudaStreamNonBlocking, lo), "stream");
        // expert decodes: placed before pending compute CTAs (a ready flag waits on them)
        ck(cudaStreamCreateWithPriority(&s_unpack_, cudaStreamNonBlocking, hi), "stream");
    }
    for (int k = 0; k < kXpRing; ++k) {
        ck(cudaEventCreateWithFlags(&ev_h2d_[k], cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&ev_xp_[k], cudaEventDisableTiming), "event");
    }
    ck(cudaEventCreateWithFlags(&ev_unp_join_, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ev_h2d_tail_, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ev_hostord2_, cudaEventDisableTiming), "event");
    ev_fork_.resize(L);
    ev_join_.resize(L);
    for (int l = 0; l < L; ++l) {
        ck(cudaEventCreateWithFlags(&ev_fork_[l], cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&ev_join_[l], cudaEventDisableTiming), "event");
    }
    ck(cudaEventCreateWithFlags(&ev_side_end_, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ev_log_end_, cudaEventDisableTiming), "event");

    d_emb_ = static_cast<uint16_t*>(dalloc(2ull * V * H));
    d_unemb_ = static_cast<uint16_t*>(dalloc(2ull * m.Vp * H));
    m.qkv_stride = static_cast<long long>(m.QKVp) * H;
    m.wo_stride = static_cast<long long>(m.Hp) * D;
    m.gate_stride = static_cast<long long>(m.Ep) * H;
    d_wqkv_ = static_cast<uint16_t*>(dalloc(2ull * L * m.qkv_stride));
    d_wo_ = static_cast<uint16_t*>(dalloc(2ull * L * m.wo_stride));
    d_gate_ = static_cast<uint16_t*>(dalloc(2ull * L * m.gate_stride));
    d_final_gain_ = static_cast<float*>(dalloc(4ull * H));
    d_attn_gain_ = static_cast<float*>(dalloc(4ull * L * H));
    d_moe_gain_ = static_cast<float*>(dalloc(4ull * L * H));
    {
        std::vector<float> ones(static_cast<size_t>(L) * H, 1.0f);  // model.cpp:126-131
        h2d(d_final_gain_, ones.data(), 4ull * H, "gain");
        h2d(d_attn_gain_, ones.data(), 4ull * L * H, "gain");
        h2d(d_moe_gain_, ones.data(), 4ull * L * H, "gain");
    }
    // RoPE table with the host libm, exactly model.cpp:311-316.
    {
        std::vector<float> rope(static_cast<size_t>(m.cap) * (D / 2) * 2);
        for (int p = 0; p < m.cap; ++p)
            for (int i = 0; i < D / 2; ++i) {
                const double theta =
                    std::pow(10000.0, -2.0 * static_cast<double>(i) / static_cast<double>(D));
                const double angle = static_cast<double>(p) * theta;
                rope[(static_cast<size_t>(p) * (D / 2) + i) * 2] = static_cast<float>(std::cos(angle));
                rope[(static_cast<size_t>(p) * (D / 2) + i) * 2 + 1] = static_cast<float>(std::sin(angle));
            }
        d_rope_ = static_cast<float*>(dalloc(rope.size() * 4));
        h2d(d_rope_, rope.data(), rope.size() * 4, "rope");
    }
    d_slots_ = static_cast<uint16_t*>(dalloc(2ull * L * C_ * m.expert_elems));
    d_slot_of_ = static_cast<int*>(dalloc(4ull * L * E));
    dset(d_slot_of_, 0xff, 4ull * L * E, "memset");
    d_dv_ = static_cast<float*>(dalloc(4ull * L * E * H));
    // EP exchange region (shared with peers through one CUDA IPC handle):
    // [tag 256 B | arrival counters L ints, padded to 256 B | exchange buffer [2][K][Hp] f32]
    // The tag (a random 128-bit value) lets a peer verify, and if need be
    // find, the region inside the block its cudaIpcOpenMemHandle mapped:
    // small cudaMallocs are sub-allocated from shared driver blocks.
    // ... | batched counters (padded) | batched exchange [2][kEpBatchMax * K][Hp] f32],
    // at fixed offsets from the exchange buffer (ep_batch_ptrs)
    {
        const size_t cnt_bytes = (4ull * L + 255) / 256 * 256;
        unsigned char* reg = static_cast<unsigned char*>(
            dalloc(256 + cnt_bytes + 4ull * 2 * K * m.Hp + cnt_bytes + 4ull * 2 * kEpBatchMax * K * m.Hp));
        std::random_device rd;
        ep_tag_[0] = 0x31585045454f4d53ull;  // "SMOEEPX1"
        ep_tag_[1] = (static_cast<uint64_t>(rd()) << 32 ^ rd()) ^ reinterpret_cast<uintptr_t>(reg) ^
                     static_cast<uint64_t>(getpid()) << 40;
        h2d(reg, ep_tag_, 16, "ep tag");
        d_ep_region_ = reg;
        d_cnt_ = reinterpret_cast<int*>(reg + 256);
        d_xbuf_ = reinterpret_cast<float*>(reg + 256 + cnt_bytes);
    }
    d_epoch_ = static_cast<int*>(dalloc(4ull * L));
    d_bepoch_ = static_cast<int*>(dalloc(4ull * L));
    d_bdone_ = static_cast<int*>(dalloc(4ull * L));
    ctl_.ep.bepoch = d_bepoch_;
    ctl_.ep.bdone = d_bdone_;
    ep_batch_ptrs(d_xbuf_, &ctl_.ep.bcnt[0], &ctl_.ep.bxbuf[0]);
    ctl_.ep.rank = 0;
    ctl_.ep.world = 1;  // EP activates at ep_connect(); until then this rank runs everything it owns
    ctl_.ep.xbuf[0] = d_xbuf_;
    ctl_.ep.cnt[0] = d_cnt_;
    ctl_.ep.epoch = d_epoch_;
    d_hybrid_ = static_cast<int*>(dalloc(4ull * L));
    // e [cap] f64 | p [cap] f32 (+pad) | split-attention control words and maxima
    d_attn_scratch_ = static_cast<double*>(dalloc(attn_scratch_bytes(m.cap)));
    dset(d_attn_scratch_, 0, attn_scratch_bytes(m.cap), "attn scratch");
    d_prompt_tok_ = static_cast<int*>(dalloc(4ull * m.cap));

    m.emb = d_emb_;
    m.unemb = d_unemb_;
    m.final_gain = d_final_gain_;
    m.attn_gain = d_attn_gain_;
    m.moe_gain = d_moe_gain_;
    m.wqkv = d_wqkv_;
    m.wo = d_wo_;
    m.gate = d_gate_;
    m.rope = d_rope_;
    m.slots = d_slots_;
    m.slot_of = d_slot_of_;
    m.dv = d_dv_;
    m.hybrid = d_hybrid_;

    auto mk_state = [&](DevState& st) {
        st.x = static_cast<float*>(dalloc(4ull * m.Hp));
        st.r = static_cast<float*>(dalloc(4ull * L * m.Hp));
        st.s = static_cast<float*>(dalloc(4ull * L * m.Hp));
        st.m = static_cast<float*>(dalloc(4ull * L * m.Hp));
        st.q = static_cast<float*>(dalloc(4ull * kMaxD));
        st.ctx = static_cast<float*>(dalloc(4ull * kMaxD));
        st.kc = static_cast<float*>(dalloc(4ull * L * m.cap * D));
        st.vc = static_cast<float*>(dalloc(4ull * L * m.cap * D));
        st.lg_true = static_cast<float*>(dalloc(4ull * L * E));
        st.id_true = static_cast<int*>(dalloc(4ull * L * K));
        st.g_true = static_cast<float*>(dalloc(4ull * L * K));
        st.id_exec = static_cast<int*>(dalloc(4ull * L * K));
        st.g_exec = static_cast<float*>(dalloc(4ull * L * K));
        st.lg_pred = static_cast<float*>(dalloc(4ull * L * E));
        st.id_pred = static_cast<int*>(dalloc(4ull * L * K));
        st.g_pred = static_cast<float*>(dalloc(4ull * L * K));
        st.quasi = static_cast<float*>(dalloc(4ull * m.Hp));
        st.h = static_cast<float*>(dalloc(4ull * K * m.Hmp));
        st.y = static_cast<float*>(dalloc(4ull * K * m.Hp));
        st.dpart = static_cast<float*>(dalloc(4ull * K * (m.Hmp / 16) * m.Hp));
        st.logits = static_cast<float*>(dalloc(4ull * m.Vp));
        st.pos = static_cast<int*>(dalloc(4));
        st.token = static_cast<int*>(dalloc(4));
        st.tok_in = static_cast<int*>(dalloc(4));
        st.counters = static_cast<int*>(dalloc(4 * 64));
        st.down_cnt = static_cast<int*>(dalloc(4ull * (m.Hp / 32)));
        st.log_cnt = static_cast<int*>(dalloc(4ull * L));
        st.ssq_x = static_cast<double*>(dalloc(8ull * (L + 1) * (m.Hp / 32)));
        st.ssq_r = static_cast<double*>(dalloc(8ull * L * (m.Hp / 32)));
        st.rd = static_cast<float*>(dalloc(4ull * L * m.Hp));
        st.pass_id = static_cast<int*>(dalloc(4));
        st.dec_ready = static_cast<int*>(dalloc(4ull * L));
        st.gu_done = static_cast<int*>(dalloc(4ull * L * K));
        st.ffn_epoch = static_cast<int*>(dalloc(4ull * L));
        st.ssq_rd = static_cast<double*>(dalloc(8ull * L * (m.Hp / 32)));
        st.ep_arrive = static_cast<int*>(dalloc(4ull * L));
        st.est_z = st.est_act = st.est_xn = nullptr;
    };
    mk_state(st_);
    mk_state(sh_);

    ctl_.req_counter = static_cast<int*>(dalloc(4));
    ctl_.req_seq = static_cast<int*>(dalloc(4ull * L));
    ctl_.ready = static_cast<int*>(dalloc(4ull * L));
    ctl_.error = static_cast<int*>(dalloc(4));
    ctl_.step = static_cast<int*>(dalloc(4));
    ctl_.tokens_out = static_cast<int*>(dalloc(4ull * (m.cap + 1)));
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, opts_.device);
    if (clk_khz <= 0) clk_khz = 2000000;
    ctl_.spin_limit = static_cast<long long>(opts_.deadlock_s * clk_khz * 1e3);
    // host-ordered copy waits under kernel-serialising tools (ncu,
    // compute-sanitizer), detected by their injection libraries / launcher
    // variables; SMOE_HOST_ORDERED = 1 / 0 forces the mode on / off
    {
        const char* ho = std::getenv("SMOE_HOST_ORDERED");
        host_ordered_ = ho ? std::atoi(ho) != 0 : profiler_attached();
        ctl_.host_ordered = host_ordered_ ? 1 : 0;
        ctl_.fast_hit = std::getenv("SMOE_NO_FAST_HIT") ? 0 : 1;
        ck(cudaEventCreateWithFlags(&ev_hostord_, cudaEventDisableTiming), "event");
    }
    dm_.attn_err = ctl_.error;
    dm_.attn_spin = ctl_.spin_limit;

    ck(cudaHostAlloc(reinterpret_cast<void**>(&h_mailbox_), sizeof(MailboxEntry) * kMailboxRing,
                     cudaHostAllocMapped | cudaHostAllocPortable),
       "mailbox");
    std::memset(h_mailbox_, 0, sizeof(MailboxEntry) * kMailboxRing);
    MailboxEntry* dmb = nullptr;
    ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dmb), h_mailbox_, 0), "mailbox map");
    ctl_.mailbox = dmb;
    ck(cudaHostAlloc(reinterpret_cast<void**>(&h_stage_), 4ull * 256 * (E + 1), cudaHostAllocPortable), "stage");
    ck(cudaHostAlloc(reinterpret_cast<void**>(&h_token_), 64, cudaHostAllocPortable), "token");
    ck(cudaHostAlloc(reinterpret_cast<void**>(&h_logits_), 4ull * m.Vp, cudaHostAllocPortable), "logits");

    ev_copy_.resize(2 * 8192);
    for (auto& e : ev_copy_) ck(cudaEventCreate(&e), "event");
    ev_step_.resize(2 * 4096);
    for (auto& e : ev_step_) ck(cudaEventCreate(&e), "event");
    ck(cudaEventCreate(&ev_origin_), "event");

    store_ = std::make_unique<ExpertStore>(static_cast<long long>(L) * el_max_, m.expert_elems, opts_.device);
    xp_stride_ = (store_->max_packed_bytes() + 255) / 256 * 256;
    d_xp_stage_ = static_cast<unsigned char*>(dalloc(static_cast<size_t>(kXpRing * xp_stride_)));
    cache_ = std::make_unique<SlotCache>(L, E, C_);
    ck(cudaDeviceSynchronize(), "alloc");
    reset(0, 0);
}

int Session::slots_for(float frac) const {
    const int El = local_experts();
    int C = static_cast<int>(std::ceil(static_cast<double>(frac) * El));
    const int lo = cfg_.K < El ? cfg_.K : El;  // one request holds at most min(k, El) local ids
    if (C < lo) C = lo;
    if (C > El) C = El;
    if (C < 1) C = 1;
    return C;
}

// The batched exchange of a rank's region sits at fixed offsets after its
// exchange buffer (same L, K, Hp on every rank): counters, then rows.
void Session::ep_batch_ptrs(float* xbuf, int** bcnt, float** bxbuf) const {
    const size_t cnt_bytes = (4ull * cfg_.L + 255) / 256 * 256;
    unsigned char* b = reinterpret_cast<unsigned char*>(xbuf) + 4ull * 2 * cfg_.K * dm_.Hp;
    *bcnt = reinterpret_cast<int*>(b);
    *bxbuf = reinterpret_cast<float*>(b + cnt_bytes);
}

void Session::ep_buffers(void** xbuf, void** cnt) {
    *xbuf = d_xbuf_;
    *cnt = d_cnt_;
}

// 128 bytes per rank: the IPC handle of the exchange region's allocation
// (64 B), the region's offset in it as this process sees it (8 B), the
// buffer's offset in the region (8 B) and the region's 16-byte tag.
void Session::ep_ipc_handles(unsigned char* out128) {
    cudaIpcMemHandle_t a;
    ck(cudaIpcGetMemHandle(&a, d_ep_region_), "ipc handle");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (addr_range_fn()(&base, &size, reinterpret_cast<CUdeviceptr>(d_ep_region_)) != CUDA_SUCCESS)
        throw std::runtime_error("cuMemGetAddressRange failed");
    const unsigned long long off = reinterpret_cast<CUdeviceptr>(d_ep_region_) - base;
    const unsigned long long xoff = reinterpret_cast<unsigned char*>(d_xbuf_) - d_ep_region_;
    std::memset(out128, 0, 128);
    std::memcpy(out128, &a, 64);
    std::memcpy(out128 + 64, &off, 8);
    std::memcpy(out128 + 72, &xoff, 8);
    std::memcpy(out128 + 80, ep_tag_, 16);
}

// Every rank passes the exchange buffers / counters of all ranks (its own at
// index ep_rank).  Replicated dense path + these peer stores = bit-exact EP.
void Session::ep_connect(void* const* xbufs, void* const* cnts) {
    sync();
    const int W = opts_.ep_world;
    for (int p = 0; p < W; ++p) {
        if (!xbufs[p] || !cnts[p]) throw std::invalid_argument("ep_connect: null peer buffer");
        // ranks of one process on different GPUs: map the peer's memory over NVLink
        cudaPointerAttributes a{};
        if (p != opts_.ep_rank && cudaPointerGetAttributes(&a, xbufs[p]) == cudaSuccess &&
            a.type == cudaMemoryTypeDevice && a.device != opts_.device) {
            int can = 0;
            ck(cudaDeviceCanAccessPeer(&can, opts_.device, a.device), "peer query");
            if (!can)
                throw std::runtime_error("ep_connect: device " + std::to_string(opts_.device) +
                                         " cannot access peer device " + std::to_string(a.device));
            const cudaError_t e = cudaDeviceEnablePeerAccess(a.device, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled)
                cudaGetLastError();
            else
                ck(e, "enable peer access");
        }
        ctl_.ep.xbuf[p] = static_cast<float*>(xbufs[p]);
        ctl_.ep.cnt[p] = static_cast<int*>(cnts[p]);
        ep_batch_ptrs(ctl_.ep.xbuf[p], &ctl_.ep.bcnt[p], &ctl_.ep.bxbuf[p]);
    }
    ctl_.ep.xbuf[opts_.ep_rank] = d_xbuf_;
    ctl_.ep.cnt[opts_.ep_rank] = d_cnt_;
    ep_batch_ptrs(d_xbuf_, &ctl_.ep.bcnt[opts_.ep_rank], &ctl_.ep.bxbuf[opts_.ep_rank]);
    ctl_.ep.rank = opts_.ep_rank;
    ctl_.ep.world = W;
    dset(d_cnt_, 0, 4ull * cfg_.L, "ep reset");
    dset(d_epoch_, 0, 4ull * cfg_.L, "ep reset");
    dset(ctl_.ep.bcnt[opts_.ep_rank], 0, 4ull * cfg_.L, "ep reset");
    dset(d_bepoch_, 0, 4ull * cfg_.L, "ep reset");
    dset(d_bdone_, 0, 4ull * cfg_.L, "ep reset");
    // the reset must land before any peer (released by the caller's barrier)
    // starts adding to these counters
    ck(cudaDeviceSynchronize(), "ep reset sync");
    drop_graphs();
}

// The peer's region: at `off` from the mapped base when the mapping starts
// where the peer's allocation does; otherwise found by its tag, scanning the
// mapped block at 256-byte steps (done once, at connect time).
unsigned char* Session::locate_ep_region(unsigned char* base, unsigned long long off,
                                         const unsigned long long tag[2]) {
    unsigned long long got[2] = {0, 0};
    CUdeviceptr b0 = 0;
    size_t size = 0;
    if (addr_range_fn()(&b0, &size, reinterpret_cast<CUdeviceptr>(base)) != CUDA_SUCCESS)
        throw std::runtime_error("cuMemGetAddressRange failed on an IPC mapping");
    unsigned char* lo = reinterpret_cast<unsigned char*>(b0);
    if (base + off + 16 <= lo + size) {
        d2h(got, base + off, 16, "ep tag read");
        if (got[0] == tag[0] && got[1] == tag[1]) return base + off;
    }
    if (size > (1ull << 31)) return nullptr;
    std::vector<unsigned long long> blk(size / 8);
    d2h(blk.data(), lo, size / 8 * 8, "ep block read");
    for (size_t i = 0; i + 1 < blk.size(); i += 32)
        if (blk[i] == tag[0] && blk[i + 1] == tag[1]) return lo + i * 8;
    return nullptr;
}

void Session::ep_connect_ipc(const unsigned char* handles) {
    const int W = opts_.ep_world;
    std::vector<void*> xb(W), cn(W);
    for (int p = 0; p < W; ++p) {
        if (p == opts_.ep_rank) {
            xb[p] = d_xbuf_;
            cn[p] = d_cnt_;
            continue;
        }
        cudaIpcMemHandle_t a;
        unsigned long long off = 0, xoff = 0, tag[2];
        std::memcpy(&a, handles + p * 128, 64);
        std::memcpy(&off, handles + p * 128 + 64, 8);
        std::memcpy(&xoff, handles + p * 128 + 72, 8);
        std::memcpy(tag, handles + p * 128 + 80, 16);
        void* base = nullptr;
        ck(cudaIpcOpenMemHandle(&base, a, cudaIpcMemLazyEnablePeerAccess), "ipc open");
        ipc_opened_.push_back(base);
        unsigned char* region = locate_ep_region(static_cast<unsigned char*>(base), off, tag);
        if (!region)
            throw std::runtime_error("ep_connect_ipc: rank " + std::to_string(p) +
                                     "'s exchange region not found in the mapped IPC block");
        cn[p] = region + 256;
        xb[p] = region + xoff;
    }
    ep_connect(xb.data(), cn.data());
}

void Session::preload_all() {
    sync();
    if (C_ != local_experts()) throw std::invalid_argument("preload_all: needs cache_fraction 1.0");
    ck(cudaStreamSynchronize(s_copy_), "copy stream");
    const long long per = dm_.expert_elems;
    std::vector<int> ids;
    for (int e = 0; e < cfg_.E; ++e)
        if (is_local(e)) ids.push_back(e);
    for (int l = 0; l < cfg_.L; ++l) {
        int h = 0, mi = 0;
        auto copies = cache_->request(l, ids.data(), static_cast<int>(ids.size()), &h, &mi);
        for (auto& [slot, expert] : copies)
            copy_expert(l, expert, d_slots_ + (static_cast<long long>(l) * C_ + slot) * per, s_copy_, "preload");
        join_unpack(s_copy_);
        ck(cudaMemcpyAsync(d_slot_of_ + static_cast<long long>(l) * cfg_.E, cache_->slot_row(l).data(),
                           4ull * cfg_.E, cudaMemcpyHostToDevice, s_copy_),
           "preload table");
        ck(cudaStreamSynchronize(s_copy_), "preload");
    }
    cache_->clear_stats();
    ctl_.resident = 1;
    drop_graphs();
}

void Session::set_cache_fraction(float frac) {
    if (!(frac > 0.0f && frac <= 1.0f)) throw std::invalid_argument("cache_fraction must be in (0, 1]");
    sync();
    const int C = slots_for(frac);
    if (C == C_) return;
    // replace the slot pool
    for (auto it = dev_allocs_.begin(); it != dev_allocs_.end(); ++it)
        if (*it == d_slots_) {
            cudaFree(*it);
            dev_allocs_.erase(it);
            break;
        }
    opts_.cache_fraction = frac;
    ctl_.resident = 0;
    C_ = C;
    dm_.C = C;
    d_slots_ = static_cast<uint16_t*>(dalloc(2ull * cfg_.L * C_ * dm_.expert_elems));
    dm_.slots = d_slots_;
    dset(d_slot_of_, 0xff, 4ull * cfg_.L * cfg_.E, "memset");
    cache_ = std::make_unique<SlotCache>(cfg_.L, cfg_.E, C_);
    drop_graphs();
}

// ------------------------------------------------------------- weights ------

// build_model (model.cpp:112-158) on the GPU: every tensor from its labelled
// counter-based stream, rounded to bf16 in the kernels' layouts.  Expert
// blocks are generated into an HBM staging area and copied into the pinned
// host store (they live off-device until the cache pulls them in).
void Session::init_weights_seeded() {
    sync();
    const ModelCfg& c = cfg_;
    DevModel& m = dm_;
    const float stddev = 0.4f / std::sqrt(static_cast<float>(c.H));
    cudaStream_t s = s_comp_;
    auto gen = [&](const std::string& label, int R, int C, int tc, int layout, int which,
                   int roff, uint16_t* out) {
        ck(launch_gen_bf16(derive_seed(c.seed, label), stddev, R, C, tc, layout, which, roff, out, s),
           "gen");
    };
    gen("embedding", c.V, c.H, c.H, kRowMajor, 0, 0, d_emb_);
    gen("unembed", c.V, c.H, c.H, kRowTiled, 0, 0, d_unemb_);
    for (int l = 0; l < c.L; ++l) {
        const std::string p = "layer" + std::to_string(l) + ".";
        uint16_t* qkv = d_wqkv_ + l * m.qkv_stride;
        gen(p + "wq", c.D, c.H, c.H, kRowTiled, 0, 0, qkv);
        gen(p + "wk", c.D, c.H, c.H, kRowTiled, 0, c.D, qkv);
        gen(p + "wv", c.D, c.H, c.H, kRowTiled, 0, 2 * c.D, qkv);
        gen(p + "wo", c.H, c.D, c.D, kRowTiled, 0, 0, d_wo_ + l * m.wo_stride);
        gen(p + "gate", c.E, c.H, c.H, kRowTiled, 0, 0, d_gate_ + l * m.gate_stride);
    }
    // experts: batches through an HBM staging buffer
    const long long per = m.expert_elems;
    const long long total = static_cast<long long>(c.L) * el_max_;
    long long batch = (1ll << 30) / (per * 2);  // ~1 GiB staging
    if (batch < 1) batch = 1;
    if (batch > total) batch = total;
    uint16_t* stage = nullptr;
    ck(cudaMalloc(&stage, static_cast<size_t>(batch) * per * 2), "staging");
    for (long long b0 = 0; b0 < total; b0 += batch) {
        const long long nb = std::min(batch, total - b0);
        ck(cudaMemsetAsync(stage, 0, static_cast<size_t>(nb) * per * 2, s), "memset");
        for (long long i = 0; i < nb; ++i) {
            const long long x = b0 + i;
            const int l = static_cast<int>(x / el_max_);
            const int e = static_cast<int>(x % el_max_) * opts_.ep_world + opts_.ep_rank;
            if (e >= c.E) continue;  // padding block of a short shard
            const std::string p = "layer" + std::to_string(l) + ".expert" + std::to_string(e) + ".";
            uint16_t* blk = stage + i * per;
            gen(p + "w_gate", c.Hm, c.H, c.H, kGateUp, 0, 0, blk);
            gen(p + "w_up", c.Hm, c.H, c.H, kGateUp, 1, 0, blk);
            gen(p + "w_down", c.H, c.Hm, m.Hmp, kRowTiled, 0, 0, blk + m.gu_elems);
        }
        ck(cudaMemcpyAsync(store_->expert(b0), stage, static_cast<size_t>(nb) * per * 2,
                           cudaMemcpyDeviceToHost, s),
           "D2H store");
    }
    ck(cudaStreamSynchronize(s), "init sync");
    cudaFree(stage);
    if (pack_store_) store_packed_ = store_->pack_all() > 0;  // xp11: ~11 bits per weight on the link (lossless)
    cache_->invalidate();
    ctl_.resident = 0;
    drop_graphs();
    dset(d_slot_of_, 0xff, 4ull * c.L * c.E, "memset");
}

void Session::load_tensor(const std::string& name, const float* data, long long n) {
    sync();
    const ModelCfg& c = cfg_;
    DevModel& m = dm_;
    auto need = [&](long long want) {
        if (n != want) throw std::invalid_argument("load_tensor: " + name + " has wrong size");
    };
    auto upload16 = [&](uint16_t* dst, const std::vector<uint16_t>& v) {
        h2d(dst, v.data(), v.size() * 2, "upload");
    };
    if (name == "embedding") {
        need(static_cast<long long>(c.V) * c.H);
        std::vector<uint16_t> v(n);
        for (long long i = 0; i < n; ++i) v[i] = f2bf(data[i]);
        upload16(d_emb_, v);
        return;
    }
    if (name == "unembed") {
        need(static_cast<long long>(c.V) * c.H);
        std::vector<uint16_t> v(static_cast<size_t>(m.Vp) * c.H, 0);
        tile_write_bf16(v.data(), data, c.V, c.H, c.H, 1, 0, 0);
        upload16(d_unemb_, v);
        return;
    }
    if (name == "final_norm_gain") {
        need(c.H);
        h2d(d_final_gain_, data, 4ull * c.H, "upload");
        return;
    }
    int l;
    std::string rest;
    if (!parse_layer(name, &l, &rest) || l < 0 || l >= c.L)
        throw std::invalid_argument("load_tensor: unknown tensor " + name);
    if (rest == "attn_norm_gain" || rest == "moe_norm_gain") {
        need(c.H);
        float* dst = (rest == "attn_norm_gain" ? d_attn_gain_ : d_moe_gain_) + static_cast<long long>(l) * c.H;
        h2d(dst, data, 4ull * c.H, "upload");
        drop_graphs();
        return;
    }
    if (rest == "wq" || rest == "wk" || rest == "wv") {
        need(static_cast<long long>(c.D) * c.H);
        std::vector<uint16_t> v(m.qkv_stride);
        uint16_t* dst = d_wqkv_ + l * m.qkv_stride;
        d2h(v.data(), dst, v.size() * 2, "download");
        const int off = rest == "wq" ? 0 : rest == "wk" ? c.D : 2 * c.D;
        tile_write_bf16(v.data(), data, c.D, c.H, c.H, 1, 0, off);
        upload16(dst, v);
        return;
    }
    if (rest == "wo") {
        need(static_cast<long long>(c.H) * c.D);
        std::vector<uint16_t> v(m.wo_stride, 0);
        tile_write_bf16(v.data(), data, c.H, c.D, c.D, 1, 0, 0);
        upload16(d_wo_ + l * m.wo_stride, v);
        return;
    }
    if (rest == "gate") {
        need(static_cast<long long>(c.E) * c.H);
        std::vector<uint16_t> v(m.gate_stride, 0);
        tile_write_bf16(v.data(), data, c.E, c.H, c.H, 1, 0, 0);
        upload16(d_gate_ + l * m.gate_stride, v);
        return;
    }
    int e;
    char which[32];
    if (std::sscanf(rest.c_str(), "expert%d.%31s", &e, which) == 2 && e >= 0 && e < c.E) {
        if (!is_local(e)) return;  // EP: another rank owns this expert
        store_->unpack(store_index(l, e));  // raw bf16 again before a partial rewrite
        uint16_t* blk = store_->expert(store_index(l, e));
        const std::string w = which;
        if (w == "w_gate" || w == "w_up") {
            need(static_cast<long long>(c.Hm) * c.H);
            tile_write_bf16(blk, data, c.Hm, c.H, c.H, 2, w == "w_up" ? 1 : 0, 0);
        } else if (w == "w_down") {
            need(static_cast<long long>(c.H) * c.Hm);
            tile_write_bf16(blk + m.gu_elems, data, c.H, c.Hm, m.Hmp, 1, 0, 0);
        } else {
            throw std::invalid_argument("load_tensor: unknown tensor " + name);
        }
        // invalidate a resident copy of this expert
        cache_->invalidate();
        ctl_.resident = 0;
        drop_graphs();
        dset(d_slot_of_, 0xff, 4ull * c.L * c.E, "memset");
        return;
    }
    throw std::invalid_argument("load_tensor: unknown tensor " + name);
}

void Session::load_default_vectors(const float* d) {
    sync();
    h2d(d_dv_, d, 4ull * cfg_.L * cfg_.E * cfg_.H, "dv upload");
    have_dv_ = true;
}

// EstimatorParams flat layout (estimator.hpp:41-72) -> f32 row tiles.
void Session::load_estimator(const EstCfg& e, const float* flat) {
    sync();
    if (e.d != cfg_.H) throw std::invalid_argument("estimator: d must equal the model hidden size");
    if (e.E != cfg_.E) throw std::invalid_argument("estimator: E must equal the model expert count");
    if (e.L != cfg_.L) throw std::invalid_argument("estimator: L must equal the model layer count");
    if (e.m <= 1 || e.n <= 1 || e.d % e.m != 0) throw std::invalid_argument("estimator: bad m/n");
    if ((e.d / e.m) % 4 != 0) throw std::invalid_argument("estimator: latent width d/m must be a multiple of 4 on this path");
    const int dm = e.d / e.m, mlp = dm * e.n;
    {
        DevModel probe = dm_;
        probe.est_d = e.d;
        probe.est_dm = dm;
        probe.est_mlp = mlp;
        const std::string v = estimator_limit_violation(probe);
        if (!v.empty()) throw std::invalid_argument("estimator: " + v);
    }
    const int dmp = round_up(dm, 32), mlpp = round_up(mlp, 32);
    const long long a_off = 0, pos_off = static_cast<long long>(dm) * e.d,
                    b_off = pos_off + static_cast<long long>(e.L) * dm,
                    c_off = b_off + static_cast<long long>(mlp) * dm,
                    g_off = c_off + static_cast<long long>(dm) * mlp, bias_off = g_off + dm,
                    h_off = bias_off + dm;
    const long long szA = static_cast<long long>(dmp) * e.d, szB = static_cast<long long>(mlpp) * dm,
                    szC = static_cast<long long>(dmp) * mlp, szH = static_cast<long long>(dm_.Ep) * dm;
    std::vector<float> buf(szA + szB + szC + szH + static_cast<long long>(e.L) * dm + 2 * dm, 0.0f);
    float* A = buf.data();
    float* B = A + szA;
    float* Cc = B + szB;
    float* Hd = Cc + szC;
    float* P = Hd + szH;
    float* G = P + static_cast<long long>(e.L) * dm;
    float* Bi = G + dm;
    tile_write_f32(A, flat + a_off, dm, e.d);
    tile_write_f32(B, flat + b_off, mlp, dm);
    tile_write_f32(Cc, flat + c_off, dm, mlp);
    tile_write_f32(Hd, flat + h_off, e.E, dm);
    std::memcpy(P, flat + pos_off, 4ull * e.L * dm);
    std::memcpy(G, flat + g_off, 4ull * dm);
    std::memcpy(Bi, flat + bias_off, 4ull * dm);
    if (!d_est_ || est_.d != e.d || est_.m != e.m || est_.n != e.n) {
        d_est_ = static_cast<float*>(dalloc(buf.size() * 4));
        auto mk = [&](DevState& st) {
            st.est_z = static_cast<float*>(dalloc(4ull * dmp));
            st.est_act = static_cast<float*>(dalloc(4ull * mlpp));
            st.est_xn = static_cast<float*>(dalloc(4ull * dmp));
        };
        mk(st_);
        mk(sh_);
    }
    h2d(d_est_, buf.data(), buf.size() * 4, "est upload");
    // the flat block as well: batched decode runs estimator_forward as chain GEMMs (train.cu)
    const size_t flat_n = static_cast<size_t>(g_off + 2 * dm) + static_cast<size_t>(e.E) * dm;
    if (!d_est_flat_ || est_flat_n_ != flat_n) {
        d_est_flat_ = static_cast<float*>(dalloc(flat_n * 4));
        est_flat_n_ = flat_n;
    }
    h2d(d_est_flat_, flat, flat_n * 4, "est upload");
    est_ = e;
    DevModel& m = dm_;
    m.est_d = e.d;
    m.est_dm = dm;
    m.est_mlp = mlp;
    m.est_eps = e.eps;
    m.est_a = d_est_;
    m.est_b = d_est_ + (A - buf.data()) + szA;
    m.est_c = d_est_ + (Cc - buf.data());
    m.est_head = d_est_ + (Hd - buf.data());
    m.est_pos = d_est_ + (P - buf.data());
    m.est_gain = d_est_ + (G - buf.data());
    m.est_bias = d_est_ + (Bi - buf.data());
    have_est_ = true;
    drop_graphs();
}

void Session::set_predictor(int kind, const int* hybrid_map) {
    sync();
    if (kind < kNone || kind > kOracle) throw std::invalid_argument("unknown predictor kind");
    const int L = cfg_.L;
    std::vector<int> map;
    if (kind == kHybrid) {
        map.assign(L, kRouterPF);
        if (hybrid_map)
            for (int l = 0; l < L - 1; ++l) {
                const int k = hybrid_map[l];
                if (k != kBaselineS && k != kRouterPF && k != kEstPF)
                    throw std::invalid_argument("hybrid map: entries must be concrete predictors");
                map[l] = k;
            }
    }
    auto needs = [&](int k) {
        if ((k == kRouterPF || k == kEstPF) && !have_dv_)
            throw std::invalid_argument(std::string(k == kRouterPF ? "router-pf" : "est-pf") +
                                        ": missing default-vector table");
        if (k == kEstPF && !have_est_) throw std::invalid_argument("est-pf: missing estimator");
    };
    if (kind == kHybrid)
        for (int l = 0; l < L - 1; ++l) needs(map[l]);
    else
        needs(kind);
    pred_kind_ = kind;
    hybrid_ = map;
    drop_graphs();
}

// ------------------------------------------------------------- decode -------

void Session::sync() {
    static const bool dbg = std::getenv("SMOE_DEBUG") != nullptr;
    if (dbg)
        std::fprintf(stderr, "[main] t=%.3f ms sync begin\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count());
    if (s_comp_) ck(cudaStreamSynchronize(s_comp_), "compute stream");
    if (dbg)
        std::fprintf(stderr, "[main] t=%.3f ms sync end\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count());
    check_device_error();
}

void Session::check_device_error() {
    int err = 0;
    d2h(&err, ctl_.error, 4, "error flag");
    const std::string se = sched_ ? sched_->error() : std::string();
    if (!se.empty()) {
        cudaMemsetAsync(ctl_.error, 0, 4, s_comp_);
        throw std::runtime_error(se);
    }
    if (err != 0) {
        cudaMemsetAsync(ctl_.error, 0, 4, s_comp_);
        if (err >= 1000 && err < 2000)
            throw std::runtime_error("deadlock suspected: compute waited " +
                                     std::to_string(static_cast<long long>(opts_.deadlock_s * 1000)) +
                                     " ms for layer " + std::to_string(err - 1000) + " expert copy");
        if (err >= 3000 && err < 4000)
            throw std::runtime_error("deadlock suspected: expert-parallel combine of layer " +
                                     std::to_string(err - 3000) + " waited " +
                                     std::to_string(static_cast<long long>(opts_.deadlock_s * 1000)) +
                                     " ms for peer ranks");
        if (err >= 4000 && err < 5000)
            throw std::runtime_error("split attention stalled at layer " + std::to_string(err - 4000) +
                                     ": its CTAs were not co-resident within " +
                                     std::to_string(static_cast<long long>(opts_.deadlock_s * 1000)) + " ms");
        if (err >= 5000 && err < 6000)
            throw std::runtime_error("deadlock suspected: batched expert-parallel combine of layer " +
                                     std::to_string(err - 5000) + " waited " +
                                     std::to_string(static_cast<long long>(opts_.deadlock_s * 1000)) +
                                     " ms for peer ranks");
        throw std::runtime_error("expert read before readiness at layer " + std::to_string(err - 2000));
    }
}

void Session::reset(int max_steps, int trace_full) {
    sync();
    const ModelCfg& c = cfg_;
    int zero = 0;
    for (DevState* st : {&st_, &sh_}) {
        h2d(st->pos, &zero, 4, "reset");
        dset(st->counters, 0, 256, "reset");
        dset(st->down_cnt, 0, 4ull * (dm_.Hp / 32), "reset");
    }
    h2d(ctl_.step, &zero, 4, "reset");
    host_pos_ = 0;
    // trace buffers
    if (max_steps != max_steps_ || trace_full != trace_full_ || !tr_.step) {
        auto drop = [&](void* p) {
            if (!p) return;
            for (auto it = dev_allocs_.begin(); it != dev_allocs_.end(); ++it)
                if (*it == p) {
                    cudaFree(p);
                    dev_allocs_.erase(it);
                    return;
                }
        };
        for (void* p : {(void*)tr_.s, (void*)tr_.r, (void*)tr_.m, (void*)tr_.lg_true, (void*)tr_.g_true,
                        (void*)tr_.g_exec, (void*)tr_.lg_pred, (void*)tr_.g_pred, (void*)tr_.y,
                        (void*)tr_.logits, (void*)tr_.id_true, (void*)tr_.id_exec, (void*)tr_.id_pred,
                        (void*)tr_.tok_in, (void*)tr_.step})
            drop(p);
        tr_ = TraceDev{};
        tr_.step = static_cast<int*>(dalloc(4));
        tr_.cap = max_steps;
        tr_.full = trace_full;
        const long long S = max_steps > 0 ? max_steps : 1;
        const long long LK = static_cast<long long>(c.L) * c.K;
        tr_.tok_in = static_cast<int*>(dalloc(4 * S));
        tr_.id_true = static_cast<int*>(dalloc(4 * S * LK));
        tr_.id_exec = static_cast<int*>(dalloc(4 * S * LK));
        tr_.id_pred = static_cast<int*>(dalloc(4 * S * LK));
        if (trace_full) {
            const long long LH = static_cast<long long>(c.L) * c.H, LE = static_cast<long long>(c.L) * c.E;
            tr_.g_true = static_cast<float*>(dalloc(4 * S * LK));
            tr_.g_exec = static_cast<float*>(dalloc(4 * S * LK));
            tr_.g_pred = static_cast<float*>(dalloc(4 * S * LK));
            tr_.s = static_cast<float*>(dalloc(4 * S * LH));
            tr_.r = static_cast<float*>(dalloc(4 * S * LH));
            tr_.m = static_cast<float*>(dalloc(4 * S * LH));
            tr_.lg_true = static_cast<float*>(dalloc(4 * S * LE));
            tr_.lg_pred = static_cast<float*>(dalloc(4 * S * LE));
            tr_.y = static_cast<float*>(dalloc(4 * S * LK * c.H));
            tr_.logits = static_cast<float*>(dalloc(4 * S * c.V));
        }
        max_steps_ = max_steps;
        trace_full_ = trace_full;
        drop_graphs();
    }
    dset(tr_.step, 0, 4, "reset");
    if (max_steps > 0) {
        const long long n = static_cast<long long>(max_steps) * c.L * c.K * 4;
        dset(tr_.id_pred, 0xff, n, "reset");
    }
    steps_ = 0;
    n_step_events_ = 0;
    ck(cudaEventRecord(ev_origin_, s_comp_), "event");
    cache_->clear_stats();
    sched_ ? sched_->clear_records() : void();
}

// One forward pass of `st` (forward_decode / speculative_forward structure,
// model.cpp:355-389 / speculation.cpp:350-399, with Alg. 1's copy requests).
void Session::enqueue_pass(DevState& st, int mode, int use_pred, int calibrating, int step_tag,
                           int record, cudaStream_t s) {
    (void)step_tag;
    const ModelCfg& c = cfg_;
    const bool is_main = (&st == &st_);
    const bool prefetch = mode == 1 && use_pred && pred_kind_ != kNone;
    auto kind_at = [&](int l) -> int {
        if (l >= c.L - 1) return kNone;
        return pred_kind_ == kHybrid ? hybrid_[l] : pred_kind_;
    };
    const DevState* shadow = pred_kind_ == kOracle ? &sh_ : nullptr;
    // Prefetch mode keeps routing off the critical path (Alg. 1): the experts
    // executed at layer l were predicted at l-1, so the true router (logging
    // only) and the predictor for l+1 run on a side stream forked after the
    // attention output, while the expert FFN proceeds on the compute stream.
    // The side work of layer l joins before the FFN of layer l+1 (which runs
    // the decision it produced) and before the end of the step.
    std::vector<char> side_at(c.L, 0);  // layers whose side work recorded ev_join_
    bool side_used = false, log_used = false;
    const bool tl = tl_ && is_main;  // timeline: CUDA events around each phase
    for (int l = 0; l < c.L; ++l) {
        const int t_attn = tl ? tl_begin(0, 0, l, s) : -1;
        ck(launch_qkv(dm_, st, l, s), "qkv");
        ck(launch_attn(dm_, st, d_attn_scratch_, l, s), "attn");
        // prefetch, l >= 1: k_wo also forms rd_l = r_l + d_l for this layer's
        // q_l (router-pf / est-pf) from the decision predicted at l-1, which it
        // and k_ffn_gu take from the predictor's device flag (dec_ready), not
        // from a stream join: a graph-captured PDL launch makes even the
        // cross-stream edge programmatic, and a join here would hold the whole
        // layer behind the predictor's tail.
        const int kq = prefetch && l > 0 ? kind_at(l) : kNone;
        const int quasi_ready = kq == kRouterPF || kq == kEstPF;
        ck(launch_wo(dm_, st, ctl_, l, s, quasi_ready), "wo");
        if (tl) tl_end(t_attn, s);
        int exec_src = 0, s_from_r = 0;
        if (!prefetch) {
            const int t_gate = tl ? tl_begin(0, 1, l, s) : -1;
            RouterLaunch rl{l, 1, kNone, 0, 1, 0, step_tag, 0};
            ck(launch_router(dm_, st, ctl_, rl, nullptr, s), "router");
            if (tl) tl_end(t_gate, s);
        } else {
            const int k = kind_at(l);
            if (l == 0) {
                const int t_gate = tl ? tl_begin(0, 1, l, s) : -1;
                RouterLaunch rl{0, 1, kNone, 0, 1, 0, step_tag, 0};
                ck(launch_router(dm_, st, ctl_, rl, nullptr, s), "router");
                if (tl) tl_end(t_gate, s);
            }
            ck(cudaEventRecord(ev_fork_[l], s), "fork");
            ck(cudaStreamWaitEvent(s_side_, ev_fork_[l], 0), "fork");
            const int t_side = tl ? tl_begin(0, 1, l, s_side_) : -1;
            if (l == 0) {
                if (k != kNone) {
                    const int q0 = k == kRouterPF || k == kEstPF;
                    if (q0) ck(launch_quasi_rd(dm_, st, 0, s_side_), "quasi");
                    RouterLaunch rp{0, 0, k, -1, 0, k != kEstPF, step_tag, q0};
                    ck(launch_router(dm_, st, ctl_, rp, shadow, s_side_), "router");
                }
            } else {
                // the predictor first: its copy request and decision gate the
                // next layer; the true router of this layer only feeds the
                // hit-rate log, so it runs after the join point
                RouterLaunch rp{l, 0, k, 1, 0, k != kNone && k != kEstPF, step_tag, quasi_ready};
                ck(launch_router(dm_, st, ctl_, rp, shadow, s_side_), "router");
            }
            if (k == kEstPF) ck(launch_estimator(dm_, st, ctl_, l, 1, step_tag, s_side_), "estimator");
            // joined before k_wo of the next layer (see above); kernels read the
            // side stream's results only after their griddepcontrol.wait (a
            // captured PDL launch makes even a cross-stream edge programmatic)
            ck(cudaEventRecord(ev_join_[l], s_side_), "join");
            if (k != kNone && l + 1 < c.L && l2_prefetch_)  // warm L2 with layer l+1's experts
                ck(launch_l2_prefetch(dm_, st, ctl_, l + 1, s_side_), "l2 prefetch");
            if (tl) tl_end(t_side, s_side_);
            if (l == c.L - 1 && c.L > 1) {
                // true routers of layers 1..L-1 (speculation.cpp:370-371: logged
                // every layer, never executed here) in ONE launch on the
                // lowest-priority log stream once r_{L-1} exists, overlapping the
                // last layer's experts.  (Launched per layer, the graph executor
                // queued each one behind the compute stream's expert kernel.)
                ck(cudaStreamWaitEvent(s_log_, ev_fork_[l], 0), "fork");
                ck(launch_log_routers(dm_, st, ctl_, 1, c.L - 1, step_tag, s_log_), "router");
                log_used = true;
            }
            side_used = true;
            side_at[l] = 1;
            if (l > 0) {
                exec_src = 1;
                s_from_r = 1;
            }
        }
        // guard join, one layer behind: the side work of layer l-2 is complete
        // before the FFN of layer l (its flags were consumed a layer earlier),
        // so spinning expert CTAs can never starve an unfinished predictor
        static const bool guard_join = std::getenv("SMOE_GUARD_JOIN") != nullptr;
        if (guard_join && l >= 2 && side_at[l - 2]) ck(cudaStreamWaitEvent(s, ev_join_[l - 2], 0), "join");
        if (host_ordered_ && !ctl_.resident) host_copy_barrier(s);
        const int t_exp = tl ? tl_begin(0, 2, l, s) : -1;
        ck(launch_ffn(dm_, st, ctl_, l, s, exec_src, s_from_r), "ffn");
        if (tl) tl_end(t_exp, s);
        if (calibrating) ck(launch_dv_accum(dm_, st, d_dv_sums_, d_dv_counts_, l, s), "dv");
        if (is_main && record && trace_full_ && tr_.cap > 0) ck(launch_trace_y(dm_, st, tr_, l, s), "trace");
    }
    if (side_used) {  // everything on the side stream
        ck(cudaEventRecord(ev_side_end_, s_side_), "join");
        ck(cudaStreamWaitEvent(s, ev_side_end_, 0), "join");
    }
    if (log_used) {  // and the logging routers
        ck(cudaEventRecord(ev_log_end_, s_log_), "join");
        ck(cudaStreamWaitEvent(s, ev_log_end_, 0), "join");
    }
    ck(launch_final(dm_, st, ctl_, record && is_main, s), "final");
    if (is_main && record && tr_.cap > 0) ck(launch_trace(dm_, st, tr_, s), "trace");
}

void Session::enqueue_step(int mode, int is_prefill, int record, int calibrating, cudaStream_t s,
                           int stream) {
    const int* tok_src = st_.token;
    const int* sp = stream ? d_stream_ : nullptr;
    if (!is_prefill && mode == 1 && pred_kind_ == kOracle) {
        // Oracle::begin_token (speculation.cpp:271-280): true path on the shadow state
        ck(launch_embed(dm_, sh_, tok_src, s, sp, ctl_.step), "embed");
        enqueue_pass(sh_, 0, 0, 0, -2, 0, s);
    }
    ck(launch_embed(dm_, st_, tok_src, s, sp, ctl_.step), "embed");
    enqueue_pass(st_, is_prefill ? 0 : mode, is_prefill ? 0 : 1, calibrating, is_prefill ? -1 : 0,
                 record, s);
}

void Session::host_copy_barrier(cudaStream_t s) {
    ck(cudaStreamSynchronize(s), "host-ordered sync");
    ck(cudaStreamSynchronize(s_side_), "host-ordered sync");
    int posted = 0;
    ck(cudaMemcpy(&posted, ctl_.req_counter, 4, cudaMemcpyDeviceToHost), "request counter");
    const auto t0 = std::chrono::steady_clock::now();
    while (sched_->next_seq() - 1 < posted) {
        if (!sched_->error().empty()) break;  // surfaced by the next sync()
        if (std::chrono::steady_clock::now() - t0 > std::chrono::duration<double>(opts_.deadlock_s))
            throw std::runtime_error("deadlock suspected: copy scheduler did not serve request " +
                                     std::to_string(posted));
        std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
    ck(cudaEventRecord(ev_hostord_, s_copy_), "event");
    ck(cudaStreamWaitEvent(s, ev_hostord_, 0), "host-ordered wait");
    ck(cudaEventRecord(ev_hostord2_, s_unpack_), "event");  // tails of a packed store
    ck(cudaStreamWaitEvent(s, ev_hostord2_, 0), "host-ordered wait");
}

void Session::set_token(int tok) {
    // synchronous small upload (host-driven entry points only)
    ck(cudaMemcpyAsync(st_.token, &tok, 4, cudaMemcpyHostToDevice, s_comp_), "token");
    ck(cudaStreamSynchronize(s_comp_), "token");
}

void Session::prefill(const int* tokens, int n) {
    if (n < 1) throw std::invalid_argument("generate: empty prompt");
    sync();
    for (int i = 0; i < n; ++i)
        if (tokens[i] < 0 || tokens[i] >= cfg_.V) throw std::invalid_argument("forward_decode: token out of vocab");
    int pos = 0;
    d2h(&pos, st_.pos, 4, "pos");
    if (pos + n >= dm_.cap) throw std::invalid_argument("prefill: KV capacity exceeded");
    h2d(d_prompt_tok_, tokens, 4ull * n, "prompt");
    for (int i = 0; i < n; ++i) {
        ck(launch_embed(dm_, st_, d_prompt_tok_ + i, s_comp_), "embed");
        enqueue_pass(st_, 0, 0, 0, -1, 1, s_comp_);
        if (pred_kind_ == kOracle) {  // Oracle::observe_prompt_token (speculation.cpp:266-269)
            ck(launch_embed(dm_, sh_, d_prompt_tok_ + i, s_comp_), "embed");
            enqueue_pass(sh_, 0, 0, 0, -2, 0, s_comp_);
        }
        ++steps_;
    }
    host_pos_ = pos + n;
    sync();
}

// Batched prefill: true routing, all tokens per layer at
// once; the executed experts of a layer are loaded once (in waves of at most
// C slots) instead of once per token.  Produces the same KV cache, next token
// and later decode steps as prefill() (tests/test_gpu.py); per-token trace
// rows of the prompt are not recorded.
void Session::prefill_batched(const int* tokens, int n) {
    if (n < 1) throw std::invalid_argument("generate: empty prompt");
    if (opts_.ep_world > 1) throw std::invalid_argument("prefill_batched: single GPU only");
    if (pred_kind_ == kOracle) {  // the Oracle replays a shadow state token by token
        prefill(tokens, n);
        return;
    }
    sync();
    ck(cudaStreamSynchronize(s_copy_), "copy stream");
    const ModelCfg& c = cfg_;
    for (int i = 0; i < n; ++i)
        if (tokens[i] < 0 || tokens[i] >= c.V) throw std::invalid_argument("forward_decode: token out of vocab");
    int pos = 0;
    d2h(&pos, st_.pos, 4, "pos");
    if (pos + n >= dm_.cap) throw std::invalid_argument("prefill: KV capacity exceeded");
    const DevModel& m = dm_;
    const long long E = c.E, K = c.K, Hp = m.Hp, D = c.D, nb = m.Hp / 32;
    if (n > pf_cap_) {  // (re)allocate for n tokens
        auto fr = [&](void* p) {
            for (auto it = dev_allocs_.begin(); it != dev_allocs_.end(); ++it)
                if (*it == p) {
                    cudaFree(p);
                    dev_allocs_.erase(it);
                    return;
                }
        };
        for (void* p : {(void*)pf_.tokens, (void*)pf_.X, (void*)pf_.ssqx, (void*)pf_.Q, (void*)pf_.ctx,
                        (void*)pf_.R, (void*)pf_.ssqr, (void*)pf_.lg, (void*)pf_.ids, (void*)pf_.gates,
                        (void*)pf_.cnt, (void*)pf_.off, (void*)pf_.fill, (void*)pf_.list, (void*)pf_.Hb,
                        (void*)pf_.Y, (void*)pf_.attn_scratch, (void*)pf_.scale, (void*)pf_.chunk_u,
                        (void*)pf_.chunk_c})
            if (p) fr(p);
        const long long P = n;
        pf_ = PrefillDev{};
        pf_.tokens = static_cast<int*>(dalloc(4ull * P));
        pf_.X = static_cast<float*>(dalloc(4ull * P * Hp));
        pf_.ssqx = static_cast<double*>(dalloc(8ull * P * nb));
        pf_.Q = static_cast<float*>(dalloc(4ull * P * D));
        pf_.ctx = static_cast<float*>(dalloc(4ull * P * D));
        pf_.R = static_cast<float*>(dalloc(4ull * P * Hp));
        pf_.ssqr = static_cast<double*>(dalloc(8ull * P * nb));
        pf_.lg = static_cast<float*>(dalloc(4ull * P * E));
        pf_.ids = static_cast<int*>(dalloc(4ull * P * K));
        pf_.gates = static_cast<float*>(dalloc(4ull * P * K));
        pf_.cnt = static_cast<int*>(dalloc(4ull * E));
        pf_.off = static_cast<int*>(dalloc(4ull * (E + 1)));
        pf_.fill = static_cast<int*>(dalloc(4ull * E));
        pf_.list = static_cast<int*>(dalloc(4ull * P * K));
        pf_.Hb = static_cast<float*>(dalloc(4ull * P * K * m.Hmp));
        pf_.Y = static_cast<float*>(dalloc(4ull * P * K * Hp));
        if (m.cap > pf_attn_smem_positions())
            pf_.attn_scratch = static_cast<double*>(dalloc(8ull * P * 2 * m.cap));
        pf_.scale = static_cast<float*>(dalloc(4ull * P));
        pf_.chunk_u = static_cast<int*>(dalloc(4ull * (P * K + E)));  // >= sum of ceil(cnt/8)
        pf_.chunk_c = static_cast<int*>(dalloc(4ull * (P * K + E)));
        pf_cap_ = n;
    }
    pf_.P = n;
    pf_.pos0 = pos;
    pf_.attn_smem_positions = pf_attn_smem_positions();
    pf_.dev_step = ctl_.step;
    pf_.trace_step = tr_.cap > 0 ? tr_.step : nullptr;
    h2d(const_cast<int*>(pf_.tokens), tokens, 4ull * n, "prompt");
    ck(launch_pf_embed(m, pf_, s_comp_), "prefill embed");
    std::vector<int> cnt(E);
    for (int l = 0; l < c.L; ++l) {
        dset(pf_.cnt, 0, 4ull * E, "prefill counts");
        ck(launch_pf_layer_dense(m, st_, pf_, l, s_comp_), "prefill layer");
        d2h(cnt.data(), pf_.cnt, 4ull * E, "prefill counts");  // (synchronises)
        pf_waves(pf_, l, cnt);
        ck(launch_pf_mix(m, pf_, s_comp_), "prefill mix");
    }
    ck(launch_pf_handoff(m, st_, pf_, s_comp_), "prefill handoff");
    ck(launch_final(dm_, st_, ctl_, 1, s_comp_), "final");
    steps_ += n;
    host_pos_ = pos + n;
    sync();
}

// The experts of one layer for a batch of tokens, in waves of at most C
// slot-resident experts: copies (cache misses) on the copy stream, then the
// gate/up and down kernels over the wave's (expert, 8-token chunk) items.
// Decode GEMV arithmetic (DESIGN "Decode arithmetic modes"): 0 exact — every
// row a sequential f32 chain in the reference's column order (bit parity);
// 1 tolerance — the same kernels with four packed FFMA partial sums per row
// (WarpPipe::run_fast), HBM-bound instead of FADD-latency bound.  The captured
// step graphs embed DevModel by value, so they are rebuilt.
void Session::set_decode_mode(int mode) {
    if (mode != 0 && mode != 1) throw std::invalid_argument("decode mode must be 0 (exact) or 1 (tolerance)");
    if (dm_.fast == mode) return;
    sync();
    drop_graphs();
    dm_.fast = mode;
}

void Session::set_prefill_mode(int mode) {
    if (mode != 0 && mode != 1) throw std::invalid_argument("prefill mode must be 0 (exact) or 1 (tensor cores)");
    if (mode == 1 && !tc_prefill_supported(dm_))
        throw std::invalid_argument("tensor-core prefill needs hidden and expert_hidden multiples of 64");
    pf_tc_ = mode;
}

void Session::pf_waves(const PrefillDev& pf, int l, const std::vector<int>& cnt) {
    const ModelCfg& c = cfg_;
    const DevModel& m = dm_;
    std::vector<int> uni;
    for (int e = 0; e < c.E; ++e)
        if (cnt[e] > 0 && is_local(e)) uni.push_back(e);  // EP: this rank's experts
    const int W = std::min<int>(C_, kMaxWave);
    for (size_t w0 = 0; w0 < uni.size(); w0 += W) {
        const int nw = static_cast<int>(std::min<size_t>(W, uni.size() - w0));
        PfWave wv{};
        wv.n = nw;
        std::vector<int> cu, cc;  // (expert, 8-token chunk) work items of the wave
        for (int u = 0; u < nw; ++u) {
            wv.e[u] = uni[w0 + u];
            for (int q = 0; q < (cnt[uni[w0 + u]] + 7) / 8; ++q) {
                cu.push_back(u);
                cc.push_back(q);
            }
        }
        const int chunks = static_cast<int>(cu.size());
        h2d(pf.chunk_u, cu.data(), 4ull * chunks, "prefill chunks");
        h2d(pf.chunk_c, cc.data(), 4ull * chunks, "prefill chunks");
        if (!ctl_.resident) {  // load the wave's experts into this layer's slots
            int hits = 0, misses = 0;
            auto copies = cache_->request(l, wv.e, nw, &hits, &misses);
            for (auto& [slot, expert] : copies)
                direct_bytes_ += copy_expert(l, expert, d_slots_ + (static_cast<long long>(l) * C_ + slot) * m.expert_elems,
                                             s_copy_, "prefill expert copy");
            join_unpack(s_copy_);
            ck(cudaStreamSynchronize(s_copy_), "prefill copies");
            h2d(d_slot_of_ + static_cast<long long>(l) * c.E, cache_->slot_row(l).data(), 4ull * c.E, "slot table");
        }
        const std::vector<int>& row = cache_->slot_row(l);
        for (int u = 0; u < nw; ++u) {
            wv.slot[u] = row[wv.e[u]];
            if (wv.slot[u] < 0) throw std::runtime_error("expert read before readiness at layer " + std::to_string(l));
        }
        if (pf_tc_ && !pf.bkc) {  // tensor-core expert GEMMs over 128-token blocks
            std::vector<int> tu, tcb;
            for (int u = 0; u < nw; ++u)
                for (int b = 0; b < (cnt[wv.e[u]] + 127) / 128; ++b) {
                    tu.push_back(u);
                    tcb.push_back(b);
                }
            const int items = static_cast<int>(tu.size());
            h2d(pf.chunk_u, tu.data(), 4ull * items, "prefill items");
            h2d(pf.chunk_c, tcb.data(), 4ull * items, "prefill items");
            const size_t need = tc_pack_bytes(m, items);
            if (need > tc_apk_cap_) {
                for (auto it = dev_allocs_.begin(); it != dev_allocs_.end(); ++it)
                    if (*it == d_tc_apk_) {
                        cudaFree(d_tc_apk_);
                        dev_allocs_.erase(it);
                        break;
                    }
                d_tc_apk_ = static_cast<uint16_t*>(dalloc(need));
                tc_apk_cap_ = need;
            }
            ck(launch_pf_experts_tc(m, pf, l, wv, items, d_tc_apk_, s_comp_), "prefill experts (tcgen05)");
        } else {
            // prefills fill whole 8-token chunks; decode batches (bkc set) get per-chunk dispatch
            ck(launch_pf_experts(m, pf, l, wv, chunks, s_comp_, pf.bkc ? 0 : 8), "prefill experts");
        }
        if (w0 + W < uni.size()) ck(cudaStreamSynchronize(s_comp_), "prefill wave");  // slots reused
    }
}

void Session::batch_generate(int B, const int* prompts, int P, int n_new, int mode, int* out_tokens,
                             float* out_logits, double* step_ms) {
    if (B < 1) throw std::invalid_argument("batch_generate: batch must be >= 1");
    if (P < 1) throw std::invalid_argument("generate: empty prompt");
    if (n_new < 1) throw std::invalid_argument("generate: n_new must be >= 1");
    if (opts_.ep_world > 1 && ctl_.ep.world != opts_.ep_world)
        throw std::invalid_argument("batch_generate: expert-parallel ranks must be connected first (ep_connect)");
    if (ctl_.ep.world > 1 && B > kEpBatchMax)
        throw std::invalid_argument("batch_generate: at most " + std::to_string(kEpBatchMax) +
                                    " sequences per step under expert parallelism");
    if (mode == 1 && pred_kind_ == kNone)
        throw std::invalid_argument("offloaded decode: prefetch mode needs a predictor");
    if (mode == 1 && pred_kind_ == kOracle)
        throw std::invalid_argument("batch_generate: the oracle predictor replays one shadow state; not batched");
    auto kind_at = [&](int l) -> int { return pred_kind_ == kHybrid ? hybrid_[l] : pred_kind_; };
    if (mode == 1)
        for (int l = 0; l + 1 < cfg_.L; ++l) {
            const int k = kind_at(l);
            if ((k == kRouterPF || k == kEstPF) && !have_dv_)
                throw std::invalid_argument("batch_generate: quasi-hidden inputs need default vectors");
            if (k == kEstPF && !have_est_) throw std::invalid_argument("batch_generate: est-pf needs an estimator");
        }
    const ModelCfg& c = cfg_;
    const DevModel& m = dm_;
    for (long long i = 0; i < static_cast<long long>(B) * P; ++i)
        if (prompts[i] < 0 || prompts[i] >= c.V) throw std::invalid_argument("forward_decode: token out of vocab");
    if (P + n_new - 1 > m.cap) throw std::invalid_argument("batch_generate: KV capacity exceeded");
    sync();
    ck(cudaStreamSynchronize(s_copy_), "copy stream");
    const long long E = c.E, K = c.K, Hp = m.Hp, D = c.D, nb = m.Hp / 32, Bl = B;
    if (B > bd_cap_) {  // buffers sized for bd_cap_ sequences, kept across calls
        for (void* p : bd_allocs_) cudaFree(p);
        bd_allocs_.clear();
        bd_cap_ = 0;
    }
    auto al = [&](size_t bytes) {
        void* p = nullptr;
        ck(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "batch alloc");
        bd_allocs_.push_back(p);
        return p;
    };
    PrefillDev& bd = bd_;
    if (bd_cap_ == 0) {
        bd = PrefillDev{};
        bd.tokens = static_cast<int*>(al(4ull * Bl));
        bd.X = static_cast<float*>(al(4ull * Bl * Hp));
        bd.ssqx = static_cast<double*>(al(8ull * Bl * nb));
        bd.Q = static_cast<float*>(al(4ull * Bl * D));
        bd.ctx = static_cast<float*>(al(4ull * Bl * D));
        bd.R = static_cast<float*>(al(4ull * Bl * Hp));
        bd.ssqr = static_cast<double*>(al(8ull * Bl * nb));
        bd.lg = static_cast<float*>(al(4ull * Bl * E));
        bd.ids = static_cast<int*>(al(4ull * Bl * K));
        bd.gates = static_cast<float*>(al(4ull * Bl * K));
        bd.cnt = static_cast<int*>(al(4ull * E));
        bd.off = static_cast<int*>(al(4ull * (E + 1)));
        bd.fill = static_cast<int*>(al(4ull * E));
        bd.list = static_cast<int*>(al(4ull * Bl * K));
        bd.Hb = static_cast<float*>(al(4ull * Bl * K * m.Hmp));
        bd.Y = static_cast<float*>(al(4ull * Bl * K * Hp));
        if (m.cap > pf_attn_smem_positions()) bd.attn_scratch = static_cast<double*>(al(8ull * Bl * 2 * m.cap));
        bd.scale = static_cast<float*>(al(4ull * Bl));
        bd.chunk_u = static_cast<int*>(al(4ull * (Bl * K + E)));
        bd.chunk_c = static_cast<int*>(al(4ull * (Bl * K + E)));
        bd.bkv_stride = static_cast<long long>(c.L) * m.cap * D;
        bd.bkc = static_cast<float*>(al(4ull * Bl * bd.bkv_stride));
        bd.bvc = static_cast<float*>(al(4ull * Bl * bd.bkv_stride));
        bd.RD = static_cast<float*>(al(4ull * Bl * Hp));
        bd.ssqrd = static_cast<double*>(al(8ull * Bl * nb));
        bd.lgp = static_cast<float*>(al(4ull * Bl * E));
        bd.pids = static_cast<int*>(al(4ull * 2 * Bl * K));
        bd.pgates = static_cast<float*>(al(4ull * 2 * Bl * K));
        bd.logits = static_cast<float*>(al(4ull * Bl * c.V));
        bd.next = static_cast<int*>(al(4ull * Bl));
        bd_nchunks_ = static_cast<int*>(al(4));
        bd_qn_ = static_cast<float*>(al(4ull * Bl * c.H));
        bd_pos_ = static_cast<int*>(al(4));
        bd_cap_ = B;
    }
    bd.P = B;
    bd.attn_smem_positions = pf_attn_smem_positions();
    float *ez = nullptr, *eu = nullptr, *ea = nullptr, *eh = nullptr, *ex = nullptr, *ey = nullptr, *ei = nullptr;
    int edm = 0, emlp = 0;
    std::vector<void*> scratch;
    struct FreeAll {
        std::vector<void*>& v;
        ~FreeAll() {
            for (void* p : v) cudaFree(p);
        }
    } free_scratch{scratch};
    auto tmp = [&](size_t bytes) {
        void* p = nullptr;
        ck(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "batch alloc");
        scratch.push_back(p);
        return static_cast<float*>(p);
    };
    if (have_est_ && mode == 1) {  // estimator_forward scratch for B tokens (freed with this call)
        edm = est_.d / est_.m;
        emlp = edm * est_.n;
        for (float** p : {&ez, &eh, &ex, &ey}) *p = tmp(4ull * Bl * edm);
        for (float** p : {&eu, &ea}) *p = tmp(4ull * Bl * emlp);
        ei = tmp(4ull * Bl);
    }
    // resident experts: every expert's slot is fixed, the work list is built on
    // the device and a layer needs no host round trip
    const bool dev_lists = ctl_.resident && c.E <= kMaxWave;
    const int max_chunks = static_cast<int>(std::min<long long>(Bl * K, E * ((Bl + 7) / 8)));
    bd.nchunks = dev_lists ? bd_nchunks_ : nullptr;  // null: host-built lists, no bound check
    std::vector<int> cnt(E), tok(B), next(B);
    std::vector<float> lg(static_cast<size_t>(Bl) * c.V);
    // one token of every sequence at position pos (forward_decode /
    // speculative_forward, model.cpp:355-398, speculation.cpp:350-399)
    // resident experts: each step mode is captured once as a CUDA graph (the
    // position and the tokens live on the device; nothing in a step needs the host)
    // (not under EP: instantiating a graph may wait for the device, which a
    // peer's combine is spinning on)
    const bool use_graph = dev_lists && ctl_.ep.world == 1 && std::getenv("SMOE_BATCH_NO_GRAPH") == nullptr;
    bd.pos_dev = use_graph ? bd_pos_ : nullptr;
    auto body = [&](int md) {
        ck(launch_pf_embed(m, bd, s_comp_), "batch embed");
        for (int l = 0; l < c.L; ++l) {
            dset(bd.cnt, 0, 4ull * E, "batch counts");
            ck(launch_pf_attn_block(m, st_, bd, l, s_comp_), "batch attention");
            if (md == 0 || l == 0)
                ck(launch_pf_route(m, bd, l, s_comp_), "batch router");
            else
                ck(launch_pf_exec_pred(m, bd, l & 1, s_comp_), "batch executed = predicted");
            if (dev_lists) {
                PfWave wv{};  // every expert (wave index = expert id); work items for this rank's only
                wv.n = c.E;
                const std::vector<int>& row = cache_->slot_row(l);
                for (int e = 0; e < c.E; ++e) {
                    wv.e[e] = e;
                    wv.slot[e] = row[e];
                }
                ck(launch_pf_experts_dev(m, bd, l, wv, max_chunks, s_comp_, ctl_.ep.world > 1 ? ctl_.ep.rank : 0,
                                         ctl_.ep.world),
                   "batch experts");
            } else {
                d2h(cnt.data(), bd.cnt, 4ull * E, "batch counts");  // (synchronises)
                pf_waves(bd, l, cnt);  // local experts only
            }
            if (ctl_.ep.world > 1) {  // every rank's expert rows of this layer, then the mix reads them
                ck(launch_pf_ep_combine(m, bd, ctl_.ep, l, ctl_.error, ctl_.spin_limit, s_comp_), "batch ep combine");
                PrefillDev bx = bd;
                bx.Y = ctl_.ep.bxbuf[ctl_.ep.rank] + static_cast<long long>(l & 1) * kEpBatchMax * K * Hp;
                ck(launch_pf_mix(m, bx, s_comp_), "batch mix");
            } else {
                ck(launch_pf_mix(m, bd, s_comp_), "batch mix");
            }
            if (md == 1 && l + 1 < c.L) {  // prediction for l+1 (speculation.cpp:174-252)
                const int k = kind_at(l), buf = (l + 1) & 1;
                if (k == kBaselineS) {
                    ck(launch_pf_predict_baseline_s(m, bd, l, buf, s_comp_), "batch predictor");
                } else if (k == kRouterPF) {
                    ck(launch_pf_predict(m, bd, l, buf, s_comp_), "batch predictor");
                } else {  // est-pf: estimator_forward (estimator.cpp:94-161) over the B q_l
                    const long long d = est_.d, L = est_.L, dm = edm, mlp = emlp;
                    const float* A = d_est_flat_;
                    const float* pos = A + dm * d + static_cast<long long>(l) * dm;
                    const float* Bw = A + dm * d + L * dm;
                    const float* Cw = Bw + mlp * dm;
                    const float* gain = Cw + dm * mlp;
                    const float* bias = gain + dm;
                    const float* head = bias + dm;
                    ck(launch_pf_quasi_q(m, bd, l, bd_qn_, s_comp_), "batch q");
                    auto gm = [&](ChainGemm g) { ck(launch_chain_gemm(g, s_comp_), "batch estimator"); };
                    gm({bd_qn_, 1, d, A, 1, d, ez, dm, 1, nullptr, B, edm, static_cast<int>(d), kEpiAddPos, pos,
                        nullptr, 1});
                    gm({ez, 1, dm, Bw, 1, dm, eu, mlp, 1, nullptr, B, emlp, edm, kEpiSilu, nullptr, ea, 1});
                    gm({ea, 1, mlp, Cw, 1, mlp, eh, dm, 1, nullptr, B, edm, emlp, kEpiAddAfter, ez, nullptr, 1});
                    ck(launch_est_layernorm(eh, gain, bias, B, edm, est_.eps, ex, ey, ei, s_comp_), "batch estimator");
                    gm({ey, 1, dm, head, 1, dm, bd.lgp, c.E, 1, nullptr, B, c.E, edm, kEpiNone, nullptr, nullptr, 1});
                    ck(launch_pf_decide_pred(m, bd, buf, s_comp_), "batch predictor");
                }
                if (!dev_lists) {
                    // Algorithm 1 for the batch: the predicted experts of l+1 (the
                    // union over the B sequences, in the order pf_waves loads them)
                    // start copying now, one layer ahead, on the copy stream; the
                    // first wave of l+1 then finds them resident or in flight
                    std::vector<int> pids(static_cast<size_t>(Bl) * K);
                    d2h(pids.data(), bd.pids + static_cast<long long>(buf) * Bl * K, 4ull * Bl * K, "batch pids");
                    std::vector<char> want(c.E, 0);
                    for (int e : pids)
                        if (e >= 0 && e < c.E) want[e] = 1;
                    std::vector<int> first;
                    const int W = std::min<int>(C_, kMaxWave);
                    for (int e = 0; e < c.E && static_cast<int>(first.size()) < W; ++e)
                        if (want[e] && is_local(e)) first.push_back(e);
                    int hits = 0, misses = 0;
                    const auto copies = cache_->request(l + 1, first.data(), static_cast<int>(first.size()), &hits, &misses);
                    for (const auto& [slot, expert] : copies) {
                        const long long b = copy_expert(
                            l + 1, expert, d_slots_ + (static_cast<long long>(l + 1) * C_ + slot) * m.expert_elems,
                            s_copy_, "batch prefetch copy");
                        batch_prefetched_bytes_ += b;
                        direct_bytes_ += b;
                    }
                    join_unpack(s_copy_);
                }
            }
        }
        ck(launch_pf_final(m, bd, s_comp_), "batch final");
    };
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    struct GraphFree {
        cudaGraphExec_t* g;
        ~GraphFree() {
            for (int i = 0; i < 2; ++i)
                if (g[i]) cudaGraphExecDestroy(g[i]);
        }
    } graph_free{gexec};
    auto step = [&](const int* toks, int pos, int md) {
        bd.pos0 = pos;
        h2d(const_cast<int*>(bd.tokens), toks, 4ull * B, "batch tokens");
        if (use_graph) {
            h2d(bd_pos_, &pos, 4, "batch position");
            if (!gexec[md]) {
                cudaGraph_t g;
                ck(cudaStreamBeginCapture(s_comp_, cudaStreamCaptureModeThreadLocal), "capture");
                body(md);
                ck(cudaStreamEndCapture(s_comp_, &g), "capture");
                const cudaError_t e = cudaGraphInstantiate(&gexec[md], g, 0);
                cudaGraphDestroy(g);
                ck(e, "instantiate");
            }
            ck(cudaGraphLaunch(gexec[md], s_comp_), "batch graph");
        } else {
            body(md);
        }
        d2h(next.data(), bd.next, 4ull * B, "batch next");
        if (out_logits) d2h(lg.data(), bd.logits, 4ull * Bl * c.V, "batch logits");
    };
    for (int i = 0; i < P; ++i) {  // prompt: true path (generate, speculation.cpp:404-409)
        for (int b = 0; b < B; ++b) tok[b] = prompts[static_cast<long long>(b) * P + i];
        step(tok.data(), i, 0);
    }
    double ms = 0.0;
    for (int i = 0; i < n_new; ++i) {
        for (int b = 0; b < B; ++b) {
            out_tokens[static_cast<long long>(b) * n_new + i] = next[b];
            if (out_logits)
                std::memcpy(out_logits + (static_cast<long long>(b) * n_new + i) * c.V,
                            lg.data() + static_cast<long long>(b) * c.V, 4ull * c.V);
        }
        if (i + 1 == n_new) break;
        tok = next;
        const auto t0 = std::chrono::steady_clock::now();
        step(tok.data(), P + i, mode);  // ends with the next-token read back
        ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    if (step_ms) *step_ms = n_new > 1 ? ms / (n_new - 1) : 0.0;
    sync();
}

void Session::decode(int mode, int n_steps, int use_graph) {
    if (n_steps < 0) throw std::invalid_argument("decode: n_steps must be >= 0");
    if (mode == 1 && pred_kind_ == kNone)
        throw std::invalid_argument("offloaded decode: prefetch mode needs a predictor");
    sync();
    int pos = 0;
    d2h(&pos, st_.pos, 4, "pos");
    if (pos + n_steps >= dm_.cap) throw std::invalid_argument("decode: KV capacity exceeded");
    size_attn_grid(pos + n_steps);
    host_pos_ = pos + n_steps;
    cudaGraphExec_t exec = use_graph ? get_graph(mode) : nullptr;
    ck(cudaEventRecord(ev_origin_, s_comp_), "event");
    for (int i = 0; i < n_steps; ++i) {
        const int ev = n_step_events_ < static_cast<int>(ev_step_.size() / 2) ? n_step_events_++ : -1;
        if (ev >= 0) ck(cudaEventRecord(ev_step_[2 * ev], s_comp_), "event");
        if (exec)
            ck(cudaGraphLaunch(exec, s_comp_), "graph launch");
        else
            enqueue_step(mode, 0, 1, 0, s_comp_);
        if (ev >= 0) ck(cudaEventRecord(ev_step_[2 * ev + 1], s_comp_), "event");
        ++steps_;
    }
    dm_.attn_fast_grid = 0;
    sync();
}

int Session::tl_begin(int lane, int kind, int layer, cudaStream_t s) {
    cudaEvent_t a, b;
    ck(cudaEventCreate(&a), "event");
    ck(cudaEventCreate(&b), "event");
    ck(cudaEventRecord(a, s), "event");
    tl_->ev.push_back({a, b});
    tl_->meta.push_back({lane, kind, layer, tl_->step, 0.0, 0.0});
    return static_cast<int>(tl_->meta.size()) - 1;
}

void Session::tl_end(int idx, cudaStream_t s) { ck(cudaEventRecord(tl_->ev[idx].second, s), "event"); }

void Session::upload_stream(const int* tokens, int n_steps) {
    for (int i = 0; i < n_steps; ++i)
        if (tokens[i] < 0 || tokens[i] >= cfg_.V)
            throw std::invalid_argument("forward_decode: token out of vocab");
    if (!d_stream_) d_stream_ = static_cast<int*>(dalloc(4ull * (dm_.cap + 2)));
    int step = 0;
    d2h(&step, ctl_.step, 4, "step");
    if (step + n_steps > dm_.cap + 1) throw std::invalid_argument("decode: stream exceeds capacity");
    h2d(d_stream_ + step, tokens, 4ull * n_steps, "stream");
}

// run_offloaded_decode's measured event log (executor.cpp:239-322): compute
// lane phases from CUDA events around each layer's attention, routing (side
// stream in prefetch mode) and expert kernels; copy lane from the scheduler's
// per-request events, assigned to the decode step whose window they start in.
void Session::decode_timeline(int mode, const int* tokens, int n_steps,
                              std::vector<TimelineEvent>& out) {
    if (mode == 1 && pred_kind_ == kNone)
        throw std::invalid_argument("offloaded decode: prefetch mode needs a predictor");
    sync();
    int pos = 0;
    d2h(&pos, st_.pos, 4, "pos");
    if (pos + n_steps >= dm_.cap) throw std::invalid_argument("decode: KV capacity exceeded");
    if (tokens) upload_stream(tokens, n_steps);
    clear_stats();
    TlRec rec;
    tl_ = &rec;
    try {
        ck(cudaEventRecord(ev_origin_, s_comp_), "event");
        for (int i = 0; i < n_steps; ++i) {
            rec.step = i;
            enqueue_step(mode, 0, 1, 0, s_comp_, tokens ? 1 : 0);
            ++steps_;
        }
        sync();
        ck(cudaStreamSynchronize(s_copy_), "copy stream");
    } catch (...) {
        tl_ = nullptr;
        for (auto& ab : rec.ev) {
            cudaEventDestroy(ab.first);
            cudaEventDestroy(ab.second);
        }
        throw;
    }
    tl_ = nullptr;
    std::vector<double> step_start(n_steps, 1e300);
    for (size_t i = 0; i < rec.meta.size(); ++i) {
        float a = 0.0f, b = 0.0f;
        ck(cudaEventElapsedTime(&a, ev_origin_, rec.ev[i].first), "elapsed");
        ck(cudaEventElapsedTime(&b, ev_origin_, rec.ev[i].second), "elapsed");
        TimelineEvent e = rec.meta[i];
        e.start_ms = a;
        e.end_ms = b;
        step_start[e.token] = std::min(step_start[e.token], e.start_ms);
        out.push_back(e);
        cudaEventDestroy(rec.ev[i].first);
        cudaEventDestroy(rec.ev[i].second);
    }
    std::map<std::pair<int, int>, double> copy_end;  // (step, layer) -> end of its copy
    for (const CopyRecord& r : sched_->records()) {
        if (r.ev < 0 || r.bytes == 0) continue;
        const double a = event_ms(r.ev, 0), b = event_ms(r.ev, 1);
        int t = -1;
        for (int i = 0; i < n_steps; ++i)
            if (a >= step_start[i] - 1e-6) t = i;
        out.push_back({1, 3, r.layer, t, a, b});
        copy_end[{t, r.layer}] = b;
    }
    // The expert kernel spins on the copy-ready flag inside its launch; the
    // reference's expert compute starts after wait_ready (executor.cpp:306-316),
    // so the compute-lane expert interval starts at max(launch, copy end).
    for (TimelineEvent& e : out) {
        if (e.lane != 0 || e.kind != 2) continue;
        auto it = copy_end.find({e.token, e.layer});
        if (it != copy_end.end() && it->second > e.start_ms)
            e.start_ms = std::min(it->second, e.end_ms);
    }
}

void Session::decode_stream(int mode, const int* tokens, int n_steps) {
    if (n_steps < 0) throw std::invalid_argument("decode: n_steps must be >= 0");
    if (mode == 1 && pred_kind_ == kNone)
        throw std::invalid_argument("offloaded decode: prefetch mode needs a predictor");
    sync();
    int pos = 0;
    d2h(&pos, st_.pos, 4, "pos");
    if (pos + n_steps >= dm_.cap) throw std::invalid_argument("decode: KV capacity exceeded");
    upload_stream(tokens, n_steps);
    size_attn_grid(pos + n_steps);
    host_pos_ = pos + n_steps;
    cudaGraphExec_t exec = get_graph(mode, 1);
    ck(cudaEventRecord(ev_origin_, s_comp_), "event");
    for (int i = 0; i < n_steps; ++i) {
        const int ev = n_step_events_ < static_cast<int>(ev_step_.size() / 2) ? n_step_events_++ : -1;
        if (ev >= 0) ck(cudaEventRecord(ev_step_[2 * ev], s_comp_), "event");
        if (exec)
            ck(cudaGraphLaunch(exec, s_comp_), "graph launch");
        else
            enqueue_step(mode, 0, 1, 0, s_comp_, 1);
        if (ev >= 0) ck(cudaEventRecord(ev_step_[2 * ev + 1], s_comp_), "event");
        ++steps_;
    }
    dm_.attn_fast_grid = 0;
    sync();
}

int Session::step_host(int mode, int token, float* logits_out) {
    if (token < 0 || token >= cfg_.V) throw std::invalid_argument("forward_decode: token out of vocab");
    if (mode == 1 && pred_kind_ == kNone)
        throw std::invalid_argument("offloaded decode: prefetch mode needs a predictor");
    // host mirror of the position (no device read on this path); if it is
    // stale the grid is only suboptimal, never wrong
    size_attn_grid(std::min(host_pos_ + 64, dm_.cap - 1));
    ++host_pos_;
    cudaGraphExec_t exec = get_graph(mode);
    h_token_[0] = token;
    ck(cudaMemcpyAsync(st_.token, h_token_, 4, cudaMemcpyHostToDevice, s_comp_), "token H2D");
    if (exec)
        ck(cudaGraphLaunch(exec, s_comp_), "graph launch");
    else
        enqueue_step(mode, 0, 1, 0, s_comp_);
    dm_.attn_fast_grid = 0;
    ck(cudaMemcpyAsync(h_logits_, st_.logits, 4ull * cfg_.V, cudaMemcpyDeviceToHost, s_comp_), "logits D2H");
    ck(cudaMemcpyAsync(h_token_ + 1, st_.token, 4, cudaMemcpyDeviceToHost, s_comp_), "token D2H");
    ck(cudaStreamSynchronize(s_comp_), "step");
    ++steps_;
    check_device_error();
    if (logits_out) std::memcpy(logits_out, h_logits_, 4ull * cfg_.V);
    return h_token_[1];
}

// accumulate_default_vectors over random_token_stream (trace.cpp:187-211,
// speculation.cpp:23-58), true routing, state reset every seq_len tokens.
void Session::calibrate(long long ntok, uint64_t seed, int seq_len, float* d_out, long long* c_out) {
    if (ntok < 1) throw std::invalid_argument("trace: empty workload");
    if (seq_len < 1) throw std::invalid_argument("trace: seq_len must be >= 1");
    if (seq_len + 1 >= dm_.cap) throw std::invalid_argument("calibrate: seq_len exceeds KV capacity");
    sync();
    const ModelCfg& c = cfg_;
    const long long LE = static_cast<long long>(c.L) * c.E;
    d_dv_sums_ = static_cast<double*>(dalloc(8ull * LE * c.H));
    d_dv_counts_ = static_cast<long long*>(dalloc(8ull * LE));
    std::vector<int> toks(ntok);
    {
        uint64_t st = derive_seed(seed, "token-stream");
        for (long long i = 0; i < ntok; ++i) {
            st += 0x9E3779B97F4A7C15ull;
            uint64_t z = st;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            z = z ^ (z >> 31);
            toks[i] = static_cast<int>(z % static_cast<uint64_t>(c.V));
        }
    }
    int* d_toks = static_cast<int*>(dalloc(4ull * ntok));
    h2d(d_toks, toks.data(), 4ull * ntok, "tokens");
    int zero = 0;
    for (long long i = 0; i < ntok; ++i) {
        if (i % seq_len == 0) ck(cudaMemcpyAsync(st_.pos, &zero, 4, cudaMemcpyHostToDevice, s_comp_), "pos");
        ck(launch_embed(dm_, st_, d_toks + i, s_comp_), "embed");
        enqueue_pass(st_, 0, 0, 1, -3, 0, s_comp_);
        if (i % 64 == 63) sync();
    }
    ck(launch_dv_freeze(d_dv_sums_, d_dv_counts_, d_dv_, LE, c.H, s_comp_), "freeze");
    sync();
    if (d_out) d2h(d_out, d_dv_, 4ull * LE * c.H, "dv");
    if (c_out) d2h(c_out, d_dv_counts_, 8ull * LE, "counts");
    for (void* p : {(void*)d_dv_sums_, (void*)d_dv_counts_, (void*)d_toks})
        for (auto it = dev_allocs_.begin(); it != dev_allocs_.end(); ++it)
            if (*it == p) {
                cudaFree(p);
                dev_allocs_.erase(it);
                break;
            }
    d_dv_sums_ = nullptr;
    d_dv_counts_ = nullptr;
    h2d(st_.pos, &zero, 4, "pos");
    have_dv_ = true;
}

// ------------------------------------------------------------- results ------

int Session::steps_done() { return steps_; }

// Tolerance-mode attention grid for decode steps that reach position
// `pos_end`: the power of two >= the CTAs the positions need (64 per CTA), so
// a short context does not launch (and wait for) the capacity's 296 CTAs.
// Any grid is correct (the kernel spreads the positions over the CTAs it
// has); graphs are cached per grid.
void Session::size_attn_grid(int pos_end) {
    if (!dm_.fast) return;
    const int need = (pos_end + 1 + 63) / 64;
    int b = 1;
    while (b < need && b < 296) b *= 2;
    dm_.attn_fast_grid = std::min(b, 296);
}

cudaGraphExec_t Session::get_graph(int mode, int stream) {
    if (host_ordered_) return nullptr;  // the step syncs on the host mid-pass: no graphs
    const long long base = mode * 10 + 1 + (stream ? 100 : 0);
    const long long key = base + 1000LL * (dm_.fast ? dm_.attn_fast_grid : 0);
    auto it = graphs_.find(key);
    if (it != graphs_.end()) return it->second;
    sync();
    cudaGraph_t g;
    cudaGraphExec_t exec = nullptr;
    const long long before = launch_counter();
    ck(cudaStreamBeginCapture(s_comp_, cudaStreamCaptureModeThreadLocal), "capture");
    enqueue_step(mode, 0, 1, 0, s_comp_, stream);
    ck(cudaStreamEndCapture(s_comp_, &g), "capture");
    graph_kernels_[base] = static_cast<int>(launch_counter() - before);
    ck(cudaGraphInstantiate(&exec, g, 0), "instantiate");
    cudaGraphDestroy(g);
    graphs_[key] = exec;
    return exec;
}

// Kernels in one captured decode step: the teacher-forced (stream) graph if
// it was built, else the greedy one; -1 before any graph exists.
void Session::path_info(int* out, int cap) const {
    // packed store: blocks packed, and the packed wire bytes per 1000 raw bytes
    long long np = 0, wire = 0, raw = 0;
    if (store_)
        for (long long i = 0; i < store_->blocks(); ++i) {
            np += store_->packed_bytes(i) != 0;
            wire += store_->wire_bytes(i);
            raw += store_->bytes_per_expert();
        }
    const int v[] = {dm_.ffn_fused || (dm_.fast && dm_.ffn_cs_fused), dm_.attn_grid, host_ordered_ ? 1 : 0,
                     ctl_.fast_hit,
                     store_ ? store_->numa_node() : -1, static_cast<int>(np),
                     raw ? static_cast<int>(1000 * wire / raw) : 0,
                     static_cast<int>(xp_unpack_launches() & 0x7fffffff)};
    for (int i = 0; i < cap && i < 8; ++i) out[i] = v[i];
}

int Session::kernels_per_step(int mode) const {
    for (const long long key : {mode * 10 + 1 + 100LL, mode * 10 + 1LL}) {
        auto it = graph_kernels_.find(key);
        if (it != graph_kernels_.end()) return it->second;
    }
    return -1;
}

void Session::clear_stats() {
    sync();
    ck(cudaStreamSynchronize(s_copy_), "copy stream");
    cache_->clear_stats();
    sched_->clear_records();
    direct_bytes_ = 0;
    n_step_events_ = 0;
}

void Session::profile_kernels(int reps, double* out) {
    sync();
    ck(cudaStreamSynchronize(s_copy_), "copy stream");
    const int L = cfg_.L;
    cudaEvent_t a, b;
    ck(cudaEventCreate(&a), "event");
    ck(cudaEventCreate(&b), "event");
    int pos = 0;
    d2h(&pos, st_.pos, 4, "pos");
    size_attn_grid(pos);  // the attention grid a decode step at this position launches
    for (int k = 0; k < 7; ++k) {
        // warm-up pass
        for (int pass = 0; pass < 2; ++pass) {
            if (pass == 1) ck(cudaEventRecord(a, s_comp_), "event");
            const int R = pass == 0 ? 1 : reps;
            for (int r = 0; r < R; ++r)
                for (int l = 0; l < L; ++l) {
                    switch (k) {
                    case 0: ck(launch_qkv(dm_, st_, l, s_comp_), "qkv"); break;
                    case 1: ck(launch_attn(dm_, st_, d_attn_scratch_, l, s_comp_), "attn"); break;
                    case 2: ck(launch_wo(dm_, st_, ctl_, l, s_comp_), "wo"); break;
                    case 3: {
                        RouterLaunch rl{l, 1, kNone, -1, 0, 0, -9, 0};
                        ck(launch_router(dm_, st_, ctl_, rl, nullptr, s_comp_), "router");
                        break;
                    }
                    case 4:
                    case 5: {
                        // one of the two FFN kernels: launch the pair, subtract below
                        ck(launch_ffn(dm_, st_, ctl_, l, s_comp_), "ffn");
                        break;
                    }
                    case 6:
                        if (l == 0) ck(launch_final(dm_, st_, ctl_, 0, s_comp_), "final");
                        break;
                    }
                }
            if (pass == 1) ck(cudaEventRecord(b, s_comp_), "event");
        }
        ck(cudaEventSynchronize(b), "event");
        float ms = 0.0f;
        ck(cudaEventElapsedTime(&ms, a, b), "elapsed");
        const double n = k == 6 ? reps : static_cast<double>(reps) * L;
        out[k] = 1000.0 * ms / n;
    }
    out[7] = out[4];  // the expert FFN as decode launches it (one fused launch when active)
    // split the FFN pair with a gate/up-only and down-only timing
    {
        ck(cudaEventRecord(a, s_comp_), "event");
        for (int r = 0; r < reps; ++r)
            for (int l = 0; l < L; ++l) ck(launch_ffn_part(dm_, st_, ctl_, l, 0, s_comp_), "ffn");
        ck(cudaEventRecord(b, s_comp_), "event");
        ck(cudaEventSynchronize(b), "event");
        float ms = 0.0f;
        ck(cudaEventElapsedTime(&ms, a, b), "elapsed");
        out[4] = 1000.0 * ms / (static_cast<double>(reps) * L);
        ck(cudaEventRecord(a, s_comp_), "event");
        for (int r = 0; r < reps; ++r)
            for (int l = 0; l < L; ++l) ck(launch_ffn_part(dm_, st_, ctl_, l, 1, s_comp_), "ffn");
        ck(cudaEventRecord(b, s_comp_), "event");
        ck(cudaEventSynchronize(b), "event");
        ck(cudaEventElapsedTime(&ms, a, b), "elapsed");
        out[5] = 1000.0 * ms / (static_cast<double>(reps) * L);
        // k_ffn_gu in the prefetch form (layers >= 1 of a prefetch pass); the
        // predicted decisions of the last prefetch pass are resident
        out[8] = out[4];
        if (L > 1) {
            ck(launch_mark_decided(st_, L, s_comp_), "mark");
            for (int l = 1; l < L; ++l) ck(launch_ffn_part(dm_, st_, ctl_, l, 2, s_comp_), "ffn");
            ck(cudaEventRecord(a, s_comp_), "event");
            for (int r = 0; r < reps; ++r)
                for (int l = 1; l < L; ++l) ck(launch_ffn_part(dm_, st_, ctl_, l, 2, s_comp_), "ffn");
            ck(cudaEventRecord(b, s_comp_), "event");
            ck(cudaEventSynchronize(b), "event");
            ck(cudaEventElapsedTime(&ms, a, b), "elapsed");
            out[8] = 1000.0 * ms / (static_cast<double>(reps) * (L - 1));
        }
    }
    dm_.attn_fast_grid = 0;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    sync();
}

double Session::measure_link(int n_copies) {
    sync();
    ck(cudaStreamSynchronize(s_copy_), "copy stream");
    const long long bytes = store_->bytes_per_expert();
    void* scratch = nullptr;
    ck(cudaMalloc(&scratch, bytes), "scratch");
    cudaEvent_t a, b;
    ck(cudaEventCreate(&a), "event");
    ck(cudaEventCreate(&b), "event");
    const long long nexp = static_cast<long long>(cfg_.L) * el_max_;
    for (int i = 0; i < 4; ++i)
        ck(cudaMemcpyAsync(scratch, store_->expert(i % nexp), bytes, cudaMemcpyHostToDevice, s_copy_), "warm");
    ck(cudaEventRecord(a, s_copy_), "event");
    for (int i = 0; i < n_copies; ++i)
        ck(cudaMemcpyAsync(scratch, store_->expert((7919LL * i) % nexp), bytes, cudaMemcpyHostToDevice,
                           s_copy_),
           "link copy");
    ck(cudaEventRecord(b, s_copy_), "event");
    ck(cudaEventSynchronize(b), "event");
    float ms = 0.0f;
    ck(cudaEventElapsedTime(&ms, a, b), "elapsed");
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(scratch);
    return static_cast<double>(bytes) * n_copies / (ms * 1e-3) / 1e9;
}

// Diagnostics: [req_counter, error, host next_seq, n_records, polls, mailbox seq of
// the next slot, then ready[0..L), req_seq[0..L)].
void Session::debug_state(int* out, int cap) {
    std::vector<int> v;
    int x = 0;
    cudaStreamSynchronize(s_comp_);
    cudaMemcpy(&x, ctl_.req_counter, 4, cudaMemcpyDeviceToHost);
    v.push_back(x);
    cudaMemcpy(&x, ctl_.error, 4, cudaMemcpyDeviceToHost);
    v.push_back(x);
    v.push_back(sched_->next_seq());
    v.push_back(static_cast<int>(sched_->records().size()));
    v.push_back(static_cast<int>(sched_->polls));
    v.push_back(static_cast<int>(h_mailbox_[sched_->next_seq() % kMailboxRing].seq));
    std::vector<int> r(cfg_.L), q(cfg_.L);
    cudaMemcpy(r.data(), ctl_.ready, 4 * cfg_.L, cudaMemcpyDeviceToHost);
    cudaMemcpy(q.data(), ctl_.req_seq, 4 * cfg_.L, cudaMemcpyDeviceToHost);
    v.insert(v.end(), r.begin(), r.end());
    v.insert(v.end(), q.begin(), q.end());
    for (int i = 0; i < cap && i < static_cast<int>(v.size()); ++i) out[i] = v[i];
}

void Session::read_tokens(int* out, int n) {
    sync();
    d2h(out, ctl_.tokens_out, 4ull * n, "tokens");
}

void Session::read_trace(const char* field, void* out, long long n) {
    sync();
    const std::string f = field;
    const void* src = nullptr;
    long long esz = 4;
    if (f == "tok_in") src = tr_.tok_in;
    else if (f == "id_true") src = tr_.id_true;
    else if (f == "id_exec") src = tr_.id_exec;
    else if (f == "id_pred") src = tr_.id_pred;
    else if (f == "g_true") src = tr_.g_true;
    else if (f == "g_exec") src = tr_.g_exec;
    else if (f == "g_pred") src = tr_.g_pred;
    else if (f == "s") src = tr_.s;
    else if (f == "r") src = tr_.r;
    else if (f == "m") src = tr_.m;
    else if (f == "lg_true") src = tr_.lg_true;
    else if (f == "lg_pred") src = tr_.lg_pred;
    else if (f == "y") src = tr_.y;
    else if (f == "logits") src = tr_.logits;
    else throw std::invalid_argument("read_trace: unknown field " + f);
    if (!src) throw std::invalid_argument("read_trace: field not captured (trace_full=0?)");
    d2h(out, src, n * esz, "trace");
}

void Session::build_distill_dataset(int first, int n, int mode, float* inputs, float* targets) {
    sync();
    if (!trace_full_ || !tr_.s) throw std::invalid_argument("distill dataset: needs reset(trace_full=1)");
    if (cfg_.L < 2) throw std::invalid_argument("distill dataset: need at least 2 layers");
    if (mode != 0 && mode != 1) throw std::invalid_argument("distill dataset: mode must be 0 (quasi) or 1 (s-next)");
    if (mode == 0 && !have_dv_) throw std::invalid_argument("distill dataset: quasi-hidden inputs need a table");
    if (n < 1 || first < 0 || first + n > tr_.cap) throw std::invalid_argument("distill dataset: steps out of range");
    const size_t ns = static_cast<size_t>(n) * (cfg_.L - 1);
    float *di = nullptr, *dt = nullptr;
    ck(cudaMalloc(&di, ns * cfg_.H * 4), "distill alloc");
    ck(cudaMalloc(&dt, ns * cfg_.E * 4), "distill alloc");
    cudaError_t err = launch_distill(dm_, tr_, first, n, mode, di, dt, s_comp_);
    if (err == cudaSuccess) err = cudaMemcpyAsync(inputs, di, ns * cfg_.H * 4, cudaMemcpyDeviceToHost, s_comp_);
    if (err == cudaSuccess) err = cudaMemcpyAsync(targets, dt, ns * cfg_.E * 4, cudaMemcpyDeviceToHost, s_comp_);
    if (err == cudaSuccess) err = cudaStreamSynchronize(s_comp_);
    cudaFree(di);
    cudaFree(dt);
    ck(err, "distill dataset");
}

void Session::predict_ahead(int first, int n, int depth, int* ids) {
    sync();
    if (!trace_full_ || !tr_.s) throw std::invalid_argument("predict_ahead: needs reset(trace_full=1)");
    if (!have_dv_) throw std::invalid_argument("predict_ahead: quasi-hidden inputs need a table");
    if (depth < 1 || depth >= cfg_.L) throw std::invalid_argument("predict_ahead: depth must be in [1, L)");
    if (n < 1 || first < 0 || first + n > tr_.cap) throw std::invalid_argument("predict_ahead: steps out of range");
    const size_t cnt = static_cast<size_t>(n) * cfg_.L * cfg_.K;
    int* d = nullptr;
    ck(cudaMalloc(&d, cnt * 4), "predict_ahead alloc");
    cudaError_t err = cudaMemsetAsync(d, 0xff, cnt * 4, s_comp_);
    if (err == cudaSuccess) err = launch_pred_ahead(dm_, tr_, first, n, depth, d, s_comp_);
    if (err == cudaSuccess) err = cudaMemcpyAsync(ids, d, cnt * 4, cudaMemcpyDeviceToHost, s_comp_);
    if (err == cudaSuccess) err = cudaStreamSynchronize(s_comp_);
    cudaFree(d);
    ck(err, "predict_ahead");
}

// ---- trace bundles in the reference's format (trace.cpp:60-122, moet.cpp) ----
namespace {
void moet_write(const std::string& path, const std::vector<unsigned long long>& dims,
                const std::vector<float>& data) {
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error("trace: cannot write " + path);
    unsigned char hdr[10] = {'M', 'O', 'E', 'T', 1, 0, 0, 0, 1, static_cast<unsigned char>(dims.size())};
    bool ok = std::fwrite(hdr, 1, 10, f) == 10;
    for (unsigned long long d : dims) {
        unsigned char b[8];
        for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>(d >> (8 * i));
        ok = ok && std::fwrite(b, 1, 8, f) == 8;
    }
    // little-endian host: the f32 payload is written as is (moet.cpp:9-13)
    ok = ok && std::fwrite(data.data(), 4, data.size(), f) == data.size();
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw std::runtime_error("trace: short write to " + path);
}
std::string json_str(const std::string& s) {
    std::string o = "\"";
    for (char ch : s) {
        if (ch == '"' || ch == '\\') o += '\\';
        o += ch;
    }
    return o + "\"";
}
}  // namespace

void Session::write_trace_bundle(const std::string& dir, int first, int n, int seq_len,
                                 const std::string& source, unsigned long long seed) {
    sync();
    if (!trace_full_ || !tr_.s) throw std::invalid_argument("write_trace_bundle: needs reset(trace_full=1)");
    if (n < 1 || first < 0 || first + n > tr_.cap) throw std::invalid_argument("trace: empty workload");
    const ModelCfg& c = cfg_;
    const long long N = n, L = c.L, H = c.H, E = c.E, K = c.K;
    auto rd = [&](const char* field, long long per, bool ints) {
        std::vector<float> out(static_cast<size_t>(N * per));
        if (ints) {
            std::vector<int> v(static_cast<size_t>(N * per));
            std::vector<int> all(static_cast<size_t>((first + N) * per));
            read_trace(field, all.data(), static_cast<long long>(all.size()));
            for (size_t i = 0; i < v.size(); ++i) out[i] = static_cast<float>(all[first * per + i]);
        } else {
            std::vector<float> all(static_cast<size_t>((first + N) * per));
            read_trace(field, all.data(), static_cast<long long>(all.size()));
            std::copy(all.begin() + first * per, all.end(), out.begin());
        }
        return out;
    };
    if (::mkdir(dir.c_str(), 0755) != 0 && errno != EEXIST)
        throw std::runtime_error("trace: cannot create " + dir);
    const unsigned long long n_ = N, L_ = L, H_ = H, E_ = E, K_ = K;
    moet_write(dir + "/token_ids.moet", {n_}, rd("tok_in", 1, true));
    moet_write(dir + "/s.moet", {n_, L_, H_}, rd("s", L * H, false));
    moet_write(dir + "/r.moet", {n_, L_, H_}, rd("r", L * H, false));
    moet_write(dir + "/m.moet", {n_, L_, H_}, rd("m", L * H, false));
    moet_write(dir + "/router_logits.moet", {n_, L_, E_}, rd("lg_true", L * E, false));
    moet_write(dir + "/expert_ids.moet", {n_, L_, K_}, rd("id_exec", L * K, true));
    moet_write(dir + "/expert_gates.moet", {n_, L_, K_}, rd("g_exec", L * K, false));
    moet_write(dir + "/expert_outputs.moet", {n_, L_, K_, H_}, rd("y", L * K * H, false));
    // manifest.json (trace.cpp:19-41; keys in nlohmann's sorted order)
    char eps[64];  // shortest round-trip form of double(eps), as nlohmann prints it
    {
        const auto res = std::to_chars(eps, eps + sizeof eps - 1, static_cast<double>(c.eps));
        *res.ptr = 0;
    }
    std::string j = "{\n  \"config\": {\n";
    j += "    \"eps\": " + std::string(eps) + ",\n";
    j += "    \"expert_hidden\": " + std::to_string(c.Hm) + ",\n";
    j += "    \"experts\": " + std::to_string(c.E) + ",\n";
    j += "    \"gating\": " + json_str(c.gating == kTopKSoftmax ? "topk-softmax" : "softmax-topk-renorm") + ",\n";
    j += "    \"head_dim\": " + std::to_string(c.D) + ",\n";
    j += "    \"hidden\": " + std::to_string(c.H) + ",\n";
    j += "    \"layers\": " + std::to_string(c.L) + ",\n";
    j += "    \"seed\": " + std::to_string(c.seed) + ",\n";
    j += "    \"top_k\": " + std::to_string(c.K) + ",\n";
    j += "    \"vocab\": " + std::to_string(c.V) + "\n  },\n  \"fields\": [\n";
    const std::vector<std::pair<std::string, std::vector<unsigned long long>>> shapes = {
        {"token_ids", {n_}}, {"s", {n_, L_, H_}}, {"r", {n_, L_, H_}}, {"m", {n_, L_, H_}},
        {"router_logits", {n_, L_, E_}}, {"expert_ids", {n_, L_, K_}},
        {"expert_gates", {n_, L_, K_}}, {"expert_outputs", {n_, L_, K_, H_}}};
    for (size_t f = 0; f < shapes.size(); ++f) {
        j += "    {\n      \"dims\": [";
        for (size_t d = 0; d < shapes[f].second.size(); ++d)
            j += (d ? "," : "") + std::to_string(shapes[f].second[d]);
        j += "],\n      \"name\": " + json_str(shapes[f].first) + "\n    }" + (f + 1 < shapes.size() ? "," : "") + "\n";
    }
    j += "  ],\n  \"seed\": " + std::to_string(seed) + ",\n  \"seq_len\": " + std::to_string(seq_len) +
         ",\n  \"source\": " + json_str(source) + ",\n  \"tokens\": " + std::to_string(N) + "\n}\n";
    FILE* f = std::fopen((dir + "/manifest.json").c_str(), "w");
    if (!f) throw std::runtime_error("trace: cannot write manifest");
    std::fputs(j.c_str(), f);
    std::fclose(f);
}

std::vector<double> Session::token_ms() {
    sync();
    std::vector<double> v;
    for (int i = 0; i < n_step_events_; ++i) {
        float ms = 0.0f;
        ck(cudaEventElapsedTime(&ms, ev_step_[2 * i], ev_step_[2 * i + 1]), "elapsed");
        v.push_back(ms);
    }
    return v;
}

double Session::step_event_ms(int i, int which) {
    float ms = 0.0f;
    ck(cudaEventElapsedTime(&ms, ev_origin_, ev_step_[2 * i + which]), "elapsed");
    return ms;
}

double Session::event_ms(int ev, int which) {
    float ms = 0.0f;
    ck(cudaEventElapsedTime(&ms, ev_origin_, ev_copy_[2 * ev + which]), "elapsed");
    return ms;
}

void Session::counters(long long* hits, long long* misses, long long* bytes, double* copy_ms,
                       int* requests) {
    sync();
    ck(cudaStreamSynchronize(s_copy_), "copy stream");
    for (int l = 0; l < cfg_.L; ++l) {
        if (hits) hits[l] = cache_->hits(l);
        if (misses) misses[l] = cache_->misses(l);
    }
    long long b = 0;
    double ms = 0.0;
    auto recs = sched_->records();
    for (const CopyRecord& r : recs) {
        b += r.bytes;
        if (r.ev >= 0 && r.bytes > 0) {
            float t = 0.0f;
            if (cudaEventElapsedTime(&t, ev_copy_[2 * r.ev], ev_copy_[2 * r.ev + 1]) == cudaSuccess) ms += t;
        }
    }
    if (bytes) *bytes = b + direct_bytes_.load();  // + host-driven (batched) copies
    if (copy_ms) *copy_ms = ms;
    if (requests) *requests = static_cast<int>(recs.size());
}

}  // namespace smoe
