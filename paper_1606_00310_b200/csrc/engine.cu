// Host side of liboctgpu: the C-ABI (include/octgpu.h), engine state,
// parameter resolution, stream seeding and GF(2) jump-ahead matrices.
// Device work lives in kernels.cu.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <limits>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "octgpu.h"
#include "octgpu_internal.h"

using namespace octgpu;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(OCTGPU_ERR_CUDA, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

#define CK(x)                                         \
    do {                                              \
        cudaError_t e_ = (x);                         \
        if (e_ != cudaSuccess) return cuda_fail(e_, #x); \
    } while (0)

// ---------------------------------------------------------------------------
// xoshiro256++ on the host (rng.hpp:25-60)

inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

inline void xo_advance(uint64_t s[4]) {
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
}

uint64_t splitmix64(uint64_t& x) {
    uint64_t z = (x += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// ---------------------------------------------------------------------------
// GF(2) 256x256 matrices: the xoshiro state transition is linear, so
// advancing a stream by N draws is s -> T^N s. Column j = image of bit j.

struct M256 {
    uint64_t c[256][4];
};

inline void mat_vec(const M256& M, const uint64_t v[4], uint64_t out[4]) {
    uint64_t r[4] = {0, 0, 0, 0};
    for (int w = 0; w < 4; ++w) {
        uint64_t bits = v[w];
        while (bits) {
            const int b = __builtin_ctzll(bits);
            bits &= bits - 1;
            const uint64_t* col = M.c[w * 64 + b];
            r[0] ^= col[0];
            r[1] ^= col[1];
            r[2] ^= col[2];
            r[3] ^= col[3];
        }
    }
    std::memcpy(out, r, sizeof r);
}

void mat_mul(const M256& A, const M256& B, M256& out) {  // out = A * B
    M256 tmp;
    for (int j = 0; j < 256; ++j) mat_vec(A, B.c[j], tmp.c[j]);
    out = tmp;
}

struct JumpCache {
    std::mutex mu;
    std::vector<M256> pow2;  // pow2[i] = T^(2^i)
    bool have_jump = false;
    std::vector<uint64_t> jump_table;  // 4-bit table of T^(2^128), for seeding

    const M256& pow(int i) {
        if (pow2.empty()) {
            M256 T;
            for (int j = 0; j < 256; ++j) {
                uint64_t s[4] = {0, 0, 0, 0};
                s[j / 64] = uint64_t(1) << (j % 64);
                xo_advance(s);
                std::memcpy(T.c[j], s, sizeof s);
            }
            pow2.push_back(T);
        }
        while (int(pow2.size()) <= i) {
            M256 sq;
            mat_mul(pow2.back(), pow2.back(), sq);
            pow2.push_back(sq);
        }
        return pow2[i];
    }

    // T^N for a 64-bit N
    M256 power(uint64_t N) {
        M256 R;
        std::memset(&R, 0, sizeof R);
        for (int j = 0; j < 256; ++j) R.c[j][j / 64] = uint64_t(1) << (j % 64);
        for (int i = 0; i < 64; ++i)
            if (N >> i & 1) mat_mul(pow(i), R, R);
        return R;
    }
};

JumpCache& jc() {
    static JumpCache c;
    return c;
}

// 4-bit table: tab[(i*16 + nib)*4 + w] = (XOR of columns 4i+b, b in nib)[w]
std::vector<uint64_t> table_of(const M256& M) {
    std::vector<uint64_t> tab(64 * 16 * 4, 0);
    for (int i = 0; i < 64; ++i)
        for (int nib = 1; nib < 16; ++nib) {
            uint64_t* e = &tab[(size_t(i) * 16 + nib) * 4];
            for (int b = 0; b < 4; ++b)
                if (nib >> b & 1)
                    for (int w = 0; w < 4; ++w) e[w] ^= M.c[4 * i + b][w];
        }
    return tab;
}

inline void table_apply(const std::vector<uint64_t>& tab, uint64_t s[4]) {
    uint64_t r[4] = {0, 0, 0, 0};
    for (int i = 0; i < 64; ++i) {
        const uint32_t nib = uint32_t(s[i >> 4] >> (4 * (i & 15))) & 15u;
        const uint64_t* e = &tab[(size_t(i) * 16 + nib) * 4];
        r[0] ^= e[0]; r[1] ^= e[1]; r[2] ^= e[2]; r[3] ^= e[3];
    }
    std::memcpy(s, r, sizeof r);
}

const std::vector<uint64_t>& seed_jump_table() {
    JumpCache& c = jc();
    std::lock_guard<std::mutex> lk(c.mu);
    if (!c.have_jump) {
        c.jump_table = table_of(c.pow(128));  // RngStream::jump() == 2^128 draws (rng.hpp:46)
        c.have_jump = true;
    }
    return c.jump_table;
}

std::vector<uint64_t> power_table(uint64_t N) {
    JumpCache& c = jc();
    std::lock_guard<std::mutex> lk(c.mu);
    return table_of(c.power(N));
}

// RngStreamSet(master_seed, n) (rng.hpp:84-94): stream i = i jumps from from_seed.
void stream_states(uint64_t seed, uint32_t n, uint64_t* out) {
    uint64_t s[4];
    for (auto& v : s) v = splitmix64(seed);
    if ((s[0] | s[1] | s[2] | s[3]) == 0) s[0] = 1;
    const auto& tab = seed_jump_table();
    for (uint32_t i = 0; i < n; ++i) {
        std::memcpy(out + 4 * size_t(i), s, sizeof s);
        if (i + 1 < n) table_apply(tab, s);
    }
}

// ---------------------------------------------------------------------------
// Parameter resolution (params.hpp:34-80, rng.cpp:7-30)

bool dyadic_plan(double r, uint32_t max_words, uint32_t& k, uint64_t& m) {
    if (!(r > 0.0 && r < 1.0)) return false;
    const double scaled = std::ldexp(r, int(max_words));
    if (scaled != std::floor(scaled)) return false;
    m = uint64_t(scaled);
    k = max_words;
    while (k > 0 && (m & 1) == 0) {
        m >>= 1;
        --k;
    }
    return true;
}

std::string fmt_r(double r) {
    return std::to_string(r);  // std::to_string as the reference message (params.hpp:36)
}

int resolve(double r, int forced, octgpu_prob& o) {
    if (r < 0.0 || r > 1.0) return fail(OCTGPU_ERR_CONFIG, "probability must be in [0,1], got " + fmt_r(r));
    o.value = r;
    o.k = 0;
    o.m = 0;
    if (r == 0.0)
        o.mode = OCTGPU_ZERO;
    else if (r == 0.5)
        o.mode = OCTGPU_HALF;
    else if (dyadic_plan(r, 16, o.k, o.m))
        o.mode = OCTGPU_DYADIC;
    else
        o.mode = OCTGPU_ARBITRARY;
    if (forced < 0 || forced == o.mode) return OCTGPU_OK;
    switch (forced) {
    case OCTGPU_ZERO:
        if (r != 0.0) return fail(OCTGPU_ERR_CONFIG, "mode zero requires probability 0");
        break;
    case OCTGPU_HALF:
        if (r != 0.5) return fail(OCTGPU_ERR_CONFIG, "mode half requires probability 0.5");
        break;
    case OCTGPU_DYADIC:
        if (dyadic_plan(r, 16, o.k, o.m)) {
            o.mode = OCTGPU_DYADIC;
            return OCTGPU_OK;
        }
        return fail(OCTGPU_ERR_CONFIG, "probability has no dyadic plan within 16 words");
    case OCTGPU_ARBITRARY:
        if (r == 0.0) return fail(OCTGPU_ERR_CONFIG, "mode arbitrary is pointless for probability 0; use zero");
        o.mode = OCTGPU_ARBITRARY;
        o.k = 0;
        o.m = 0;
        return OCTGPU_OK;
    default:
        return fail(OCTGPU_ERR_CONFIG, "unknown probability mode " + std::to_string(forced));
    }
    return OCTGPU_OK;
}

uint32_t draws(const octgpu_prob& p, uint32_t w) {
    switch (p.mode) {
    case OCTGPU_ZERO: return 0;
    case OCTGPU_HALF: return 1;
    case OCTGPU_DYADIC: return p.k;
    default: return w;
    }
}

// Checks a caller-supplied ProbSpec and lowers it to the device form.
int lower(const octgpu_prob& p, ProbDev& d) {
    d = ProbDev{M_ZERO, 0, 0, 0};
    const double r = p.value;
    if (!(r >= 0.0 && r <= 1.0)) return fail(OCTGPU_ERR_CONFIG, "probability must be in [0,1], got " + fmt_r(r));
    switch (p.mode) {
    case OCTGPU_ZERO:
        if (r != 0.0) return fail(OCTGPU_ERR_CONFIG, "mode zero requires probability 0");
        d.mode = M_ZERO;
        return OCTGPU_OK;
    case OCTGPU_HALF:
        if (r != 0.5) return fail(OCTGPU_ERR_CONFIG, "mode half requires probability 0.5");
        d.mode = M_HALF;
        return OCTGPU_OK;
    case OCTGPU_DYADIC: {
        if (p.k < 1 || p.k > 64 || (p.m & 1) == 0 || std::ldexp(double(p.m), -int(p.k)) != r)
            return fail(OCTGPU_ERR_CONFIG, "inconsistent dyadic plan");
        d.mode = M_DYADIC;
        d.k = p.k;
        d.m = p.m;
        return OCTGPU_OK;
    }
    case OCTGPU_ARBITRARY: {
        if (r == 0.0) return fail(OCTGPU_ERR_CONFIG, "mode arbitrary is pointless for probability 0; use zero");
        // to_unit(x) < r  <=>  (x >> 11) < ceil(r * 2^53)  <=>  x < ceil(r * 2^53) << 11
        const double scaled = std::ldexp(r, 53);  // exact
        const uint64_t thr = uint64_t(std::ceil(scaled));
        if (thr >= (uint64_t(1) << 53)) {
            d.mode = M_ONE;  // r == 1: all bits accepted
        } else {
            d.mode = M_ARB;
            d.T = thr << 11;
        }
        return OCTGPU_OK;
    }
    default:
        return fail(OCTGPU_ERR_CONFIG, "unknown probability mode " + std::to_string(p.mode));
    }
}

inline bool is_const(const ProbDev& d) { return d.mode == M_ZERO || d.mode == M_ONE; }

int validate(uint32_t X, uint32_t Y, uint32_t w) {  // lattice.hpp:31-39
    if (w != 32 && w != 64) return fail(OCTGPU_ERR_CONFIG, "word size must be 32 or 64, got " + std::to_string(w));
    if (X == 0 || X % (2 * w) != 0)
        return fail(OCTGPU_ERR_CONFIG, "X must be a positive multiple of 2*w = " + std::to_string(2 * w) +
                                           ", got " + std::to_string(X));
    if (Y < 2 || Y % 2 != 0) return fail(OCTGPU_ERR_CONFIG, "Y must be even and >= 2, got " + std::to_string(Y));
    return OCTGPU_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// Engine

struct octgpu_engine {
    uint32_t X = 0, Y = 0, w = 64, n = 0;
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    void* planes[2] = {nullptr, nullptr};  // ping-pong plane sets (word-major)
    uint64_t* rng[2] = {nullptr, nullptr};  // ping-pong SoA row states
    int pcur = 0;  // current plane set
    int rcur = 0;  // current rng state set
    uint64_t t = 0;
    int phase = 0;
    uint64_t master_seed = 0;
    uint64_t pending = 0;  // draws owed to every row stream (constant-xi sweeps)
    void* stage = nullptr;  // reference-layout staging buffer
    void* scratch = nullptr;
    MeasureResult* res_dev = nullptr;
    MeasureResult* res_host = nullptr;
    std::map<uint64_t, uint64_t*> jtabs;  // draws per sweep -> device 4-bit table of T^draws
    uint64_t* pend_tab = nullptr;          // table of T^pending (materialize), device
    uint64_t* pend_host = nullptr;         // ... and its pinned upload buffer
    cudaEvent_t pend_ev = nullptr;         // the last jump that read them
    uint64_t launches = 0;
    // fused-MCS implementation: 2 = bulk-copy staged (k_mcs_bulk), 1 = register-prefetch (k_mcs)
    int mcs_impl = 2;
    int bulk_ks = 2, bulk_S = 2;
    int bulk_key = -1;  // (p, q) mode pair the bulk plan was made for
    CUtensorMap tm[2][2];  // [plane set][box: ks words, ks+1 words] for k_mcs_bulk
    int tm_ks = -1;
    CUtensorMap tmd[2][2];  // the same for k_mcs_deep (deep_box_rows rows x 2 / 3 words)
    bool tmd_ok = false;
    int deep = 1;  // temporally blocked passes (k_mcs_deep) where supported; OCTGPU_DEEP=0 disables
    // multi-MCS peer-memory stripe passes fused with their halo exchange: -1 = when a neighbour is on another
    // device (decided at connect), 0 / 1 = OCTGPU_FUSED_LINK
    int fused_link = -1, fused_link_env = -1;
    bool ghost_kernel = true;  // deep passes' ghost-row mirror: a copy kernel (OCTGPU_GHOST=memcpy: cudaMemcpy2DAsync)
    bool deep_long = true;  // 4-MCS passes for remainders of 3-MCS schedules (OCTGPU_DEEP_LONG=0: 2 / 1-MCS passes)
    int deep_l = kDeepSweepsConst;  // sweeps of a constant-xi deep pass (OCTGPU_DEEP_L = 4 keeps 2 MCS per pass)
    bool graphs = true;  // replay CUDA graphs for long step() calls (OCTGPU_GRAPH=0 disables)
    uint32_t prefetch = 0;  // TMA kernels: L2 prefetch distance in ring stages (OCTGPU_PREFETCH)
    long long p2p_timeout = kP2PTimeoutCycles;  // peer halo wait limit (OCTGPU_P2P_TIMEOUT_MS)
    int rng_kind = OCTGPU_RNG_XOSHIRO;  // octgpu_set_rng
    uint64_t tile_shift = 0;  // != 0: random per-pass row origin of the block tiling (DTr-style, result-neutral)
    std::map<std::string, std::pair<cudaGraphExec_t, uint64_t>> graph_cache;  // exec, kernels per replay
    int deep_S = 5;    // k_mcs_deep ring stages (OCTGPU_DEEP_S): with one word per stage (kDeepKS) S = 5 measured best
    // Row-stripe mode (multi-GPU): this engine owns global rows [y0, y0 + L) of
    // a Ytot-row periodic lattice, held at local rows 1..L with one halo row
    // above (0), two below (L+1, L+2) and padding; Y is then the allocated row
    // count. Periodic mode: Y = Ytot, y0 = 0, L = Ytot.
    bool stripe = false;
    bool pooled = false;  // plane sets from the device's stream-ordered memory pool
    uint32_t Ytot = 0, y0 = 0, L = 0;
    // device-side P2P halo exchange (p2p.cu): passes completed (device counter,
    // exposed to the neighbours), timeout flag, and the neighbours' memory
    uint64_t* done = nullptr;
    uint32_t* p2p_err = nullptr;
    uint64_t passes = 0;
    bool p2p = false;
    octgpu_peer prev{}, next{};
    std::vector<void*> ipc_opened;  // peer allocations mapped with cudaIpcOpenMemHandle

    // k_mcs_deep (ls sweeps per pass): the same periodic lattice with core rows starting at virtual row ls - 1
    Geom deep_geom(int ls) const { return Geom{Y, n, size_t(n) * Y, uint32_t(ls - 1), L + uint32_t(ls - 1), L, 0, kGhostRows}; }
    Geom geom() const {
        // stripe: local row 0 = global y0 - kStripeHA (parity of y0 + 1)
        if (!stripe) return Geom{Y, n, size_t(n) * Y, 1, L + 1, L, 0, kGhostRows};
        Geom g{Y, n, size_t(n) * Y, kStripeHA, kStripeHA + L, 0, (y0 + 1) & 1u, 0};
        g.gy0 = (y0 + Ytot - kStripeHA % Ytot) % Ytot;
        g.gytot = Ytot;
        return g;
    }
    uint32_t core_rows() const { return L; }
    // rows of the reference-layout staging buffer: the lattice rows (periodic) or
    // every allocated row (stripe; the host slices rows 1..L)
    uint32_t host_rows() const { return stripe ? Y : L; }
    size_t host_bytes() const { return 4 * size_t(n) * host_rows() * word_bytes(); }
    uint32_t first_row() const { return stripe ? kStripeHA : 0; }  // local index of the first core row
    size_t word_bytes() const { return w / 8; }
    size_t set_bytes() const { return 4 * size_t(n) * Y * word_bytes(); }
    size_t rng_bytes() const { return 4 * size_t(Y) * sizeof(uint64_t); }
};

namespace {

int use_device(octgpu_engine* e) {
    CK(cudaSetDevice(e->device));
    return OCTGPU_OK;
}

// Reference-layout staging buffer for import / export transposes. A periodic
// engine uses its idle ping-pong plane set (the next MCS rewrites every row of
// it), saving a 1-GiB allocation at 2^16^2; a stripe keeps its own buffer,
// since a neighbour may push its boundary row into the idle set at any time
// (p2p.cu).
int ensure_stage(octgpu_engine* e, void** out) {
    if (!e->stripe) {
        *out = e->planes[e->pcur ^ 1];
        return OCTGPU_OK;
    }
    if (!e->stage) CK(cudaMalloc(&e->stage, e->set_bytes()));
    *out = e->stage;
    return OCTGPU_OK;
}

int get_table(octgpu_engine* e, uint64_t draws_n, uint64_t** out) {
    auto it = e->jtabs.find(draws_n);
    if (it != e->jtabs.end()) {
        *out = it->second;
        return OCTGPU_OK;
    }
    std::vector<uint64_t> tab = power_table(draws_n);
    uint64_t* d = nullptr;
    CK(cudaMalloc(&d, tab.size() * sizeof(uint64_t)));
    CK(cudaMemcpy(d, tab.data(), tab.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
    e->jtabs[draws_n] = d;
    *out = d;
    return OCTGPU_OK;
}

void trace_create(const char* what, bool start);

// Apply owed draws to every row stream (lazy advance of constant-xi sweeps). The table of T^pending is
// not cached (every pending count is different): it goes through one engine-owned pinned + device buffer
// pair, reused once the previous jump that read it has completed (pend_ev).
int dev_alloc(octgpu_engine* e, void** out, size_t bytes);
cudaError_t host_pinned(void** out, size_t bytes);
constexpr size_t kPendTabBytes = size_t(64) * 16 * 4 * sizeof(uint64_t);

int materialize(octgpu_engine* e) {
    if (!e->pending) return OCTGPU_OK;
    const size_t bytes = kPendTabBytes;
    if (!e->pend_tab) {
        int rc = dev_alloc(e, reinterpret_cast<void**>(&e->pend_tab), bytes);
        if (rc) return rc;
        CK(host_pinned(reinterpret_cast<void**>(&e->pend_host), bytes));
        CK(cudaEventCreateWithFlags(&e->pend_ev, cudaEventDisableTiming));
    } else {
        CK(cudaEventSynchronize(e->pend_ev));
    }
    trace_create("mat-alloc", false);
    const std::vector<uint64_t> tab = power_table(e->pending);
    trace_create("mat-power", false);
    std::memcpy(e->pend_host, tab.data(), bytes);
    CK(cudaMemcpyAsync(e->pend_tab, e->pend_host, bytes, cudaMemcpyHostToDevice, e->stream));
    CK(launch_apply_jump(e->rng[e->rcur], e->Y, e->pend_tab, e->stream));
    CK(cudaEventRecord(e->pend_ev, e->stream));
    ++e->launches;
    e->pending = 0;
    return OCTGPU_OK;
}

// AoS states of the core rows -> SoA at local rows first_row().. (stride Y)
int upload_states(octgpu_engine* e, const uint64_t* aos) {
    std::vector<uint64_t> soa(4 * size_t(e->Y), 0);
    const uint32_t r0 = e->first_row();
    for (uint32_t y = 0; y < e->core_rows(); ++y)
        for (int j = 0; j < 4; ++j) soa[size_t(j) * e->Y + r0 + y] = aos[4 * size_t(y) + j];
    CK(cudaMemcpyAsync(e->rng[e->rcur], soa.data(), e->rng_bytes(), cudaMemcpyHostToDevice, e->stream));
    if (!e->stripe) {
        CK(launch_refresh_ghosts(e->w, e->planes[e->pcur], e->rng[e->rcur], e->geom(), e->stream));
        ++e->launches;
    }
    CK(cudaStreamSynchronize(e->stream));
    trace_create("states", false);
    return OCTGPU_OK;
}

// Pick the fused-MCS variant: k_mcs_bulk (TMA-staged, warp-specialised) for
// w = 64 lattices with n >= 8 words and, when periodic, at least kGhostRows
// rows; k_mcs (register prefetch) otherwise.
int plan_mcs(octgpu_engine* e) {
    e->mcs_impl = (e->w == 64 && e->n >= 8 && (e->stripe || e->L >= kGhostRows)) ? 2 : 1;
    if (const char* v = getenv("OCTGPU_MCS_IMPL")) e->mcs_impl = (atoi(v) == 1) ? 1 : e->mcs_impl;
    if (const char* v = getenv("OCTGPU_DEEP")) e->deep = atoi(v);
    if (const char* v = getenv("OCTGPU_GRAPH")) e->graphs = atoi(v) != 0;
    if (const char* v = getenv("OCTGPU_TILE_SHIFT")) e->tile_shift = strtoull(v, nullptr, 10);
    if (const char* v = getenv("OCTGPU_P2P_TIMEOUT_MS")) e->p2p_timeout = std::max(1LL, atoll(v)) * 2'000'000LL;
    if (const char* v = getenv("OCTGPU_PREFETCH")) e->prefetch = uint32_t(std::max(0, std::min(64, atoi(v))));
    if (const char* v = getenv("OCTGPU_DEEP_S")) e->deep_S = std::max(2, std::min(8, atoi(v)));
    if (const char* v = getenv("OCTGPU_FUSED_LINK")) e->fused_link = e->fused_link_env = atoi(v) != 0 ? 1 : 0;
    if (const char* v = getenv("OCTGPU_DEEP_LONG")) e->deep_long = atoi(v) != 0;
    if (const char* v = getenv("OCTGPU_GHOST")) e->ghost_kernel = std::string(v) != "memcpy";
    if (const char* v = getenv("OCTGPU_DEEP_L")) e->deep_l = atoi(v) == kDeepSweepsLive ? kDeepSweepsLive : kDeepSweepsConst;
    return OCTGPU_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

// 3-D view of a plane set: dim 0 = rows (contiguous, Y allocated rows), dim 1 =
// words (stride Y*8 B), dim 2 = planes (stride n*Y*8 B); tiles of kTmaBoxRows rows x
// (ks | ks+1) words x 1 plane, no swizzle, out-of-bounds words read as zero.
int ensure_tmaps(octgpu_engine* e) {
    if (e->tm_ks == e->bulk_ks) return OCTGPU_OK;
    auto enc = tensor_map_encoder();
    if (!enc) return fail(OCTGPU_ERR_CUDA, "cuTensorMapEncodeTiled is not available from the driver");
    for (int b = 0; b < 2; ++b)
        for (int v = 0; v < 2; ++v) {
            const cuuint64_t dims[3] = {e->Y, e->n, 4};
            const cuuint64_t strides[2] = {cuuint64_t(e->Y) * 8, cuuint64_t(e->n) * e->Y * 8};
            const cuuint32_t box[3] = {kTmaBoxRows, cuuint32_t(e->bulk_ks + v), 1};
            const cuuint32_t estr[3] = {1, 1, 1};
            const CUresult r = enc(&e->tm[b][v], CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, e->planes[b], dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return fail(OCTGPU_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
        }
    e->tm_ks = e->bulk_ks;
    return OCTGPU_OK;
}

int ensure_tmaps_deep(octgpu_engine* e) {
    if (e->tmd_ok) return OCTGPU_OK;
    auto enc = tensor_map_encoder();
    if (!enc) return fail(OCTGPU_ERR_CUDA, "cuTensorMapEncodeTiled is not available from the driver");
    for (int b = 0; b < 2; ++b)
        for (int v = 0; v < 2; ++v) {
            const cuuint64_t dims[3] = {e->Y, e->n, 4};
            const cuuint64_t strides[2] = {cuuint64_t(e->Y) * 8, cuuint64_t(e->n) * e->Y * 8};
            const cuuint32_t box[3] = {cuuint32_t(deep_box_rows()), cuuint32_t(kDeepKS + v), 1};
            const cuuint32_t estr[3] = {1, 1, 1};
            const CUresult r = enc(&e->tmd[b][v], CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, e->planes[b], dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return fail(OCTGPU_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
        }
    e->tmd_ok = true;
    return OCTGPU_OK;
}

// Pipeline depth of k_mcs_bulk: KS words per stage, S stages. Measured on
// B200 at 2^16^2 and 2^17^2 for every (KS, S) in {1, 2, 4} x {2..6}
// (profiles/r1_pipeline_sweep.json): the shallowest double-buffered ring,
// KS = 2, S = 2 (18.6 KB per block), is fastest in every memory-bound mode
// (c2 0.351 ms vs 0.40-0.45 ms for deeper rings) and neutral in the
// issue-bound arbitrary mode. The consumers then stall almost only on the
// "full" barriers, i.e. on DRAM (95% of the measured copy bandwidth).
int plan_bulk(octgpu_engine* e, const ProbDev& p, const ProbDev& q) {
    const int key = p.mode * 8 + q.mode;
    if (e->bulk_key == key) return OCTGPU_OK;
    e->bulk_ks = 2;
    e->bulk_S = 2;
    if (const char* v = getenv("OCTGPU_MCS_KS")) e->bulk_ks = atoi(v) >= 4 ? 4 : atoi(v) == 2 ? 2 : 1;
    if (const char* v = getenv("OCTGPU_MCS_S")) e->bulk_S = std::max(2, std::min(8, atoi(v)));
    int smem_blk = 0;
    CK(cudaDeviceGetAttribute(&smem_blk, cudaDevAttrMaxSharedMemoryPerBlockOptin, e->device));
    if (int64_t(mcs_bulk_smem(e->bulk_ks, e->bulk_S)) > smem_blk)
        return fail(OCTGPU_ERR_CONFIG, "k_mcs_bulk pipeline does not fit in shared memory");
    e->bulk_key = key;
    return ensure_tmaps(e);
}

int alloc_p2p(octgpu_engine* e) {
    // separate allocations: each is exported on its own with cudaIpcGetMemHandle
    CK(cudaMalloc(reinterpret_cast<void**>(&e->done), 256));
    CK(cudaMalloc(reinterpret_cast<void**>(&e->p2p_err), 256));
    CK(cudaMemset(e->done, 0, 256));
    CK(cudaMemset(e->p2p_err, 0, 256));
    return OCTGPU_OK;
}

// The library's stream-ordered pool for periodic plane sets, one per device, created on first use with a
// release threshold of "keep everything": an engine re-created in the same process (resume, e2e runs) reuses
// the memory instead of paying cudaMalloc's page mapping again (40-130 ms for 2 GiB at 2^16^2).
std::mutex g_pool_mu;
std::map<int, cudaMemPool_t> g_pools;

int engine_pool(int device, cudaMemPool_t* out) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto it = g_pools.find(device);
    if (it == g_pools.end()) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        cudaMemPool_t pool = nullptr;
        CK(cudaMemPoolCreate(&pool, &props));
        uint64_t keep = ~uint64_t(0);
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        it = g_pools.emplace(device, pool).first;
    }
    *out = it->second;
    return OCTGPU_OK;
}

// Device buffers of an engine: from the library pool on the engine's stream when the engine is pooled
// (periodic), else cudaMalloc (stripes export theirs over CUDA IPC).
int dev_alloc(octgpu_engine* e, void** out, size_t bytes) {
    if (!e->pooled) {
        CK(cudaMalloc(out, bytes));
        return OCTGPU_OK;
    }
    cudaMemPool_t pool = nullptr;
    int rc = engine_pool(e->device, &pool);
    if (rc) return rc;
    cudaError_t ae = cudaMallocFromPoolAsync(out, bytes, pool, e->stream);
    if (ae == cudaErrorMemoryAllocation) {  // trim what earlier engines left and retry once
        cudaGetLastError();
        CK(cudaStreamSynchronize(e->stream));
        CK(cudaMemPoolTrimTo(pool, 0));
        ae = cudaMallocFromPoolAsync(out, bytes, pool, e->stream);
    }
    CK(ae);
    return OCTGPU_OK;
}

void dev_free(octgpu_engine* e, void* ptr) {
    if (!ptr) return;
    if (e->pooled)  // on the engine's own stream: a user stream may already be gone
        cudaFreeAsync(ptr, e->own_stream);
    else
        cudaFree(ptr);
}

// Small pinned host buffers (measure results, jump tables) are recycled process-wide: cudaMallocHost
// costs ~1 ms per call, paid again by every engine otherwise.
std::mutex g_pinned_mu;
std::multimap<size_t, void*> g_pinned_free;

cudaError_t host_pinned(void** out, size_t bytes) {
    {
        std::lock_guard<std::mutex> lk(g_pinned_mu);
        auto it = g_pinned_free.find(bytes);
        if (it != g_pinned_free.end()) {
            *out = it->second;
            g_pinned_free.erase(it);
            return cudaSuccess;
        }
    }
    return cudaMallocHost(out, bytes);
}

void host_pinned_release(void* ptr, size_t bytes) {
    if (!ptr) return;
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    g_pinned_free.emplace(bytes, ptr);
}

int alloc_engine(octgpu_engine* e) {
    CK(cudaSetDevice(e->device));
    CK(cudaStreamCreateWithFlags(&e->own_stream, cudaStreamNonBlocking));
    trace_create("stream", false);
    e->stream = e->own_stream;
    // Plane sets of a periodic engine come from the device's stream-ordered pool, kept (release threshold
    // = max) across engines: an engine re-created in the same process (resume, e2e runs) reuses the
    // memory instead of paying cudaMalloc's page mapping again (40-130 ms for 2 GiB at 2^16^2). Stripes
    // keep cudaMalloc: their plane sets are exported with cudaIpcGetMemHandle (p2p.cu).
    // The pool is the library's own (cudaMemPoolCreate), not the device's default pool, so the keep-all
    // release threshold does not leak into other users of cudaMallocAsync (PyTorch, NCCL). Memory a freed
    // engine leaves in it is returned with octgpu_release_pool(device), and automatically when a later
    // plane-set allocation of this library would otherwise fail.
    e->pooled = !e->stripe;
    for (int i = 0; i < 2; ++i) {
        int rc = dev_alloc(e, &e->planes[i], e->set_bytes());
        if (!rc) rc = dev_alloc(e, reinterpret_cast<void**>(&e->rng[i]), e->rng_bytes());
        if (rc) return rc;
    }
    trace_create("planes", false);
    // the small buffers too: a synchronous cudaMalloc / cudaMemset / cudaMallocHost each cost 0.5-1.5 ms
    // of an engine re-created inside a timed region
    int rc = dev_alloc(e, &e->scratch, measure_scratch_bytes(e->Y));
    if (!rc) rc = dev_alloc(e, reinterpret_cast<void**>(&e->res_dev), sizeof(MeasureResult));
    if (rc) return rc;
    CK(cudaMemsetAsync(e->scratch, 0, measure_scratch_bytes(e->Y), e->stream));  // k_col_scan's ticket starts at 0
    CK(host_pinned(reinterpret_cast<void**>(&e->res_host), sizeof(MeasureResult)));
    trace_create("small", false);
    return plan_mcs(e);
}

int lower_params(const octgpu_params* prm, ProbDev& p, ProbDev& q) {
    if (!prm) return fail(OCTGPU_ERR_CONFIG, "null parameters");
    int rc = lower(prm->p, p);
    if (rc) return rc;
    return lower(prm->q, q);
}

__int128 i128_of(uint64_t lo, int64_t hi) { return (__int128)(((unsigned __int128)(uint64_t)hi << 64) | lo); }

}  // namespace

extern "C" {

const char* octgpu_last_error(void) { return g_err.c_str(); }
const char* octgpu_version(void) { return "octgpu 0.1.0 (octsca 0.1.0 drop-in, sm_100a)"; }

int octgpu_resolve(double r, int forced_mode, octgpu_prob* out) {
    if (!out) return fail(OCTGPU_ERR_CONFIG, "null output");
    return resolve(r, forced_mode, *out);
}

uint32_t octgpu_draws_per_word(const octgpu_prob* p, uint32_t w) { return p ? draws(*p, w) : 0; }

int octgpu_validate_lattice(uint32_t X, uint32_t Y, uint32_t w) { return validate(X, Y, w); }

void octgpu_height_moments(uint32_t X, uint32_t Y, const int32_t* h, double* out) {
    // measure.cpp:24-51, same operation order (compiled with -ffp-contract=off)
    const size_t N = size_t(X) * Y;
    double mean = 0.0, m2 = 0.0, m3 = 0.0, m4 = 0.0, skew, kurt;
    if (N == 0) {
        for (int i = 0; i < 6; ++i) out[i] = 0.0;
        return;
    }
    const double n = double(N);
    for (size_t i = 0; i < N; ++i) mean += h[i];
    mean /= n;
    for (size_t i = 0; i < N; ++i) {
        const double d = h[i] - mean;
        const double d2 = d * d;
        m2 += d2;
        m3 += d2 * d;
        m4 += d2 * d2;
    }
    m2 /= n;
    m3 /= n;
    m4 /= n;
    if (m2 > 0.0) {
        skew = m3 / std::pow(m2, 1.5);
        kurt = m4 / (m2 * m2) - 3.0;
    } else {
        skew = std::numeric_limits<double>::quiet_NaN();
        kurt = std::numeric_limits<double>::quiet_NaN();
    }
    out[0] = mean; out[1] = m2; out[2] = m3; out[3] = m4; out[4] = skew; out[5] = kurt;
}

int octgpu_stream_states(uint64_t master_seed, uint32_t n, uint64_t* out) {
    if (n < 1) return fail(OCTGPU_ERR_CONFIG, "stream count must be >= 1");
    stream_states(master_seed, n, out);
    return OCTGPU_OK;
}

uint32_t octgpu_log_schedule(uint64_t t_max, uint32_t ppd, uint64_t* out, uint32_t cap) {
    if (t_max < 1 || ppd < 1) {
        fail(OCTGPU_ERR_CONFIG, t_max < 1 ? "t_max must be >= 1" : "points_per_decade must be >= 1");
        return 0;
    }
    std::vector<uint64_t> times;
    uint64_t prev = 0;
    for (uint32_t k = 0;; ++k) {
        const double exact = std::pow(10.0, double(k) / double(ppd));
        if (exact > double(t_max) * (1.0 + 1e-12)) break;
        uint64_t tt = uint64_t(std::llround(exact));
        if (tt <= prev) tt = prev + 1;
        if (tt > t_max) break;
        times.push_back(tt);
        prev = tt;
    }
    if (times.empty() || times.back() != t_max) times.push_back(t_max);
    for (size_t i = 0; i < times.size() && i < cap; ++i) out[i] = times[i];
    return uint32_t(times.size());
}

}  // extern "C"

namespace {

int refresh_ghosts(octgpu_engine* e);

// OCTGPU_TRACE_CREATE=1: stderr timings of the engine-creation phases (diagnostics)
void trace_create(const char* what, bool start) {
    static const bool on = getenv("OCTGPU_TRACE_CREATE") != nullptr;
    static std::chrono::steady_clock::time_point last;
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    if (!start) fprintf(stderr, "[octgpu create] %-10s %8.3f ms\n", what,
                        std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
}

// Allocates an engine over global rows [y0, y0 + L) of an X x Ytot lattice
// (stripe) or the whole periodic lattice (!stripe).
int make_engine(uint32_t X, uint32_t Ytot, uint32_t w, bool stripe, uint32_t y0, uint32_t L, int device,
                uint64_t master_seed, octgpu_engine** out) {
    auto* e = new octgpu_engine;
    e->X = X; e->w = w; e->n = X / (2 * w); e->device = device; e->master_seed = master_seed;
    e->Ytot = Ytot; e->stripe = stripe; e->y0 = stripe ? y0 : 0; e->L = stripe ? L : Ytot;
    // stripe: halo rows 0..HA-1, core HA..HA+L-1, halos below HA+L..HA+L+HB-1, then >= 34
    // rows of padding (k_mcs reads up to 33 rows past a warp's first row; the TMA kernels
    // zero-fill past the allocation); even for 16-B alignment
    e->Y = stripe ? ((L + kStripeHA + kStripeHB + 34 + 1) & ~1u) : Ytot + kGhostRows;
    trace_create("", true);
    int rc = alloc_engine(e);
    trace_create("alloc", false);
    if (!rc && stripe) rc = alloc_p2p(e);
    if (rc) {
        std::string keep = g_err;
        octgpu_destroy(e);
        g_err = keep;
        return rc;
    }
    *out = e;
    return OCTGPU_OK;
}

// Upload core-row planes given in the reference layout ([4][core rows][n]).
int load_planes(octgpu_engine* e, const void* planes) {
    void* stage = nullptr;
    int rc = ensure_stage(e, &stage);
    if (rc) return rc;
    const size_t wb = e->word_bytes(), row_bytes = size_t(e->n) * wb;
    if (!e->stripe) {
        CK(cudaMemcpyAsync(stage, planes, e->host_bytes(), cudaMemcpyHostToDevice, e->stream));
    } else {  // core rows of each plane into their place in the staged layout; halo and padding rows zero
        CK(cudaMemsetAsync(stage, 0, e->host_bytes(), e->stream));
        for (int p = 0; p < 4; ++p)
            CK(cudaMemcpyAsync(static_cast<unsigned char*>(stage) + (size_t(p) * e->Y + kStripeHA) * row_bytes,
                               static_cast<const unsigned char*>(planes) + size_t(p) * e->L * row_bytes,
                               e->L * row_bytes, cudaMemcpyHostToDevice, e->stream));
    }
    if (getenv("OCTGPU_TRACE_CREATE")) {
        CK(cudaStreamSynchronize(e->stream));
        trace_create("upload", false);
    }
    CK(launch_import(e->w, stage, e->planes[e->pcur], e->geom(), e->host_rows(), e->stream));
    ++e->launches;
    rc = refresh_ghosts(e);
    if (rc) return rc;
    // no host sync here: every caller follows with upload_states, which transposes the states on the host
    // while the planes are still in flight and then synchronises the stream (the caller's buffer is read
    // until then)
    if (getenv("OCTGPU_TRACE_CREATE")) {
        CK(cudaStreamSynchronize(e->stream));
        trace_create("import", false);
    }
    return OCTGPU_OK;
}

int flat_fill(octgpu_engine* e) {  // new_flat: odd planes all ones, even planes zero (slope_field.hpp:110-118)
    const size_t pb = e->set_bytes() / 4;
    char* base = static_cast<char*>(e->planes[e->pcur]);
    for (int p = 0; p < 4; ++p) CK(cudaMemsetAsync(base + p * pb, (p & 1) ? 0xff : 0x00, pb, e->stream));
    return OCTGPU_OK;
}

// Rewrite the ghost rows of the current plane set and rng states (periodic
// lattices; every operation except k_mcs_bulk leaves them stale).
int refresh_ghosts(octgpu_engine* e) {
    if (e->stripe) return OCTGPU_OK;
    CK(launch_refresh_ghosts(e->w, e->planes[e->pcur], e->rng[e->rcur], e->geom(), e->stream));
    ++e->launches;
    return OCTGPU_OK;
}

int fail_destroy(octgpu_engine* e, int rc) {
    std::string keep = g_err;
    octgpu_destroy(e);
    g_err = keep;
    return rc;
}

}  // namespace

extern "C" {

int octgpu_create(uint32_t X, uint32_t Y, uint32_t w, uint64_t seed, int device, octgpu_engine** out) {
    if (!out) return fail(OCTGPU_ERR_CONFIG, "null output");
    *out = nullptr;
    int rc = validate(X, Y, w);
    if (rc) return rc;
    octgpu_engine* e = nullptr;
    rc = make_engine(X, Y, w, false, 0, Y, device, seed, &e);
    if (rc) return rc;
    rc = flat_fill(e);
    if (!rc) {
        std::vector<uint64_t> st(4 * size_t(Y));
        stream_states(seed, Y, st.data());
        rc = upload_states(e, st.data());
    }
    if (rc) return fail_destroy(e, rc);
    *out = e;
    return OCTGPU_OK;
}

int octgpu_create_from(uint32_t X, uint32_t Y, uint32_t w, uint64_t t_mcs, int phase, const void* planes,
                       const uint64_t* states, uint32_t n_states, uint64_t master_seed, int device,
                       octgpu_engine** out) {
    if (!out || !planes || !states) return fail(OCTGPU_ERR_CONFIG, "null argument");
    *out = nullptr;
    int rc = validate(X, Y, w);
    if (rc) return rc;
    if (phase != 0 && phase != 1) return fail(OCTGPU_ERR_CONFIG, "phase must be 0 or 1");
    if (n_states < Y) return fail(OCTGPU_ERR_INVARIANT, "stream set smaller than row count");
    octgpu_engine* e = nullptr;
    rc = make_engine(X, Y, w, false, 0, Y, device, master_seed, &e);
    if (rc) return rc;
    e->t = t_mcs;
    e->phase = phase;
    rc = load_planes(e, planes);
    if (!rc) rc = upload_states(e, states);
    if (rc) return fail_destroy(e, rc);
    *out = e;
    return OCTGPU_OK;
}

int octgpu_create_stripe(uint32_t X, uint32_t Y, uint32_t w, uint32_t y0, uint32_t y1, uint64_t t_mcs, int phase,
                         const void* planes, const uint64_t* states, uint64_t master_seed, int device,
                         octgpu_engine** out) {
    if (!out) return fail(OCTGPU_ERR_CONFIG, "null output");
    *out = nullptr;
    int rc = validate(X, Y, w);
    if (rc) return rc;
    if (!(y0 < y1 && y1 <= Y) || y1 - y0 < kStripeHB)
        return fail(OCTGPU_ERR_CONFIG, "stripe rows [" + std::to_string(y0) + "," + std::to_string(y1) +
                                           ") must hold at least " + std::to_string(kStripeHB) +
                                           " rows of the lattice");
    if (phase != 0 && phase != 1) return fail(OCTGPU_ERR_CONFIG, "phase must be 0 or 1");
    if ((planes == nullptr) != (states == nullptr))
        return fail(OCTGPU_ERR_CONFIG, "give both planes and states, or neither (flat start)");
    const uint32_t L = y1 - y0;
    octgpu_engine* e = nullptr;
    rc = make_engine(X, Y, w, true, y0, L, device, master_seed, &e);
    if (rc) return rc;
    e->t = t_mcs;
    e->phase = phase;
    if (planes) {
        rc = load_planes(e, planes);
        if (!rc) rc = upload_states(e, states);
    } else {
        rc = flat_fill(e);
        if (!rc) {  // RngStreamSet(seed, Y) rows y0..y1-1
            std::vector<uint64_t> st(4 * size_t(y1));
            stream_states(master_seed, y1, st.data());
            rc = upload_states(e, st.data() + 4 * size_t(y0));
        }
    }
    if (rc) return fail_destroy(e, rc);
    *out = e;
    return OCTGPU_OK;
}

int octgpu_set_state(octgpu_engine* e, uint64_t t_mcs, int phase, const void* planes, const uint64_t* states,
                     uint32_t n_states) {
    if (!e || !planes || !states) return fail(OCTGPU_ERR_CONFIG, "null argument");
    if (phase != 0 && phase != 1) return fail(OCTGPU_ERR_CONFIG, "phase must be 0 or 1");
    if (n_states < e->core_rows()) return fail(OCTGPU_ERR_INVARIANT, "stream set smaller than row count");
    int rc = use_device(e);
    if (!rc) rc = load_planes(e, planes);
    if (!rc) {
        e->pending = 0;
        rc = upload_states(e, states);
    }
    if (rc) {
        cudaStreamSynchronize(e->stream);  // no copy may still read the caller's buffers after we return
        return rc;
    }
    e->t = t_mcs;
    e->phase = phase;
    return OCTGPU_OK;
}

void octgpu_destroy(octgpu_engine* e) {
    if (!e) return;
    cudaSetDevice(e->device);
    if (e->stream) cudaStreamSynchronize(e->stream);
    for (int i = 0; i < 2; ++i) {
        dev_free(e, e->planes[i]);
        dev_free(e, e->rng[i]);
    }
    for (auto& kv : e->graph_cache) cudaGraphExecDestroy(kv.second.first);
    for (auto& kv : e->jtabs) cudaFree(kv.second);
    dev_free(e, e->pend_tab);
    host_pinned_release(e->pend_host, kPendTabBytes);
    if (e->pend_ev) cudaEventDestroy(e->pend_ev);
    for (void* ptr : e->ipc_opened) cudaIpcCloseMemHandle(ptr);
    if (e->done) cudaFree(e->done);
    if (e->p2p_err) cudaFree(e->p2p_err);
    if (e->stage) cudaFree(e->stage);
    dev_free(e, e->scratch);
    dev_free(e, e->res_dev);
    host_pinned_release(e->res_host, sizeof(MeasureResult));
    if (e->own_stream) {
        cudaStreamSynchronize(e->own_stream);
        cudaStreamDestroy(e->own_stream);
    }
    delete e;
}

int octgpu_release_pool(int device) {
    cudaMemPool_t pool = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        auto it = g_pools.find(device);
        if (it == g_pools.end()) return OCTGPU_OK;
        pool = it->second;
    }
    CK(cudaSetDevice(device));
    CK(cudaDeviceSynchronize());  // frees of destroyed engines are stream-ordered
    CK(cudaMemPoolTrimTo(pool, 0));
    return OCTGPU_OK;
}

int octgpu_set_stream(octgpu_engine* e, void* s) {
    if (!e) return fail(OCTGPU_ERR_CONFIG, "null engine");
    int rc = use_device(e);
    if (rc) return rc;
    CK(cudaStreamSynchronize(e->stream));
    e->stream = s ? static_cast<cudaStream_t>(s) : e->own_stream;
    return OCTGPU_OK;
}

int octgpu_sync(octgpu_engine* e) {
    if (!e) return fail(OCTGPU_ERR_CONFIG, "null engine");
    int rc = use_device(e);
    if (rc) return rc;
    CK(cudaStreamSynchronize(e->stream));
    CK(cudaGetLastError());
    if (e->p2p) {  // a peer-memory halo wait that timed out (p2p.cu)
        uint32_t err = 0;
        CK(cudaMemcpy(&err, e->p2p_err, sizeof(err), cudaMemcpyDeviceToHost));
        if (err) return fail(OCTGPU_ERR_CUDA, "peer halo exchange timed out waiting for a neighbour stripe");
    }
    return OCTGPU_OK;
}

namespace {

// k_mcs_deep ring depth: deep_S (3) unless two blocks per SM would no longer fit
// in shared memory (live passes park xoshiro states and pre-drawn xi there) -> 2.
int deep_ring(octgpu_engine* e, const ProbDev& p, const ProbDev& q, int ls, bool ctr = false) {
    int smem_sm = 0;
    if (cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, e->device) != cudaSuccess)
        return 2;
    int S = e->deep_S;
    while (S > 2 && size_t(kDeepMinBlocks) * (mcs_deep_smem(p.mode, q.mode, ls, S, ctr) + 1024) > size_t(smem_sm)) --S;
    return S;
}

// sweeps per k_mcs_deep pass: 6 (3 MCS) where the kernel takes it (constant xi), else 4 (row stripes too: their
// halo rows are sized for kStripeSweeps = 6)
int deep_sweeps(const octgpu_engine* e, const ProbDev& p, const ProbDev& q, bool ctr) {
    return (e->deep_l == kDeepSweepsConst && mcs_deep_supported_l(p.mode, q.mode, kDeepSweepsConst, ctr))
               ? kDeepSweepsConst
               : kDeepSweepsLive;
}

// k_mcs_deep does not mirror its plane stores into a periodic lattice's ghost rows: rows 0..ghost-1 of the
// new plane set are copied there after the pass (every (plane, word) column holds its rows contiguously, so
// one strided device copy of ghost x 8 bytes per column)
cudaError_t mirror_ghost_planes(octgpu_engine* e, void* planes) {
    if (e->stripe || kGhostRows > e->L) return cudaSuccess;
    if (e->ghost_kernel) {  // k_ghost_copy: 0.5% faster per pass than the 2-D memcpy (c2 0.1287 vs 0.1294 ms/MCS)
        ++e->launches;
        return launch_ghost_copy(planes, e->Y, e->L, kGhostRows, 4 * e->n, e->stream);
    }
    char* base = static_cast<char*>(planes);
    const size_t pitch = size_t(e->Y) * e->word_bytes();
    return cudaMemcpy2DAsync(base + size_t(e->L) * e->word_bytes(), pitch, base, pitch, size_t(kGhostRows) * e->word_bytes(),
                             size_t(4) * e->n, cudaMemcpyDeviceToDevice, e->stream);
}

// Sweeps of the next deep pass with `left` MCS to go: full-length passes (lsmax); in a 3-MCS schedule a remainder
// of 1 or 2 is absorbed by one or two 4-MCS passes (L = 8 runs at the 3-MCS pass's cost per MCS, while a 2-MCS
// pass costs ~1.6x per MCS and a one-MCS pass ~2.6x: 20 MCS = 4 x 3 + 2 x 4, not 6 x 3 + 2); then 2, then 0.
int pass_sweeps(const octgpu_engine* e, const ProbDev& p, const ProbDev& q, bool ctr, int lsmax, uint64_t left) {
    if (lsmax == kDeepSweepsConst && e->deep_long && !e->stripe &&
        mcs_deep_supported_l(p.mode, q.mode, kDeepSweepsLong, ctr)) {
        const uint64_t r = left % 3;
        if ((r == 1 && left >= 4) || (r == 2 && left >= 8)) return kDeepSweepsLong;
    }
    if (left >= uint64_t(lsmax / 2)) return lsmax;
    return left >= 2 ? kDeepSweepsLive : 0;
}

// Periodic lattices: does octgpu_step run k_mcs_deep passes for these parameters? (D = draws per word of a
// xoshiro sweep; ctr = the counter-based streams)
bool deep_policy(const octgpu_engine* e, const ProbDev& p, const ProbDev& q, uint64_t D, bool ctr) {
    if (e->mcs_impl != 2 || !mcs_deep_supported(p.mode, q.mode) || e->deep == 0) return false;
    if (e->deep == 2) return true;
    const uint64_t sites = uint64_t(e->X) * e->L;
    const bool live = !(is_const(p) && is_const(q));
    // 2-MCS passes with counter streams: no stream state to park, so every cheap mode qualifies from 2^28
    if (ctr || !live) return sites >= (uint64_t(1) << 28);
    // live xoshiro streams: one draw per word (p = 1/2, q = 0: 0.318 -> 0.249 ms/MCS at 2^16^2) and the
    // half/half pair (p = q = 1/2, BASELINE configs[2]: 0.388 -> 0.347); a dyadic stream or three draws per
    // word spill at the 128-register budget and stay on the one-MCS kernel (p = 3/4: 0.395 vs 0.521)
    const bool cheap_live = D == 1 || (p.mode == M_HALF && q.mode == M_HALF);
    return cheap_live && sites >= (uint64_t(1) << 30);
}

// One fused pass (k_mcs_deep: 2 or 3 MCS; else 1 MCS) from the current plane / rng set into the other,
// with the host-side bookkeeping of what the pass does.
// Random tile-origin shift (the DTr idea of BASELINE.json's north_star, applied to the block tiling): the
// first core row of the block decomposition moves by s rows, drawn per pass from (tile_shift seed, t).
// Sites of one sublattice share no slopes (engine_vec.hpp:95-97), so any tiling gives the same result;
// the shift only moves block / warp / halo boundaries (tested: shifted == unshifted, bit for bit).
// s is even and keeps every TMA window inside the ghost rows.
Geom shifted(const octgpu_engine* e, Geom g, uint32_t window) {
    g.pf = e->prefetch;
    if (!e->tile_shift || e->stripe || e->mcs_impl != 2) return g;
    uint64_t z = e->tile_shift + 0x9e3779b97f4a7c15ull * (e->t + 1);  // splitmix64 finaliser
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    // even shifts: a TMA box must start 16-B aligned in its innermost (row) dimension
    const uint32_t smax = (kGhostRows - window - 2) / 2;
    const uint32_t s = 2 * uint32_t(z % (smax + 1));
    g.c0 += s;
    g.c1 += s;
    return g;
}

// ls = sweeps of a k_mcs_deep pass (4 or 6), 0 = one-MCS kernel
int step_pass(octgpu_engine* e, const ProbDev& p, const ProbDev& q, bool live, int ls, const uint64_t* jtab,
              uint64_t per_sweep) {
    const int ps = e->pcur, rs = e->rcur;
    const bool deep = ls > 0;
    if (deep) {
        int rc = ensure_tmaps_deep(e);
        if (rc) return rc;
        CK(launch_mcs_deep(e->planes[ps], e->planes[ps ^ 1], e->rng[rs], e->rng[rs ^ 1], e->phase,
                           shifted(e, e->deep_geom(ls), uint32_t(deep_box_rows())), p, q, jtab, ls,
                           deep_ring(e, p, q, ls), &e->tmd[ps][0], &e->tmd[ps][1], e->stream));
        CK(mirror_ghost_planes(e, e->planes[ps ^ 1]));
    } else if (e->mcs_impl == 2) {
        int rc = plan_bulk(e, p, q);
        if (rc) return rc;
        CK(launch_mcs_bulk(e->planes[ps], e->planes[ps ^ 1], e->rng[rs], e->rng[rs ^ 1], e->phase,
                           shifted(e, e->geom(), kTmaBoxRows), p, q, jtab, e->bulk_ks, e->bulk_S, &e->tm[ps][0],
                           &e->tm[ps][1], e->stream));
    } else {
        CK(launch_mcs(e->w, e->planes[ps], e->planes[ps ^ 1], e->rng[rs], e->rng[rs ^ 1], e->phase, e->geom(), p, q,
                      live, jtab, e->stream));
    }
    const uint32_t mcs = deep ? uint32_t(ls / 2) : 1u;
    ++e->launches;
    e->pcur ^= 1;
    if (live)
        e->rcur ^= 1;
    else
        e->pending += 2 * uint64_t(mcs) * per_sweep;  // constant xi: streams advance lazily
    e->t += mcs;  // whole MCS: the phase returns to its value (engine_vec.hpp:172-177)
    return OCTGPU_OK;
}

std::string graph_key(const octgpu_engine* e, const ProbDev& p, const ProbDev& q, int ls, const uint64_t* jtab) {
    char buf[256];
    std::snprintf(buf, sizeof buf, "%d/%u/%llx/%llx|%d/%u/%llx/%llx|%d|%d%d%d|%p|%d%d%d", p.mode, p.k,
                  (unsigned long long)p.m, (unsigned long long)p.T, q.mode, q.k, (unsigned long long)q.m,
                  (unsigned long long)q.T, ls, e->pcur, e->rcur, e->phase, static_cast<const void*>(jtab),
                  ls ? deep_ring(const_cast<octgpu_engine*>(e), p, q, ls) : 0, e->bulk_ks, e->bulk_S);
    return buf;
}

}  // namespace

namespace {

// n MCS with counter-based xi (octgpu_set_rng), sweeps in the engine_vec.hpp:171-177 order (phase, then !phase),
// global sweep index sigma = 2 t + 0 / 1: the fused TMA kernel (k_mcs_bulk<CTR>, 1 MCS per pass) where the
// lattice takes it, else two in-place k_sweep_ctr sweeps per MCS.
int step_counter(octgpu_engine* e, const ProbDev& p, const ProbDev& q, uint64_t n_mcs) {
    if (e->mcs_impl == 2) {
        int rc = plan_bulk(e, p, q);
        if (rc) return rc;
    }
    // 2-MCS passes (k_mcs_deep<CTR>): no stream state to park, so every cheap mode qualifies; same size
    // threshold as the constant-xi xoshiro passes
    const bool deep = deep_policy(e, p, q, 0, true);
    if (deep) {
        int rc = ensure_tmaps_deep(e);
        if (rc) return rc;
        const int lsmax = deep_sweeps(e, p, q, true);
        while (n_mcs >= 2) {  // full-length passes, then a 2-MCS pass for a remainder of 2
            const int ls = pass_sweeps(e, p, q, true, lsmax, n_mcs);
            const uint64_t mpp = uint64_t(ls / 2);
            const int ps = e->pcur;
            CK(launch_mcs_deep_ctr(e->planes[ps], e->planes[ps ^ 1], e->phase,
                                   shifted(e, e->deep_geom(ls), uint32_t(deep_box_rows())), p, q, e->master_seed,
                                   2 * e->t, ls, deep_ring(e, p, q, ls, true), &e->tmd[ps][0], &e->tmd[ps][1],
                                   e->stream));
            CK(mirror_ghost_planes(e, e->planes[ps ^ 1]));
            ++e->launches;
            e->pcur ^= 1;
            e->t += mpp;
            n_mcs -= mpp;
        }
    }
    if (e->mcs_impl == 2 && e->bulk_ks == 2) {
        for (uint64_t i = 0; i < n_mcs; ++i) {
            const int ps = e->pcur;
            CK(launch_mcs_bulk_ctr(e->planes[ps], e->planes[ps ^ 1], e->phase, shifted(e, e->geom(), kTmaBoxRows), p,
                                   q, e->master_seed, 2 * e->t, e->bulk_S, &e->tm[ps][0], &e->tm[ps][1], e->stream));
            ++e->launches;
            e->pcur ^= 1;
            ++e->t;
        }
        return OCTGPU_OK;
    }
    for (uint64_t i = 0; i < n_mcs; ++i) {
        for (int h = 0; h < 2; ++h) {
            CK(launch_sweep_ctr(e->w, e->planes[e->pcur], e->phase, e->geom(), p, q, e->master_seed, 2 * e->t + h,
                                e->stream));
            ++e->launches;
            e->phase ^= 1;
        }
        ++e->t;
    }
    return refresh_ghosts(e);  // k_sweep_ctr works in place and does not maintain ghost rows
}

}  // namespace

int octgpu_step(octgpu_engine* e, const octgpu_params* prm, uint64_t n_mcs) {
    if (!e) return fail(OCTGPU_ERR_CONFIG, "null engine");
    if (e->stripe) return fail(OCTGPU_ERR_CONFIG, "octgpu_step is not available on a row stripe (use the octgpu_stripe_* calls)");
    ProbDev p, q;
    int rc = lower_params(prm, p, q);
    if (rc) return rc;
    if (n_mcs == 0) return OCTGPU_OK;
    rc = use_device(e);
    if (rc) return rc;
    if (e->rng_kind == OCTGPU_RNG_COUNTER) return step_counter(e, p, q, n_mcs);
    const bool live = !(is_const(p) && is_const(q));
    const uint64_t D = draws(prm->p, e->w) + (q.mode != M_ZERO ? draws(prm->q, e->w) : 0);
    const uint64_t per_sweep = uint64_t(e->n) * D;
    uint64_t* jtab = nullptr;
    if (live) {
        rc = materialize(e);
        if (rc) return rc;
        rc = get_table(e, per_sweep, &jtab);
        if (rc) return rc;
    }
    // Temporal blocking pays where the one-MCS kernel is DRAM-bound: constant xi
    // (zero / one) and one draw per word (p = 1/2 with q = 0, the paper's benchmark
    // case: 0.367 -> 0.316 ms/MCS at 2^16^2). With more draws per word the four
    // streams per lane make it issue-bound and slower than k_mcs_bulk (p = q = 1/2:
    // 0.41 -> 0.47; p = 3/4: 0.40 -> 0.51; profiles/r1_deep_modes.json).
    // OCTGPU_DEEP=2 forces it for every cheap mode, OCTGPU_DEEP=0 disables it.
    // Small lattices underfill the GPU and are latency-bound, where the longer 2-MCS
    // pipeline loses (tools/step_timer.py: constant xi wins from 2^28 sites, p = 1/2
    // from 2^30); OCTGPU_DEEP=2 forces the deep pass for any size (tests).
    const bool deep = deep_policy(e, p, q, D, false);
    const int lsmax = deep ? deep_sweeps(e, p, q, false) : 0;  // sweeps per full-length pass (0: one-MCS kernel)
    const uint64_t mpp = deep ? uint64_t(lsmax / 2) : 1;  // MCS per pass
    uint64_t left = n_mcs;
    // Long runs on small / medium lattices replay a CUDA graph of kGraphPasses passes
    // (an even number, so the plane / rng sets end where they started and the captured
    // arguments repeat): no per-launch CPU work, which is what bounds small lattices.
    // Measured steady state (tools/step_timer.py, KWARM=300): 1024^2 p=1/2 10.3 -> 7.7 us/MCS,
    // 4096^2 p=1 10.0 -> 9.0, 16384^2 p=1 27.7 -> 26.7 us. The first capture + instantiate
    // in a process costs tens of ms, so lattices whose passes are long anyway (> 2^28
    // sites, where a pass is >= 0.1 ms) keep plain launches.
    const uint64_t period = mpp * kGraphPasses;
    const bool graph_ok = e->graphs && !e->tile_shift && uint64_t(e->X) * e->L <= (uint64_t(1) << 28) &&
                          e->stream != cudaStreamLegacy && e->stream != cudaStreamPerThread;
    if (graph_ok && left >= 2 * period) {
        // first pass outside any capture: plans, tensor maps and kernel attributes exist afterwards
        rc = step_pass(e, p, q, live, lsmax, jtab, per_sweep);
        if (rc) return rc;
        left -= mpp;
        const std::string key = graph_key(e, p, q, lsmax, jtab);
        auto it = e->graph_cache.find(key);
        if (it == e->graph_cache.end()) {
            const int pc = e->pcur, rcs = e->rcur;
            const uint64_t pend = e->pending, t0 = e->t, l0 = e->launches;
            cudaGraph_t graph = nullptr;
            CK(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
            int crc = OCTGPU_OK;
            for (int k = 0; k < kGraphPasses && !crc; ++k) crc = step_pass(e, p, q, live, lsmax, jtab, per_sweep);
            const cudaError_t ce = cudaStreamEndCapture(e->stream, &graph);
            const uint64_t kernels = e->launches - l0;  // what one replay launches (passes + ghost copies)
            e->pcur = pc;  // capturing enqueued nothing: undo the bookkeeping
            e->rcur = rcs;
            e->pending = pend;
            e->t = t0;
            e->launches = l0;
            if (crc) {
                if (graph) cudaGraphDestroy(graph);
                return crc;
            }
            CK(ce);
            cudaGraphExec_t exec = nullptr;
            const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
            cudaGraphDestroy(graph);
            CK(ie);
            it = e->graph_cache.emplace(key, std::make_pair(exec, kernels)).first;
        }
        while (left >= period) {
            CK(cudaGraphLaunch(it->second.first, e->stream));
            if (!live) e->pending += 2 * period * per_sweep;
            e->t += period;
            e->launches += it->second.second;
            left -= period;
        }
    }
    while (left > 0) {
        // full-length passes, then a 2-MCS pass for a remainder of 2 (of a 3-MCS schedule), then one MCS
        const int ls = !deep ? 0 : pass_sweeps(e, p, q, false, lsmax, left);
        rc = step_pass(e, p, q, live, ls, jtab, per_sweep);
        if (rc) return rc;
        left -= ls ? uint64_t(ls / 2) : 1;
    }
    return OCTGPU_OK;
}

int octgpu_sweep(octgpu_engine* e, int parity, const octgpu_params* prm, void* mask_log) {
    if (!e) return fail(OCTGPU_ERR_CONFIG, "null engine");
    if (e->stripe) return fail(OCTGPU_ERR_CONFIG, "octgpu_sweep is not available on a row stripe (use the octgpu_stripe_* calls)");
    if (e->rng_kind != OCTGPU_RNG_XOSHIRO)
        return fail(OCTGPU_ERR_CONFIG, "single sweeps draw from the per-row xoshiro streams; the counter-based "
                                       "rng steps whole MCS only (octgpu_step)");
    if (parity != e->phase)  // engine_vec.hpp:150-152
        return fail(OCTGPU_ERR_INVARIANT, "sweep parity " + std::to_string(parity) +
                                              " does not match field phase " + std::to_string(e->phase));
    ProbDev p, q;
    int rc = lower_params(prm, p, q);
    if (rc) return rc;
    rc = use_device(e);
    if (rc) return rc;
    const bool live = !(is_const(p) && is_const(q));
    const uint64_t D = draws(prm->p, e->w) + (q.mode != M_ZERO ? draws(prm->q, e->w) : 0);
    if (live) {
        rc = materialize(e);
        if (rc) return rc;
    }
    void* mlog = nullptr;
    const size_t log_bytes = size_t(e->L) * e->n * e->word_bytes();
    if (mask_log) CK(cudaMalloc(&mlog, log_bytes));
    const cudaError_t le =
        launch_sweep(e->w, e->planes[e->pcur], e->rng[e->rcur], parity, e->geom(), p, q, live, mlog, e->stream);
    if (le != cudaSuccess) {
        if (mlog) cudaFree(mlog);
        return cuda_fail(le, "sweep");
    }
    ++e->launches;
    if (!live) e->pending += uint64_t(e->n) * D;
    e->phase ^= 1;
    rc = refresh_ghosts(e);  // k_sweep works in place and does not maintain ghost rows
    if (rc) return rc;
    if (mask_log) {
        CK(cudaMemcpyAsync(mask_log, mlog, log_bytes, cudaMemcpyDeviceToHost, e->stream));
        CK(cudaStreamSynchronize(e->stream));
        CK(cudaFree(mlog));
    }
    return OCTGPU_OK;
}

int octgpu_set_tile_shift(octgpu_engine* e, uint64_t seed) {
    if (!e) return fail(OCTGPU_ERR_CONFIG, "null engine");
    e->tile_shift = seed;
    return OCTGPU_OK;
}

int octgpu_set_rng(octgpu_engine* e, int kind) {
    if (!e) return fail(OCTGPU_ERR_CONFIG, "null engine");
    if (kind != OCTGPU_RNG_XOSHIRO && kind != OCTGPU_RNG_COUNTER)
        return fail(OCTGPU_ERR_CONFIG, "unknown rng kind " + std::to_string(kind));
    if (kind == OCTGPU_RNG_COUNTER && e->stripe && e->mcs_impl != 2)
        return fail(OCTGPU_ERR_CONFIG, "the counter-based rng on a row stripe needs w = 64 and >= 8 words per row");
    e->rng_kind = kind;
    return OCTGPU_OK;
}

int octgpu_get_rng(const octgpu_engine* e) { return e ? e->rng_kind : -1; }

uint64_t octgpu_t(const octgpu_engine* e) { return e ? e->t : 0; }
int octgpu_phase(const octgpu_engine* e) { return e ? e->phase : 0; }
uint64_t octgpu_master_seed(const octgpu_engine* e) { return e ? e->master_seed : 0; }
uint64_t octgpu_launch_count(const octgpu_engine* e) { return e ? e->launches : 0; }

int octgpu_get_planes(octgpu_engine* e, void* out) {
    if (!e || !out) return fail(OCTGPU_ERR_CONFIG, "null argument");
    int rc = use_device(e);
    void* stage = nullptr;
    if (!rc) rc = ensure_stage(e, &stage);
    if (rc) return rc;
    CK(launch_export(e->w, e->planes[e->pcur], stage, e->geom(), e->host_rows(), e->stream));
    ++e->launches;
    if (!e->stripe) {
        trace_create("planes", true);
        CK(cudaMemcpyAsync(out, stage, e->host_bytes(), cudaMemcpyDeviceToHost, e->stream));
        CK(cudaStreamSynchronize(e->stream));
        trace_create("planes-d2h", false);
        return OCTGPU_OK;
    }
    // a stripe's core rows of each plane are contiguous in the staged reference layout: one copy per plane
    // straight into the caller's buffer (pinned buffers take the DMA path at full PCIe rate)
    const size_t row_bytes = size_t(e->n) * e->word_bytes();
    for (int p = 0; p < 4; ++p)
        CK(cudaMemcpyAsync(static_cast<unsigned char*>(out) + size_t(p) * e->L * row_bytes,
                           static_cast<const unsigned char*>(stage) + (size_t(p) * e->Y + kStripeHA) * row_bytes,
                           e->L * row_bytes, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    return OCTGPU_OK;
}

int octgpu_get_states(octgpu_engine* e, uint64_t* out) {
    if (!e || !out) return fail(OCTGPU_ERR_CONFIG, "null argument");
    trace_create("states", true);
    int rc = use_device(e);
    if (!rc) rc = materialize(e);
    if (rc) return rc;
    std::vector<uint64_t> soa(4 * size_t(e->Y));
    CK(cudaMemcpyAsync(soa.data(), e->rng[e->rcur], e->rng_bytes(), cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    trace_create("states-d2h", false);
    const uint32_t r0 = e->first_row();
    for (uint32_t y = 0; y < e->core_rows(); ++y)
        for (int j = 0; j < 4; ++j) out[4 * size_t(y) + j] = soa[size_t(j) * e->Y + r0 + y];
    trace_create("states-aos", false);
    return OCTGPU_OK;
}

int octgpu_field_checksum(octgpu_engine* e, uint64_t* out) {
    if (!e || !out) return fail(OCTGPU_ERR_CONFIG, "null argument");
    std::vector<unsigned char> buf(e->host_bytes());
    int rc = octgpu_get_planes(e, buf.data());
    if (rc) return rc;
    uint64_t h = 0xcbf29ce484222325ULL;  // FNV-1a, slope_field.hpp:232-246
    auto mix = [&h](uint64_t v) {
        for (int i = 0; i < 8; ++i) {
            h ^= (v >> (8 * i)) & 0xff;
            h *= 0x100000001b3ULL;
        }
    };
    const size_t nw = 4 * size_t(e->n) * e->L;
    if (e->w == 64) {
        const uint64_t* p = reinterpret_cast<const uint64_t*>(buf.data());
        for (size_t i = 0; i < nw; ++i) mix(p[i]);
    } else {
        const uint32_t* p = reinterpret_cast<const uint32_t*>(buf.data());
        for (size_t i = 0; i < nw; ++i) mix(uint64_t(p[i]));
    }
    mix(e->t);
    *out = h;
    return OCTGPU_OK;
}

namespace {

int run_measure(octgpu_engine* e) {
    int rc = use_device(e);
    if (rc) return rc;
    CK(launch_measure(e->w, e->planes[e->pcur], e->geom(), e->X, e->scratch, e->res_dev, e->stream));
    e->launches += 3;
    CK(cudaMemcpyAsync(e->res_host, e->res_dev, sizeof(MeasureResult), cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    const MeasureResult& r = *e->res_host;
    // reconstruct_heights' checks, in its order (slope_field.hpp:209-226)
    if (r.curl_count) {
        const uint64_t x = r.curl_first % e->X, y = r.curl_first / e->X;
        return fail(OCTGPU_ERR_INVARIANT, "curl violation at plaquette (" + std::to_string(x) + "," +
                                              std::to_string(y) + "); " + std::to_string(r.curl_count) +
                                              " plaquettes inconsistent");
    }
    if (r.row0_sum != 0) return fail(OCTGPU_ERR_INVARIANT, "row 0 of sigma_x- does not balance to zero");
    // curl-free => all column sums are equal, so column 0 is the first failing one
    if (r.col0_sum != 0) return fail(OCTGPU_ERR_INVARIANT, "column 0 of sigma_y- does not balance to zero");
    return OCTGPU_OK;
}

}  // namespace

namespace {
// MeasurementRecord from the exact sums S_k = sum h^k (measure.cpp:24-56 semantics):
// mean = S1/N exactly rounded (the reference's double sum is exact here); central
// moments about the nearest integer c, exact in int128, then one extended-precision
// correction for d = mean - c (|d| <= 1/2).
void fill_moments(uint64_t t, uint64_t N, const __int128 S[4], octgpu_moments* out) {
    out->t = t;
    out->n_sites = N;
    for (int k = 0; k < 4; ++k) {
        out->s_lo[k] = uint64_t((unsigned __int128)S[k]);
        out->s_hi[k] = int64_t((unsigned __int128)S[k] >> 64);
    }
    out->mean_h = double(S[0]) / double(N);
    const __int128 NN = N;
    __int128 c = S[0] / NN;
    if (2 * (S[0] - c * NN) > NN) c += 1;
    if (2 * (S[0] - c * NN) < -NN) c -= 1;
    const __int128 c2 = c * c, c3 = c2 * c, c4 = c3 * c;
    const __int128 T1 = S[0] - c * NN;
    const __int128 T2 = S[1] - 2 * c * S[0] + c2 * NN;
    const __int128 T3 = S[2] - 3 * c * S[1] + 3 * c2 * S[0] - c3 * NN;
    const __int128 T4 = S[3] - 4 * c * S[2] + 6 * c2 * S[1] - 4 * c3 * S[0] + c4 * NN;
    const long double n = (long double)N;
    const long double d = (long double)T1 / n;
    const long double t2 = (long double)T2 / n, t3 = (long double)T3 / n, t4 = (long double)T4 / n;
    const bool flat = (NN * T2 == T1 * T1);  // m2 == 0 exactly
    const long double m2 = flat ? 0.0L : t2 - d * d;
    const long double m3 = t3 - 3 * d * t2 + 2 * d * d * d;
    const long double m4 = t4 - 4 * d * t3 + 6 * d * d * t2 - 3 * d * d * d * d;
    out->W2 = double(m2);
    if (!flat && m2 > 0) {
        out->skew = double(m3 / powl(m2, 1.5L));
        out->kurt = double(m4 / (m2 * m2) - 3.0L);
    } else {
        out->skew = NAN;
        out->kurt = NAN;
    }
}
}  // namespace

int octgpu_stripes_combine(const octgpu_stripe_moments* parts, uint32_t n_parts, uint32_t X, uint32_t Y,
                           octgpu_moments* out) {
    // parts in row order (SweepPlan order; parts[0] holds global row 0), as StripeGroup and the C++
    // GpuStripeGroup pass them; reconstruct_heights' checks in its order (slope_field.hpp:209-226)
    if (!parts || !out || n_parts == 0) return fail(OCTGPU_ERR_CONFIG, "null argument / no stripes");
    uint64_t N = 0, curl = 0, first = ~0ull;
    for (uint32_t i = 0; i < n_parts; ++i) {
        N += parts[i].n_sites;
        curl += parts[i].curl_count;
        if (parts[i].curl_count && parts[i].curl_first < first) first = parts[i].curl_first;
    }
    if (N != uint64_t(X) * Y) return fail(OCTGPU_ERR_CONFIG, "stripes do not cover the lattice");
    if (curl)
        return fail(OCTGPU_ERR_INVARIANT, "curl violation at plaquette (" + std::to_string(first % X) + "," +
                                              std::to_string(first / X) + "); " + std::to_string(curl) +
                                              " plaquettes inconsistent");
    if (parts[0].row_first_sum != 0) return fail(OCTGPU_ERR_INVARIANT, "row 0 of sigma_x- does not balance to zero");
    long long col = 0;
    for (uint32_t i = 0; i < n_parts; ++i) col += parts[i].col_sum;
    if (col != 0) return fail(OCTGPU_ERR_INVARIANT, "column 0 of sigma_y- does not balance to zero");
    // h_global = h_local + c on each stripe, c = (sum of col_sum above) - sigma_y-(0, 0)
    const long long sigma00 = parts[0].sy_first;
    __int128 S[4] = {0, 0, 0, 0};
    long long prefix = 0;
    for (uint32_t i = 0; i < n_parts; ++i) {
        const octgpu_stripe_moments& m = parts[i];
        const __int128 c = prefix - sigma00;
        __int128 loc[5] = {(__int128)m.n_sites, 0, 0, 0, 0};
        for (int k = 0; k < 4; ++k) loc[k + 1] = i128_of(m.s_lo[k], m.s_hi[k]);
        static const int C[5][5] = {{1}, {1, 1}, {1, 2, 1}, {1, 3, 3, 1}, {1, 4, 6, 4, 1}};
        for (int k = 1; k <= 4; ++k) {
            __int128 acc = 0, cp = 1;  // sum_j C(k,j) c^(k-j) loc_j, j = k..0
            for (int j = k; j >= 0; --j) {
                acc += C[k][j] * cp * loc[j];
                cp *= c;
            }
            S[k - 1] += acc;
        }
        prefix += m.col_sum;
    }
    fill_moments(parts[0].t, N, S, out);
    return OCTGPU_OK;
}

int octgpu_measure(octgpu_engine* e, octgpu_moments* out) {
    if (!e || !out) return fail(OCTGPU_ERR_CONFIG, "null argument");
    if (e->stripe) return fail(OCTGPU_ERR_CONFIG, "octgpu_measure is not available on a row stripe (use the octgpu_stripe_* calls)");
    int rc = run_measure(e);
    if (rc) return rc;
    const MeasureResult& r = *e->res_host;
    const uint64_t N = uint64_t(e->X) * e->L;
    __int128 S[4];
    for (int k = 0; k < 4; ++k) S[k] = i128_of(r.s_lo[k], r.s_hi[k]);
    fill_moments(e->t, N, S, out);
    return OCTGPU_OK;
}

int octgpu_heights(octgpu_engine* e, int32_t* out) {
    if (!e || !out) return fail(OCTGPU_ERR_CONFIG, "null argument");
    if (e->stripe) return fail(OCTGPU_ERR_CONFIG, "octgpu_heights is not available on a row stripe (use the octgpu_stripe_* calls)");
    int rc = run_measure(e);
    if (rc) return rc;
    const size_t bytes = size_t(e->X) * e->L * sizeof(int32_t);
    int32_t* d = nullptr;
    CK(cudaMalloc(&d, bytes));
    cudaError_t le = launch_heights(e->w, e->planes[e->pcur], e->geom(), e->X, e->scratch, d, e->stream);
    ++e->launches;
    if (le == cudaSuccess) le = cudaMemcpyAsync(out, d, bytes, cudaMemcpyDeviceToHost, e->stream);
    if (le == cudaSuccess) le = cudaStreamSynchronize(e->stream);
    cudaFree(d);
    if (le != cudaSuccess) return cuda_fail(le, "heights");
    return OCTGPU_OK;
}

int octgpu_balances(octgpu_engine* e, int64_t* rows_out, int64_t* cols_out) {
    if (!e || (!rows_out && !cols_out)) return fail(OCTGPU_ERR_CONFIG, "null argument");
    int rc = use_device(e);
    if (rc) return rc;
    // periodic: rows 0..Y-1 in order; stripe: its core rows (global rows y0 .. y0 + L - 1)
    const uint32_t r0 = e->first_row(), R = e->L;
    const Geom g = e->geom();
    long long* d = nullptr;
    const size_t nr = rows_out ? R : 0, nc = cols_out ? e->X : 0;
    CK(cudaMalloc(&d, (nr + 2 * nc) * sizeof(long long)));
    cudaError_t le = launch_balances(e->w, e->planes[e->pcur], g, r0, R, e->X, rows_out ? d : nullptr,
                                     cols_out ? d + nr : nullptr, d + nr + nc, e->stream);
    e->launches += (rows_out ? 1 : 0) + (cols_out ? 2 : 0);
    if (le == cudaSuccess && rows_out)
        le = cudaMemcpyAsync(rows_out, d, nr * sizeof(long long), cudaMemcpyDeviceToHost, e->stream);
    if (le == cudaSuccess && cols_out)
        le = cudaMemcpyAsync(cols_out, d + nr, nc * sizeof(long long), cudaMemcpyDeviceToHost, e->stream);
    if (le == cudaSuccess) le = cudaStreamSynchronize(e->stream);
    cudaFree(d);
    if (le != cudaSuccess) return cuda_fail(le, "balances");
    return OCTGPU_OK;
}

// ---------------------------------------------------------------------------
// Row stripes (multi-GPU): see include/octgpu.h

int octgpu_stripe_sizes(const octgpu_engine* e, uint64_t* to_prev, uint64_t* to_next, uint64_t* boundary) {
    if (!e || !e->stripe) return fail(OCTGPU_ERR_CONFIG, "not a row stripe");
    const uint64_t row = 4ull * e->n * e->word_bytes() + 32;  // 4 plane-rows + the row's rng state
    if (to_prev) *to_prev = kStripeHB * row;
    if (to_next) *to_next = kStripeHA * row;
    if (boundary) *boundary = uint64_t(e->n) * e->word_bytes();
    return OCTGPU_OK;
}

int octgpu_halo_pack(octgpu_engine* e, void* to_prev, void* to_next) {
    if (!e || !e->stripe || !to_prev || !to_next) return fail(OCTGPU_ERR_CONFIG, "not a row stripe / null buffer");
    int rc = use_device(e);
    if (rc) return rc;
    const Geom g = e->geom();
    // first HB core rows (+ states) become the next-lower rank's halo rows below
    CK(launch_rows_gather(e->w, e->planes[e->pcur], e->rng[e->rcur], g, kStripeHA, kStripeHB, to_prev, e->stream));
    // last HA core rows (+ states) become the next-higher rank's halo rows above
    CK(launch_rows_gather(e->w, e->planes[e->pcur], e->rng[e->rcur], g, e->L, kStripeHA, to_next, e->stream));
    e->launches += 2;
    return OCTGPU_OK;
}

int octgpu_halo_unpack(octgpu_engine* e, const void* from_prev, const void* from_next) {
    if (!e || !e->stripe || !from_prev || !from_next) return fail(OCTGPU_ERR_CONFIG, "not a row stripe / null buffer");
    int rc = use_device(e);
    if (rc) return rc;
    const Geom g = e->geom();
    CK(launch_rows_scatter(e->w, e->planes[e->pcur], e->rng[e->rcur], g, 0, kStripeHA, from_prev, e->stream));
    CK(launch_rows_scatter(e->w, e->planes[e->pcur], e->rng[e->rcur], g, kStripeHA + e->L, kStripeHB, from_next,
                           e->stream));
    e->launches += 2;
    return OCTGPU_OK;
}

namespace {
// k_mcs_deep can carry a stripe through 2 MCS per halo exchange (constant-xi modes)
bool stripe_deep_ok(const octgpu_engine* e, const ProbDev& p, const ProbDev& q) {
    // xoshiro: constant xi only (a live deep pass would not advance the halo rows' streams, which p2p.cu
    // relies on); counter streams have no state, so every cheap mode qualifies
    // The size threshold uses the WHOLE lattice (X * Ytot), a quantity every stripe of a group shares: with
    // the stripe's own row count, an uneven SweepPlan split straddling the threshold would give ranks
    // different pass lengths (a hang with NCCL, drifting pass counters over peer memory).
    const bool size_ok = e->deep == 2 || uint64_t(e->X) * e->Ytot >= (uint64_t(1) << 28);
    const bool xi_ok = e->rng_kind == OCTGPU_RNG_COUNTER || (is_const(p) && is_const(q));
    return e->deep && size_ok && e->mcs_impl == 2 && mcs_deep_supported(p.mode, q.mode) && xi_ok;
}

// sweeps of a stripe pass of n_mcs MCS: 0 = the one-MCS kernel; 4 / 6 = k_mcs_deep (2 MCS for cheap modes with
// constant xi or counter streams, 3 where the kernel takes L = 6). -1: not a valid pass length.
int stripe_pass_sweeps(const octgpu_engine* e, const ProbDev& p, const ProbDev& q, uint32_t n_mcs) {
    if (n_mcs == 1) return 0;
    if (!stripe_deep_ok(e, p, q)) return -1;
    const bool ctr = e->rng_kind == OCTGPU_RNG_COUNTER;
    if (n_mcs == 2) return kDeepSweepsLive;
    if (n_mcs == 3 && deep_sweeps(e, p, q, ctr) == kDeepSweepsConst) return kDeepSweepsConst;
    return -1;
}

// one fused stripe pass with counter-based xi (ls = 0: k_mcs_bulk<CTR>, else k_mcs_deep<CTR> of ls sweeps)
int stripe_kernel_ctr(octgpu_engine* e, const ProbDev& p, const ProbDev& q, int ls) {
    const bool deep = ls > 0;
    const Geom g = e->geom();
    const int ps = e->pcur;
    if (deep) {
        int rc = ensure_tmaps_deep(e);
        if (rc) return rc;
        CK(launch_mcs_deep_ctr(e->planes[ps], e->planes[ps ^ 1], e->phase, g, p, q, e->master_seed, 2 * e->t, ls,
                               deep_ring(e, p, q, ls, true), &e->tmd[ps][0], &e->tmd[ps][1], e->stream));
    } else {
        int rc = plan_bulk(e, p, q);
        if (rc) return rc;
        if (e->bulk_ks != 2) return fail(OCTGPU_ERR_CONFIG, "the counter-based rng needs OCTGPU_MCS_KS=2");
        CK(launch_mcs_bulk_ctr(e->planes[ps], e->planes[ps ^ 1], e->phase, g, p, q, e->master_seed, 2 * e->t,
                               e->bulk_S, &e->tm[ps][0], &e->tm[ps][1], e->stream));
    }
    return OCTGPU_OK;
}
}  // namespace

int octgpu_pass_plan(octgpu_engine* e, const octgpu_params* prm, int* kernel, int* sweeps_per_launch) {
    if (!e || !kernel || !sweeps_per_launch) return fail(OCTGPU_ERR_CONFIG, "null engine / output");
    ProbDev p, q;
    const int rc = lower_params(prm, p, q);
    if (rc) return rc;
    const bool ctr = e->rng_kind == OCTGPU_RNG_COUNTER;
    int k = e->mcs_impl == 2 ? OCTGPU_KERNEL_BULK : OCTGPU_KERNEL_MCS, ls = 2;
    if (e->stripe) {
        if (stripe_deep_ok(e, p, q)) {
            k = OCTGPU_KERNEL_DEEP;
            ls = deep_sweeps(e, p, q, ctr);
        }
    } else {
        const uint64_t D = draws(prm->p, e->w) + (q.mode != M_ZERO ? draws(prm->q, e->w) : 0);
        if (deep_policy(e, p, q, D, ctr)) {
            k = OCTGPU_KERNEL_DEEP;
            ls = deep_sweeps(e, p, q, ctr);
        } else if (ctr && !(e->mcs_impl == 2 && e->bulk_ks == 2)) {
            k = OCTGPU_KERNEL_SWEEP;
            ls = 1;
        }
    }
    *kernel = k;
    *sweeps_per_launch = ls;
    return OCTGPU_OK;
}

int octgpu_stripe_max_mcs(octgpu_engine* e, const octgpu_params* prm) {
    if (!e || !e->stripe) {
        fail(OCTGPU_ERR_CONFIG, "not a row stripe");
        return 0;
    }
    ProbDev p, q;
    if (lower_params(prm, p, q)) return 0;
    return stripe_deep_ok(e, p, q) ? deep_sweeps(e, p, q, e->rng_kind == OCTGPU_RNG_COUNTER) / 2 : 1;
}

int octgpu_stripe_mcs_n(octgpu_engine* e, const octgpu_params* prm, uint32_t n_mcs, void* boundary_out) {
    if (!e || !e->stripe || !boundary_out) return fail(OCTGPU_ERR_CONFIG, "not a row stripe / null buffer");
    ProbDev p, q;
    int rc = lower_params(prm, p, q);
    if (!rc) rc = use_device(e);
    if (rc) return rc;
    const int ls = stripe_pass_sweeps(e, p, q, n_mcs);
    if (ls < 0)
        return fail(OCTGPU_ERR_CONFIG, "a stripe pass covers 1 MCS, or up to octgpu_stripe_max_mcs() with constant "
                                       "xi (2 or 3)");
    const bool deep = ls > 0;
    const bool ctr = e->rng_kind == OCTGPU_RNG_COUNTER;
    const bool live = !ctr && !(is_const(p) && is_const(q));
    const uint64_t D = draws(prm->p, e->w) + (q.mode != M_ZERO ? draws(prm->q, e->w) : 0);
    const uint64_t per_sweep = uint64_t(e->n) * D;
    uint64_t* jtab = nullptr;
    if (live) {
        rc = materialize(e);
        if (!rc) rc = get_table(e, per_sweep, &jtab);
        if (rc) return rc;
    }
    const Geom g = e->geom();
    const int ps = e->pcur, rs = e->rcur;
    if (ctr) {
        rc = stripe_kernel_ctr(e, p, q, ls);
        if (rc) return rc;
    } else if (deep) {
        rc = ensure_tmaps_deep(e);
        if (rc) return rc;
        CK(launch_mcs_deep(e->planes[ps], e->planes[ps ^ 1], e->rng[rs], e->rng[rs ^ 1], e->phase, g, p, q, jtab, ls,
                           deep_ring(e, p, q, ls), &e->tmd[ps][0], &e->tmd[ps][1], e->stream));
    } else if (e->mcs_impl == 2) {
        rc = plan_bulk(e, p, q);
        if (rc) return rc;
        CK(launch_mcs_bulk(e->planes[ps], e->planes[ps ^ 1], e->rng[rs], e->rng[rs ^ 1], e->phase, g, p, q, jtab,
                           e->bulk_ks, e->bulk_S, &e->tm[ps][0], &e->tm[ps][1], e->stream));
    } else
        CK(launch_mcs(e->w, e->planes[ps], e->planes[ps ^ 1], e->rng[rs], e->rng[rs ^ 1], e->phase, g, p, q, live,
                      jtab, e->stream));
    // Y(f) of the first halo row below is final here (its own f sweeps + the s sweeps of
    // our last core row): the next rank's first core row, which its own pass never writes
    CK(launch_planerow_copy(e->w, e->planes[ps ^ 1], 2 + e->phase, g, kStripeHA + e->L, boundary_out, true,
                            e->stream));
    e->launches += 2;
    e->pcur ^= 1;
    if (live)
        e->rcur ^= 1;
    else if (!ctr)
        e->pending += 2 * uint64_t(n_mcs) * per_sweep;
    e->t += n_mcs;
    return OCTGPU_OK;
}

int octgpu_stripe_mcs(octgpu_engine* e, const octgpu_params* prm, void* boundary_out) {
    return octgpu_stripe_mcs_n(e, prm, 1, boundary_out);
}

int octgpu_stripe_finish(octgpu_engine* e, const void* boundary_in) {
    if (!e || !e->stripe || !boundary_in) return fail(OCTGPU_ERR_CONFIG, "not a row stripe / null buffer");
    int rc = use_device(e);
    if (rc) return rc;
    CK(launch_planerow_copy(e->w, e->planes[e->pcur], 2 + e->phase, e->geom(), kStripeHA,
                            const_cast<void*>(boundary_in), false, e->stream));
    ++e->launches;
    return OCTGPU_OK;
}

int octgpu_measure_stripe(octgpu_engine* e, octgpu_stripe_moments* out) {
    if (!e || !e->stripe || !out) return fail(OCTGPU_ERR_CONFIG, "not a row stripe / null output");
    int rc = use_device(e);
    if (rc) return rc;
    CK(launch_measure(e->w, e->planes[e->pcur], e->geom(), e->X, e->scratch, e->res_dev, e->stream));
    e->launches += 3;
    CK(cudaMemcpyAsync(e->res_host, e->res_dev, sizeof(MeasureResult), cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    rc = octgpu_sync(e);  // reports a timed-out peer halo wait
    if (rc) return rc;
    const MeasureResult& r = *e->res_host;
    out->t = e->t;
    out->n_sites = uint64_t(e->X) * e->L;
    for (int k = 0; k < 4; ++k) {
        out->s_lo[k] = r.s_lo[k];
        out->s_hi[k] = r.s_hi[k];
    }
    out->col_sum = r.col0_sum;
    out->sy_first = r.sy_first;
    out->row_first_sum = r.row0_sum;
    out->curl_count = r.curl_count;
    out->curl_first = r.curl_count ? r.curl_first + uint64_t(e->y0) * e->X : ~0ull;
    return OCTGPU_OK;
}

// ---------------------------------------------------------------------------
// Device-side halo exchange over peer memory (p2p.cu)

namespace {
struct IpcBlob {
    cudaIpcMemHandle_t h[5];  // planes[0], planes[1], rng[0], rng[1], done
    uint32_t alloc_rows, rows, n, w;
    int32_t device;
};
static_assert(sizeof(IpcBlob) <= OCTGPU_IPC_BYTES, "IPC blob");

PeerView peer_view(const octgpu_engine* e, const octgpu_peer& p) {
    return PeerView{reinterpret_cast<const void*>(p.planes[e->pcur]), reinterpret_cast<const uint64_t*>(p.rng[e->rcur]),
                    reinterpret_cast<const uint64_t*>(p.done), p.alloc_rows, p.rows, e->p2p_timeout};
}

int p2p_pull(octgpu_engine* e, bool with_rng) {
    CK(launch_halo_pull(e->w, e->planes[e->pcur], e->rng[e->rcur], e->geom(), peer_view(e, e->prev),
                        peer_view(e, e->next), e->passes, e->p2p_err, with_rng, e->stream));
    ++e->launches;
    return OCTGPU_OK;
}

}  // namespace

int octgpu_stripe_peer(const octgpu_engine* e, octgpu_peer* out) {
    if (!e || !e->stripe || !out) return fail(OCTGPU_ERR_CONFIG, "not a row stripe / null output");
    *out = octgpu_peer{};
    for (int i = 0; i < 2; ++i) {
        out->planes[i] = reinterpret_cast<uint64_t>(e->planes[i]);
        out->rng[i] = reinterpret_cast<uint64_t>(e->rng[i]);
    }
    out->done = reinterpret_cast<uint64_t>(e->done);
    out->alloc_rows = e->Y;
    out->rows = e->L;
    out->n = e->n;
    out->w = e->w;
    out->device = e->device;
    return OCTGPU_OK;
}

int octgpu_stripe_ipc_export(const octgpu_engine* e, void* out) {
    if (!e || !e->stripe || !out) return fail(OCTGPU_ERR_CONFIG, "not a row stripe / null output");
    IpcBlob b{};
    CK(cudaSetDevice(e->device));
    void* ptrs[5] = {e->planes[0], e->planes[1], e->rng[0], e->rng[1], e->done};
    for (int i = 0; i < 5; ++i) CK(cudaIpcGetMemHandle(&b.h[i], ptrs[i]));
    b.alloc_rows = e->Y;
    b.rows = e->L;
    b.n = e->n;
    b.w = e->w;
    b.device = e->device;
    std::memset(out, 0, OCTGPU_IPC_BYTES);
    std::memcpy(out, &b, sizeof(b));
    return OCTGPU_OK;
}

int octgpu_stripe_ipc_open(octgpu_engine* e, const void* blob, octgpu_peer* out) {
    if (!e || !e->stripe || !blob || !out) return fail(OCTGPU_ERR_CONFIG, "not a row stripe / null argument");
    IpcBlob b;
    std::memcpy(&b, blob, sizeof(b));
    CK(cudaSetDevice(e->device));
    void* ptrs[5];
    for (int i = 0; i < 5; ++i) {
        CK(cudaIpcOpenMemHandle(&ptrs[i], b.h[i], cudaIpcMemLazyEnablePeerAccess));
        e->ipc_opened.push_back(ptrs[i]);
    }
    *out = octgpu_peer{};
    for (int i = 0; i < 2; ++i) {
        out->planes[i] = reinterpret_cast<uint64_t>(ptrs[i]);
        out->rng[i] = reinterpret_cast<uint64_t>(ptrs[2 + i]);
    }
    out->done = reinterpret_cast<uint64_t>(ptrs[4]);
    out->alloc_rows = b.alloc_rows;
    out->rows = b.rows;
    out->n = b.n;
    out->w = b.w;
    out->device = b.device;
    return OCTGPU_OK;
}

int octgpu_stripe_connect(octgpu_engine* e, const octgpu_peer* prev, const octgpu_peer* next) {
    if (!e || !e->stripe || !prev || !next) return fail(OCTGPU_ERR_CONFIG, "not a row stripe / null peer");
    if (e->mcs_impl != 2)
        return fail(OCTGPU_ERR_CONFIG, "the peer-memory halo exchange needs w = 64 and X >= 1024 (TMA kernels)");
    for (const octgpu_peer* p : {prev, next}) {
        if (p->n != e->n || p->w != e->w) return fail(OCTGPU_ERR_CONFIG, "peer stripe has a different row width");
        if (p->rows < kStripeHB) return fail(OCTGPU_ERR_CONFIG, "peer stripe holds fewer rows than the halo");
    }
    int rc = use_device(e);
    if (rc) return rc;
    for (const octgpu_peer* p : {prev, next})
        if (p->device != e->device) {
            const cudaError_t pe = cudaDeviceEnablePeerAccess(p->device, 0);
            if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) CK(pe);
            cudaGetLastError();
        }
    if (e->pending) return fail(OCTGPU_ERR_CONFIG, "connect stripes before stepping them");
    e->prev = *prev;
    e->next = *next;
    e->p2p = true;
    // Fused passes leave the boundary blocks waiting inside the MCS kernel: right when each stripe has its own
    // GPU; stripes sharing one GPU (streams / processes time-sharing its SMs) would hold SM slots the awaited
    // neighbour needs (measured on one B200: 3 launches +1.7 / +3.3 / +6.0% vs fused +21 / +21 / +18% per MCS
    // over the periodic engine at 2 / 4 / 8 stripes, tools/stripe_overhead.py).
    if (e->fused_link < 0) e->fused_link = (prev->device != e->device || next->device != e->device) ? 1 : 0;
    return p2p_pull(e, true);  // halo rows with their streams; later passes advance those streams locally
}

int octgpu_stripe_disconnect(octgpu_engine* e) {
    if (!e || !e->stripe) return fail(OCTGPU_ERR_CONFIG, "not a row stripe");
    int rc = use_device(e);
    if (rc) return rc;
    CK(cudaStreamSynchronize(e->stream));
    for (void* ptr : e->ipc_opened) CK(cudaIpcCloseMemHandle(ptr));
    e->ipc_opened.clear();
    e->p2p = false;
    e->prev = e->next = octgpu_peer{};
    e->fused_link = e->fused_link_env;  // decided again at the next connect
    return OCTGPU_OK;
}

int octgpu_stripe_pull(octgpu_engine* e) {
    if (!e || !e->stripe || !e->p2p) return fail(OCTGPU_ERR_CONFIG, "not a connected row stripe");
    int rc = use_device(e);
    if (rc) return rc;
    return p2p_pull(e, false);
}

namespace {
// One fused 2-MCS stripe pass (constant xi or counter streams: no stream state crosses the stripe boundary).
int stripe_pass_fused(octgpu_engine* e, const ProbDev& p, const ProbDev& q, bool ctr, bool live,
                      uint64_t per_sweep, int ls) {
    const Geom g = e->geom();
    const int ps = e->pcur, rs = e->rcur;
    StripeLink lk{};
    lk.prev = peer_view(e, e->prev);
    lk.next = peer_view(e, e->next);
    lk.need = e->passes;
    lk.err = e->p2p_err;
    lk.done = e->done;
    lk.ticket = reinterpret_cast<uint32_t*>(e->done + 1);
    lk.value = e->passes + 1;
    lk.next_planes = reinterpret_cast<void*>(e->next.planes[ps ^ 1]);
    lk.next_Y = e->next.alloc_rows;
    lk.push_plane = 2 + e->phase;
    lk.active = 1;
    uint64_t* jtab = nullptr;
    if (live) {  // lazy stream advance: no neighbour reads our states after connect
        int rc = materialize(e);
        if (!rc) rc = get_table(e, per_sweep, &jtab);
        if (rc) return rc;
    }
    if (ls > 0) {  // k_mcs_deep, 2 or 3 MCS
        int rc = ensure_tmaps_deep(e);
        if (rc) return rc;
        if (ctr)
            CK(launch_mcs_deep_ctr(e->planes[ps], e->planes[ps ^ 1], e->phase, g, p, q, e->master_seed, 2 * e->t, ls,
                                   deep_ring(e, p, q, ls, true), &e->tmd[ps][0], &e->tmd[ps][1], e->stream, &lk));
        else
            CK(launch_mcs_deep(e->planes[ps], e->planes[ps ^ 1], e->rng[rs], e->rng[rs ^ 1], e->phase, g, p, q,
                               nullptr, ls, deep_ring(e, p, q, ls), &e->tmd[ps][0], &e->tmd[ps][1], e->stream, &lk));
    } else {  // k_mcs_bulk, one MCS
        int rc = plan_bulk(e, p, q);
        if (rc) return rc;
        if (ctr) {
            if (e->bulk_ks != 2) return fail(OCTGPU_ERR_CONFIG, "the counter-based rng needs OCTGPU_MCS_KS=2");
            CK(launch_mcs_bulk_ctr(e->planes[ps], e->planes[ps ^ 1], e->phase, g, p, q, e->master_seed, 2 * e->t,
                                   e->bulk_S, &e->tm[ps][0], &e->tm[ps][1], e->stream, &lk));
        } else {
            CK(launch_mcs_bulk(e->planes[ps], e->planes[ps ^ 1], e->rng[rs], e->rng[rs ^ 1], e->phase, g, p, q, jtab,
                               e->bulk_ks, e->bulk_S, &e->tm[ps][0], &e->tm[ps][1], e->stream, &lk));
        }
    }
    const uint64_t mcs = ls > 0 ? uint64_t(ls / 2) : 1;
    ++e->launches;
    e->pcur ^= 1;
    if (live)
        e->rcur ^= 1;
    else if (!ctr)
        e->pending += 2 * mcs * per_sweep;
    e->t += mcs;
    ++e->passes;
    return OCTGPU_OK;
}
}  // namespace

int octgpu_stripe_pass(octgpu_engine* e, const octgpu_params* prm, uint32_t n_mcs) {
    if (!e || !e->stripe || !e->p2p) return fail(OCTGPU_ERR_CONFIG, "not a connected row stripe");
    ProbDev p, q;
    int rc = lower_params(prm, p, q);
    if (!rc) rc = use_device(e);
    if (rc) return rc;
    const int ls = stripe_pass_sweeps(e, p, q, n_mcs);
    if (ls < 0)
        return fail(OCTGPU_ERR_CONFIG, "a stripe pass covers 1 MCS, or up to octgpu_stripe_max_mcs() with constant "
                                       "xi (2 or 3)");
    const bool deep = ls > 0;
    const bool ctr = e->rng_kind == OCTGPU_RNG_COUNTER;
    const bool live = !ctr && !(is_const(p) && is_const(q));
    const uint64_t D = draws(prm->p, e->w) + (q.mode != M_ZERO ? draws(prm->q, e->w) : 0);
    const uint64_t per_sweep = uint64_t(e->n) * D;
    // ONE launch with the halo exchange fused into the MCS kernel (stripe_link.cuh) when a neighbour is on another
    // GPU; otherwise pull, kernel, push + signal (p2p.cu)
    if (e->fused_link == 1 && e->mcs_impl == 2) return stripe_pass_fused(e, p, q, ctr, live, per_sweep, ls);
    // 1. wait for the neighbours' previous pass, pull their boundary rows
    rc = p2p_pull(e, false);
    if (rc) return rc;
    // 2. lazy stream advance (after the wait: no neighbour reads our states any more)
    uint64_t* jtab = nullptr;
    if (live) {
        rc = materialize(e);
        if (!rc) rc = get_table(e, per_sweep, &jtab);
        if (rc) return rc;
    }
    // 3. the MCS kernel
    const Geom g = e->geom();
    const int ps = e->pcur, rs = e->rcur;
    if (ctr) {
        rc = stripe_kernel_ctr(e, p, q, ls);
        if (rc) return rc;
    } else if (deep) {
        rc = ensure_tmaps_deep(e);
        if (rc) return rc;
        CK(launch_mcs_deep(e->planes[ps], e->planes[ps ^ 1], e->rng[rs], e->rng[rs ^ 1], e->phase, g, p, q, jtab, ls,
                           deep_ring(e, p, q, ls), &e->tmd[ps][0], &e->tmd[ps][1], e->stream));
    } else {
        rc = plan_bulk(e, p, q);
        if (rc) return rc;
        CK(launch_mcs_bulk(e->planes[ps], e->planes[ps ^ 1], e->rng[rs], e->rng[rs ^ 1], e->phase, g, p, q, jtab,
                           e->bulk_ks, e->bulk_S, &e->tm[ps][0], &e->tm[ps][1], e->stream));
    }
    e->pcur ^= 1;
    if (live)
        e->rcur ^= 1;
    else if (!ctr)
        e->pending += 2 * uint64_t(n_mcs) * per_sweep;
    e->t += n_mcs;
    ++e->passes;
    // 4. the boundary plane-row into the next stripe's new plane set, then publish the pass
    CK(launch_push_signal(e->w, e->planes[e->pcur], 2 + e->phase, g,
                          reinterpret_cast<void*>(e->next.planes[e->pcur]), e->next.alloc_rows, e->done, e->passes,
                          e->stream));
    e->launches += 2;
    return OCTGPU_OK;
}

uint32_t octgpu_stripe_y0(const octgpu_engine* e) { return e ? e->y0 : 0; }
uint32_t octgpu_stripe_rows(const octgpu_engine* e) { return e ? e->L : 0; }

}  // extern "C"
