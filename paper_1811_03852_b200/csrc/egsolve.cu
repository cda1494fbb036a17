// egsolve.cu — the C ABI (include/egsolve.h) over the sm_100a kernels in kernels.cuh.
//
// Host responsibilities only: validation, workspace carving, launch geometry, the restart /
// verification state machine of DESIGN.md §Algorithm (mirrors), CUDA-graph
// replay of the iteration, NCCL halo exchange and group-sum all-gather for latitude bands (or the
// in-process loopback transport that runs the same decomposition on one GPU for tests), and
// per-kernel CUDA-event profiling.  All arithmetic of the method runs in the kernels.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "egsolve.h"
#include "kernels.cuh"
#include "march.cuh"
#include "sor_tma.cuh"
#include "march64.cuh"

using namespace eg;

namespace {

enum KernelId {
    KID_SCALE = 0, KID_START, KID_FIN, KID_THOMAS_P, KID_STENCIL_A, KID_THOMAS_S, KID_STENCIL_B,
    KID_UPDATE, KID_APPLY, KID_PRECOND, KID_CONVERT, KID_PHASE_A, KID_PHASE_B, KID_SOR, KID_VERIFY, KID_UPDATE_X, KID_EDGE,
    KID_COUNT
};
const char* kKernelNames[KID_COUNT] = {"scale", "start", "finalize", "thomas_p", "stencil_dot_A",
                                       "thomas_s", "stencil_dot_B", "update_xr", "apply",
                                       "precondition", "convert", "phase_A", "phase_B", "trisor_half",
                                       "verify", "update_x", "edge_rows"};

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct Layout {
    size_t off_bands, off_diag, off_bhat, off_x64, off_x32, off_xg, off_vec, off_z, off_pv, off_slots, off_hslots,
        off_gsum, off_edge, off_p2p, off_state, base_total, off_split, off_batch, total;
    size_t vsz;      // sizeof(V)
    size_t xsz;      // sizeof(X)
    int64_t n, row, nyl;
    int tiles, G;
};

constexpr size_t kP2PGall = 2 * 48 * sizeof(unsigned long long);  // gather words [2][8][3][2]

int vsize(int mode) { return mode == EG_FP64 ? 8 : 4; }
int xsize(int mode) { return mode == EG_FP32 ? 4 : 8; }

bool make_layout(const eg_grid* g, int64_t nyl, int mode, Layout* L, uint32_t features = 0) {
    const size_t A = 256;
    L->row = g->nx * g->nz;
    L->nyl = nyl;
    L->n = nyl * L->row;
    L->vsz = vsize(mode);
    L->xsz = xsize(mode);
    L->tiles = (int)((g->nx + RW - 1) / RW);
    L->G = (int)std::min<int64_t>(8, g->ny);
    const size_t n = (size_t)L->n, row = (size_t)L->row;
    size_t o = 0;
    L->off_bands = o; o = align_up(o + 6 * n * L->vsz, A);
    L->off_diag = o;  o = align_up(o + n * 8, A);
    L->off_bhat = o;  o = align_up(o + n * 8, A);
    L->off_x64 = o;   o = align_up(o + n * 8, A);
    L->off_x32 = o;   o = align_up(o + (mode == EG_FP32 ? n * 4 : 0), A);
    L->off_xg = o;    o = align_up(o + 2 * row * 8, A);
    L->off_vec = o;   o = align_up(o + 6 * align_up(n * L->vsz, A), A);
    L->off_z = o;     o = align_up(o + 2 * align_up((n + 2 * row) * L->vsz, A), A);
    // ready flags of the fused phases: one per (row, tile) of 128 (fp32) or 64 (FP64) columns
    L->off_pv = o;    o = align_up(o + (size_t)nyl * ((g->nx + 63) / 64) * sizeof(int), A);
    // reduction slots per row: 128-column tiles (unfused kernels) or 64-longitude strips (phases)
    L->off_slots = o; o = align_up(o + 3 * (size_t)nyl * L->tiles * 8, A);
    // FP64 phase kernels: 4 warp sums per (row, 128-column slot) (march64.cuh)
    L->off_hslots = o; o = align_up(o + (mode == EG_FP64 ? 3 * 4 * (size_t)nyl * L->tiles * 8 : 0), A);
    L->off_gsum = o;  o = align_up(o + 2 * 8 * 3 * 8, A);
    // P2P transport (latitude bands): gather buffers [2][8][3][2] stamped words, the ghost-row
    // flags [z, z_s][side][64-column tiles] and the tri-SOR halo flags [2][side][tiles] — written by
    // the other ranks through peer memory — and this rank's tri-SOR halo counter
    L->off_p2p = o;   o = align_up(o + kP2PGall + (8 * (size_t)((g->nx + 63) / 64) + 4) * sizeof(int), A);
    // latitude bands: k_edge_rows' scratch rows [z, z_s][row 0, row nyl-1][row] and the band-edge
    // copies of p and v [p, v][row 0, row nyl-1][row] (fused schedule), then k_edge_stencil's arrival
    // counters [2 rows][tiles]
    L->off_edge = o;  o = align_up(o + 8 * row * L->vsz + 2 * (size_t)L->tiles * sizeof(int), A);
    L->off_state = o; o = align_up(o + sizeof(DevState), A);
    L->base_total = o;
    // EG_FEATURE_TRISOR: colour-split (E,W,N,S), (U,D) and f for the red-black tri-SOR sweeps
    // and the colour-split x of the fp32 TMA sweeps (ghosted rows: n + 2 rows)
    L->off_split = o; if (features & EG_FEATURE_TRISOR) o = align_up(o + (8 * n + 2 * row) * L->vsz, A);
    L->off_batch = o; if (features & EG_FEATURE_BATCH) o = align_up(o + 4 * n * 8, A);
    L->total = o;
    return true;
}

struct PendingEv { int kid; cudaEvent_t a, b; double bytes; };

}  // namespace

// In-process loopback transport (eg_loopback_id): the ranks of a latitude-band decomposition are
// handles in ONE process on ONE GPU, each driven by its own host thread, all created on the same
// stream.  An exchange posts this rank's buffers, meets the other ranks at a host barrier, enqueues
// device-to-device copies from the neighbours' buffers on the shared stream and meets them again
// (so no rank moves on and overwrites a posted buffer before everyone has enqueued its reads).
// Every kernel of every rank runs in enqueue order on that one stream: no kernel ever waits for
// another rank's kernel (B200_PROFILING.md: ranks must not spin on each other on one GPU).
struct LoopGroup {
    int n = 0;
    int refs = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    bool broken = false;
    bool have_st = false;
    cudaStream_t st = nullptr;
    std::vector<const unsigned char*> first, last;  // posted edge rows
    std::vector<const double*> gsum;                // posted group sums
    std::vector<unsigned char*> ws;                 // the ranks' workspaces (P2P transport)
    std::vector<int> split;                         // the ranks have the colour-split tri-SOR region
};
constexpr int kMaxIt = 1 << 26;  // epochs (8 per iteration at most) stay far below 2^31
constexpr char kLoopMagic[8] = {'E', 'G', 'L', 'O', 'O', 'P', 'B', 'K'};

// The fused phase kernels need every CTA of a launch resident (their CTAs wait on each other's
// ready flags).  Two of them launched concurrently from different streams of this process could
// each end up partly resident and wait forever, so solves that use them are serialised here
// (eg_solve is blocking: every kernel of a solve has finished when the lock is released).
// Loopback ranks share one stream already and meet at host barriers inside a solve: not locked.
// One lock per device: solves on different GPUs never compete for SMs (and NCCL ranks driven as
// threads of one process must not block each other).
constexpr int kMaxDevices = 64;
std::recursive_mutex g_fused_solve_mu[kMaxDevices];

// all n ranks arrive or the wait times out (a rank that failed never comes): false = broken group
bool lb_barrier(LoopGroup* G) {
    std::unique_lock<std::mutex> lk(G->m);
    if (G->broken) return false;
    const uint64_t my = G->gen;
    if (++G->arrived == G->n) {
        G->arrived = 0;
        ++G->gen;
        G->cv.notify_all();
        return true;
    }
    const bool ok = G->cv.wait_for(lk, std::chrono::seconds(120), [&] { return G->gen != my || G->broken; });
    if (!ok || G->broken) {
        G->broken = true;
        G->cv.notify_all();
        return false;
    }
    return true;
}

struct eg_solver {
    eg_grid grid{};
    int64_t j_begin = 0, j_end = 0;
    int rank = 0, nranks = 1;
    int mode = EG_MIXED;
    cudaStream_t st = nullptr;
    cudaStream_t cap_st = nullptr;  // private stream used only to capture the iteration graph
    Layout L{};
    Geo geo{};
    unsigned char* ws = nullptr;
    // carved pointers
    void* B4 = nullptr;    // [n][4] scaled (E, W, N, S)
    void* B2 = nullptr;    // [n][2] scaled (U, D)
    double* diag = nullptr;
    double* bhat = nullptr;
    double* x64 = nullptr;
    float* x32 = nullptr;
    double* xg = nullptr;  // [2][row] ghost rows of x (X-typed)
    void* vec[6]{};        // r, rh, p, v, s, t
    void* zext[2]{};       // ghosted z, zs (row -1 .. nyl)
    int* ready_flags = nullptr;  // [nyl][tiles] ready flags of the fused (marching) phase kernels
    bool use_march = false;     // fused phases (fp32 working precision; march.cuh)
    MarchGeo mg{};
    MarchMaps maps{};
    SorMaps sor_maps{};     // TMA maps of the fp32 tri-SOR sweeps (colour-split arrays)
    bool sor_tma = false;   // later tri-SOR sweeps on k_sor_tma (fp32, colour-split copies)
    SorMaps64 sor_maps64{};
    bool sor_tma64 = false; // later tri-SOR sweeps on k_sor_tma64 (FP64, colour-split copies)
    int nsm = 148;
    size_t smem_march = 0;
    int64_t epoch_base = 1;     // first epoch of the next solve (flags are reset before 2^30)
    int gseq = 0;               // DevState.gseq carried from solve to solve (P2P gather buffers)
    int device = 0;             // the CUDA device the handle was created on
    int precond = EG_PRECOND_TRIDIAG;  // NEXT-1: EG_PRECOND_TRISOR selects red-black tri-SOR
    void* split = nullptr;             // colour-split B4 | B2 | f for tri-SOR (NULL: not available)
    double* batch = nullptr;           // eg_solve_batch staging: b[2] | x[2] (NULL: not available)
    cudaStream_t cin = nullptr, cout = nullptr;  // eg_solve_batch copy streams (owned)
    cudaEvent_t ev_in[2]{}, ev_x[2]{}, ev_out[2]{};
    bool split_valid = false;          // the split bands match the current operator
    int sor_sweeps = 3;
    double sor_omega = 1.5;
    double* slots = nullptr;
    double* hslots = nullptr;    // FP64 phase kernels' half-slots [3][nyl][tiles][4]
    MarchMaps64 maps64{};        // TMA maps of the FP64 phase kernels
    double* gsum = nullptr;  // [G][3] local
    double* gall = nullptr;  // [G][3] all ranks
    DevState* dstate = nullptr;
    DevState* hstate = nullptr;  // pinned, mapped host mirror
    void* hstate_dev = nullptr;  // its device address
    int wth = 128;               // Thomas CTA width (columns)
    int cpt = 1;                 // columns per thread of the Thomas / update kernels (2 if nx even)
    bool update_kb2 = false;     // k_update with 2-level batches (more CTAs per SM; few-wave grids)
    bool pdl = false;            // programmatic dependent launches in the iteration (EG_PDL=1)
    bool split_update = false;   // x half of the update beside reduction 3 (NCCL / loopback-copy bands)
    size_t smem_th = 0;
    bool use_tm = false;         // fp32 Thomas with TMEM-resident factors (nz <= 128)
    bool use_tm64 = false;       // fp64 Thomas with TMEM-resident factors (nz <= 80)
    bool th_tma64 = false;       // fp64 phase-A Thomas on the TMA-fed kernel (nz <= 72; 6 % faster)
    ThomasMaps64 thmaps64{};
    size_t smem_tm = 0;
    // graphs of one iteration, keyed on the iterate pointer (two: eg_solve_batch alternates buffers)
    cudaGraphExec_t graphs[2]{};
    void* graphs_x[2]{};
    int graph_next = 0;  // entry replaced on the next miss
    cudaGraphExec_t graph = nullptr;  // the entry for the current solve
    void* graph_x = nullptr;
    // NCCL, or the loopback group (tests)
    ncclComm_t comm = nullptr;
    LoopGroup* lb = nullptr;
    // P2P transport: the producing kernels store ghost rows and group sums straight
    // into the other ranks' workspaces (NVLink peer memory opened by CUDA IPC, or the loopback
    // group's own buffers) and the consumers wait on epoch-stamped flags; no NCCL call, no copy in
    // the iteration.  p2p_want: EG_P2P != 0; pp.on once the peer table is built.
    bool p2p_want = false;
    P2P pp{};
    std::vector<void*> ipc_open;  // peer workspaces this handle opened (closed at destroy)
    // latitude bands: the ghost-row exchange runs on cst beside the phase kernel (ev_edge: the edge
    // rows are computed; ev_halo: the ghost rows have arrived); the x half of the update runs on xst
    // beside reduction 3 (ev_b: reduction 2 done; ev_xu: x updated)
    cudaStream_t cst = nullptr, xst = nullptr;
    cudaEvent_t ev_edge = nullptr, ev_halo = nullptr, ev_b = nullptr, ev_xu = nullptr;
    // profiling
    bool profiling = false;
    std::vector<cudaEvent_t> evpool;
    std::vector<PendingEv> pending;
    double prof_ms[KID_COUNT]{};
    double prof_bytes[KID_COUNT]{};  // algorithmic HBM bytes of the profiled launches
    int64_t prof_n[KID_COUNT]{};
    bool next_fresh = false;         // the next iteration starts from p = v = 0 (reads r only)
    bool next_xzero = false;         // the next update starts from x = 0 (does not read x)
    std::string err;
};

namespace {

int fail(eg_solver* s, int code, const char* fmt, ...) {
    if (s) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        s->err = buf;
    }
    return code;
}

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(s, EG_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,            \
                        cudaGetErrorString(e_));                                              \
    } while (0)

#define NK(call)                                                                              \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess)                                                                \
            return fail(s, EG_ERR_NCCL, "%s:%d %s: %s", __FILE__, __LINE__, #call,            \
                        ncclGetErrorString(r_));                                              \
    } while (0)

// -------- profiling helpers --------
cudaEvent_t take_event(eg_solver* s) {
    if (s->evpool.empty()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    cudaEvent_t e = s->evpool.back();
    s->evpool.pop_back();
    return e;
}

double alg_bytes(const eg_solver* s, int kid);
double start_bytes(const eg_solver* s, int entry, int xzero, bool write);
double sor_alg_bytes(const eg_solver* s, int kind, int sweep, int colour);

struct ProfScope {
    eg_solver* s;
    int kid;
    double bytes;
    cudaEvent_t a = nullptr;
    ProfScope(eg_solver* s_, int k, double b = -1.0) : s(s_), kid(k), bytes(b) {
        if (s->profiling) {
            a = take_event(s);
            cudaEventRecord(a, s->st);
        }
    }
    ~ProfScope() {
        if (s->profiling) {
            cudaEvent_t b = take_event(s);
            cudaEventRecord(b, s->st);
            s->pending.push_back({kid, a, b, bytes >= 0.0 ? bytes : alg_bytes(s, kid)});
        }
    }
};

void drain_profile(eg_solver* s) {
    for (auto& p : s->pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
            s->prof_ms[p.kid] += ms;
            s->prof_bytes[p.kid] += p.bytes;
            s->prof_n[p.kid] += 1;
        }
        s->evpool.push_back(p.a);
        s->evpool.push_back(p.b);
    }
    s->pending.clear();
}

template <int MODE>
Vecs<MODE> vecs(eg_solver* s, void* x_it) {
    using V = typename Prec<MODE>::V;
    using X = typename Prec<MODE>::X;
    Vecs<MODE> v;
    v.B4 = (const V*)s->B4;
    v.B2 = (const V*)s->B2;
    v.diag = s->diag;
    v.bhat = s->bhat;
    v.x = (X*)x_it;
    v.xg_lo = (const X*)s->xg;
    v.xg_hi = (const X*)((unsigned char*)s->xg + s->L.row * 8);
    v.r = (V*)s->vec[0]; v.rh = (V*)s->vec[1]; v.p = (V*)s->vec[2];
    v.v = (V*)s->vec[3]; v.s = (V*)s->vec[4]; v.t = (V*)s->vec[5];
    v.z = (V*)s->zext[0] + s->L.row;
    v.zs = (V*)s->zext[1] + s->L.row;
    v.slots = s->slots;
    v.st = s->dstate;
    return v;
}

// A cooperative launch (cudaLaunchAttributeCooperative, also as a captured graph kernel node): the
// runtime guarantees every CTA of the grid is resident at once, or fails the launch
// (cudaErrorCooperativeLaunchTooLarge) instead of letting CTAs that wait on other CTAs' ready flags
// hang.  Used for the fused phase kernels, whose CTAs wait on their neighbours' rows.
template <typename... Exp, typename... Act>
cudaError_t launch_ex(bool coop, bool pdl, void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                      Act&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (coop) {
        at[na].id = cudaLaunchAttributeCooperative;
        at[na].val.cooperative = 1;
        ++na;
    }
    if (pdl) {  // programmatic dependent launch: may start before the previous kernel finished; the
                // kernel waits for it (griddepcontrol.wait) before touching its results
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Act>(args)...);
}
template <typename... Exp, typename... Act>
cudaError_t launch_coop(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Act&&... args) {
    return launch_ex(true, false, kernel, grid, block, smem, st, std::forward<Act>(args)...);
}

// -------- multi-GPU plumbing (latitude bands) --------
// exchange the boundary rows of a ghosted array with the j-neighbours
bool multi(const eg_solver* s) { return s->comm != nullptr || s->lb != nullptr; }

int lb_fail(eg_solver* s) {
    return fail(s, EG_ERR_NCCL, "loopback group: a rank failed or did not arrive within 120 s");
}

// ---- P2P transport: the peer table ----
// base[r]: rank r's workspace as this process addresses it.  Every rank's layout follows from the
// grid, the precision and its band (valid_dist's group-aligned split), so only the bases travel.
void p2p_table(eg_solver* s, unsigned char* const* base, int split_all) {
    P2P& pp = s->pp;
    pp = P2P{};
    pp.rank = s->rank;
    pp.nranks = s->nranks;
    pp.tiles = (int)((s->grid.nx + ER_COLS - 1) / ER_COLS);  // one flag per edge-row CTA
    const char* tm = getenv("EG_P2P_TIMEOUT_MS");  // tests: a short limit for the fault-injection case
    pp.timeout_ns = (long long)(tm && atoll(tm) > 0 ? atoll(tm) : 60000) * 1000000ll;
    const char* fl = getenv("EG_P2P_FAULT");
    pp.fault = fl && fl[0] == '1';
    const int G = s->L.G, per = G / s->nranks;
    auto layout_of = [&](int r, Layout* Lr) {
        const int64_t b0 = (int64_t)(r * per) * s->grid.ny / G, b1 = (int64_t)((r + 1) * per) * s->grid.ny / G;
        make_layout(&s->grid, b1 - b0, s->mode, Lr);
    };
    auto zext_of = [&](int r, const Layout& Lr, int a) {
        return base[r] + Lr.off_z + (size_t)a * align_up((Lr.n + 2 * Lr.row) * Lr.vsz, 256);
    };
    for (int r = 0; r < s->nranks; ++r) {
        Layout Lr;
        layout_of(r, &Lr);
        pp.gall[r] = (unsigned long long*)(base[r] + Lr.off_p2p);
        int* hfl = (int*)(base[r] + Lr.off_p2p + kP2PGall);
        // the colour-split x (tri-SOR sweeps), row 0 at split + 7 n + row (off_split = base_total
        // whatever the features; every rank has the region, or none: split_all)
        unsigned char* xs0 = base[r] + Lr.off_split + (size_t)(7 * Lr.n + Lr.row) * Lr.vsz;
        if (r == s->rank - 1) {  // our row 0 -> its ghost row nyl
            pp.fdst_lo = hfl;
            pp.tdst_lo = hfl + 4 * pp.tiles;
            for (int a = 0; a < 2; ++a) pp.dst_lo[a] = zext_of(r, Lr, a) + (size_t)(Lr.row + Lr.n) * Lr.vsz;
            pp.dst_lo_x = s->split ? (void*)(xs0 + (size_t)Lr.n * Lr.vsz) : nullptr;
            pp.dst_lo_xg = base[r] + Lr.off_xg + (size_t)Lr.row * 8;  // its ghost row nyl of x
        }
        if (r == s->rank + 1) {  // our row nyl-1 -> its ghost row -1
            pp.fdst_hi = hfl;
            pp.tdst_hi = hfl + 4 * pp.tiles;
            for (int a = 0; a < 2; ++a) pp.dst_hi[a] = zext_of(r, Lr, a);
            pp.dst_hi_x = s->split ? (void*)(xs0 - (size_t)Lr.row * Lr.vsz) : nullptr;
            pp.dst_hi_xg = base[r] + Lr.off_xg;  // its ghost row -1 of x
        }
    }
    pp.hflag = (const int*)(s->ws + s->L.off_p2p + kP2PGall);
    pp.tflag = pp.hflag + 4 * pp.tiles;
    pp.tcount = (int*)(s->ws + s->L.off_p2p + kP2PGall) + 8 * pp.tiles;
    pp.tsor = split_all;
    pp.on = 1;
}

typedef CUresult (*MemGetAddressRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);

// CUDA IPC of a pointer INSIDE an allocation (a PyTorch caching-allocator block): the handle names
// the allocation's base (cuMemGetAddressRange), the offset travels beside it
struct IpcRec {
    cudaIpcMemHandle_t h;
    uint64_t off;
    int32_t ok, pad;
};
static_assert(sizeof(IpcRec) == 80, "IpcRec is the 80-byte record of eg_debug_ipc_export");
IpcRec ipc_export(const void* ptr) {
    IpcRec r{};
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CUdeviceptr a0 = 0;
    size_t sz = 0;
    if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &fn, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess && fn && ((MemGetAddressRangeFn)fn)(&a0, &sz, (CUdeviceptr)ptr) == CUDA_SUCCESS &&
        cudaIpcGetMemHandle(&r.h, (void*)a0) == cudaSuccess) {
        r.off = (uint64_t)((CUdeviceptr)ptr - a0);
        r.ok = 1;
    }
    cudaGetLastError();
    return r;
}
// -> the peer's pointer in this process (base opened with lazy peer access + offset), or NULL;
// *opened: the base to pass to cudaIpcCloseMemHandle
unsigned char* ipc_open(const IpcRec& r, void** opened) {
    *opened = nullptr;
    if (!r.ok) return nullptr;
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, r.h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    *opened = p;
    return (unsigned char*)p + r.off;
}

// NCCL ranks (separate processes, one GPU each): export the workspace's allocation by CUDA IPC,
// all-gather the handles, open the peers' (NVLink peer access enabled lazily).  Every rank must
// succeed or all keep the NCCL exchange (the result is agreed by an all-reduce).  Collective.
int p2p_setup_nccl(eg_solver* s) {
    using Rec = IpcRec;
    const int P = s->nranks;
    std::vector<unsigned char*> base(P, nullptr);
    base[s->rank] = s->ws;
    int ok = 1, split_same = 1;
    if (P > 1) {
        Rec mine = ipc_export(s->ws);
        mine.pad = s->split ? 1 : 0;  // has the colour-split tri-SOR region
        std::vector<Rec> all(P);
        Rec* d = nullptr;
        CK(cudaMalloc(&d, sizeof(Rec) * (P + 1)));
        int rc = EG_OK;
        if (cudaMemcpy(d + P, &mine, sizeof(Rec), cudaMemcpyHostToDevice) != cudaSuccess) rc = EG_ERR_CUDA;
        if (rc == EG_OK && ncclAllGather(d + P, d, sizeof(Rec), ncclChar, s->comm, s->st) != ncclSuccess) rc = EG_ERR_NCCL;
        if (rc == EG_OK && (cudaStreamSynchronize(s->st) != cudaSuccess ||
                            cudaMemcpy(all.data(), d, sizeof(Rec) * P, cudaMemcpyDeviceToHost) != cudaSuccess))
            rc = EG_ERR_CUDA;
        for (int r = 0; rc == EG_OK && r < P; ++r) {
            if (all[r].pad != mine.pad) split_same = 0;
            if (!all[r].ok) { ok = 0; continue; }
            if (r == s->rank || !ok) continue;
            void* p = nullptr;
            base[r] = ipc_open(all[r], &p);
            if (!base[r]) { ok = 0; continue; }
            s->ipc_open.push_back(p);
        }
        // agree: P2P only if every rank opened every peer
        int* dok = (int*)(d + P);
        if (rc == EG_OK && cudaMemcpy(dok, &ok, sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess) rc = EG_ERR_CUDA;
        if (rc == EG_OK && ncclAllReduce(dok, dok, 1, ncclInt, ncclMin, s->comm, s->st) != ncclSuccess) rc = EG_ERR_NCCL;
        if (rc == EG_OK && (cudaStreamSynchronize(s->st) != cudaSuccess ||
                            cudaMemcpy(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess))
            rc = EG_ERR_CUDA;
        cudaFree(d);
        if (rc != EG_OK) return fail(s, rc, "P2P setup: handle exchange failed");
    }
    if (!ok) {  // keep the NCCL exchange
        for (void* p : s->ipc_open) cudaIpcCloseMemHandle(p);
        s->ipc_open.clear();
        return EG_OK;
    }
    CK(cudaMemsetAsync(s->ws + s->L.off_p2p, 0, s->L.off_state - s->L.off_p2p, s->st));
    CK(cudaStreamSynchronize(s->st));
    // (split-ness differs between ranks: the tri-SOR halos stay on NCCL; ranks agree, all saw the records)
    p2p_table(s, base.data(), split_same);
    // every rank has cleared its flags before any rank's first push (which comes after this barrier)
    int* one = nullptr;
    CK(cudaMalloc(&one, sizeof(int)));
    ncclResult_t nr = ncclAllReduce(one, one, 1, ncclInt, ncclSum, s->comm, s->st);
    cudaError_t ce = cudaStreamSynchronize(s->st);
    cudaFree(one);
    if (nr != ncclSuccess || ce != cudaSuccess) return fail(s, EG_ERR_NCCL, "P2P setup: barrier failed");
    return EG_OK;
}

// loopback ranks (one process): the table is built at the first solve, when every rank exists
int p2p_setup_loop(eg_solver* s) {
    LoopGroup* G = s->lb;
    G->ws[s->rank] = s->ws;
    G->split[s->rank] = s->split ? 1 : 0;
    CK(cudaMemsetAsync(s->ws + s->L.off_p2p, 0, s->L.off_state - s->L.off_p2p, s->st));
    if (!lb_barrier(G)) return lb_fail(s);  // every rank's clear is enqueued before any push
    int same = 1;
    for (int r = 0; r < s->nranks; ++r) same &= G->split[r] == G->split[s->rank];
    p2p_table(s, G->ws.data(), same);
    return EG_OK;
}

// the flag reset at an epoch wrap-around (solve_impl), with every rank's pushes of earlier solves
// done before it and none of the next solve's before it: a collective
int p2p_reset_flags(eg_solver* s) {
    if (s->lb) {
        if (!lb_barrier(s->lb)) return lb_fail(s);
    } else {
        CK(cudaStreamSynchronize(s->st));
        int* one = nullptr;
        CK(cudaMalloc(&one, sizeof(int)));
        ncclResult_t nr = ncclAllReduce(one, one, 1, ncclInt, ncclSum, s->comm, s->st);
        cudaError_t ce = cudaStreamSynchronize(s->st);
        cudaFree(one);
        if (nr != ncclSuccess || ce != cudaSuccess) return fail(s, EG_ERR_NCCL, "P2P flag reset: barrier failed");
    }
    CK(cudaMemsetAsync(s->ws + s->L.off_p2p, 0, s->L.off_state - s->L.off_p2p, s->st));
    if (s->lb) {
        if (!lb_barrier(s->lb)) return lb_fail(s);
    } else {
        CK(cudaStreamSynchronize(s->st));
        int* one = nullptr;
        CK(cudaMalloc(&one, sizeof(int)));
        ncclResult_t nr = ncclAllReduce(one, one, 1, ncclInt, ncclSum, s->comm, s->st);
        cudaError_t ce = cudaStreamSynchronize(s->st);
        cudaFree(one);
        if (nr != ncclSuccess || ce != cudaSuccess) return fail(s, EG_ERR_NCCL, "P2P flag reset: barrier failed");
    }
    return EG_OK;
}

// async: the exchange runs on the communication stream s->cst, ordered after everything enqueued on
// s->st so far (ev_edge); the caller joins it (edge_join) before the first kernel that reads a
// ghost row.  Otherwise it runs on s->st.
// row0 / last_row: the band's row 0 and row nyl-1 as sent (last_row = NULL: row nyl-1 of row0's array)
int halo(eg_solver* s, void* row0, void* ghost_lo, void* ghost_hi, size_t esz, bool async = false,
         void* last_row = nullptr, bool cst_ordered = false) {
    if (s->nranks == 1) return EG_OK;
    const size_t rowb = (size_t)s->L.row * esz;
    ncclDataType_t ty = esz == 8 ? ncclDouble : ncclFloat;
    unsigned char* first = (unsigned char*)row0;
    unsigned char* last = last_row ? (unsigned char*)last_row : first + (size_t)(s->L.nyl - 1) * rowb;
    cudaStream_t xs = async ? s->cst : s->st;
    if (s->lb) {
        LoopGroup* G = s->lb;
        G->first[s->rank] = first;
        G->last[s->rank] = last;
        if (!lb_barrier(G)) return lb_fail(s);
        // every rank's edge rows are enqueued on the shared stream before this point
        if (async && !cst_ordered) {
            CK(cudaEventRecord(s->ev_edge, s->st));
            CK(cudaStreamWaitEvent(xs, s->ev_edge, 0));
        }
        if (s->rank > 0) CK(cudaMemcpyAsync(ghost_lo, G->last[s->rank - 1], rowb, cudaMemcpyDeviceToDevice, xs));
        if (s->rank < s->nranks - 1)
            CK(cudaMemcpyAsync(ghost_hi, G->first[s->rank + 1], rowb, cudaMemcpyDeviceToDevice, xs));
        if (async) CK(cudaEventRecord(s->ev_halo, xs));
        if (!lb_barrier(G)) return lb_fail(s);
        return EG_OK;
    }
    if (async && !cst_ordered) {
        CK(cudaEventRecord(s->ev_edge, s->st));
        CK(cudaStreamWaitEvent(xs, s->ev_edge, 0));
    }
    NK(ncclGroupStart());
    if (s->rank > 0) {
        NK(ncclSend(first, s->L.row, ty, s->rank - 1, s->comm, xs));
        NK(ncclRecv(ghost_lo, s->L.row, ty, s->rank - 1, s->comm, xs));
    }
    if (s->rank < s->nranks - 1) {
        NK(ncclSend(last, s->L.row, ty, s->rank + 1, s->comm, xs));
        NK(ncclRecv(ghost_hi, s->L.row, ty, s->rank + 1, s->comm, xs));
    }
    NK(ncclGroupEnd());
    if (async) CK(cudaEventRecord(s->ev_halo, xs));
    return EG_OK;
}

int halo_ghosted(eg_solver* s, void* zrow0, bool async = false) {
    const size_t esz = s->L.vsz, rowb = (size_t)s->L.row * esz;
    unsigned char* r0 = (unsigned char*)zrow0;
    return halo(s, r0, r0 - rowb, r0 + (size_t)s->L.nyl * rowb, esz, async);
}


// the rows of a band whose stencil needs a neighbouring rank's ghost row (edge) or none (interior)
int edge_rows(const eg_solver* s, RowMap* rm) {
    const int lo = s->rank > 0, hi = s->rank < s->nranks - 1;
    const int nyl = (int)s->L.nyl;
    if (nyl == 1) { *rm = RowMap{0, 0}; return lo | hi; }
    if (lo && hi) { *rm = RowMap{0, nyl - 1}; return 2; }
    *rm = RowMap{lo ? 0 : nyl - 1, 0};
    return lo | hi;
}
int interior_rows(const eg_solver* s, RowMap* rm) {
    const int lo = s->rank > 0, hi = s->rank < s->nranks - 1;
    *rm = RowMap{lo, 1};
    return std::max(0, (int)s->L.nyl - lo - hi);
}

// P2P transport, loopback ranks: after the pushes, meet the other ranks, so that every rank's
// pushes are enqueued on the shared stream ahead of any rank's wait (no kernel then ever spins on
// another rank's kernel on the one GPU)
int p2p_push_join(eg_solver* s) {
    if (s->lb && !lb_barrier(s->lb)) return lb_fail(s);
    return EG_OK;
}

// stencil of the interior rows (edge = false: the 5-kernel schedule while the ghost rows travel) or
// of the band-edge rows after their ghost rows arrived (the phase kernel / the interior launch left
// them out: k_edge_stencil, which with the P2P transport first waits for the neighbours'
// pushes of array a: 0 = z, 1 = z_s), same arithmetic and reduction slots as the full launch
template <int MODE, int DOTS>
int stencil_rows(eg_solver* s, const typename Prec<MODE>::V* z, typename Prec<MODE>::V* y,
                 const typename Prec<MODE>::V* aux, bool edge, int a = 0, bool copy_v = false) {
    RowMap rm;
    const int n = edge ? edge_rows(s, &rm) : interior_rows(s, &rm);
    if (n == 0) return EG_OK;
#ifdef EG_MUTATE_NO_EDGE_STENCIL  // mutation check of the loopback tests (scripts/build_variant.sh)
    if (edge) return EG_OK;
#endif
    Vecs<MODE> v = vecs<MODE>(s, s->x64);
    if (edge) {
        // (fused schedule, phase A: v of the edge rows also into their band-edge copies for k_edge_rows)
        typename Prec<MODE>::V* ycopy =
            copy_v ? (typename Prec<MODE>::V*)(s->ws + s->L.off_edge) + 6 * s->L.row : nullptr;
        HWait hw{nullptr, 0, 0, 0, 0};
        if (s->pp.on)
            hw = HWait{s->pp.hflag + a * 2 * s->pp.tiles, s->pp.tiles, s->rank > 0, s->rank < s->nranks - 1,
                       s->pp.timeout_ns};
        k_edge_stencil<MODE, DOTS><<<dim3((unsigned)s->L.tiles, (unsigned)n, (unsigned)((s->grid.nz + 3) / 4)), 512,
                                     es_smem_bytes<MODE>(), s->st>>>(s->geo, v, z, y, aux, rm, hw,
                                                                     (int*)(s->ws + s->L.off_edge + 8 * s->L.row * s->L.vsz), ycopy);
    } else {
        k_stencil<MODE, DOTS><<<dim3((unsigned)s->L.tiles, (unsigned)n), RW, 0, s->st>>>(s->geo, v, z, y, aux, rm);
    }
    CK(cudaGetLastError());
    return EG_OK;
}

// quad: the slots are the FP64 phase kernels' half-slots (4 warp sums each, Geo.quad)
template <int MODE, int WHICH>
int finalize(eg_solver* s, int first, int tiles = 0, bool quad = false) {
    ProfScope ps(s, KID_FIN);
    Geo geo = s->geo;
    if (tiles > 0) geo.tiles = tiles;  // slots per row of the producing kernel
    geo.quad = quad ? 1 : 0;
    const double* slots = quad ? s->hslots : s->slots;
    if (!multi(s) || (s->pp.on && !s->lb)) {  // one launch: group sums (+ P2P all-gather) and logic
        CK(launch_ex(false, s->pdl, k_fin<MODE, WHICH>, dim3((unsigned)(geo.g_hi - geo.g_lo)), dim3(FIN_THREADS), 0, s->st,
                     geo, slots, s->dstate, s->gsum, first, s->pp));
        return EG_OK;
    }
    constexpr int NQ = fin_nq(WHICH);
    k_fin_groups<MODE, WHICH><<<(unsigned)(s->geo.g_hi - s->geo.g_lo), FIN_THREADS, 0, s->st>>>(geo, slots, s->dstate, s->gsum,
                                                                                                  s->pp);
    CK(cudaGetLastError());
    const int gl = s->geo.g_hi - s->geo.g_lo;
    if (s->pp.on) {  // the group kernels pushed the sums; the logic kernel waits for all of them
        // (loopback: every rank's pushes are enqueued on the shared stream before any wait)
        if (s->lb && !lb_barrier(s->lb)) return lb_fail(s);
    } else if (s->lb) {  // all-gather: rank r's block lands at gall + r * gl * NQ, as ncclAllGather places it
        LoopGroup* G = s->lb;
        G->gsum[s->rank] = s->gsum;
        if (!lb_barrier(G)) return lb_fail(s);
        for (int r = 0; r < s->nranks; ++r)
            CK(cudaMemcpyAsync(s->gall + (size_t)r * gl * NQ, G->gsum[r], (size_t)gl * NQ * sizeof(double),
                               cudaMemcpyDeviceToDevice, s->st));
        if (!lb_barrier(G)) return lb_fail(s);
    } else {
        NK(ncclAllGather(s->gsum, s->gall, (size_t)gl * NQ, ncclDouble, s->comm, s->st));
    }
    k_fin_logic<MODE, WHICH><<<1, 32, 0, s->st>>>(geo, s->gall, s->dstate, first, s->pp);
    CK(cudaGetLastError());
    return EG_OK;
}

#ifdef MA_VERIFY
// debug builds: after every fused phase kernel, recompute its outputs with the 5-kernel kernels on
// copies and count bitwise mismatches per array (0 z, 1 p, 2 v, 3 s, 4 z_s, 5 t, 6 slots)
__device__ unsigned long long g_vfy_cnt[8];
__device__ long long g_vfy_rec[256];
__device__ int g_vfy_nrec;
template <class T>
__global__ void k_vfy_cmp(const T* __restrict__ a, const T* __restrict__ b, int64_t n, int id) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const bool same = sizeof(T) == 4 ? __float_as_uint((float)a[q]) == __float_as_uint((float)b[q])
                                         : __double_as_longlong((double)a[q]) == __double_as_longlong((double)b[q]);
        if (!same) {
            atomicAdd(&g_vfy_cnt[id], 1ull);
            const int r = atomicAdd(&g_vfy_nrec, 1);
            if (r < 64) {
                g_vfy_rec[4 * r] = id; g_vfy_rec[4 * r + 1] = q;
                g_vfy_rec[4 * r + 2] = __double_as_longlong((double)a[q]);
                g_vfy_rec[4 * r + 3] = __double_as_longlong((double)b[q]);
            }
        }
    }
}
struct VfyBufs { float *p, *v, *z, *s, *zs, *t; double* slots; int64_t n; };
VfyBufs g_vfy{};
#endif

// the ghost-row exchange of z (a = 0) / z_s (a = 1) after the Thomas kernel wrote all rows: a push
// kernel (P2P) or the overlapped NCCL / loopback exchange (joined by edge_join)
template <class V>
int halo_start_t(eg_solver* s, V* z, int a) {
    if (!s->pp.on) return halo_ghosted(s, z, true);
    k_push_rows<V><<<dim3((unsigned)((s->grid.nx + ER_COLS - 1) / ER_COLS), 2u), 256, 0, s->st>>>(s->geo, z, s->dstate, s->pp, a);
    CK(cudaGetLastError());
    return p2p_push_join(s);
}
int halo_start(eg_solver* s, float* z, int a) { return halo_start_t<float>(s, z, a); }
int halo_start(eg_solver* s, double* z, int a) { return halo_start_t<double>(s, z, a); }

// Fused schedule, latitude bands: z (KIND 1) / z_s (KIND 2) of the band's edge rows, k_edge_rows
// into the scratch rows, then either its own pushes into the neighbours' ghost rows (P2P) or the
// NCCL / loopback exchange of the scratch rows, all on s->cst (ev_halo marks the end) beside the
// phase kernel.  Phase B writes s, z_s, t and reads r, v: nothing k_edge_rows<2> reads; phase A
// rewrites p and v, so k_edge_rows<1> reads their band-edge copies instead.  Profiled solves keep
// everything on s->st ahead of the phase kernel, where the CUDA events are (and so does the
// loopback copy transport).
// The edge rows on the communication stream?  (Loopback copies: the copies read the neighbours'
// scratch rows, ordered after their k_edge_rows only if those ran on the one shared stream.)
bool edge_on_cst(const eg_solver* s, int kind) { (void)kind; return !(s->profiling || (s->lb && !s->pp.on)); }

// On s->cst, iteration_fused records ev_edge right after the finaliser and launches the phase
// kernel BEFORE this (so that the cooperative phase kernel takes its SMs first and k_edge_rows fills
// the spare ones, instead of holding SMs the cooperative launch then has to wait for).  z (KIND 1)
// reads p and v of the edge rows from their band-edge copies (pv_edge), which phase A does not touch.
template <int MODE, int KIND>
int edge_exchange(eg_solver* s, Vecs<MODE>& v, typename Prec<MODE>::V* z) {
    using V = typename Prec<MODE>::V;
    const dim3 gedge((unsigned)((s->grid.nx + ER_COLS - 1) / ER_COLS), 2u);
    V* scratch = (V*)(s->ws + s->L.off_edge) + (size_t)(KIND - 1) * 2 * s->L.row;
    const bool on_cst = edge_on_cst(s, KIND);
    cudaStream_t xs = on_cst ? s->cst : s->st;
    if (on_cst) CK(cudaStreamWaitEvent(xs, s->ev_edge, 0));  // ev_edge: after the finaliser that set alpha
    {
        ProfScope ps(s, KID_EDGE, 0.0);
        k_edge_rows<MODE, KIND><<<gedge, ER_THREADS, er_smem_bytes(s->grid.nz), xs>>>(
            s->geo, v, (float*)scratch, s->pp, KIND == 1 ? (float*)(s->ws + s->L.off_edge) + 4 * s->L.row : nullptr);
        CK(cudaGetLastError());
    }
    int rc;
    if (s->pp.on) {
        if (!s->profiling) CK(cudaEventRecord(s->ev_halo, xs));
        return p2p_push_join(s);
    }
    // (from s->st: halo() orders the exchange on s->cst after k_edge_rows itself; on s->cst it
    // follows k_edge_rows there and must not wait for the phase kernel already on s->st)
    const size_t rowb = (size_t)s->L.row * sizeof(V);
    unsigned char* zr = (unsigned char*)z;
    if ((rc = halo(s, scratch, zr - rowb, zr + (size_t)s->L.nyl * rowb, sizeof(V), !s->profiling, scratch + s->L.row,
                   on_cst)))
        return rc;
    return EG_OK;
}
// before the band-edge rows' stencil: the join of the communication stream (cst_used: the
// exchange or k_edge_rows ran there).  (The P2P wait is the stencil kernel's own.)
int edge_join(eg_solver* s, int a, bool cst_used) {
    (void)a;
    if (cst_used && !s->profiling && s->nranks > 1) CK(cudaStreamWaitEvent(s->st, s->ev_halo, 0));
    return EG_OK;
}

// -------- the iteration (rows a3-a10) --------
// a9 + a10: the update and reduction 3.  One GPU and the P2P transport: one k_update.  Latitude
// bands over NCCL / loopback copies (split_update): the x half runs on s->xst beside the r half and
// reduction 3 (its all-gather), joined at the end of the iteration — before anything reads x or
// overwrites z / z_s.  (The P2P all-gather costs a few microseconds: hiding it does not pay for
// the second kernel's tail and the stream fork / join, profiles/r02_transport_cost.txt.)
template <int MODE>
int update_and_reduce(eg_solver* s, Vecs<MODE>& v) {
    const dim3 gr((unsigned)s->L.tiles, (unsigned)s->L.nyl);
    const double bx = 2.0 * s->L.xsz + 2.0 * s->L.vsz;     // x, z, z_s in; x out
    const double xz_bytes = s->next_xzero ? (double)s->L.xsz * s->L.n : 0.0;
    int rc;
    if (!s->split_update) {
        ProfScope ps(s, KID_UPDATE, s->next_xzero ? alg_bytes(s, KID_UPDATE) - xz_bytes : -1.0);
        s->next_xzero = false;
        if (s->cpt == 2 && s->update_kb2) CK(launch_ex(false, s->pdl, k_update<MODE, 2, 0, 2>, gr, dim3(RW / 2), 0, s->st, s->geo, v));
        else if (s->cpt == 2) CK(launch_ex(false, s->pdl, k_update<MODE, 2, 0, 0>, gr, dim3(RW / 2), 0, s->st, s->geo, v));
        else CK(launch_ex(false, s->pdl, k_update<MODE, 1, 0, 0>, gr, dim3(RW), 0, s->st, s->geo, v));
        return finalize<MODE, W_C>(s, 0);
    }
    // (profiled solves keep both halves on s->st, where the CUDA events are)
    cudaStream_t xs = s->profiling ? s->st : s->xst;
    if (!s->profiling) {
        CK(cudaEventRecord(s->ev_b, s->st));
        CK(cudaStreamWaitEvent(xs, s->ev_b, 0));
    }
    {
        ProfScope ps(s, KID_UPDATE_X, bx * s->L.n - xz_bytes);
        s->next_xzero = false;
        if (s->cpt == 2) k_update<MODE, 2, 2><<<gr, RW / 2, 0, xs>>>(s->geo, v);
        else k_update<MODE, 1, 2><<<gr, RW, 0, xs>>>(s->geo, v);
        CK(cudaGetLastError());
    }
    if (!s->profiling) CK(cudaEventRecord(s->ev_xu, xs));
    {
        ProfScope ps(s, KID_UPDATE, alg_bytes(s, KID_UPDATE) - bx * s->L.n);
        if (s->cpt == 2) k_update<MODE, 2, 1><<<gr, RW / 2, 0, s->st>>>(s->geo, v);
        else k_update<MODE, 1, 1><<<gr, RW, 0, s->st>>>(s->geo, v);
        CK(cudaGetLastError());
    }
    if ((rc = finalize<MODE, W_C>(s, 0))) return rc;
    if (!s->profiling) CK(cudaStreamWaitEvent(s->st, s->ev_xu, 0));
    return EG_OK;
}

// fused schedule: phase A (a3 + a4), phase B (a6 + a7), update (a9), three finalisers
template <int MODE>
int iteration_fused(eg_solver* s, void* x_it) {
    Vecs<MODE> v = vecs<MODE>(s, x_it);
    int rc;
    if constexpr (MODE != 0) {
        const unsigned grid = (unsigned)(s->mg.strips * s->L.tiles);
        const bool z_beside = s->nranks > 1 && edge_on_cst(s, 1);
        if (z_beside) CK(cudaEventRecord(s->ev_edge, s->st));  // z edge rows: after the last finaliser
        else if (s->nranks > 1 && (rc = edge_exchange<MODE, 1>(s, v, v.z))) return rc;
#ifdef MA_VERIFY
        const int64_t n = s->L.n;
        if (g_vfy.n != n) return fail(s, EG_ERR_CUDA, "MA_VERIFY buffers not allocated for this size");
        CK(cudaMemcpyAsync(g_vfy.p, v.p, n * 4, cudaMemcpyDeviceToDevice, s->st));
        CK(cudaMemcpyAsync(g_vfy.v, v.v, n * 4, cudaMemcpyDeviceToDevice, s->st));
        const dim3 gtm_((unsigned)((s->grid.nx + 127) / 128), (unsigned)s->L.nyl);
        const dim3 gr_((unsigned)s->L.tiles, (unsigned)s->L.nyl);
        const int64_t nsl = (int64_t)s->L.nyl * s->L.tiles;
#endif
        {
            // the first iteration after a (re)start has p = v = 0: phase A then reads r only
            ProfScope ps(s, KID_PHASE_A, s->next_fresh ? alg_bytes(s, KID_PHASE_A) - 2.0 * s->L.vsz * s->L.n : -1.0);
            s->next_fresh = false;
            CK(launch_ex(true, s->pdl, k_march<MODE, 1>, grid, MA_THREADS, s->smem_march, s->st, s->geo, v, s->mg, s->ready_flags,
                           s->maps));
        }
        if (z_beside && (rc = edge_exchange<MODE, 1>(s, v, v.z))) return rc;
        if (s->nranks > 1) {  // the band-edge rows' stencil, once their ghost rows are in
            if ((rc = edge_join(s, 0, true))) return rc;
            if ((rc = stencil_rows<MODE, 1>(s, v.z, v.v, v.rh, true, 0, true))) return rc;
        }
#ifdef MA_VERIFY
        {
            Vecs<MODE> w = v;
            w.p = (typename Prec<MODE>::V*)g_vfy.p; w.v = (typename Prec<MODE>::V*)g_vfy.v; w.slots = g_vfy.slots;
            k_thomas_tm<MODE, 1><<<gtm_, 128, s->smem_tm, s->st>>>(s->geo, w, nullptr, (typename Prec<MODE>::V*)g_vfy.z);
            k_stencil<MODE, 1><<<gr_, RW, 0, s->st>>>(s->geo, w, (typename Prec<MODE>::V*)g_vfy.z, w.v, w.rh, ALL_ROWS);
            k_vfy_cmp<float><<<592, 256, 0, s->st>>>((const float*)v.z, g_vfy.z, n, 0);
            k_vfy_cmp<float><<<592, 256, 0, s->st>>>((const float*)v.p, g_vfy.p, n, 1);
            k_vfy_cmp<float><<<592, 256, 0, s->st>>>((const float*)v.v, g_vfy.v, n, 2);
            k_vfy_cmp<double><<<64, 256, 0, s->st>>>(v.slots, g_vfy.slots, nsl, 6);
            CK(cudaGetLastError());
        }
#endif
        if ((rc = finalize<MODE, W_A>(s, 0))) return rc;
        const bool zs_beside = s->nranks > 1 && edge_on_cst(s, 2);
        if (zs_beside) CK(cudaEventRecord(s->ev_edge, s->st));  // z_s edge rows: after this finaliser
        else if (s->nranks > 1 && (rc = edge_exchange<MODE, 2>(s, v, v.zs))) return rc;
        {
            ProfScope ps(s, KID_PHASE_B);
            CK(launch_ex(true, s->pdl, k_march<MODE, 2>, grid, MA_THREADS, s->smem_march, s->st, s->geo, v, s->mg, s->ready_flags,
                           s->maps));
        }
        if (zs_beside && (rc = edge_exchange<MODE, 2>(s, v, v.zs))) return rc;
        if (s->nranks > 1) {
            if ((rc = edge_join(s, 1, true))) return rc;
            if ((rc = stencil_rows<MODE, 2>(s, v.zs, v.t, v.s, true, 1))) return rc;
        }
#ifdef MA_VERIFY
        {
            Vecs<MODE> w = v;
            w.s = (typename Prec<MODE>::V*)g_vfy.s; w.slots = g_vfy.slots;
            k_thomas_tm<MODE, 2><<<gtm_, 128, s->smem_tm, s->st>>>(s->geo, w, nullptr, (typename Prec<MODE>::V*)g_vfy.zs);
            k_stencil<MODE, 2><<<gr_, RW, 0, s->st>>>(s->geo, w, (typename Prec<MODE>::V*)g_vfy.zs,
                                                     (typename Prec<MODE>::V*)g_vfy.t, w.s, ALL_ROWS);
            k_vfy_cmp<float><<<592, 256, 0, s->st>>>((const float*)v.s, g_vfy.s, n, 3);
            k_vfy_cmp<float><<<592, 256, 0, s->st>>>((const float*)v.zs, g_vfy.zs, n, 4);
            k_vfy_cmp<float><<<592, 256, 0, s->st>>>((const float*)v.t, g_vfy.t, n, 5);
            k_vfy_cmp<double><<<64, 256, 0, s->st>>>(v.slots, g_vfy.slots, 3 * nsl, 6);
            CK(cudaGetLastError());
        }
#endif
        if ((rc = finalize<MODE, W_B>(s, 0))) return rc;
        if ((rc = update_and_reduce<MODE>(s, v))) return rc;
    } else {  // FP64: march64.cuh (64-column tiles, half-slot dot partials), one GPU
        const unsigned grid = (unsigned)(s->mg.strips * ((s->grid.nx + M6_TILE - 1) / M6_TILE));
        {
            ProfScope ps(s, KID_PHASE_A, s->next_fresh ? alg_bytes(s, KID_PHASE_A) - 2.0 * s->L.vsz * s->L.n : -1.0);
            s->next_fresh = false;
            CK(launch_coop(k_march64<1>, grid, M6_THREADS, s->smem_march, s->st, s->geo, v, s->mg, s->ready_flags,
                           s->hslots, s->maps64));
        }
        if ((rc = finalize<MODE, W_A>(s, 0, 0, true))) return rc;
        {
            ProfScope ps(s, KID_PHASE_B);
            CK(launch_coop(k_march64<2>, grid, M6_THREADS, s->smem_march, s->st, s->geo, v, s->mg, s->ready_flags,
                           s->hslots, s->maps64));
        }
        if ((rc = finalize<MODE, W_B>(s, 0, 0, true))) return rc;
        if ((rc = update_and_reduce<MODE>(s, v))) return rc;
    }
    return EG_OK;
}

// the halo after a tri-SOR half-sweep of the ghosted array arr (which: 0 z, 1 z_s, 2 colour-split
// x): the P2P push + wait (k_push_sweep / k_wait_sweep; loopback: a barrier between them) or the
// NCCL / loopback exchange.  in_solve: the sweep kernels skip halted iterations (so do these).
int sweep_halo(eg_solver* s, void* arr, int which, bool in_solve, size_t esz = 0) {
    if (s->nranks == 1) return EG_OK;
    if (!(s->pp.on && (s->pp.tsor || which != 2))) {
        if (which != 3) return halo_ghosted(s, arr);
        return halo(s, arr, s->xg, (unsigned char*)s->xg + s->L.row * 8, esz);
    }
    if (esz == 0) esz = s->L.vsz;
    const dim3 gp((unsigned)((s->grid.nx + ER_COLS - 1) / ER_COLS), 2u);
    if (esz == 8) k_push_sweep<double><<<gp, 256, 0, s->st>>>(s->geo, (const double*)arr, s->dstate, s->pp, which, in_solve);
    else k_push_sweep<float><<<gp, 256, 0, s->st>>>(s->geo, (const float*)arr, s->dstate, s->pp, which, in_solve);
    CK(cudaGetLastError());
    int rc;
    if ((rc = p2p_push_join(s))) return rc;
    k_wait_sweep<<<1, 256, 0, s->st>>>(s->dstate, s->pp, in_solve, s->rank > 0, s->rank < s->nranks - 1);
    CK(cudaGetLastError());
    return EG_OK;
}

// the colour-split band copies of the tri-SOR sweeps for the current operator (set_operator writes
// them itself once tri-SOR is selected; otherwise this pass derives them).  Called before an
// iteration graph is captured, so that the one-time pass is never part of the replayed graph.
template <int MODE>
int ensure_split(eg_solver* s) {
    using V = typename Prec<MODE>::V;
    if (!s->split || s->split_valid) return EG_OK;
    V* b4s = (V*)s->split;
    const dim3 grid((unsigned)((s->grid.nx + 255) / 256), (unsigned)s->grid.nz, (unsigned)s->L.nyl);
    k_split_bands<V><<<grid, 256, 0, s->st>>>(s->geo, (const V*)s->B4, (const V*)s->B2, b4s, b4s + 4 * s->L.n);
    CK(cudaGetLastError());
    s->split_valid = true;
    return EG_OK;
}

// NEXT-1: M^-1 f by `sor_sweeps` red-black tri-SOR sweeps (Eq. 7) into the ghosted array z (row 0
// pointer).  KIND 1 / 2: the first sweep also forms and stores p (s); later sweeps read it back.
template <int MODE, int KIND>
int apply_trisor(eg_solver* s, Vecs<MODE>& v, const typename Prec<MODE>::V* fin, typename Prec<MODE>::V* z) {
    using V = typename Prec<MODE>::V;
    const dim3 gs((unsigned)((s->grid.nx / 2 + s->wth - 1) / s->wth), (unsigned)s->L.nyl);
    const V* fsrc = KIND == 0 ? fin : (KIND == 1 ? v.p : v.s);
    int rc;
    Split<V> sp{nullptr, nullptr, nullptr};
    if (s->split) {  // colour-split bands (refreshed after every set_operator) and f
        V* b4s = (V*)s->split;
        V* b2s = b4s + 4 * s->L.n;
        if ((rc = ensure_split<MODE>(s))) return rc;
        sp = Split<V>{b4s, b2s, b2s + 2 * s->L.n};
    }
    // the colour-split x of the TMA sweeps: ghosted, after f in the split region; row 0 pointer
    V* xsv = s->split ? (V*)s->split + 7 * s->L.n + s->L.row : nullptr;
    float* xsr = (float*)xsv;  // (the fp32 kernels' view)
    for (int sw = 0; sw < s->sor_sweeps; ++sw)
        for (int colour = 0; colour < 2; ++colour) {
            bool xs_half = false;  // this half-sweep wrote the colour-split x (else the natural z)
            {
                ProfScope ps(s, KID_SOR, sor_alg_bytes(s, KIND, sw, colour));
                bool tma = false;
                if constexpr (MODE != 0) {
                    tma = s->sor_tma && s->split;
                    if (tma) {  // fp32 with colour-split copies: x colour-split until the last half-sweep
                        const int so_smem = SO_STAGES * SO_STAGE_FLOATS * 4 + 128;
                        const int fin_ = sw == s->sor_sweeps - 1 && colour == 1;
                        if (sw == 0 && colour == 0)  // red half + f of both colours
                            k_sor_first_red<MODE, KIND><<<gs, s->wth, s->smem_th, s->st>>>(s->geo, v, (const float*)fin,
                                                                                         (float*)z, s->sor_omega, sp, xsr);
                        else if (sw == 0)
                            k_sor_tma<MODE, true><<<2 * s->nsm, SO_THREADS, so_smem, s->st>>>(
                                s->geo, v, xsr, (float*)z, colour, fin_, s->sor_omega, KIND != 0, s->sor_maps);
                        else
                            k_sor_tma<MODE, false><<<2 * s->nsm, SO_THREADS, so_smem, s->st>>>(
                                s->geo, v, xsr, (float*)z, colour, fin_, s->sor_omega, KIND != 0, s->sor_maps);
                        xs_half = !fin_;
                    }
                }
                if constexpr (MODE == 0) {
                    tma = s->sor_tma64 && s->split;
                    if (tma) {  // FP64: the same structure (colour-split x until the last half-sweep)
                        const int fin_ = sw == s->sor_sweeps - 1 && colour == 1;
                        if (sw == 0 && colour == 0)
                            k_sor_first_red<MODE, KIND><<<gs, s->wth, s->smem_th, s->st>>>(s->geo, v, fin, z, s->sor_omega, sp,
                                                                                         xsv);
                        else if (sw == 0)
                            k_sor_tma64<true><<<s->nsm, S6_THREADS, S6_SMEM, s->st>>>(s->geo, v, (double*)xsv, (double*)z,
                                                                                    colour, fin_, s->sor_omega, KIND != 0,
                                                                                    s->sor_maps64);
                        else
                            k_sor_tma64<false><<<s->nsm, S6_THREADS, S6_SMEM, s->st>>>(s->geo, v, (double*)xsv, (double*)z,
                                                                                     colour, fin_, s->sor_omega, KIND != 0,
                                                                                     s->sor_maps64);
                        xs_half = !fin_;
                    }
                }
                if (!tma) {
                    if (sw == 0)
                        k_sor_half<MODE, KIND, true><<<gs, s->wth, s->smem_th, s->st>>>(s->geo, v, fin, z, colour,
                                                                                         s->sor_omega, 0, sp);
                    else
                        k_sor_half<MODE, 0, false><<<gs, s->wth, s->smem_th, s->st>>>(s->geo, v, fsrc, z, colour,
                                                                                       s->sor_omega, KIND != 0, sp);
                }
                CK(cudaGetLastError());
            }
            if ((rc = sweep_halo(s, xs_half ? (void*)xsr : (void*)z, xs_half ? 2 : (z == v.zs ? 1 : 0), KIND != 0)))
                return rc;
        }
    return EG_OK;
}

template <int MODE>
int iteration_trisor(eg_solver* s, void* x_it) {
    Vecs<MODE> v = vecs<MODE>(s, x_it);
    const dim3 gr((unsigned)s->L.tiles, (unsigned)s->L.nyl);
    int rc;
    if ((rc = apply_trisor<MODE, 1>(s, v, nullptr, v.z))) return rc;
    {
        ProfScope ps(s, KID_STENCIL_A);
        k_stencil<MODE, 1><<<gr, RW, 0, s->st>>>(s->geo, v, v.z, v.v, v.rh, ALL_ROWS);
        CK(cudaGetLastError());
    }
    if ((rc = finalize<MODE, W_A>(s, 0))) return rc;
    if ((rc = apply_trisor<MODE, 2>(s, v, nullptr, v.zs))) return rc;
    {
        ProfScope ps(s, KID_STENCIL_B);
        k_stencil<MODE, 2><<<gr, RW, 0, s->st>>>(s->geo, v, v.zs, v.t, v.s, ALL_ROWS);
        CK(cudaGetLastError());
    }
    if ((rc = finalize<MODE, W_B>(s, 0))) return rc;
    return update_and_reduce<MODE>(s, v);
}

template <int MODE>
int iteration(eg_solver* s, void* x_it) {
    using V = typename Prec<MODE>::V;
    if (s->precond == EG_PRECOND_TRISOR) return iteration_trisor<MODE>(s, x_it);
    if (s->use_march) return iteration_fused<MODE>(s, x_it);
    Vecs<MODE> v = vecs<MODE>(s, x_it);
    const dim3 gt((unsigned)((s->grid.nx + s->wth - 1) / s->wth), (unsigned)s->L.nyl);
    const dim3 gr((unsigned)s->L.tiles, (unsigned)s->L.nyl);
    const int tth = s->wth / s->cpt;
    int rc;
    const dim3 gtm((unsigned)((s->grid.nx + 127) / 128), (unsigned)s->L.nyl);
    {
        ProfScope ps(s, KID_THOMAS_P);
        if constexpr (MODE != 0) {
            if (s->use_tm) CK(launch_ex(false, s->pdl, k_thomas_tm<MODE, 1>, dim3(gtm), dim3(128), s->smem_tm, s->st, s->geo, v, nullptr, v.z));
            else if (s->cpt == 2) CK(launch_ex(false, s->pdl, k_thomas<MODE, 1, 2>, dim3(gt), dim3(tth), s->smem_th, s->st, s->geo, v, nullptr, v.z));
            else CK(launch_ex(false, s->pdl, k_thomas<MODE, 1, 1>, dim3(gt), dim3(tth), s->smem_th, s->st, s->geo, v, nullptr, v.z));
        } else {
            if (s->th_tma64) CK(launch_ex(false, s->pdl, k_thomas_tma64<1>, dim3(s->nsm), dim3(T6_THREADS), T6_SMEM, s->st, s->geo, v, v.z, s->thmaps64));
            else if (s->use_tm64) CK(launch_ex(false, s->pdl, k_thomas_tm64<1>, dim3(gtm), dim3(128), TM64_SMEM, s->st, s->geo, v, nullptr, v.z));
            else if (s->cpt == 2) CK(launch_ex(false, s->pdl, k_thomas<MODE, 1, 2>, dim3(gt), dim3(tth), s->smem_th, s->st, s->geo, v, nullptr, v.z));
            else CK(launch_ex(false, s->pdl, k_thomas<MODE, 1, 1>, dim3(gt), dim3(tth), s->smem_th, s->st, s->geo, v, nullptr, v.z));
        }
        CK(cudaGetLastError());
    }
    {
        ProfScope ps(s, KID_STENCIL_A);
        if (s->nranks > 1) {  // interior rows while the ghost rows travel, then the band-edge rows
            if ((rc = halo_start(s, v.z, 0))) return rc;
            if ((rc = stencil_rows<MODE, 1>(s, v.z, v.v, v.rh, false))) return rc;
            if ((rc = edge_join(s, 0, !s->pp.on))) return rc;
            if ((rc = stencil_rows<MODE, 1>(s, v.z, v.v, v.rh, true, 0))) return rc;
        } else {
            CK(launch_ex(false, s->pdl, k_stencil<MODE, 1>, dim3(gr), dim3(RW), 0, s->st, s->geo, v, v.z, v.v, v.rh, ALL_ROWS));
            CK(cudaGetLastError());
        }
    }
    if ((rc = finalize<MODE, W_A>(s, 0))) return rc;
    {
        ProfScope ps(s, KID_THOMAS_S);
        if constexpr (MODE != 0) {
            if (s->use_tm) CK(launch_ex(false, s->pdl, k_thomas_tm<MODE, 2>, dim3(gtm), dim3(128), s->smem_tm, s->st, s->geo, v, nullptr, v.zs));
            else if (s->cpt == 2) CK(launch_ex(false, s->pdl, k_thomas<MODE, 2, 2>, dim3(gt), dim3(tth), s->smem_th, s->st, s->geo, v, nullptr, v.zs));
            else CK(launch_ex(false, s->pdl, k_thomas<MODE, 2, 1>, dim3(gt), dim3(tth), s->smem_th, s->st, s->geo, v, nullptr, v.zs));
        } else {
            // (the TMA-fed kernel is slower for this lighter solve, 3.68 vs 3.40 ms at C5: one CTA per SM
            // cannot hide the FP64 recurrence the 2-CTA TMEM kernel overlaps)
            if (s->use_tm64) CK(launch_ex(false, s->pdl, k_thomas_tm64<2>, dim3(gtm), dim3(128), TM64_SMEM, s->st, s->geo, v, nullptr, v.zs));
            else if (s->cpt == 2) CK(launch_ex(false, s->pdl, k_thomas<MODE, 2, 2>, dim3(gt), dim3(tth), s->smem_th, s->st, s->geo, v, nullptr, v.zs));
            else CK(launch_ex(false, s->pdl, k_thomas<MODE, 2, 1>, dim3(gt), dim3(tth), s->smem_th, s->st, s->geo, v, nullptr, v.zs));
        }
        CK(cudaGetLastError());
    }
    {
        ProfScope ps(s, KID_STENCIL_B);
        if (s->nranks > 1) {
            if ((rc = halo_start(s, v.zs, 1))) return rc;
            if ((rc = stencil_rows<MODE, 2>(s, v.zs, v.t, v.s, false))) return rc;
            if ((rc = edge_join(s, 1, !s->pp.on))) return rc;
            if ((rc = stencil_rows<MODE, 2>(s, v.zs, v.t, v.s, true, 1))) return rc;
        } else {
            CK(launch_ex(false, s->pdl, k_stencil<MODE, 2>, dim3(gr), dim3(RW), 0, s->st, s->geo, v, v.zs, v.t, v.s, ALL_ROWS));
            CK(cudaGetLastError());
        }
    }
    if ((rc = finalize<MODE, W_B>(s, 0))) return rc;
    if ((rc = update_and_reduce<MODE>(s, v))) return rc;
    (void)sizeof(V);
    return EG_OK;
}

// start / restart / verification (rows a2, a11)
template <int MODE>
int start(eg_solver* s, void* x_it, const double* b, int entry, int xzero, const double* shadow = nullptr) {
    using X = typename Prec<MODE>::X;
    Vecs<MODE> v = vecs<MODE>(s, x_it);
    int rc;
    if (!xzero && s->nranks > 1) {  // fp64 (X) ghost rows of x
        X* x = (X*)x_it;
        if ((rc = sweep_halo(s, x, 3, false, sizeof(X)))) return rc;
    }
    const dim3 gr((unsigned)s->L.tiles, (unsigned)s->L.nyl);
    s->next_fresh = true;
    s->next_xzero = entry && xzero;
    {
        ProfScope ps(s, KID_START, start_bytes(s, entry, xzero, true));
        if (entry && xzero) k_start<MODE, true, true><<<gr, RW, 0, s->st>>>(s->geo, v, b);
        else if (entry) k_start<MODE, true, false><<<gr, RW, 0, s->st>>>(s->geo, v, b);
        else k_start<MODE, false, false><<<gr, RW, 0, s->st>>>(s->geo, v, b);
        CK(cudaGetLastError());
    }
    if ((rc = finalize<MODE, W_START>(s, entry))) return rc;
    if (shadow) {  // the caller's rhat0 replaces rhat0 = r0 (the first start only; restarts use r, A-11)
        ProfScope ps(s, KID_START, (8.0 + 2.0 * s->L.vsz) * s->L.n);
        k_shadow<MODE><<<gr, RW, 0, s->st>>>(s->geo, v, shadow);
        CK(cudaGetLastError());
    }
    return shadow ? finalize<MODE, W_SHADOW>(s, 0) : EG_OK;
}

// true residual of the current x only, r / rhat0 untouched (A-6 verification, final true_R)
template <int MODE>
int verify(eg_solver* s, void* x_it) {
    using X = typename Prec<MODE>::X;
    Vecs<MODE> v = vecs<MODE>(s, x_it);
    int rc;
    if (s->nranks > 1) {
        X* x = (X*)x_it;
        if ((rc = sweep_halo(s, x, 3, false, sizeof(X)))) return rc;
    }
    const dim3 gr((unsigned)s->L.tiles, (unsigned)s->L.nyl);
    {
        ProfScope ps(s, KID_VERIFY, start_bytes(s, 0, 0, false));
        // two columns per thread for fp32 bands (2.65 -> 2.20 ms at C5); FP64 measured slower with it
        if (s->cpt == 2 && MODE != 0) k_verify2<MODE><<<gr, RW / 2, 0, s->st>>>(s->geo, v);
        else k_start<MODE, false, false, false><<<gr, RW, 0, s->st>>>(s->geo, v, nullptr);
        CK(cudaGetLastError());
    }
    return finalize<MODE, W_VERIFY>(s, 0);
}

// DevState <-> its host mirror by a one-CTA copy kernel through mapped pinned memory, not by
// cudaMemcpyAsync: a small DMA copy would queue behind the multi-GB transfers eg_solve_batch keeps
// in flight on the copy engines
__global__ void k_copy_words(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, int n) {
    for (int w = threadIdx.x; w < n; w += blockDim.x) dst[w] = src[w];
}

int state_to_host(eg_solver* s, const void* dev, void* host, size_t bytes) {
    const size_t off = (const unsigned char*)host - (const unsigned char*)s->hstate;
    k_copy_words<<<1, 256, 0, s->st>>>((const uint32_t*)dev, (uint32_t*)((unsigned char*)s->hstate_dev + off),
                                       (int)(bytes / 4));
    CK(cudaGetLastError());
    return EG_OK;
}

int read_state(eg_solver* s) {
    int rc = state_to_host(s, s->dstate, s->hstate, sizeof(DevState));
    if (rc) return rc;
    CK(cudaStreamSynchronize(s->st));
    if (s->profiling) drain_profile(s);
    if (s->hstate->halt == H_PEER_TIMEOUT)
        return fail(s, EG_ERR_NCCL, "P2P transport: a neighbouring rank's push did not arrive within %lld ms",
                    (long long)(s->pp.timeout_ns / 1000000));
    return EG_OK;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// x = 0 not stored yet (DevState.xzero, no update since an x0 = 0 entry): store it before anything
// else reads x (restart, verification, the output)
template <int MODE>
int materialise_x0(eg_solver* s, void* x_it) {
    if (!s->hstate->xzero) return EG_OK;
    CK(cudaMemsetAsync(x_it, 0, (size_t)s->L.n * sizeof(typename Prec<MODE>::X), s->st));
    CK(cudaMemsetAsync(&s->dstate->xzero, 0, sizeof(int), s->st));
    s->hstate->xzero = 0;
    return EG_OK;
}

template <int MODE>
int solve_impl(eg_solver* s, const double* b, const double* x0, const eg_solve_params* prm, double* x,
               double* history, eg_solve_info* info) {
    using X = typename Prec<MODE>::X;
    const int64_t n = s->L.n;
    int rc = EG_OK;
    s->profiling = (prm->flags & EG_SOLVE_PROFILE) != 0;
    // (loopback ranks meet at host barriers inside every exchange: launched directly, never replayed)
    bool use_graph = !(prm->flags & (EG_SOLVE_NO_GRAPH | EG_SOLVE_PROFILE)) && s->lb == nullptr;
    eg_solve_info inf{};

    // ---- inputs: b (host -> staged into bhat, scaled in place), x iterate ----
    const double* bdev = b;
    if (!is_device_ptr(b)) {
        CK(cudaMemcpyAsync(s->bhat, b, n * 8, cudaMemcpyHostToDevice, s->st));
        bdev = s->bhat;
    }
    const bool xdev = is_device_ptr(x);
    void* x_it;
    if (MODE == 2) x_it = s->x32;
    else x_it = xdev ? (void*)x : (void*)s->x64;
    if (x0) {
        if (MODE == 2) {
            const double* x0d = x0;
            if (!is_device_ptr(x0)) {
                CK(cudaMemcpyAsync(s->x64, x0, n * 8, cudaMemcpyHostToDevice, s->st));
                x0d = s->x64;
            }
            ProfScope ps(s, KID_CONVERT);
            k_convert<double, float><<<1184, 256, 0, s->st>>>(x0d, s->x32, n);
            CK(cudaGetLastError());
        } else if (x0 != x_it) {
            CK(cudaMemcpyAsync(x_it, x0, n * 8, cudaMemcpyDefault, s->st));
        }
    }

    // ---- device state ----
    DevState* h = s->hstate;
    memset(h, 0, sizeof(DevState));
    h->tol = prm->tol;
    h->maxit = prm->maxit;
    h->restart_every = prm->restart_every;
    h->eps_v = MODE == 0 ? 0x1.0p-53 : 0x1.0p-24;
    h->omega = h->omega_v = 1.0;
    h->xzero = x0 == nullptr ? 1 : 0;  // entry from x = 0 does not store x (the first update starts from 0)
    // ready flags are stamped with epochs that only ever grow: reserve this solve's range
    // (at most ~5 finalisers per iteration) and wrap around with a flag reset well before overflow
    // (eg_solve sets epoch_base past the last epoch used; the reservation covers error exits)
    const int64_t reserve = 8 * ((int64_t)prm->maxit + 4);
    if (s->lb && s->p2p_want && !s->pp.on && (rc = p2p_setup_loop(s))) return rc;
    const char* ew = getenv("EG_EPOCH_WRAP_TEST");  // tests: force the wrap-around path now
    if (s->epoch_base + reserve > ((int64_t)1 << 30) || (ew && ew[0] == '1')) {
        CK(cudaMemsetAsync(s->ready_flags, 0, (size_t)s->L.nyl * ((s->grid.nx + 63) / 64) * sizeof(int), s->st));
        if (s->pp.on && (rc = p2p_reset_flags(s))) return rc;
        s->epoch_base = 1;
    }
    h->epoch = (int)s->epoch_base;
    s->epoch_base += reserve;
    h->gseq = s->gseq;  // the P2P gather buffers alternate with it across solves
    k_copy_words<<<1, 256, 0, s->st>>>((const uint32_t*)s->hstate_dev, (uint32_t*)s->dstate, (int)(sizeof(DevState) / 4));
    CK(cudaGetLastError());

    if ((rc = start<MODE>(s, x_it, bdev, 1, x0 == nullptr, prm->rhat0))) return rc;
    if ((rc = read_state(s))) return rc;
    if (h->halt == H_DEGENERATE) rc = EG_ERR_DEGENERATE_RHS;
    else if (h->halt == H_NONFINITE) rc = EG_ERR_NONFINITE;
    if (history && rc == EG_OK) history[0] = h->hist[0];
    int copied = 0;
    int bd_at = -1;
    const int chunk_max = prm->check_every > 0 ? std::min(prm->check_every, HIST_CAP) : 8;

    if (s->precond == EG_PRECOND_TRISOR && rc == EG_OK && (rc = ensure_split<MODE>(s))) return rc;
    // graph for this iterate pointer (two cached entries)
    s->graph = nullptr;
    for (int gi = 0; gi < 2; ++gi)
        if (s->graphs[gi] && s->graphs_x[gi] == x_it) s->graph = s->graphs[gi];
    if (use_graph && rc == EG_OK && s->graph == nullptr) {
        const int gi = s->graph_next;
        s->graph_next ^= 1;
        if (s->graphs[gi]) { cudaGraphExecDestroy(s->graphs[gi]); s->graphs[gi] = nullptr; }
        cudaGraph_t gph;
        if (!s->cap_st) CK(cudaStreamCreateWithFlags(&s->cap_st, cudaStreamNonBlocking));
        cudaStream_t user = s->st;
        s->st = s->cap_st;  // the user's stream may be the legacy stream, which cannot capture
        cudaError_t cb = cudaStreamBeginCapture(s->st, cudaStreamCaptureModeThreadLocal);
        int irc = cb == cudaSuccess ? iteration<MODE>(s, x_it) : EG_OK;
        cudaGraph_t tmp = nullptr;
        cudaError_t ce = cb == cudaSuccess ? cudaStreamEndCapture(s->st, &tmp) : cb;
        gph = tmp;
        s->st = user;
        cudaError_t ie = cudaErrorUnknown;
        if (cb == cudaSuccess && irc == EG_OK && ce == cudaSuccess && gph) ie = cudaGraphInstantiate(&s->graphs[gi], gph, 0);
        if (gph) cudaGraphDestroy(gph);
        if (ie == cudaSuccess) {
            s->graphs_x[gi] = x_it;
            s->graph = s->graphs[gi];
        } else {  // the graph is an optimisation only: launch the iteration's kernels directly
            cudaGetLastError();
            s->graphs[gi] = nullptr;
            use_graph = false;
        }
    }

    while (rc == EG_OK) {
        if (h->halt == H_START_CONVERGED) { inf.converged = 1; break; }
        if (h->halt == H_START_MAXIT) break;
        // run iterations until the device raises a halt flag
        while (h->halt == H_RUN) {
            const int left = h->maxit - h->iter;
            const int k = std::max(1, std::min(chunk_max, left));
            for (int c = 0; c < k; ++c) {
                if (use_graph) CK(cudaGraphLaunch(s->graph, s->st));
                else if ((rc = iteration<MODE>(s, x_it))) return rc;
            }
            if ((rc = read_state(s))) return rc;
            if (h->iter < copied || h->iter > h->maxit || h->iter - copied > HIST_CAP)
                return fail(s, EG_ERR_CUDA, "device solver state is inconsistent (iter %d)", h->iter);
            if (history)
                for (int i = copied + 1; i <= h->iter; ++i) history[i] = h->hist[i % HIST_CAP];
            copied = h->iter;
        }
        const int halt = h->halt;
        if (halt == H_NONFINITE) { rc = EG_ERR_NONFINITE; break; }
        if (halt == H_BD_ABORT || halt == H_BD_END) {
            inf.breakdowns++;
            if (bd_at == h->iter) { rc = EG_ERR_BREAKDOWN; break; }
            bd_at = h->iter;
        }
        // H_CONVERGED -> verify the true residual (A-6); H_MAXIT -> final true residual only;
        // H_RESTART / breakdown / failed verification -> restart: r = round(bhat - Ahat x) with fp64
        // accumulation (A-11), which re-checks R_true < tol itself.
        if (halt == H_CONVERGED || halt == H_MAXIT) {
            if ((rc = materialise_x0<MODE>(s, x_it))) return rc;
            if ((rc = verify<MODE>(s, x_it))) return rc;
            if ((rc = read_state(s))) return rc;
            if (h->halt == H_NONFINITE) { rc = EG_ERR_NONFINITE; break; }
            if (halt == H_MAXIT) break;
            if (h->halt == H_START_CONVERGED) { inf.converged = 1; break; }
            if (h->iter >= h->maxit) break;
        }
        inf.restarts++;  // counted before the restart re-checks R_true (as the oracle does)
        if ((rc = materialise_x0<MODE>(s, x_it))) return rc;
        if ((rc = start<MODE>(s, x_it, bdev, 0, 0))) return rc;
        if ((rc = read_state(s))) return rc;
        if (h->halt == H_START_CONVERGED) { inf.converged = 1; break; }
        if (h->halt == H_START_MAXIT) break;
    }

    if (rc != EG_ERR_CUDA && rc != EG_ERR_NCCL) {  // x = 0 if no update has stored it
        const int rc0 = materialise_x0<MODE>(s, x_it);
        if (rc0) return rc0;
    }
    // ---- output x (fp64) ----
    if (MODE == 2) {
        double* dst = xdev ? x : s->x64;
        {
            ProfScope ps(s, KID_CONVERT);
            k_convert<float, double><<<1184, 256, 0, s->st>>>(s->x32, dst, n);
            CK(cudaGetLastError());
        }
        if (!xdev) CK(cudaMemcpyAsync(x, s->x64, n * 8, cudaMemcpyDeviceToHost, s->st));
    } else if (!xdev) {
        CK(cudaMemcpyAsync(x, x_it, n * 8, cudaMemcpyDeviceToHost, s->st));
    }
    CK(cudaStreamSynchronize(s->st));
    if (s->profiling) drain_profile(s);
    inf.iters = h->iter;
    inf.final_R = h->final_R;
    inf.true_R = h->true_R;
    inf.status = rc;
    if (info) *info = inf;
    (void)sizeof(X);
    return rc;
}

template <int MODE>
int create_impl(eg_solver* s, const double* const bands[7]) {
    using V = typename Prec<MODE>::V;
    s->split_valid = false;  // the colour-split bands are re-derived on the next tri-SOR sweep
    Bands7 in;
    for (int d = 0; d < 7; ++d) in.b[d] = bands[d];
    int* err = (int*)&s->dstate->err;
    CK(cudaMemsetAsync(s->dstate, 0, sizeof(DevState), s->st));
    const dim3 grid((unsigned)((s->grid.nx + 255) / 256), (unsigned)s->grid.nz, (unsigned)s->L.nyl);
    {
        // with the tri-SOR preconditioner selected, the colour-split band copies are written here too
        // (one pass instead of a later k_split_bands re-reading the packed bands)
        V* b4s = (s->split && s->precond == EG_PRECOND_TRISOR) ? (V*)s->split : nullptr;
        V* b2s = b4s ? b4s + 4 * s->L.n : nullptr;
        ProfScope ps(s, KID_SCALE, alg_bytes(s, KID_SCALE) + (b4s ? 6.0 * s->L.vsz * s->L.n : 0.0));
        k_scale<V><<<grid, 256, 0, s->st>>>(s->geo, in, (V*)s->B4, (V*)s->B2, s->diag, err, b4s, b2s);
        s->split_valid = b4s != nullptr;
        CK(cudaGetLastError());
    }
    int rc = state_to_host(s, err, &s->hstate->err, sizeof(int));
    if (rc) return rc;
    CK(cudaStreamSynchronize(s->st));
    const int herr = s->hstate->err;
    if (herr & 2) return fail(s, EG_ERR_SINGULAR_DIAG, "a_C is zero or non-finite at some point");
    if (herr & 1)
        return fail(s, EG_ERR_ARG, "non-finite band, or nonzero band at an absent neighbour");
    return EG_OK;
}

template <int MODE>
int apply_impl(eg_solver* s, const void* x, void* y) {
    Vecs<MODE> v = vecs<MODE>(s, s->x64);
    using V = typename Prec<MODE>::V;
    const V* zin = (const V*)x;
    int rc;
    if (s->nranks > 1) {  // stage into a ghosted buffer and exchange halo rows
        // (NCCL / loopback copies, written by the receiver itself, even with the P2P transport: two
        // applies in a row have no global sum between them, so a pushing neighbour could overwrite a
        // ghost row this rank's stencil has not read yet.  z_s, not z: a tri-SOR eg_precondition
        // pushes into z and could likewise overtake this stencil; the pushes into z_s all come
        // inside a solve, after a global sum this rank takes part in only after its apply.)
        CK(cudaMemcpyAsync(v.zs, x, s->L.n * sizeof(V), cudaMemcpyDeviceToDevice, s->st));
        if ((rc = halo_ghosted(s, v.zs))) return rc;
        zin = v.zs;
    }
    const dim3 gr((unsigned)s->L.tiles, (unsigned)s->L.nyl);
    ProfScope ps(s, KID_APPLY);
    k_stencil<MODE, 0><<<gr, RW, 0, s->st>>>(s->geo, v, zin, (V*)y, nullptr, ALL_ROWS);
    CK(cudaGetLastError());
    return EG_OK;
}

template <int MODE>
int precond_impl(eg_solver* s, const void* r, void* z) {
    using V = typename Prec<MODE>::V;
    Vecs<MODE> v = vecs<MODE>(s, s->x64);
    if (s->precond == EG_PRECOND_TRISOR) {  // sweep in the ghosted buffer, then copy out
        int rc = apply_trisor<MODE, 0>(s, v, (const V*)r, v.z);
        if (rc) return rc;
        CK(cudaMemcpyAsync(z, v.z, s->L.n * sizeof(V), cudaMemcpyDeviceToDevice, s->st));
        return EG_OK;
    }
    const dim3 gt((unsigned)((s->grid.nx + s->wth - 1) / s->wth), (unsigned)s->L.nyl);
    ProfScope ps(s, KID_PRECOND);
    if constexpr (MODE != 0) {
        if (s->use_tm) {
            const dim3 gtm((unsigned)((s->grid.nx + 127) / 128), (unsigned)s->L.nyl);
            k_thomas_tm<MODE, 0><<<gtm, 128, s->smem_tm, s->st>>>(s->geo, v, (const V*)r, (V*)z);
            CK(cudaGetLastError());
            return EG_OK;
        }
    }
    if constexpr (MODE == 0) {
        if (s->use_tm64) {
            const dim3 gtm((unsigned)((s->grid.nx + 127) / 128), (unsigned)s->L.nyl);
            k_thomas_tm64<0><<<gtm, 128, TM64_SMEM, s->st>>>(s->geo, v, (const V*)r, (V*)z);
            CK(cudaGetLastError());
            return EG_OK;
        }
    }
    if (s->cpt == 2) k_thomas<MODE, 0, 2><<<gt, s->wth / 2, s->smem_th, s->st>>>(s->geo, v, (const V*)r, (V*)z);
    else k_thomas<MODE, 0, 1><<<gt, s->wth, s->smem_th, s->st>>>(s->geo, v, (const V*)r, (V*)z);
    CK(cudaGetLastError());
    return EG_OK;
}

template <int MODE, int CPT>
int set_thomas_smem_c(eg_solver* s) {
    CK(cudaFuncSetAttribute(k_thomas<MODE, 0, CPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem_th));
    CK(cudaFuncSetAttribute(k_thomas<MODE, 1, CPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem_th));
    CK(cudaFuncSetAttribute(k_thomas<MODE, 2, CPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem_th));
    return EG_OK;
}

template <int MODE>
int set_thomas_smem(eg_solver* s) {
    CK(cudaFuncSetAttribute(k_sor_half<MODE, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem_th));
    CK(cudaFuncSetAttribute(k_sor_half<MODE, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem_th));
    CK(cudaFuncSetAttribute(k_sor_half<MODE, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem_th));
    CK(cudaFuncSetAttribute(k_sor_half<MODE, 0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem_th));
    CK(cudaFuncSetAttribute(k_edge_stencil<MODE, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)es_smem_bytes<MODE>()));
    CK(cudaFuncSetAttribute(k_edge_stencil<MODE, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)es_smem_bytes<MODE>()));
    int rc = set_thomas_smem_c<MODE, 1>(s);
    if (!rc) rc = set_thomas_smem_c<MODE, 2>(s);
    if constexpr (MODE != 0) {
        if (!rc && s->use_tm) {
            CK(cudaFuncSetAttribute(k_thomas_tm<MODE, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem_tm));
            CK(cudaFuncSetAttribute(k_thomas_tm<MODE, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem_tm));
            CK(cudaFuncSetAttribute(k_thomas_tm<MODE, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem_tm));
            CK(cudaFuncSetAttribute(k_edge_rows<MODE, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)er_smem_bytes(s->grid.nz)));
            CK(cudaFuncSetAttribute(k_edge_rows<MODE, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)er_smem_bytes(s->grid.nz)));
        }
    }
    return rc;
}

// TMA tensor maps of the arrays the fused phases stream ([nyl][nz][nx] views, 128 x MA_KS x 1 boxes)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool encode_map_box(EncodeTiledFn enc, CUtensorMap* m, void* base, int64_t inner, int64_t nz, int64_t nyl, int esz,
                    int box0, int box1) {
    const cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)nz, (cuuint64_t)nyl};
    const cuuint64_t strides[2] = {(cuuint64_t)(inner * esz), (cuuint64_t)(inner * nz * esz)};
    const cuuint32_t box[3] = {(cuuint32_t)box0, (cuuint32_t)box1, 1u};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    return enc(m, esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, base, dims, strides,
               box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool encode_map(EncodeTiledFn enc, CUtensorMap* m, void* base, int64_t inner, int64_t nz, int64_t nyl, int esz,
                int box0) {
    return encode_map_box(enc, m, base, inner, nz, nyl, esz, box0, MA_KS);
}

bool make_march_maps(eg_solver* s) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
        return false;
    EncodeTiledFn enc = (EncodeTiledFn)fn;
    const int64_t nx = s->grid.nx, nz = s->grid.nz, nyl = s->L.nyl;
    bool ok = encode_map(enc, &s->maps.r, s->vec[0], nx, nz, nyl, 4, 128);
    ok = ok && encode_map(enc, &s->maps.rh, s->vec[1], nx, nz, nyl, 4, 128);
    ok = ok && encode_map(enc, &s->maps.p, s->vec[2], nx, nz, nyl, 4, 128);
    ok = ok && encode_map(enc, &s->maps.v, s->vec[3], nx, nz, nyl, 4, 128);
    ok = ok && encode_map(enc, &s->maps.b2, s->B2, nx, nz, nyl, 8, 128);       // (U, D) as one 8-byte element
    ok = ok && encode_map(enc, &s->maps.b4, s->B4, 2 * nx, nz, nyl, 8, 256);   // (E, W), (N, S)
    return ok;
}

bool make_march_maps64(eg_solver* s) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
        return false;
    EncodeTiledFn enc = (EncodeTiledFn)fn;
    const int64_t nx = s->grid.nx, nz = s->grid.nz, nyl = s->L.nyl;
    MarchMaps64& m = s->maps64;
    bool ok = encode_map_box(enc, &m.r, s->vec[0], nx, nz, nyl, 8, M6_TILE, M6_KS);
    ok = ok && encode_map_box(enc, &m.rh, s->vec[1], nx, nz, nyl, 8, M6_TILE, M6_KS);
    ok = ok && encode_map_box(enc, &m.p, s->vec[2], nx, nz, nyl, 8, M6_TILE, M6_KS);
    ok = ok && encode_map_box(enc, &m.v, s->vec[3], nx, nz, nyl, 8, M6_TILE, M6_KS);
    ok = ok && encode_map_box(enc, &m.b2, s->B2, 2 * nx, nz, nyl, 8, 2 * M6_TILE, M6_KS);  // (U, D)
    ok = ok && encode_map_box(enc, &m.b4, s->B4, 4 * nx, nz, nyl, 8, 4 * M6_TILE, M6_KS);  // (E, W, N, S)
    return ok;
}

bool make_sor_maps(eg_solver* s) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn || !s->split)
        return false;
    EncodeTiledFn enc = (EncodeTiledFn)fn;
    const int64_t nx = s->grid.nx, nz = s->grid.nz, nyl = s->L.nyl;
    float* b4s = (float*)s->split;
    float* b2s = b4s + 4 * s->L.n;
    float* fs = b2s + 2 * s->L.n;
    float* xs = fs + s->L.n;  // the colour-split x from its row -1: rows are addressed as jl + 1
    SorMaps& m = s->sor_maps;
    bool ok = encode_map_box(enc, &m.xo6, xs, nx, nz, nyl + 2, 4, 128, SO_KS + 2);
    ok = ok && encode_map_box(enc, &m.x4, xs, nx, nz, nyl + 2, 4, 128, SO_KS);
    ok = ok && encode_map_box(enc, &m.xh, xs, nx, nz, nyl + 2, 4, 4, SO_KS);
    ok = ok && encode_map_box(enc, &m.f, fs, nx, nz, nyl, 4, 128, SO_KS);
    ok = ok && encode_map_box(enc, &m.b4, b4s, 2 * nx, nz, nyl, 8, 256, SO_KS);
    ok = ok && encode_map_box(enc, &m.b2, b2s, nx, nz, nyl, 8, 128, SO_KS);
    return ok;
}

bool make_sor_maps64(eg_solver* s) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn || !s->split)
        return false;
    EncodeTiledFn enc = (EncodeTiledFn)fn;
    const int64_t nx = s->grid.nx, nz = s->grid.nz, nyl = s->L.nyl;
    double* b4s = (double*)s->split;
    double* b2s = b4s + 4 * s->L.n;
    double* fs = b2s + 2 * s->L.n;
    double* xs = fs + s->L.n;  // the colour-split x from its row -1: rows are addressed as jl + 1
    SorMaps64& m = s->sor_maps64;
    bool ok = encode_map_box(enc, &m.xo6, xs, nx, nz, nyl + 2, 8, 128, S6_KS + 2);
    ok = ok && encode_map_box(enc, &m.x4, xs, nx, nz, nyl + 2, 8, 128, S6_KS);
    ok = ok && encode_map_box(enc, &m.xh, xs, nx, nz, nyl + 2, 8, 4, S6_KS);
    ok = ok && encode_map_box(enc, &m.f, fs, nx, nz, nyl, 8, 128, S6_KS);
    ok = ok && encode_map_box(enc, &m.b4, b4s, 4 * nx, nz, nyl, 8, 256, S6_KS);
    ok = ok && encode_map_box(enc, &m.b2, b2s, 2 * nx, nz, nyl, 8, 256, S6_KS);
    return ok;
}

bool make_thomas_maps64(eg_solver* s) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
        return false;
    EncodeTiledFn enc = (EncodeTiledFn)fn;
    const int64_t nx = s->grid.nx, nz = s->grid.nz, nyl = s->L.nyl;
    ThomasMaps64& m = s->thmaps64;
    bool ok = encode_map_box(enc, &m.a, s->vec[0], nx, nz, nyl, 8, 128, T6_KS);      // r
    ok = ok && encode_map_box(enc, &m.p, s->vec[2], nx, nz, nyl, 8, 128, T6_KS);     // p
    ok = ok && encode_map_box(enc, &m.v, s->vec[3], nx, nz, nyl, 8, 128, T6_KS);     // v
    ok = ok && encode_map_box(enc, &m.ud, s->B2, 2 * nx, nz, nyl, 8, 256, T6_KS);   // (U, D)
    return ok;
}

bool valid_dist(const eg_grid* g, const eg_dist* d, int64_t* jb, int64_t* je, int* rank, int* nranks) {
    if (!d) { *jb = 0; *je = g->ny; *rank = 0; *nranks = 1; return true; }
    *jb = d->j_begin; *je = d->j_end; *rank = d->rank; *nranks = d->nranks;
    if (d->nranks < 1 || d->rank < 0 || d->rank >= d->nranks) return false;
    if (d->j_begin < 0 || d->j_end > g->ny || d->j_end <= d->j_begin) return false;
    if (d->nranks == 1) return d->j_begin == 0 && d->j_end == g->ny;
    const int G = (int)std::min<int64_t>(8, g->ny);
    if (G % d->nranks) return false;
    const int per = G / d->nranks;
    const int64_t b0 = (int64_t)(d->rank * per) * g->ny / G, b1 = (int64_t)((d->rank + 1) * per) * g->ny / G;
    return d->j_begin == b0 && d->j_end == b1;
}

bool valid_grid(const eg_grid* g) {
    return g && g->nx >= 3 && g->ny >= 1 && g->nz >= 1 && g->nx * g->nz < (int64_t)1 << 31 &&
           g->ny < 65536 && g->nz < 65536;
}

// algorithmic HBM bytes of one red-black tri-SOR half-sweep, per grid point in units
// of V: the colour's f (or the inputs of its update) and bands, the values of x it reads, the
// colour's x (and p / s, and the colour-split f) it writes.  Layout independent: the colour-split
// copies change how much of each loaded sector is used, not what the sweep needs.
double sor_alg_bytes(const eg_solver* s, int kind, int sweep, int colour) {
    const double V = (double)s->L.vsz, n = (double)s->L.n;
    // the TMA sweeps' last half writes z in natural order, both colours (+ V / 2)
    const double fin_z = ((s->sor_tma || s->sor_tma64) && s->split && sweep == s->sor_sweeps - 1 && colour == 1) ? 0.5 * V * n : 0.0;
    if (sweep > 0) return 5 * V * n + fin_z;                           // f, 6 bands / 2; x; x / 2
    const double fin = kind == 0 ? 0.5 : (kind == 1 ? 1.5 : 1.0);     // fin | r, p, v | r, v (one colour)
    const double out = 0.5 + (kind != 0 ? 0.5 : 0.0) + (s->split ? 0.5 : 0.0);  // x, p / s, f split
    return (fin + (colour == 0 ? 1.0 : 3.0 + 0.5) + out) * V * n + fin_z;  // red: (U,D) only; black: + (E,W,N,S), red x
}

// algorithmic HBM bytes of one k_start launch, by variant:
//   entry from x0 = 0: b, diag in; bhat, r, rhat0 out (x is neither read nor stored)
//   entry from x0:     b, diag, x, 6 bands in; bhat, r, rhat0 out
//   restart:           bhat, x, 6 bands in; r, rhat0 out
//   verification:      bhat, x, 6 bands in; nothing out (the true residual norm only)
double start_bytes(const eg_solver* s, int entry, int xzero, bool write) {
    const double V = (double)s->L.vsz, X = (double)s->L.xsz, n = (double)s->L.n;
    const double out = write ? 2.0 * V : 0.0;
    if (entry && xzero) return (8.0 + 8.0 + 8.0 + out) * n;
    if (entry) return (8.0 + 8.0 + X + 6.0 * V + 8.0 + out) * n;
    return (8.0 + X + 6.0 * V + out) * n;
}

// algorithmic HBM bytes of one launch, V = vector / band bytes, X = x bytes
double alg_bytes(const eg_solver* s, int kid) {
    const double V = (double)s->L.vsz, X = (double)s->L.xsz, n = (double)s->L.n;
    double per = 0;
    switch (kid) {
        case KID_SCALE: per = 7 * 8 + 6 * V + 8; break;            // 7 fp64 in; 6 V + diag out
        case KID_START: per = 8 + X + 6 * V + 2 * V; break;        // restart (start_bytes has every variant)
        case KID_THOMAS_P: per = 5 * V + 2 * V; break;             // r,p,v,U,D; p,z
        case KID_STENCIL_A: per = 8 * V + V; break;                // z,6 bands,rhat0; v
        case KID_THOMAS_S: per = 4 * V + 2 * V; break;             // r,v,U,D; s,z_s
        case KID_STENCIL_B: per = 8 * V + V; break;                // z_s,6 bands,s; t
        case KID_UPDATE: per = X + 5 * V + X + V; break;           // x,z,z_s,s,t,rhat0; x,r
        case KID_APPLY: per = 7 * V + V; break;
        case KID_PRECOND: per = 3 * V + V; break;
        case KID_CONVERT: per = 12; break;
        case KID_VERIFY: return start_bytes(s, 0, 0, false);
        case KID_PHASE_A: per = 4 * V + 6 * V + 3 * V; break;      // r,p,v,rhat0 + B4,B2; p',z,v'
        case KID_PHASE_B: per = 2 * V + 6 * V + 3 * V; break;      // r,v' + B4,B2; s,z_s,t
        case KID_SOR: per = 5 * V; break;  // a later sweep's half: f, bands of one colour; all of x; x of one colour
        default: per = 0;
    }
    return per * n;
}

}  // namespace

// =================================== C ABI ===================================

extern "C" {

int eg_workspace_bytes(const eg_grid* grid, const eg_dist* dist, eg_precision prec, size_t* bytes) {
    int64_t jb, je;
    int rank, nranks;
    if (!valid_grid(grid) || !bytes || prec < EG_FP64 || prec > EG_FP32) return EG_ERR_ARG;
    if (!valid_dist(grid, dist, &jb, &je, &rank, &nranks)) return EG_ERR_ARG;
    Layout L;
    make_layout(grid, je - jb, prec, &L);
    *bytes = L.total;
    return EG_OK;
}

int eg_workspace_bytes_ex(const eg_grid* grid, const eg_dist* dist, eg_precision prec, uint32_t features,
                          size_t* bytes) {
    int64_t jb, je;
    int rank, nranks;
    if (!valid_grid(grid) || !bytes || prec < EG_FP64 || prec > EG_FP32 || (features & ~(EG_FEATURE_TRISOR | EG_FEATURE_BATCH)))
        return EG_ERR_ARG;
    if (!valid_dist(grid, dist, &jb, &je, &rank, &nranks)) return EG_ERR_ARG;
    Layout L;
    make_layout(grid, je - jb, prec, &L, features);
    *bytes = L.total;
    return EG_OK;
}

int eg_solver_create(const eg_grid* grid, const eg_dist* dist, const double* const bands[7],
                     eg_precision prec, void* workspace, size_t workspace_bytes, void* stream,
                     eg_solver** out) {
    return eg_solver_create_ex(grid, dist, bands, prec, 0u, workspace, workspace_bytes, stream, out);
}

int eg_solver_create_ex(const eg_grid* grid, const eg_dist* dist, const double* const bands[7],
                        eg_precision prec, uint32_t features, void* workspace, size_t workspace_bytes,
                        void* stream, eg_solver** out) {
    if (!out) return EG_ERR_ARG;
    *out = nullptr;
    if (!valid_grid(grid) || !bands || prec < EG_FP64 || prec > EG_FP32 || !workspace ||
        (features & ~(EG_FEATURE_TRISOR | EG_FEATURE_BATCH)))
        return EG_ERR_ARG;
    for (int d = 0; d < 7; ++d)
        if (!bands[d]) return EG_ERR_ARG;
    eg_solver* s = new eg_solver();
    s->grid = *grid;
    s->mode = prec;
    s->st = (cudaStream_t)stream;
    cudaGetDevice(&s->device);
    if (!valid_dist(grid, dist, &s->j_begin, &s->j_end, &s->rank, &s->nranks)) {
        delete s;
        return EG_ERR_ARG;
    }
    // the optional regions are the ones the caller asked for (features), in layout order: the
    // colour-split tri-SOR copies, then the batch staging; the workspace must hold them all
    const bool room_split = (features & EG_FEATURE_TRISOR) && grid->nx % 2 == 0;
    const bool room_batch = (features & EG_FEATURE_BATCH) != 0;
    make_layout(grid, s->j_end - s->j_begin, prec, &s->L, features);
    if (workspace_bytes < s->L.total || ((uintptr_t)workspace & 255)) {
        delete s;
        return EG_ERR_WORKSPACE;
    }
    s->ws = (unsigned char*)workspace;
    const Layout& L = s->L;
    s->B4 = s->ws + L.off_bands;
    s->B2 = s->ws + L.off_bands + (size_t)4 * L.n * L.vsz;
    s->diag = (double*)(s->ws + L.off_diag);
    s->bhat = (double*)(s->ws + L.off_bhat);
    s->x64 = (double*)(s->ws + L.off_x64);
    s->x32 = (float*)(s->ws + L.off_x32);
    s->xg = (double*)(s->ws + L.off_xg);
    for (int d = 0; d < 6; ++d) s->vec[d] = s->ws + L.off_vec + (size_t)d * align_up(L.n * L.vsz, 256);
    for (int d = 0; d < 2; ++d)
        s->zext[d] = s->ws + L.off_z + (size_t)d * align_up((L.n + 2 * L.row) * L.vsz, 256);
    s->ready_flags = (int*)(s->ws + L.off_pv);
    s->split = room_split ? (void*)(s->ws + L.off_split) : nullptr;
    s->batch = room_batch ? (double*)(s->ws + L.off_batch) : nullptr;
    s->slots = (double*)(s->ws + L.off_slots);
    s->hslots = (double*)(s->ws + L.off_hslots);
    s->gsum = (double*)(s->ws + L.off_gsum);
    s->gall = s->gsum + 8 * 3;
    s->dstate = (DevState*)(s->ws + L.off_state);
    if (cudaHostAlloc(&s->hstate, sizeof(DevState), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(&s->hstate_dev, s->hstate, 0) != cudaSuccess) {
        if (s->hstate) cudaFreeHost(s->hstate);
        delete s;
        return EG_ERR_CUDA;
    }
    Geo& g = s->geo;
    g.nx = grid->nx; g.ny = grid->ny; g.nz = grid->nz;
    g.row = L.row; g.nyl = L.nyl; g.j0 = s->j_begin; g.n = L.n; g.tiles = L.tiles;
    g.G = L.G;
    g.g_lo = s->rank * (L.G / s->nranks);
    g.g_hi = (s->rank + 1) * (L.G / s->nranks);
    // Thomas CTA width: keep 2*nz*W*sizeof(V) of factors in shared memory <= ~76 KB
    s->wth = 128;
    while (s->wth > 32 && 2 * (size_t)grid->nz * s->wth * L.vsz > 77824) s->wth /= 2;
    s->smem_th = 2 * (size_t)grid->nz * s->wth * L.vsz;
    s->cpt = (grid->nx % 2 == 0) ? 2 : 1;
    {
        // grids of < ~4 waves (8 CTAs of the default update per SM): 2-level batches, 12 CTAs per SM
        // (measured: C4 band of 144 rows -4 % update time, C3 -1 %; C4 / C5 whole grids +1 %)
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const char* pd = getenv("EG_PDL");
        s->pdl = pd && pd[0] == '1';
        const char* ukb = getenv("EG_UPDATE_KB2");  // A/B knob: 1 = on, 0 = off
        s->update_kb2 = ukb ? ukb[0] == '1' : (int64_t)L.tiles * L.nyl < (int64_t)4 * 8 * nsm;
    }
    // TMEM-factor Thomas (fp32 working precision, nz <= 128); EG_NO_TMEM=1 selects the shared-memory one
    {
        const char* no_tm = getenv("EG_NO_TMEM");
        s->use_tm = prec != EG_FP64 && grid->nz <= 128 && !(no_tm && no_tm[0] == '1');
        s->use_tm64 = prec == EG_FP64 && grid->nz <= 80 && !(no_tm && no_tm[0] == '1');
        s->smem_tm = std::max<size_t>(TM_SMEM, (size_t)grid->nz * 128 * sizeof(float));
    }
    if (s->smem_th > 227 * 1024) {
        int rc = fail(s, EG_ERR_ARG, "nz=%lld too large for the shared-memory Thomas kernel", (long long)grid->nz);
        eg_solver_destroy(s);
        return rc;
    }
    int rc = prec == EG_FP64 ? set_thomas_smem<0>(s) : prec == EG_MIXED ? set_thomas_smem<1>(s) : set_thomas_smem<2>(s);
    // k_edge_stencil's arrival counters start at 0 (each launch leaves them at 0)
    if (rc == EG_OK && cudaMemsetAsync(s->ws + L.off_edge + 8 * L.row * L.vsz, 0, 2 * (size_t)L.tiles * sizeof(int), s->st) != cudaSuccess)
        rc = fail(s, EG_ERR_CUDA, "edge-stencil counters");
    if (rc == EG_OK && s->use_tm64) {
        for (const void* f : {(const void*)k_thomas_tm64<0>, (const void*)k_thomas_tm64<1>, (const void*)k_thomas_tm64<2>})
            if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, TM64_SMEM) != cudaSuccess)
                rc = fail(s, EG_ERR_CUDA, "k_thomas_tm64 attributes");
    }
    // EG_FORCE_NCCL=1 runs a single GPU through the multi-rank path (1-rank communicator: local
    // group sums -> ncclAllGather -> logic kernel, all inside the captured graph) so that path is
    // exercised by the single-GPU parity tests.
    const char* force = getenv("EG_FORCE_NCCL");
    const bool force_nccl = s->nranks == 1 && force && force[0] == '1';
    const bool loop = rc == EG_OK && s->nranks > 1 && dist->nccl_unique_id &&
                      memcmp(dist->nccl_unique_id, kLoopMagic, sizeof kLoopMagic) == 0;
    if (loop) {  // in-process loopback group (eg_loopback_id)
        LoopGroup* G = nullptr;
        int32_t gn = 0;
        memcpy(&G, (const char*)dist->nccl_unique_id + 8, sizeof G);
        memcpy(&gn, (const char*)dist->nccl_unique_id + 16, sizeof gn);
        if (!G || gn != s->nranks) {
            rc = fail(s, EG_ERR_ARG, "loopback id is for %d ranks, dist says %d", gn, s->nranks);
        } else {
            std::lock_guard<std::mutex> lk(G->m);
            if (G->have_st && G->st != s->st) {
                rc = fail(s, EG_ERR_ARG, "the ranks of a loopback group must share one stream");
            } else {
                G->have_st = true;
                G->st = s->st;
                s->lb = G;
            }
        }
    } else if (rc == EG_OK && (s->nranks > 1 || force_nccl)) {
        ncclUniqueId id;
        ncclResult_t r = ncclSuccess;
        if (force_nccl) r = ncclGetUniqueId(&id);
        else if (!dist->nccl_unique_id) rc = EG_ERR_ARG;
        else memcpy(&id, dist->nccl_unique_id, sizeof id);
        if (rc == EG_OK && r == ncclSuccess) r = ncclCommInitRank(&s->comm, s->nranks, id, s->rank);
        if (r != ncclSuccess) rc = fail(s, EG_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    }
    {  // P2P transport for latitude bands (and the 1-rank NCCL path); EG_P2P=0 keeps NCCL / copies
        const char* pe = getenv("EG_P2P");
        s->p2p_want = (s->comm || s->lb) && !(pe && pe[0] == '0');
        if (rc == EG_OK && s->p2p_want && s->comm) rc = p2p_setup_nccl(s);
        const char* su = getenv("EG_SPLIT_UPDATE");  // A/B knob: 1 = split, 0 = one kernel
        s->split_update = su ? (su[0] == '1' && (s->comm || s->lb)) : ((s->comm || s->lb) && !s->pp.on && !(s->lb && s->p2p_want));
    }
    if (rc == EG_OK && (s->comm || s->lb)) {  // latitude bands: the overlap streams and events
        if (cudaStreamCreateWithFlags(&s->cst, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&s->xst, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->ev_edge, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->ev_halo, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->ev_b, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->ev_xu, cudaEventDisableTiming) != cudaSuccess)
            rc = fail(s, EG_ERR_CUDA, "overlap streams / events");
    }
    if (rc == EG_OK) {  // fused marching phases (march.cuh): fp32 vectors, one GPU; EG_NO_FUSE=1 disables
        const char* nf = getenv("EG_NO_FUSE");
        int dev = 0, nsm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const int64_t nz8 = (grid->nz + MA_KB - 1) / MA_KB * MA_KB;
        const size_t ring = 3 * (size_t)nz8 * MA_RING_W * sizeof(float);
        const size_t budget = 227 * 1024 - 3072 - 128;  // dynamic + static shared memory per CTA
        // two stage rings (elimination / stencil inputs) share what the z ring leaves
        const int na = ring < budget ? (int)((budget - ring) / ma_stage_bytes(1)) : 0;
        const int nb = ring < budget ? (int)((budget - ring) / ma_stage_bytes(2)) : 0;
        // below ~2^18 local points the launch-latency-bound 5-kernel schedule is faster
        // (profiles/r01_schedule_compare.txt); EG_FUSE=1 forces the fused one (tests)
        const char* ff = getenv("EG_FUSE");
        const bool big = s->L.n >= (int64_t)1 << 18 || (ff && ff[0] == '1');
        s->use_march = s->use_tm && grid->nx % 4 == 0 && nz8 <= 8 * MA_MAX_CH && 7 * nz8 <= 512 &&
                       s->L.tiles <= nsm && na >= 4 && big && !(nf && nf[0] == '1');
        if (s->use_march) {
            s->mg.fst_a = std::min(MA_MAX_STAGES, na - na / 2);
            s->mg.sst_a = std::min(MA_MAX_STAGES, na / 2);
            s->mg.fst_b = std::min(MA_MAX_STAGES, nb - nb / 2);
            s->mg.sst_b = std::min(MA_MAX_STAGES, nb / 2);
            const char* fa = getenv("EG_MARCH_FST_A");  // tuning: elimination-ring stages (rest: stencil)
            const char* fb = getenv("EG_MARCH_FST_B");
            if (fa && atoi(fa) >= 2 && na - atoi(fa) >= 2) {
                s->mg.fst_a = std::min(MA_MAX_STAGES, atoi(fa));
                s->mg.sst_a = std::min(MA_MAX_STAGES, na - atoi(fa));
            }
            if (fb && atoi(fb) >= 2 && nb - atoi(fb) >= 2) {
                s->mg.fst_b = std::min(MA_MAX_STAGES, atoi(fb));
                s->mg.sst_b = std::min(MA_MAX_STAGES, nb - atoi(fb));
            }
            // with NCCL ranks, leave a few SMs to the ghost-row exchange that runs beside the phase kernel
            // latitude bands: leave a few SMs to k_edge_rows (and NCCL's kernels), which run beside the
            // phase kernel on the communication stream
            const int sms = s->nranks > 1 ? std::max(s->L.tiles, nsm - 4) : nsm;
            s->mg.strips = (int)std::min<int64_t>(s->L.nyl, sms / s->L.tiles);
            s->mg.skip_lo = s->rank > 0;
            s->mg.skip_hi = s->rank < s->nranks - 1;
            const char* fs = getenv("EG_MARCH_STRIPS");  // tests: fewer, longer strips
            if (fs && atoi(fs) >= 1) s->mg.strips = std::min(s->mg.strips, atoi(fs));
            // tests only: more strips than SMs (a grid that cannot be co-resident; the cooperative
            // launch must refuse it with EG_ERR_CUDA rather than hang)
            const char* fo = getenv("EG_MARCH_STRIPS_UNSAFE");
            if (fo && atoi(fo) >= 1) s->mg.strips = (int)std::min<int64_t>(s->L.nyl, atoi(fo));
            // at least ~116 KB so that exactly one CTA (and one 512-column TMEM allocation) fits an SM
            const size_t st_a = (size_t)(s->mg.fst_a + s->mg.sst_a) * ma_stage_bytes(1);
            const size_t st_b = (size_t)(s->mg.fst_b + s->mg.sst_b) * ma_stage_bytes(2);
            s->smem_march = std::max<size_t>(std::max(st_a, st_b) + ring + 128, 116 * 1024);
            cudaError_t e1 = prec == EG_MIXED
                ? cudaFuncSetAttribute(k_march<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem_march)
                : cudaFuncSetAttribute(k_march<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem_march);
            cudaError_t e2 = prec == EG_MIXED
                ? cudaFuncSetAttribute(k_march<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem_march)
                : cudaFuncSetAttribute(k_march<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem_march);
            int occ = 0;
            cudaError_t e3 = prec == EG_MIXED
                ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_march<1, 2>, MA_THREADS, s->smem_march)
                : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_march<2, 2>, MA_THREADS, s->smem_march);
            cudaError_t e4 = cudaMemsetAsync(s->ready_flags, 0, (size_t)s->L.nyl * s->L.tiles * sizeof(int), s->st);
            if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess || e4 != cudaSuccess)
                rc = fail(s, EG_ERR_CUDA, "march setup: %s", cudaGetErrorString(cudaGetLastError()));
            else if (occ != 1 || !make_march_maps(s))  // co-residency of every CTA makes the flag waits safe
                s->use_march = false;
        }
    }
    if (rc == EG_OK && prec == EG_FP64 && !(s->comm || s->lb)) {
        // FP64 fused phases (march64.cuh): one GPU, nx even, 6 ceil4(nz) <= 512 TMEM columns, 64-column
        // tiles <= #SMs; EG_NO_FUSE=1 disables, EG_FUSE=1 forces below 2^18 points
        const char* nf = getenv("EG_NO_FUSE");
        const char* ff = getenv("EG_FUSE");
        int dev = 0, nsm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const int64_t nz4 = (grid->nz + M6_KS - 1) / M6_KS * M6_KS;
        const int t64 = (int)((grid->nx + M6_TILE - 1) / M6_TILE);
        const size_t ring = 3 * (size_t)nz4 * M6_RING_W * sizeof(double);
        const size_t budget = 227 * 1024 - 4096 - 128;  // dynamic + static shared memory per CTA
        const bool big = s->L.n >= (int64_t)1 << 18 || (ff && ff[0] == '1');
        bool ok = grid->nx % 2 == 0 && nz4 <= M6_MAX_NZ4 && t64 <= nsm && ring < budget && big && !(nf && nf[0] == '1');
        if (ok) {
            // stage rings: as many stencil stages as elimination ones, the rest to the elimination ring
            auto split = [&](int kind, int* nf_, int* ns_) {
                const size_t room = budget - ring;
                const int ns = (int)std::min<size_t>(M6_MAX_STAGES, room / (m6_f_bytes(kind) + m6_s_bytes(kind)));
                const int nfs = (int)std::min<size_t>(M6_MAX_STAGES, (room - ns * (size_t)m6_s_bytes(kind)) / m6_f_bytes(kind));
                *nf_ = nfs;
                *ns_ = ns;
            };
            split(1, &s->mg.fst_a, &s->mg.sst_a);
            split(2, &s->mg.fst_b, &s->mg.sst_b);
            ok = s->mg.fst_a >= 2 && s->mg.sst_a >= 2 && s->mg.fst_b >= 2 && s->mg.sst_b >= 2;
        }
        // 64-column tiles x strips must keep >= 90 % of the SMs busy: one CTA per SM moves ~1/nsm of the
        // bandwidth, and the fused kernel saves only 18 % of the 5-kernel bytes (measured: C4, 24 x 6 =
        // 144 CTAs, 6 % faster; C5, 40 x 3 = 120 CTAs, 5 % slower).  EG_FUSE=1 forces it.
        const int64_t ctas = (int64_t)t64 * std::min<int64_t>(s->L.nyl, nsm / t64);
        if (ok && !(ff && ff[0] == '1') && ctas * 10 < (int64_t)nsm * 9) ok = false;
        if (ok) {
            s->mg.strips = (int)std::min<int64_t>(s->L.nyl, nsm / t64);
            const char* fs = getenv("EG_MARCH_STRIPS");
            if (fs && atoi(fs) >= 1) s->mg.strips = std::min(s->mg.strips, atoi(fs));
            const char* fo = getenv("EG_MARCH_STRIPS_UNSAFE");
            if (fo && atoi(fo) >= 1) s->mg.strips = (int)std::min<int64_t>(s->L.nyl, atoi(fo));
            s->mg.skip_lo = s->mg.skip_hi = 0;
            const size_t st_a = (size_t)s->mg.fst_a * m6_f_bytes(1) + (size_t)s->mg.sst_a * m6_s_bytes(1);
            const size_t st_b = (size_t)s->mg.fst_b * m6_f_bytes(2) + (size_t)s->mg.sst_b * m6_s_bytes(2);
            s->smem_march = std::max<size_t>(std::max(st_a, st_b) + ring + 128, 116 * 1024);
            int occ = 0;
            cudaError_t e1 = cudaFuncSetAttribute(k_march64<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem_march);
            cudaError_t e2 = cudaFuncSetAttribute(k_march64<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem_march);
            cudaError_t e3 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_march64<1>, M6_THREADS, s->smem_march);
            cudaError_t e4 = cudaMemsetAsync(s->ready_flags, 0, (size_t)s->L.nyl * t64 * sizeof(int), s->st);
            cudaError_t e5 = cudaMemsetAsync(s->hslots, 0, 3 * 4 * (size_t)s->L.nyl * s->L.tiles * sizeof(double), s->st);
            if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess || e4 != cudaSuccess || e5 != cudaSuccess)
                rc = fail(s, EG_ERR_CUDA, "FP64 march setup: %s", cudaGetErrorString(cudaGetLastError()));
            else
                s->use_march = occ == 1 && make_march_maps64(s);
        }
    }
    // The TMA box of the colour-split f starts at column nx/2 for the second colour: a TMA box must
    // start on a 16-byte boundary of its row (measured: an illegal-instruction fault otherwise), so
    // the sweeps need nx/2 * sizeof(V) % 16 == 0, i.e. nx % 8 == 0 (fp32) / nx % 4 == 0 (FP64).
    if (rc == EG_OK && s->split && prec != EG_FP64 && grid->nx % 8 == 0 && grid->nz <= SO_MAX_NZ8 && s->use_tm) {
        // later tri-SOR sweeps on the TMA-fed kernel (EG_NO_SOR_TMA=1 keeps k_sor_half)
        const char* ns = getenv("EG_NO_SOR_TMA");
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&s->nsm, cudaDevAttrMultiProcessorCount, dev);
        const int smem = SO_STAGES * SO_STAGE_FLOATS * 4 + 128;
        cudaError_t e1 = cudaSuccess;
        auto attr = [&](const void* f, int bytes) {
            if (e1 == cudaSuccess) e1 = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        };
        if (prec == EG_MIXED) {
            attr((const void*)k_sor_tma<1, true>, smem); attr((const void*)k_sor_tma<1, false>, smem);
            attr((const void*)k_sor_first_red<1, 0>, (int)s->smem_th); attr((const void*)k_sor_first_red<1, 1>, (int)s->smem_th);
            attr((const void*)k_sor_first_red<1, 2>, (int)s->smem_th);
        } else {
            attr((const void*)k_sor_tma<2, true>, smem); attr((const void*)k_sor_tma<2, false>, smem);
            attr((const void*)k_sor_first_red<2, 0>, (int)s->smem_th); attr((const void*)k_sor_first_red<2, 1>, (int)s->smem_th);
            attr((const void*)k_sor_first_red<2, 2>, (int)s->smem_th);
        }
        s->sor_tma = e1 == cudaSuccess && !(ns && ns[0] == '1') && make_sor_maps(s);
    }
    if (rc == EG_OK && prec == EG_FP64 && grid->nx % 2 == 0 && grid->nz <= SO_MAX_NZ8) {
        // FP64 Thomas of the iteration on the TMA-fed kernel (EG_NO_THOMAS_TMA=1 keeps k_thomas_tm64)
        const char* nt = getenv("EG_NO_THOMAS_TMA");
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&s->nsm, cudaDevAttrMultiProcessorCount, dev);
        const cudaError_t e1 = cudaFuncSetAttribute(k_thomas_tma64<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, T6_SMEM);
        s->th_tma64 = e1 == cudaSuccess && !(nt && nt[0] == '1') && make_thomas_maps64(s);
    }
    if (rc == EG_OK && s->split && prec == EG_FP64 && grid->nx % 4 == 0 && grid->nz <= SO_MAX_NZ8) {
        // FP64: later tri-SOR sweeps on k_sor_tma64 (EG_NO_SOR_TMA=1 keeps k_sor_half)
        const char* ns = getenv("EG_NO_SOR_TMA");
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&s->nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaError_t e1 = cudaSuccess;
        auto attr = [&](const void* f, int bytes) {
            if (e1 == cudaSuccess) e1 = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        };
        attr((const void*)k_sor_tma64<true>, S6_SMEM); attr((const void*)k_sor_tma64<false>, S6_SMEM);
        attr((const void*)k_sor_first_red<0, 0>, (int)s->smem_th); attr((const void*)k_sor_first_red<0, 1>, (int)s->smem_th);
        attr((const void*)k_sor_first_red<0, 2>, (int)s->smem_th);
        s->sor_tma64 = e1 == cudaSuccess && !(ns && ns[0] == '1') && make_sor_maps64(s);
    }
#ifdef MA_VERIFY
    if (rc == EG_OK && g_vfy.n != s->L.n) {
        const int64_t n = s->L.n;
        g_vfy.n = n;
        if (cudaMalloc(&g_vfy.p, 6 * n * sizeof(float)) != cudaSuccess ||
            cudaMalloc(&g_vfy.slots, 3 * s->L.nyl * s->L.tiles * sizeof(double)) != cudaSuccess)
            rc = EG_ERR_CUDA;
        g_vfy.v = g_vfy.p + n; g_vfy.z = g_vfy.v + n; g_vfy.s = g_vfy.z + n; g_vfy.zs = g_vfy.s + n; g_vfy.t = g_vfy.zs + n;
    }
#endif
    if (rc == EG_OK)
        rc = prec == EG_FP64 ? create_impl<0>(s, bands) : prec == EG_MIXED ? create_impl<1>(s, bands) : create_impl<2>(s, bands);
    if (rc != EG_OK) {
        eg_solver_destroy(s);
        return rc;
    }
    *out = s;
    return EG_OK;
}

int eg_solver_set_operator(eg_solver* s, const double* const bands[7]) {
    if (!s || !bands) return EG_ERR_ARG;
    for (int d = 0; d < 7; ++d)
        if (!bands[d]) return EG_ERR_ARG;
    return s->mode == EG_FP64 ? create_impl<0>(s, bands) : s->mode == EG_MIXED ? create_impl<1>(s, bands) : create_impl<2>(s, bands);
}

int eg_solver_set_preconditioner(eg_solver* s, int kind, int sweeps, double omega) {
    if (!s) return EG_ERR_ARG;
    if (kind == EG_PRECOND_TRIDIAG) {
        s->precond = kind;
    } else if (kind == EG_PRECOND_TRISOR) {
        if (s->grid.nx % 2 != 0 || sweeps < 1 || !(omega > 0.0 && omega < 2.0))
            return fail(s, EG_ERR_ARG, "tri-SOR needs nx even, sweeps >= 1 and 0 < omega < 2");
        s->precond = kind;
        s->sor_sweeps = sweeps;
        s->sor_omega = omega;
    } else {
        return fail(s, EG_ERR_ARG, "unknown preconditioner %d", kind);
    }
    for (int gi = 0; gi < 2; ++gi)  // the captured iteration depends on the preconditioner
        if (s->graphs[gi]) {
            cudaGraphExecDestroy(s->graphs[gi]);
            s->graphs[gi] = nullptr;
            s->graphs_x[gi] = nullptr;
        }
    s->graph = nullptr;
    return EG_OK;
}

// the [p, p + bytes) ranges of two buffers overlap
bool overlaps(const void* a, const void* b, size_t bytes) {
    const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return x < y + bytes && y < x + bytes;
}

int eg_apply_operator(eg_solver* s, const void* x, void* y) {
    if (!s || !x || !y) return EG_ERR_ARG;
    if (overlaps(x, y, (size_t)s->L.n * s->L.vsz))  // the stencil reads x's neighbours while y is written
        return fail(s, EG_ERR_ARG, "eg_apply_operator: x and y overlap");
    s->profiling = false;
    return s->mode == EG_FP64 ? apply_impl<0>(s, x, y) : s->mode == EG_MIXED ? apply_impl<1>(s, x, y) : apply_impl<2>(s, x, y);
}

int eg_precondition(eg_solver* s, const void* r, void* z) {
    if (!s || !r || !z) return EG_ERR_ARG;
    if (overlaps(r, z, (size_t)s->L.n * s->L.vsz))
        return fail(s, EG_ERR_ARG, "eg_precondition: r and z overlap");
    s->profiling = false;
    return s->mode == EG_FP64 ? precond_impl<0>(s, r, z) : s->mode == EG_MIXED ? precond_impl<1>(s, r, z) : precond_impl<2>(s, r, z);
}

int eg_solve(eg_solver* s, const double* b, const double* x0, const eg_solve_params* params, double* x,
             double* history, eg_solve_info* info) {
    if (!s || !b || !x || !params || params->maxit < 0 || !(params->tol >= 0.0))
        return s ? fail(s, EG_ERR_ARG, "bad solve arguments") : EG_ERR_ARG;
    if (params->maxit > kMaxIt) return fail(s, EG_ERR_ARG, "maxit > %d", kMaxIt);
    if (params->rhat0 && !is_device_ptr(params->rhat0)) return fail(s, EG_ERR_ARG, "rhat0 must be device memory");
    std::unique_lock<std::recursive_mutex> lk(g_fused_solve_mu[s->device % kMaxDevices], std::defer_lock);
    if (s->use_march && !s->lb) lk.lock();
    int rc = s->mode == EG_FP64 ? solve_impl<0>(s, b, x0, params, x, history, info)
           : s->mode == EG_MIXED ? solve_impl<1>(s, b, x0, params, x, history, info)
                                 : solve_impl<2>(s, b, x0, params, x, history, info);
    // every finaliser launch bumps the epoch, including launches of a replayed chunk past a halt: the
    // next solve starts past the last epoch this one used (the host mirror is read after the last one)
    s->epoch_base = std::max<int64_t>(s->epoch_base, (int64_t)s->hstate->epoch + 1);
    s->gseq = s->hstate->gseq;
    if (rc != EG_OK && info) info->status = rc;
    return rc;
}

int eg_solve_batch(eg_solver* s, int count, const double* const* b, double* const* x,
                   const double* const bands[7], const eg_solve_params* params, double* history,
                   eg_solve_info* info, int* done) {
    if (done) *done = 0;
    if (!s || count < 0 || (count > 0 && (!b || !x)) || !params || params->maxit < 0 || !(params->tol >= 0.0))
        return s ? fail(s, EG_ERR_ARG, "bad batch arguments") : EG_ERR_ARG;
    for (int k = 0; k < count; ++k)
        if (!b[k] || !x[k]) return fail(s, EG_ERR_ARG, "NULL b / x in the batch");
    if (!s->batch) return fail(s, EG_ERR_WORKSPACE, "eg_solve_batch needs an EG_FEATURE_BATCH workspace");
    if (params->maxit > kMaxIt) return fail(s, EG_ERR_ARG, "maxit > %d", kMaxIt);
    std::unique_lock<std::recursive_mutex> lk(g_fused_solve_mu[s->device % kMaxDevices], std::defer_lock);
    if (s->use_march && !s->lb) lk.lock();
    if (!s->cin) {
        CK(cudaStreamCreateWithFlags(&s->cin, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&s->cout, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            CK(cudaEventCreateWithFlags(&s->ev_in[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&s->ev_x[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&s->ev_out[i], cudaEventDisableTiming));
        }
    }
    const size_t nb = (size_t)s->L.n * sizeof(double);
    double* db[2] = {s->batch, s->batch + s->L.n};
    double* dx[2] = {s->batch + 2 * s->L.n, s->batch + 3 * s->L.n};
    auto upload = [&](int k) -> int {  // b[k] -> db[k % 2] on the input copy stream
        CK(cudaMemcpyAsync(db[k & 1], b[k], nb, cudaMemcpyDefault, s->cin));
        CK(cudaEventRecord(s->ev_in[k & 1], s->cin));
        return EG_OK;
    };
    int rc = count > 0 ? upload(0) : EG_OK;
    const size_t hs = (size_t)params->maxit + 1;
    for (int k = 0; k < count && rc == EG_OK; ++k) {
        const int i = k & 1;
        // db[(k+1) % 2] was read by solve k-1, which has returned: refill it while solve k runs
        if (k + 1 < count && (rc = upload(k + 1))) break;
        if (bands && (rc = eg_solver_set_operator(s, bands))) break;  // overlaps the upload of b[k]
        CK(cudaStreamWaitEvent(s->st, s->ev_in[i], 0));
        if (k >= 2) CK(cudaStreamWaitEvent(s->st, s->ev_out[i], 0));  // dx[i]'s download (solve k-2)
        rc = eg_solve(s, db[i], nullptr, params, dx[i], history ? history + (size_t)k * hs : nullptr,
                      info ? info + k : nullptr);
        if (rc) break;
        CK(cudaEventRecord(s->ev_x[i], s->st));
        CK(cudaStreamWaitEvent(s->cout, s->ev_x[i], 0));
        CK(cudaMemcpyAsync(x[k], dx[i], nb, cudaMemcpyDefault, s->cout));  // overlaps solve k+1
        CK(cudaEventRecord(s->ev_out[i], s->cout));
        if (done) *done = k + 1;
    }
    CK(cudaStreamSynchronize(s->cout));
    CK(cudaStreamSynchronize(s->cin));
    return rc;
}

void eg_solver_destroy(eg_solver* s) {
    if (!s) return;
    for (int gi = 0; gi < 2; ++gi)
        if (s->graphs[gi]) cudaGraphExecDestroy(s->graphs[gi]);
    if (s->cap_st) cudaStreamDestroy(s->cap_st);
    if (s->cin) cudaStreamDestroy(s->cin);
    if (s->cout) cudaStreamDestroy(s->cout);
    if (s->cst) cudaStreamDestroy(s->cst);
    if (s->xst) cudaStreamDestroy(s->xst);
    for (cudaEvent_t e : {s->ev_edge, s->ev_halo, s->ev_b, s->ev_xu})
        if (e) cudaEventDestroy(e);
    for (int i = 0; i < 2; ++i) {
        if (s->ev_in[i]) cudaEventDestroy(s->ev_in[i]);
        if (s->ev_x[i]) cudaEventDestroy(s->ev_x[i]);
        if (s->ev_out[i]) cudaEventDestroy(s->ev_out[i]);
    }
    for (void* p : s->ipc_open) cudaIpcCloseMemHandle(p);
    if (s->comm) ncclCommDestroy(s->comm);
    if (s->lb) {  // the last member frees the group
        LoopGroup* G = s->lb;
        bool last;
        {
            std::lock_guard<std::mutex> lk(G->m);
            last = --G->refs == 0;
        }
        if (last) delete G;
    }
    for (auto& p : s->pending) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
    for (auto e : s->evpool) cudaEventDestroy(e);
    if (s->hstate) cudaFreeHost(s->hstate);
    delete s;
}

const char* eg_last_error(const eg_solver* s) { return s ? s->err.c_str() : ""; }

const char* eg_status_str(int status) {
    switch (status) {
        case EG_OK: return "EG_OK";
        case EG_ERR_ARG: return "EG_ERR_ARG";
        case EG_ERR_SINGULAR_DIAG: return "EG_ERR_SINGULAR_DIAG";
        case EG_ERR_DEGENERATE_RHS: return "EG_ERR_DEGENERATE_RHS";
        case EG_ERR_BREAKDOWN: return "EG_ERR_BREAKDOWN";
        case EG_ERR_NONFINITE: return "EG_ERR_NONFINITE";
        case EG_ERR_CUDA: return "EG_ERR_CUDA";
        case EG_ERR_NCCL: return "EG_ERR_NCCL";
        case EG_ERR_WORKSPACE: return "EG_ERR_WORKSPACE";
        default: return "EG_ERR_UNKNOWN";
    }
}

int eg_nccl_unique_id(char out[128]) {
    if (!out) return EG_ERR_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return EG_ERR_NCCL;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    memcpy(out, &id, 128);
    return EG_OK;
}

int eg_loopback_id(int nranks, char out[128]) {
    if (!out || nranks < 1) return EG_ERR_ARG;
    LoopGroup* G = new LoopGroup();
    G->n = G->refs = nranks;
    G->first.assign(nranks, nullptr);
    G->last.assign(nranks, nullptr);
    G->gsum.assign(nranks, nullptr);
    G->ws.assign(nranks, nullptr);
    G->split.assign(nranks, 0);
    memset(out, 0, 128);
    memcpy(out, kLoopMagic, sizeof kLoopMagic);
    memcpy(out + 8, &G, sizeof G);
    const int32_t n32 = nranks;
    memcpy(out + 16, &n32, sizeof n32);
    return EG_OK;
}

int eg_debug_ipc_export(const void* ptr, unsigned char out[80]) {
    if (!ptr || !out) return EG_ERR_ARG;
    const IpcRec r = ipc_export(ptr);
    memcpy(out, &r, sizeof r);
    return r.ok ? EG_OK : EG_ERR_CUDA;
}
int eg_debug_ipc_open(const unsigned char in[80], void** ptr, void** opened) {
    if (!in || !ptr || !opened) return EG_ERR_ARG;
    IpcRec r;
    memcpy(&r, in, sizeof r);
    *ptr = ipc_open(r, opened);
    return *ptr ? EG_OK : EG_ERR_CUDA;
}
int eg_debug_ipc_close(void* opened) {
    return cudaIpcCloseMemHandle(opened) == cudaSuccess ? EG_OK : EG_ERR_CUDA;
}

int eg_solver_transport(const eg_solver* s) {
    if (!s) return -EG_ERR_ARG;
    if (s->lb) return s->p2p_want ? EG_TRANSPORT_LOOPBACK_P2P : EG_TRANSPORT_LOOPBACK;
    if (s->comm) return s->pp.on ? EG_TRANSPORT_P2P : EG_TRANSPORT_NCCL;
    return EG_TRANSPORT_NONE;
}

int eg_num_kernels(void) { return KID_COUNT; }

const char* eg_kernel_name(int kid) { return (kid >= 0 && kid < KID_COUNT) ? kKernelNames[kid] : ""; }

int eg_profile_get(const eg_solver* s, int kid, double* total_ms, int64_t* launches,
                   double* alg_bytes_per_launch) {
    if (!s || kid < 0 || kid >= KID_COUNT) return EG_ERR_ARG;
    if (total_ms) *total_ms = s->prof_ms[kid];
    if (launches) *launches = s->prof_n[kid];
    if (alg_bytes_per_launch)  // the profiled launches' average, else the steady-state figure
        *alg_bytes_per_launch = s->prof_n[kid] > 0 ? s->prof_bytes[kid] / (double)s->prof_n[kid] : alg_bytes(s, kid);
    return EG_OK;
}

#ifdef MA_TRACE
// debug builds only (not declared in include/egsolve.h): per-CTA cycle counters of the last march
int eg_debug_march_trace(unsigned long long* out, int n) {
    return cudaMemcpyFromSymbol(out, g_ma_trace, (size_t)n * sizeof(unsigned long long)) == cudaSuccess ? 0 : EG_ERR_CUDA;
}
#endif


#ifdef MA_VERIFY
int eg_debug_verify(unsigned long long* cnt8, long long* rec128, int* nrec) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(cnt8, g_vfy_cnt, 8 * sizeof(unsigned long long));
    cudaMemcpyFromSymbol(rec128, g_vfy_rec, 256 * sizeof(long long));
    cudaMemcpyFromSymbol(nrec, g_vfy_nrec, sizeof(int));
    unsigned long long z8[8] = {0};
    int z = 0;
    cudaMemcpyToSymbol(g_vfy_cnt, z8, sizeof(z8));
    cudaMemcpyToSymbol(g_vfy_nrec, &z, sizeof(z));
    return EG_OK;
}
#endif


int eg_profile_reset(eg_solver* s) {
    if (!s) return EG_ERR_ARG;
    for (int k = 0; k < KID_COUNT; ++k) { s->prof_ms[k] = 0; s->prof_bytes[k] = 0; s->prof_n[k] = 0; }
    return EG_OK;
}

}  // extern "C"
