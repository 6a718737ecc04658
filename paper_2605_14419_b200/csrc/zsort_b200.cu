// zsort_b200.cu -- host orchestration and the C ABI (include/zsort_b200.h).
//
// zsb_sort replaces core.zsort -> _kernels.zsort_driver -> _run_worklist
// (core.py:348-400, _kernels.py:321-450).  One partition level is the
// launch sequence  K1 moments -> K2 hist -> K3 scan -> K4 scatter -> classify
// -> plan, all on the caller's stream; the host reads back one small control
// block per level (how many oversized buckets recurse, how many finish runs
// to launch), then launches K5 over that level's finish runs.  Recursion
// levels batch every oversized bucket of the previous level into one
// segmented launch (device-side segment table, no per-segment host work).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <mutex>
#include <unordered_map>

#include "../../include/zsort_b200.h"
#include "dist_kernels.cuh"
#include "gen_kernels.cuh"
#include "sort_kernels.cuh"

using namespace zsb;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

// ---- optional per-phase device timing (CUDA events on the sort's stream)
enum Phase { PH_MOMENTS = 0, PH_HIST, PH_SCAN, PH_SCATTER, PH_CLASSIFY, PH_FINISH, PH_SEGSTATS, PH_MISC, PH_SLOTS };

struct Timing {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    std::vector<int> slot_of;  // per recorded pair
    size_t used = 0;
    double ms[PH_SLOTS] = {0};
    long long launches[PH_SLOTS] = {0};
    long long records[PH_SLOTS] = {0};  // records each phase's launches processed (histogram, scatter, finish)
    long long launch_total = 0;
};
thread_local Timing g_t;

struct PhaseScope {
    int slot;
    cudaStream_t st;
    bool active;
    PhaseScope(int s, cudaStream_t stream, int nlaunch = 1) : slot(s), st(stream), active(g_t.on) {
        g_t.launch_total += nlaunch;
        g_t.launches[s] += nlaunch;
        if (!active) return;
        if (g_t.used + 2 > g_t.pool.size()) {
            for (int i = 0; i < 64; i++) {
                cudaEvent_t e;
                cudaEventCreate(&e);
                g_t.pool.push_back(e);
            }
        }
        cudaEventRecord(g_t.pool[g_t.used], st);
    }
    ~PhaseScope() {
        if (!active) return;
        cudaEventRecord(g_t.pool[g_t.used + 1], st);
        g_t.slot_of.push_back(slot);
        g_t.used += 2;
    }
};

// launches outside any PhaseScope (multi-GPU phases): counted under misc
inline void count_launches(int nl) {
    g_t.launch_total += nl;
    g_t.launches[PH_MISC] += nl;
}

// after a stream sync: fold recorded pairs into the per-phase totals
void timing_collect() {
    if (!g_t.on) return;
    for (size_t i = 0; i < g_t.slot_of.size(); i++) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, g_t.pool[2 * i], g_t.pool[2 * i + 1]) == cudaSuccess) g_t.ms[g_t.slot_of[i]] += ms;
    }
    g_t.slot_of.clear();
    g_t.used = 0;
}

#define ZSB_CUDA(call)                                                                                  \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess)                                                                          \
            return fail(ZSB_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));              \
    } while (0)

#define ZSB_LAUNCH(what)                                                                                \
    do {                                                                                                \
        cudaError_t e_ = cudaGetLastError();                                                            \
        if (e_ != cudaSuccess) return fail(ZSB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Tuning constants: the defaults are the measured best on B200 (DESIGN.md
// §4, knob table); experiments rebuild the library with -D<NAME>=<value>
// (tools/build_variant.sh).  Nothing in the library reads the environment.
#ifndef ZSB_K1MAX
#define ZSB_K1MAX 1024  // cap on the fitted level-1 bucket count
#endif
#ifndef ZSB_TEAM_L1
#define ZSB_TEAM_L1 0  // 1: level-1 buckets up to TEAM * cap are team runs (k sized for them); measured slower
#endif
#ifndef ZSB_LPT
#define ZSB_LPT 1  // the finish takes a level's runs longest first (order from classify) when they sit in L2
#endif
#ifndef ZSB_CHILD_FROM_CDF
#define ZSB_CHILD_FROM_CDF 1  // children of the equalised level 1 ranged by its CDF: no level-2 moments pass
#endif
#ifndef ZSB_HIST_RING_ALL
#define ZSB_HIST_RING_ALL 0  // 1: recursion-level histograms also stage keys through the TMA ring (measured C4 +2 %)
#endif
#ifndef ZSB_K1_TEAM
#define ZSB_K1_TEAM 2048  // cap on the level-1 bucket count when buckets are sized for team runs
#endif
#ifndef ZSB_SW16_ABOVE
#define ZSB_SW16_ABOVE 512  // bucket counts above this use 16-warp, 8192-record scatter rounds
#endif
#ifndef ZSB_TILES_PER_SM
#define ZSB_TILES_PER_SM 0  // level-1 tiles per SM; 0: 1 for 16-warp scatter rounds, 2 for 8-warp
#endif
#ifndef ZSB_WIN_PCT
#define ZSB_WIN_PCT 75  // level-1 finish window, % of the run capacity
#endif
#ifndef ZSB_CHILD_FILL
#define ZSB_CHILD_FILL 2  // recursion children: k = pow2 >= fill * len / cap
#endif
#ifndef ZSB_GREEDY
#define ZSB_GREEDY 1  // greedy finish runs on recursion levels (else fixed windows)
#endif
#ifndef ZSB_MIN_TILE
#define ZSB_MIN_TILE 8192  // recursion tile floor (raised up to 4x on long levels)
#endif
#ifndef ZSB_L2_PREFETCH
#define ZSB_L2_PREFETCH -1  // L2 prefetch of each CTA's next finish run: -1 auto (records > 128 MB), 0/1 forced
#endif
#ifndef ZSB_NO_SAMPLE
#define ZSB_NO_SAMPLE 0  // 1: exact K1 + exact coarse histogram at level 1 instead of the sample
#endif
#ifndef ZSB_NO_EQUALIZE
#define ZSB_NO_EQUALIZE 0  // 1: plain fitted z-score at level 1 (no CDF equalisation)
#endif
#ifndef ZSB_REFINE_LAUNCH
#define ZSB_REFINE_LAUNCH 0  // 1: refine iterations as a launch of their own instead of inside the finish grid
#endif

int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

constexpr int K_LEVEL1_MAX = KSCAT_MAX;  // fan-out of one scatter pass
constexpr int KMAX_CHILD = 1024;

int finish_cap(int pb) { return FT * (pb == 8 ? FinItems<8>::F : (pb == 4 ? FinItems<4>::F : FinItems<0>::F)); }

// Finish windows: classify cuts a segment into windows of this many records;
// a run is the buckets starting inside one window, plus the last of them if it
// has at most cap - window records (else that bucket is a run of its own).  A
// wider window packs small buckets into fuller runs (fewer, longer finish
// runs); measured on B200 (C4): 50% 4.80 ms, 66% 4.52 ms, 75% 4.43 ms.
int64_t fin_window(int64_t cap) {
    return std::max<int64_t>(256, std::min<int64_t>(cap - 256, cap * ZSB_WIN_PCT / 100));
}

int64_t cluster_count(int64_t n, double alpha) {  // core.py:146-148
    double v = std::nearbyint(alpha * std::sqrt((double)n));
    int64_t k = (int64_t)v;
    return k < 2 ? 2 : k;
}

int64_t pow2_at_least(int64_t x) {
    int64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

// Level-1 plan: bucket count and tiling of the whole input.
struct Plan1 {
    int64_t k, tile_len, ntiles, cap, half;  // half: finish window width (see fin_window)
};

Plan1 plan_level1(int64_t n, int pb, const zsb_config &cfg) {
    Plan1 P;
    P.cap = finish_cap(pb);
    P.half = fin_window(P.cap);
    if (cfg.mapping == ZSB_MAP_PAPER) {
        P.k = std::min<int64_t>(cluster_count(n, cfg.alpha), K_LEVEL1_MAX);
    } else {
        const int64_t kmax = ZSB_K1MAX;  // runs of >= 4 records per 4096-record round
        P.k = std::min<int64_t>(std::max<int64_t>(16, pow2_at_least((4 * n + P.cap - 1) / P.cap)), kmax);
        // large inputs: buckets of ~half a team run (K5t finishes them without a second level)
        const int64_t tcap = (int64_t)TEAM * P.cap;
        if (TEAM_ON && ZSB_TEAM_L1 && n / P.k > tcap / 2) P.k = std::min<int64_t>(pow2_at_least((2 * n + tcap - 1) / tcap), ZSB_K1_TEAM);
    }
    const int tps = ZSB_TILES_PER_SM > 0 ? ZSB_TILES_PER_SM : (scat_warps((int)P.k, ZSB_SW16_ABOVE) == 8 ? 2 : 1);
    int64_t target_tiles = (int64_t)num_sms() * tps;
    int64_t tl = std::max<int64_t>(4 * P.k, (n + target_tiles - 1) / target_tiles);
    tl = std::max<int64_t>(tl, 2048);
    tl = (tl + 255) & ~(int64_t)255;
    P.tile_len = tl;
    P.ntiles = (n + tl - 1) / tl;
    return P;
}

// zsort_rec plan: the caller's k (clamped to one pass's fan-out), level-1 tiling.
Plan1 plan_rec(int64_t n, int pb, int64_t k) {
    zsb_config c = zsb_config{0.6, 96, 65000, 32, 0, ZSB_MAP_PAPER};
    Plan1 P = plan_level1(n, pb, c);
    P.k = std::max<int64_t>(2, std::min<int64_t>(k, K_LEVEL1_MAX));
    int64_t tl = std::max<int64_t>(std::max<int64_t>(4 * P.k, 2048), P.tile_len);
    tl = (tl + 255) & ~(int64_t)255;
    P.tile_len = tl;
    P.ntiles = (n + tl - 1) / tl;
    return P;
}

struct Layout {
    size_t tmp_k, tmp_p, mat, status, seg_a, seg_b, acc, kfirst, wfirst, bstart, entries, order, teams, refine[4], parts,
        ctrl, dbg, fine, lut, total;
    int64_t mat_cap, seg_cap, ent_cap, status_cap, slot_cap, ref_cap, team_cap_list;
};

constexpr int MOM_GRID_PER_SM = 4;
constexpr int OCC_CHUNKS = 1024;  // occurrence search: chunks of pass 1

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

Layout make_layout(int64_t n, int pb, const Plan1 &P, bool need_tmp) {
    Layout L;
    const int64_t cap = P.cap;
    L.mat_cap = std::max<int64_t>(P.k * P.ntiles, n / 4 + 24 * (n / cap + 1) + 4096) + 16;
    L.seg_cap = n / cap + 4;
    L.ent_cap = 2 * (n / P.half + 1) + 2 * L.seg_cap + 4096;
    L.slot_cap = std::max<int64_t>(P.k + 1, 24 * (n / cap + 1) + 2 * L.seg_cap) + 16;
    L.ref_cap = n / (FIN_INS + 1) + 1024;
    L.status_cap = L.mat_cap / SCAN_TILE + 4;
    size_t o = 0;
    L.tmp_k = o;
    if (need_tmp) o = align_up(o + (size_t)n * 8);
    L.tmp_p = o;
    if (need_tmp) o = align_up(o + (size_t)n * pb);
    L.mat = o;
    o = align_up(o + (size_t)L.mat_cap * 4);
    L.status = o;
    o = align_up(o + (size_t)L.status_cap * 8);
    L.seg_a = o;
    o = align_up(o + (size_t)L.seg_cap * sizeof(SegParams));
    L.seg_b = o;
    o = align_up(o + (size_t)L.seg_cap * sizeof(SegParams));
    L.acc = o;
    o = align_up(o + (size_t)L.seg_cap * sizeof(SegAcc));
    L.kfirst = o;
    o = align_up(o + (size_t)(L.seg_cap + 2) * 8);
    L.wfirst = o;
    o = align_up(o + (size_t)(L.seg_cap + 2) * 8);
    L.bstart = o;
    o = align_up(o + (size_t)L.slot_cap * 8);
    L.entries = o;
    o = align_up(o + (size_t)L.ent_cap * sizeof(Entry));
    L.order = o;  // finish order of a level's runs (longest first)
    o = align_up(o + (size_t)L.ent_cap * 4);
    L.team_cap_list = n / cap + 16;  // team runs hold > cap records each
    L.teams = o;
    o = align_up(o + (size_t)L.team_cap_list * sizeof(Entry));
    for (int q = 0; q < 4; q++) {
        L.refine[q] = o;
        o = align_up(o + (size_t)L.ref_cap * sizeof(Entry));
    }
    L.parts = o;
    o = align_up(o + (size_t)num_sms() * MOM_GRID_PER_SM * sizeof(MomPartial));
    L.ctrl = o;
    o = align_up(o + C_SLOTS * 8);
    L.dbg = o;
    o = align_up(o + 16 * 8);
    L.fine = o;
    o = align_up(o + (size_t)KF_MAX * 4);
    L.lut = o;
    o = align_up(o + (size_t)(KF_MAX + 1) * 8);
    L.total = o;
    return L;
}

template <typename F>
void smem_optin(F *func, size_t bytes) {
    // Raise the kernel's dynamic shared-memory cap once to the largest value it
    // can take (device opt-in maximum minus its static shared memory), not to
    // `bytes`: concurrent callers on other host threads then never lower the
    // cap under a launch in flight.  The attribute is a cap, it reserves nothing.
    if (bytes <= 48 * 1024) return;
    static std::mutex mu;
    static std::unordered_map<const void *, int> done;
    int dev = 0;
    cudaGetDevice(&dev);
    const void *key = (const void *)((uintptr_t)(const void *)func ^ ((uintptr_t)dev << 56));
    std::lock_guard<std::mutex> g(mu);
    if (done.count(key)) return;
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, func);
    cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
    done[key] = 1;
}

__global__ void k_init_level1(SegParams *seg, int64_t *kfirst, int64_t *wfirst, int64_t nwin, int64_t n, int64_t k,
                              int64_t tile_len, int64_t ntiles, int src, double center, double sd, double zmin,
                              double scale, int mode, int level = 1) {
    SegParams p{};
    p.center = center;
    p.std = sd;
    p.zmin = zmin;
    p.scale = scale;
    p.start = 0;
    p.len = n;
    p.tile_first = 0;
    p.mat_base = 0;
    p.scan_base = 0;
    p.tile_len = tile_len;
    p.k = (int32_t)k;
    p.ntiles = (int32_t)ntiles;
    p.mode = mode;
    p.level = level;
    p.src = src;
    *seg = p;
    kfirst[0] = 0;
    kfirst[1] = k + 1;
    if (wfirst) {
        wfirst[0] = 0;
        wfirst[1] = nwin;
    }
}

__global__ void k_bucket_totals(const uint32_t *mat, int64_t k, int64_t ntiles, int64_t *counts) {
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= k) return;
    int64_t s = 0;
    for (int64_t t = 0; t < ntiles; t++) s += mat[b * ntiles + t];
    counts[b] = s;
}

struct Ctx {
    Buffers B;
    unsigned char *ws;
    Layout L;
    Plan1 P;
    cudaStream_t st;
    int64_t n;
};

#ifdef ZSB_PHASE_PROFILE
// Instrumentation build only (-DZSB_PHASE_PROFILE): per-CTA clock64 phase
// profiles of the scatter and the largest finish launch, dumped to stderr.
long long *g_scat_prof = nullptr;
int64_t g_scat_prof_n = 0;
long long *scat_prof(int64_t n) {
    if (n < g_scat_prof_n) return nullptr;
    if (g_scat_prof) cudaFree(g_scat_prof);
    cudaMalloc(&g_scat_prof, (size_t)n * 8 * 8);
    cudaMemset(g_scat_prof, 0, (size_t)n * 8 * 8);
    g_scat_prof_n = n;
    return g_scat_prof;
}

void scat_prof_dump() {
    if (!g_scat_prof) return;
    std::vector<long long> h((size_t)g_scat_prof_n * 8);
    cudaMemcpy(h.data(), g_scat_prof, h.size() * 8, cudaMemcpyDeviceToHost);
    double acc[6] = {0};
    for (int64_t b = 0; b < g_scat_prof_n; b++)
        for (int q = 0; q < 6; q++) acc[q] += (double)h[(size_t)b * 8 + q];
    fprintf(stderr, "[zsb] scatter phases per CTA (cycles, summed over rounds): - %.0f buckets+rank+prev-writes %.0f "
                    "scan %.0f place+next-keys %.0f last-writes %.0f loop %.0f\n", acc[0] / g_scat_prof_n, acc[1] / g_scat_prof_n,
            acc[2] / g_scat_prof_n, acc[3] / g_scat_prof_n, acc[4] / g_scat_prof_n, acc[5] / g_scat_prof_n);
    cudaFree(g_scat_prof);
    g_scat_prof = nullptr;
    g_scat_prof_n = 0;
}
#else
inline long long *scat_prof(int64_t) { return nullptr; }
#endif

// L2 prefetch of the next finish run by the copy engine: only when the
// level's records exceed the L2; below it the scatter's evict_last runs are
// still resident and the prefetch only adds traffic (measured on B200: C2
// +5 us, C4 -47 us).  (The same prefetch of the scatter's next round of keys
// won 1 % at C4/X9 but cost C2 its register allocation: not used.)
int fin_prefetch(int64_t n, int pb) {
    if (ZSB_L2_PREFETCH >= 0) return ZSB_L2_PREFETCH;
    return (double)n * (8 + pb) > 128.0 * (1 << 20) ? 1 : 0;
}

template <int KK, int PB, int L1>
int launch_partition_l(Ctx &c, SegParams *segs, int nseg, int64_t tiles, int64_t mat_entries, int kmax, int dst_sel,
                     bool segs_level1 = false, cudaEvent_t after_scan = nullptr, int phases = 3) {
    uint32_t *mat = (uint32_t *)(c.ws + c.L.mat);
    unsigned long long *ctrl = (unsigned long long *)(c.ws + c.L.ctrl);
    unsigned long long *status = (unsigned long long *)(c.ws + c.L.status);
    // keys through the TMA ring on every level (recursion tiles: 8-32 K keys)
    const bool ring = segs_level1 || ZSB_HIST_RING_ALL;
    const size_t kbytes = hist_smem(kmax, ring);
    smem_optin(k_hist<KK, L1>, kbytes);
    const int64_t sblocks = (mat_entries + SCAN_TILE - 1) / SCAN_TILE;
    if (phases & 1) {
    {
        PhaseScope ph(PH_HIST, c.st);
        k_hist<KK, L1><<<(unsigned)tiles, HT, kbytes, c.st>>>(c.B, segs, nseg, mat, ctrl + C_STATUS, ring ? 1 : 0, status,
                                                         (int)(sblocks + 1), ctrl);
    }
    ZSB_LAUNCH("k_hist");
    {
        PhaseScope ph(PH_SCAN, c.st);
        k_scan<<<(unsigned)sblocks, NT, 0, c.st>>>(mat, mat_entries, status, ctrl);
    }
    ZSB_LAUNCH("k_scan");
    if (after_scan) ZSB_CUDA(cudaEventRecord(after_scan, c.st));
    }
    if (!(phases & 2)) return ZSB_OK;
    const size_t cdf_bytes = (c.B.cdf && segs_level1) ? (size_t)(CDF_KNOTS + 1) * 8 : 0;
    const size_t smax = (size_t)227 * 1024 - 1024;
    // 16 warps (8192-record rounds) above ZSB_SW16_ABOVE buckets: two counter
    // sets (rounds pipelined) when they fit shared memory, else one
    const bool want16 = scat_warps(kmax, ZSB_SW16_ABOVE) == 16;
    const int nset16 = !want16 ? 0 : (scat_layout(kmax, PB, 16, 2).total + cdf_bytes <= smax ? 2
                                       : (scat_layout(kmax, PB, 16, 1).total + cdf_bytes <= smax ? 1 : 0));
    if (nset16 == 0) {
        const size_t sbytes = scat_layout(kmax, PB, 8).total + cdf_bytes;
        smem_optin(k_scatter<KK, PB, 8, 2, L1>, sbytes);
        PhaseScope ph(PH_SCATTER, c.st);
        k_scatter<KK, PB, 8, 2, L1><<<(unsigned)tiles, 256, sbytes, c.st>>>(c.B, segs, nseg, mat, dst_sel,
                                                                        scat_prof(tiles));
    } else if (nset16 == 2) {
        const size_t sbytes = scat_layout(kmax, PB, 16, 2).total + cdf_bytes;
        smem_optin(k_scatter<KK, PB, 16, 2, L1>, sbytes);
        PhaseScope ph(PH_SCATTER, c.st);
        k_scatter<KK, PB, 16, 2, L1><<<(unsigned)tiles, 512, sbytes, c.st>>>(c.B, segs, nseg, mat, dst_sel,
                                                                         scat_prof(tiles));
    } else {
        const size_t sbytes = scat_layout(kmax, PB, 16, 1).total + cdf_bytes;
        smem_optin(k_scatter<KK, PB, 16, 1, L1>, sbytes);
        PhaseScope ph(PH_SCATTER, c.st);
        k_scatter<KK, PB, 16, 1, L1><<<(unsigned)tiles, 512, sbytes, c.st>>>(c.B, segs, nseg, mat, dst_sel,
                                                                         scat_prof(tiles));
    }
    ZSB_LAUNCH("k_scatter");
    return ZSB_OK;
}

template <int KK, int PB>
int launch_partition(Ctx &c, SegParams *segs, int nseg, int64_t tiles, int64_t mat_entries, int kmax, int dst_sel,
                     bool segs_level1 = false, cudaEvent_t after_scan = nullptr) {
    return segs_level1 ? launch_partition_l<KK, PB, 1>(c, segs, nseg, tiles, mat_entries, kmax, dst_sel, true, after_scan)
                       : launch_partition_l<KK, PB, 0>(c, segs, nseg, tiles, mat_entries, kmax, dst_sel, false,
                                                       after_scan);
}

#ifdef ZSB_PHASE_PROFILE
long long *g_fin_prof = nullptr;
int64_t g_fin_prof_n = 0;
long long *fin_prof(int64_t n) {
    if (n <= g_fin_prof_n) return nullptr;  // first launch of the largest size
    if (g_fin_prof) cudaFree(g_fin_prof);
    cudaMalloc(&g_fin_prof, (size_t)n * 8 * 8);
    cudaMemset(g_fin_prof, 0, (size_t)n * 8 * 8);
    g_fin_prof_n = n;
    return g_fin_prof;
}

void fin_prof_dump() {
    if (!g_fin_prof) return;
    std::vector<long long> h((size_t)g_fin_prof_n * 8);
    cudaMemcpy(h.data(), g_fin_prof, h.size() * 8, cudaMemcpyDeviceToHost);
    double acc[8] = {0};
    int64_t cnt = 0;
    for (int64_t b = 0; b < g_fin_prof_n; b++) {
        const long long *t = &h[(size_t)b * 8];
        if (!t[6]) continue;  // all-equal or empty runs exit early
        cnt++;
        for (int q = 1; q <= 6; q++) acc[q] += (double)(t[q] - t[q - 1]);
        acc[7] += (double)(t[7] - t[0]);
    }
    fprintf(stderr, "[zsb] finish phases over %lld runs (cycles): load %.0f (staged after %.0f) minmax+params %.0f "
                    "hist %.0f scan %.0f place %.0f rank+store %.0f\n", (long long)cnt, acc[1] / cnt, acc[7] / cnt,
            acc[2] / cnt, acc[3] / cnt, acc[4] / cnt, acc[5] / cnt, acc[6] / cnt);
    cudaFree(g_fin_prof);
    g_fin_prof = nullptr;
    g_fin_prof_n = 0;
}
#else
inline long long *fin_prof(int64_t) { return nullptr; }
#endif

// Refine lists: two per level parity (a level's finish writes list 2*par,
// its refine pass list 2*par + 1), so a level's leftovers survive the next
// level's finish, which is enqueued before the host has read them.
constexpr int REF_SLOT[4] = {C_NREF0, C_NREF1, C_NREF2, C_NREF3};
constexpr int TICK_SLOT[4] = {C_FTICK0, C_FTICK1, C_FTICK2, C_FTICK3};

// Finish over `list`: count from device memory (count_dev, clamped to
// count_const; persistent CTAs with a work ticket) or the host constant
// count_const (one run per CTA); refine runs go to refine list `ref_out`.
// With `fuse_par` >= 0 the launch is cooperative and the same grid then runs
// the refine iterations of level parity `fuse_par` (no second launch).
template <int KK, int PB>
int launch_finish(Ctx &c, const Entry *list, const unsigned long long *count_dev, int64_t count_const,
                  int64_t count_bound, int ref_out, int tick, int fuse_par = -1, const int32_t *order = nullptr) {
    if (count_bound <= 0) return ZSB_OK;
    FinLayout FL = fin_layout((int)c.P.cap, PB);
    smem_optin(k_finish<KK, PB>, FL.total);
    Entry *refine = (Entry *)(c.ws + c.L.refine[ref_out]);
    unsigned long long *ctrl = (unsigned long long *)(c.ws + c.L.ctrl);
    const int64_t grid = count_dev ? std::min<int64_t>(count_bound, (int64_t)num_sms() * FIN_CTAS) : count_bound;
    RefineArgs ra{};
    ra.order = order;
    if (fuse_par >= 0) {
        ra.list_b = (Entry *)(c.ws + c.L.refine[2 * fuse_par + 1]);
        ra.count_b = ctrl + REF_SLOT[2 * fuse_par + 1];
        ra.cap_list = c.L.ref_cap;
        ra.ticket_b = ctrl + TICK_SLOT[2 * fuse_par + 1];
        ra.runs_total = ctrl + C_ST_INSERTION;
    }
    {
        PhaseScope ph(PH_FINISH, c.st);
        Buffers Bv = c.B;
        const Entry *lst = list;
        const unsigned long long *cd = count_dev;
        int64_t cc = count_const;
        int cap = (int)c.P.cap, fi = FIN_INS;  // refine lists hold <= n / (FIN_INS + 1) runs
        long long *prof = fin_prof(count_bound);
        unsigned long long *rc = ctrl + REF_SLOT[ref_out];
        unsigned long long *tk = count_dev ? ctrl + TICK_SLOT[tick] : nullptr;
        int pf = fin_prefetch(c.n, PB);
        void *args[] = {&Bv, &lst, &cd, &cc, &cap, &refine, &rc, &fi, &prof, &tk, &pf, &ra};
        if (fuse_par >= 0)
            ZSB_CUDA(cudaLaunchCooperativeKernel((const void *)k_finish<KK, PB>, dim3((unsigned)grid), dim3(FT), args,
                                                 FL.total, c.st));
        else
            ZSB_CUDA(cudaLaunchKernel((const void *)k_finish<KK, PB>, dim3((unsigned)grid), dim3(FT), args, FL.total,
                                      c.st));
    }
    ZSB_LAUNCH("k_finish");
    return ZSB_OK;
}

// Team finish (K5t): clusters of TEAM CTAs, as many as stay resident (B200:
// 15 clusters of 8 = 120 SMs with one 1024-thread CTA per SM).  0: the device
// cannot hold one cluster (teams off; oversized buckets recurse instead).
template <int KK, int PB>
int team_grid() {
    static std::mutex mu;
    static std::unordered_map<int, int> grid;  // per device
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    auto it = grid.find(dev);
    if (it != grid.end()) return it->second;
    if (!TEAM_ON) return 0;  // -DZSB_TEAM=0: no team runs, oversized buckets always recurse
    FinLayout FL = fin_layout(finish_cap(PB), PB);
    smem_optin(k_team<KK, PB>, FL.total);
    if (TEAM > 8) cudaFuncSetAttribute((const void *)k_team<KK, PB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = TEAM;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(TEAM * 16);
    cfg.blockDim = dim3(FT);
    cfg.dynamicSmemBytes = FL.total;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, (const void *)k_team<KK, PB>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        ncl = 0;
    }
    grid[dev] = ncl * TEAM;
    return ncl * TEAM;
}

template <int KK, int PB>
int launch_team(Ctx &c, const Entry *runs, const unsigned long long *count_dev, int ref_out) {
    const int grid = team_grid<KK, PB>();
    if (grid <= 0) return ZSB_OK;
    FinLayout FL = fin_layout((int)c.P.cap, PB);
    unsigned long long *ctrl = (unsigned long long *)(c.ws + c.L.ctrl);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = TEAM;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(FT);
    cfg.dynamicSmemBytes = FL.total;
    cfg.stream = c.st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    {
        PhaseScope ph(PH_FINISH, c.st);
        ZSB_CUDA(cudaLaunchKernelEx(&cfg, k_team<KK, PB>, c.B, runs, count_dev, (int64_t)c.L.team_cap_list,
                                    (int)c.P.cap, (Entry *)(c.ws + c.L.refine[ref_out]), ctrl + REF_SLOT[ref_out],
                                    (int)FIN_INS, ctrl + C_TTICK, ctrl + C_ST_INSERTION));
    }
    ZSB_LAUNCH("k_team");
    return ZSB_OK;
}

// Refine pass of a level (parity `par`): the refine runs its finish left in
// list 2*par, and their own refine runs, ping-ponging between lists 2*par and
// 2*par + 1 on the device until a pass leaves none (cooperative launch, one
// CTA per SM; the finish's shared memory admits no second CTA).
template <int KK, int PB>
int launch_refine(Ctx &c, int par) {
    FinLayout FL = fin_layout((int)c.P.cap, PB);
    smem_optin(k_refine<KK, PB>, FL.total);
    unsigned long long *ctrl = (unsigned long long *)(c.ws + c.L.ctrl);
    Entry *la = (Entry *)(c.ws + c.L.refine[2 * par]), *lb = (Entry *)(c.ws + c.L.refine[2 * par + 1]);
    unsigned long long *ca = ctrl + REF_SLOT[2 * par], *cb = ctrl + REF_SLOT[2 * par + 1];
    unsigned long long *tick = ctrl + TICK_SLOT[2 * par + 1], *tot = ctrl + C_ST_INSERTION;
    int64_t cl = c.L.ref_cap;
    int cap = (int)c.P.cap, fi = FIN_INS;
    int pf = fin_prefetch(c.n, PB);
    Buffers Bv = c.B;
    void *args[] = {&Bv, &la, &ca, &lb, &cb, &cl, &cap, &fi, &tick, &tot, &pf};
    {
        PhaseScope ph(PH_FINISH, c.st);
        ZSB_CUDA(cudaLaunchCooperativeKernel((const void *)k_refine<KK, PB>, dim3(num_sms() * FIN_CTAS), dim3(FT), args, FL.total,
                                             c.st));
    }
    ZSB_LAUNCH("k_refine");
    return ZSB_OK;
}

// Pinned host mirror of the control block and the level event (per host thread).
struct HostSync {
    unsigned long long *ctrl = nullptr;
    cudaEvent_t ev = nullptr;       // classify done (control block copied)
    cudaEvent_t ev_scan = nullptr;  // level scan done: classify may start
    cudaStream_t side = nullptr;    // classify runs here, beside the scatter
    int dev = -1;
};
thread_local HostSync g_hs;

int host_sync_init() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (g_hs.ctrl && g_hs.dev == dev) return ZSB_OK;
    if (!g_hs.ctrl) ZSB_CUDA(cudaHostAlloc((void **)&g_hs.ctrl, C_SLOTS * 8, cudaHostAllocDefault));
    if (g_hs.ev) cudaEventDestroy(g_hs.ev);
    if (g_hs.ev_scan) cudaEventDestroy(g_hs.ev_scan);
    if (g_hs.side) cudaStreamDestroy(g_hs.side);
    ZSB_CUDA(cudaEventCreateWithFlags(&g_hs.ev, cudaEventDisableTiming));
    ZSB_CUDA(cudaEventCreateWithFlags(&g_hs.ev_scan, cudaEventDisableTiming));
    ZSB_CUDA(cudaStreamCreateWithFlags(&g_hs.side, cudaStreamNonBlocking));
    g_hs.dev = dev;
    return ZSB_OK;
}

// zsort_rec's start (core.py:403-437, _kernels.py:453-473): one segment at
// level depth + 1 centred on the caller's estimated mean, bucketed with the
// caller's k and scale (paper Eq. 1) at that first level.
struct RecStart {
    double center, scale;
    int64_t k;
    int32_t level;
};

template <int KK, int PB>
int run_sort(Ctx &c, const zsb_config &cfg, int64_t *h_stats, const RecStart *rec = nullptr) {
    const int64_t n = c.n;
    unsigned long long *ctrl = (unsigned long long *)(c.ws + c.L.ctrl);
    SegParams *seg_cur = (SegParams *)(c.ws + c.L.seg_a);
    SegParams *seg_next = (SegParams *)(c.ws + c.L.seg_b);
    SegAcc *acc = (SegAcc *)(c.ws + c.L.acc);
    int64_t *kfirst = (int64_t *)(c.ws + c.L.kfirst);
    int64_t *wfirst = (int64_t *)(c.ws + c.L.wfirst);
    int64_t *bstart = (int64_t *)(c.ws + c.L.bstart);
    Entry *entries = (Entry *)(c.ws + c.L.entries);
    uint32_t *mat = (uint32_t *)(c.ws + c.L.mat);
    int64_t stats[ZSB_STAT_SLOTS] = {0, 0, 0, 0, 0};
    if (int rc = host_sync_init()) return rc;
    unsigned long long *hc = g_hs.ctrl;  // pinned: the copies below are truly asynchronous
    const bool fused_l1 =
        !rec && c.n > c.P.cap && cfg.mapping == ZSB_MAP_FITTED && !ZSB_NO_EQUALIZE && !ZSB_NO_SAMPLE;
    if (!fused_l1) ZSB_CUDA(cudaMemsetAsync(ctrl, 0, C_SLOTS * 8, c.st));  // else k_level1_map clears it
    auto full_sync = [&]() -> int {  // control block -> host, wait for everything enqueued
        ZSB_CUDA(cudaMemcpyAsync(hc, ctrl, C_SLOTS * 8, cudaMemcpyDeviceToHost, c.st));
        ZSB_CUDA(cudaStreamSynchronize(c.st));
        timing_collect();
        return ZSB_OK;
    };

    // Finish the runs of `list` and, right behind, their refine runs (device
    // iteration, count on the device) without a host round trip; parity
    // `par` selects the refine lists.
    auto enqueue_finish = [&](const Entry *list, const unsigned long long *count_dev, int64_t count_const,
                              int64_t bound, int par, bool zeroed = false, const int32_t *ord = nullptr) -> int {
        if (!zeroed) ZSB_CUDA(cudaMemsetAsync(ctrl + REF_SLOT[2 * par], 0, 32, c.st));  // two counts, two tickets
        if (ZSB_REFINE_LAUNCH) {  // the refine iterations as a launch of their own
            int rc = launch_finish<KK, PB>(c, list, count_dev, count_const, bound, 2 * par, 2 * par, -1, ord);
            if (rc) return rc;
            return launch_refine<KK, PB>(c, par);
        }
        return launch_finish<KK, PB>(c, list, count_dev, count_const, bound, 2 * par, 2 * par, par, ord);
    };
    // The sort is stream-ordered: once its last level is enqueued the call
    // returns, unless the caller asked for SortStats (or phase timing is on),
    // which needs one host round trip (~18 us on B200).
    auto finish_call = [&]() -> int {
        if (h_stats || g_t.on) {
            if (int rc = full_sync()) return rc;
            stats[ZSB_STAT_INSERTION] += (int64_t)hc[C_ST_INSERTION];  // refine runs
            stats[ZSB_STAT_MAX_DEPTH] = (int64_t)hc[C_ST_MAXDEPTH];
            stats[ZSB_STAT_FALLBACKS] = (int64_t)hc[C_ST_FALLBACKS];
            stats[ZSB_STAT_SCATTERS] = (int64_t)hc[C_ST_SCATTERS];
        }
        if (h_stats) memcpy(h_stats, stats, sizeof(stats));
        return ZSB_OK;
    };

    if (n <= c.P.cap) {  // one shared-memory finish (core.py:369-374; threshold widened to the smem capacity)
        {
            PhaseScope ph(PH_MISC, c.st);
            k_single_entry<<<1, 1, 0, c.st>>>(entries, n);
        }
        ZSB_LAUNCH("k_single_entry");
        int rc = enqueue_finish(entries, nullptr, 1, 1, 0);
        if (rc) return rc;
        stats[ZSB_STAT_INSERTION] = 1;
        if (KK == KEY_F64) {  // the finish is this path's only NaN screen: wait for its verdict
            if (int rs = full_sync()) return rs;
            if (hc[C_STATUS] == 3) return fail(ZSB_ERR_NAN, "NaN keys have no order");
        }
        return finish_call();
    }

    MapCfg mc{rec ? (int32_t)ZSB_MAP_PAPER : cfg.mapping, (int32_t)cfg.depth_guard, rec ? rec->level : 0, 0,
              rec ? rec->scale : 0.0};
    ClassCfg cc{(int32_t)c.P.cap, (int32_t)c.P.half, (int32_t)cfg.depth_guard, cfg.mapping,
                (int32_t)std::max(1, std::min(16, ZSB_CHILD_FILL)), ZSB_GREEDY,
                0, ZSB_CHILD_FROM_CDF};
    // team runs (K5t) finish the few oversized buckets of recursion levels,
    // which would otherwise cost whole extra levels (level 1: ZSB_TEAM_L1)
    const int32_t team_cap = team_grid<KK, PB>() > 0 ? (int32_t)(TEAM * c.P.cap) : 0;
    Entry *teams = (Entry *)(c.ws + c.L.teams);
    int32_t *order = (int32_t *)(c.ws + c.L.order);
    const int64_t nwin1 = (n + c.P.half - 1) / c.P.half;
    const bool equalize = !rec && cfg.mapping == ZSB_MAP_FITTED && !ZSB_NO_EQUALIZE;
    unsigned int *fine = (unsigned int *)(c.ws + c.L.fine);
    float2 *cdf_tab = (float2 *)(c.ws + c.L.lut);
    if (fused_l1) {
        // fitted mapping: one cooperative launch maps level 1 (sampled, exact fallback)
        int64_t nchunks = std::min<int64_t>(SAMP_CHUNKS_MAX, (n + SAMP_CHUNK - 1) / SAMP_CHUNK);
        int64_t stride = n / nchunks;
        const uint64_t *keys = c.B.in_k;
        int64_t n_ = n, k_ = c.P.k, tl = c.P.tile_len, nt = c.P.ntiles, nw = nwin1;
        SampPartial *sparts = (SampPartial *)(c.ws + c.L.parts);
        MomPartial *mparts = (MomPartial *)(c.ws + c.L.parts) + 2 * num_sms();
        int kf = KF_MAX;
        void *args[] = {&keys, &n_, &seg_cur, &kfirst, &wfirst, &nw, &k_, &tl, &nt, &nchunks, &stride,
                        &sparts, &mparts, &fine, &cdf_tab, &ctrl, &mc, &kf};
        PhaseScope ph(PH_MOMENTS, c.st);
        ZSB_CUDA(cudaLaunchCooperativeKernel((const void *)k_level1_map<KK>, dim3(num_sms()), dim3(LT), args, 0, c.st));
    } else if (rec) {
        // the caller's centre; the fused stats pass of the loop's first
        // iteration (k_seg_moments) gathers min, max and the squared
        // deviation around it (_kernels.py:74-88, 453-473)
        PhaseScope ph(PH_MISC, c.st);
        k_init_level1<<<1, 1, 0, c.st>>>(seg_cur, kfirst, wfirst, nwin1, n, c.P.k, c.P.tile_len, c.P.ntiles, 0,
                                         rec->center, 1.0, 0.0, 1.0, MODE_ZSCORE, rec->level);
    } else {
        {
            PhaseScope ph(PH_MISC, c.st);
            k_init_level1<<<1, 1, 0, c.st>>>(seg_cur, kfirst, wfirst, nwin1, n, c.P.k, c.P.tile_len, c.P.ntiles, 0,
                                             0.0, 1.0, 0.0, 1.0, MODE_ZSCORE);
        }
        ZSB_LAUNCH("k_init_level1");
        if (equalize) ZSB_CUDA(cudaMemsetAsync(fine, 0, (size_t)KF_MAX * 4, c.st));
        int grid = std::max(1, std::min<int>(num_sms() * MOM_GRID_PER_SM, (int)((n + NT - 1) / NT)));
        {
            PhaseScope ph(PH_MOMENTS, c.st);
            k_moments<KK><<<grid, NT, 0, c.st>>>(c.B.in_k, n, (MomPartial *)(c.ws + c.L.parts), ctrl, seg_cur, mc,
                                                 nullptr);
        }
        ZSB_LAUNCH("k_moments");
        if (equalize) {
            // exact histogram equalisation of level 1 (acts only if K1 chose z-score mode)
            {
                PhaseScope ph(PH_MOMENTS, c.st, 2);
                k_fine_hist<KK><<<num_sms() * 2, 512, (size_t)KF_MAX * 4, c.st>>>(c.B.in_k, n, seg_cur, KF_MAX, fine);
                k_build_cdf<<<1, 1024, 0, c.st>>>(fine, KF_MAX, n, seg_cur, cdf_tab);
            }
            ZSB_LAUNCH("k_fine_hist/k_build_cdf");
        }
    }

    int nseg = 1;
    int64_t tiles = c.P.ntiles, mat_entries = c.P.k * c.P.ntiles, total_slots = c.P.k + 1, total_windows = nwin1;
    int kmax = (int)c.P.k;
    int level = 1, par = 0;
    int64_t level_records = n;  // records the level's histogram and scatter pass over
    bool need_stats = true;  // the next level's children need the moments pass (read from classify)
    if (rec) {  // the segment's own stats pass, then the level loop as for a recursion level
        SegAcc a0{~0ull, 0ull, 0.0, 0.0};
        ZSB_CUDA(cudaMemcpyAsync(acc, &a0, sizeof(a0), cudaMemcpyHostToDevice, c.st));
    }
    while (true) {
        cc.team_cap = (level > 1 || ZSB_TEAM_L1) ? team_cap : 0;
        if ((level > 1 && need_stats) || rec) {
            {
                PhaseScope ph(PH_SEGSTATS, c.st, 2);
                k_seg_moments<KK><<<(unsigned)tiles, NT, 0, c.st>>>(c.B, seg_cur, nseg, acc);
                k_seg_params<KK><<<(nseg + 127) / 128, 128, 0, c.st>>>(seg_cur, nseg, acc, mc, ctrl);
            }
            ZSB_LAUNCH("k_seg_moments/params");
        }
        const int dst_sel = (level == 1) ? 1 : ((level % 2 == 0) ? 2 : 1);
        int rc = launch_partition<KK, PB>(c, seg_cur, nseg, tiles, mat_entries, kmax, dst_sel, level == 1,
                                          g_hs.ev_scan);
        if (rc) return rc;
        g_t.records[PH_HIST] += level_records;
        g_t.records[PH_SCATTER] += level_records;
        // classify needs the scanned counts, not the scattered records: it runs
        // on the side stream while the scatter runs (C_NCHILD / C_NENTRY were
        // cleared by K2)
        ZSB_CUDA(cudaStreamWaitEvent(g_hs.side, g_hs.ev_scan, 0));
        {
            PhaseScope ph(PH_CLASSIFY, g_hs.side);
            const int64_t need = std::max<int64_t>(1, (std::max(total_slots, total_windows) + 1023) / 1024);
            const int cgrid = (int)std::min<int64_t>(need, (int64_t)num_sms());
            int nseg_ = nseg, key_kind = KK, kmc = KMAX_CHILD, mt = ZSB_MIN_TILE;
            int64_t ts = total_slots, tw = total_windows;
            Buffers Bv = c.B;
            unsigned long long *ref_zero = ctrl + REF_SLOT[2 * par];
            void *args[] = {&seg_cur, &nseg_, &kfirst, &wfirst, &mat, &bstart, &seg_next, &acc, &entries, &ctrl,
                            &cc, &ts, &tw, &Bv, &key_kind, &kmc, &mt, &ref_zero, &teams, &order};
            ZSB_CUDA(cudaLaunchCooperativeKernel((const void *)k_classify, dim3(cgrid), dim3(1024), args, 0, g_hs.side));
        }
        ZSB_LAUNCH("k_classify");
        // The host needs this level's outcome (children, sizes of the next
        // level); the finish of this level does not: it is enqueued before the
        // host waits (count on the device), so the GPU goes straight on.
        ZSB_CUDA(cudaMemcpyAsync(hc, ctrl, C_SLOTS * 8, cudaMemcpyDeviceToHost, g_hs.side));
        ZSB_CUDA(cudaEventRecord(g_hs.ev, g_hs.side));
        ZSB_CUDA(cudaStreamWaitEvent(c.st, g_hs.ev, 0));  // the finish (and every later level) after classify
        // team runs first: their parts' refine runs join the finish's refine list
        if (cc.team_cap) {
            rc = launch_team<KK, PB>(c, teams, ctrl + C_NTEAM, 2 * par);
            if (rc) return rc;
        }
        // longest runs first when the level's records sit in L2 (C2: finish -5 %);
        // past L2 the window order keeps the finish's DRAM reads local (C4: +3 % with it)
        const bool lpt = ZSB_LPT && !fin_prefetch(n, PB);
        rc = enqueue_finish(entries, ctrl + C_NENTRY, c.L.ent_cap, c.L.ent_cap, par, true, lpt ? order : nullptr);
        if (rc) return rc;
        ZSB_CUDA(cudaEventSynchronize(g_hs.ev));
        if (hc[C_STATUS] == 3) {
            cudaStreamSynchronize(c.st);
            return fail(ZSB_ERR_NAN, "NaN keys have no order");
        }
        const int64_t nentry = (int64_t)hc[C_NENTRY];
        if (nentry > c.L.ent_cap) {
            cudaStreamSynchronize(c.st);
            return fail(ZSB_ERR_WORKSPACE, "finish list overflow");
        }
        stats[ZSB_STAT_INSERTION] += nentry;
        const int64_t nchild = (int64_t)hc[C_NCHILD];
        need_stats = hc[C_NEED_STATS] != 0;
#ifdef ZSB_DEBUG_LOG
        {  // host time since the call started: when this level's classify was seen
            static thread_local std::chrono::steady_clock::time_point t_call;
            if (level == 1) t_call = std::chrono::steady_clock::now();
            const double us =
                std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_call).count();
            fprintf(stderr, "[zsb] level %d: nseg %d tiles %lld kmax %d -> children %lld entries %lld fallbacks %llu"
                            " (host +%.0f us)\n",
                    level, nseg, (long long)tiles, kmax, (long long)nchild, (long long)nentry, hc[C_ST_FALLBACKS], us);
        }
#endif
        if (nchild == 0) break;
        if (nchild > c.L.seg_cap) return fail(ZSB_ERR_WORKSPACE, "segment table overflow");
        nseg = (int)nchild;
        tiles = (int64_t)hc[C_TILES_NEXT];
        mat_entries = (int64_t)hc[C_MAT_NEXT];
        kmax = (int)hc[C_KMAX_NEXT];
        total_slots = (int64_t)hc[C_NEXT_BIG];
        total_windows = (int64_t)hc[C_WIN_NEXT];
        level_records = (int64_t)hc[C_REC_NEXT];
        par ^= 1;
        if (mat_entries > c.L.mat_cap) return fail(ZSB_ERR_WORKSPACE, "count matrix overflow");
        if (total_slots > c.L.slot_cap) return fail(ZSB_ERR_WORKSPACE, "bucket slot overflow");
        std::swap(seg_cur, seg_next);
        level++;
        if (level > 200) return fail(ZSB_ERR_CUDA, "partition did not terminate");
    }
#ifdef ZSB_PHASE_PROFILE
    fin_prof_dump();
    scat_prof_dump();
#endif
    g_t.records[PH_FINISH] += n;  // every record is finished exactly once (finish, team and refine runs)
    return finish_call();
}

int check_common(const void *d_keys, int32_t kd, int32_t pb, int64_t n) {
    if (kd != ZSB_KEY_I64 && kd != ZSB_KEY_F64) return fail(ZSB_ERR_DTYPE, "key dtype must be int64 or float64");
    if (pb != 0 && pb != 4 && pb != 8) return fail(ZSB_ERR_DTYPE, "payload must be 0, 4 or 8 bytes wide");
    if (n < 0) return fail(ZSB_ERR_ARG, "n must be >= 0");
    if (n >= ((int64_t)1 << 32)) return fail(ZSB_ERR_ARG, "n must be < 2^32 per device");
    if (n > 0 && !d_keys) return fail(ZSB_ERR_ARG, "null key pointer");
    return ZSB_OK;
}

zsb_config default_cfg() {
    zsb_config c;
    c.alpha = 0.6;
    c.insertion_threshold = 96;
    c.counting_range_threshold = 65000;
    c.depth_guard = 32;
    c.collect_stats = 0;
    c.mapping = ZSB_MAP_FITTED;
    return c;
}

int check_cfg(const zsb_config &c) {  // core.py:81-89
    if (!(c.alpha > 0 && c.alpha <= 2)) return fail(ZSB_ERR_ARG, "alpha must be in (0, 2]");
    if (c.insertion_threshold < 1) return fail(ZSB_ERR_ARG, "insertion_threshold must be >= 1");
    if (c.counting_range_threshold < 1) return fail(ZSB_ERR_ARG, "counting_range_threshold must be >= 1");
    if (c.depth_guard < 3) return fail(ZSB_ERR_ARG, "depth_guard must be >= 3");
    if (c.mapping != ZSB_MAP_FITTED && c.mapping != ZSB_MAP_PAPER) return fail(ZSB_ERR_ARG, "bad mapping");
    return ZSB_OK;
}

template <template <int, int> class F, typename... A>
int dispatch(int kd, int pb, A &&...args) {
#ifdef ZSB_ONLY_F64_P4  // experiment builds (tools/build_variant.sh): one key/payload combination, 1/6 the compile
    if (kd == ZSB_KEY_F64 && pb == 4) return F<1, 4>::run(args...);
    return fail(ZSB_ERR_ARG, "this experiment build holds only float64 keys with a 4-byte payload");
#else
    if (kd == ZSB_KEY_I64) {
        if (pb == 0) return F<0, 0>::run(args...);
        if (pb == 4) return F<0, 4>::run(args...);
        return F<0, 8>::run(args...);
    }
    if (pb == 0) return F<1, 0>::run(args...);
    if (pb == 4) return F<1, 4>::run(args...);
    return F<1, 8>::run(args...);
#endif
}

template <int KK, int PB>
struct SortOp {
    static int run(Ctx &c, const zsb_config &cfg, int64_t *h_stats, const RecStart *rec) {
        return run_sort<KK, PB>(c, cfg, h_stats, rec);
    }
};

// -------------------------------------------------------------- K8 check

template <int KK, typename IT>
__global__ void k_check(const uint64_t *in_k, const uint64_t *out_k, const IT *idx, int64_t n, int64_t base,
                        unsigned int *bitmap, unsigned long long *viol) {
    unsigned long long bad = 0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = (int64_t)idx[j] - base;
        uint64_t ok = ord_key<KK>(out_k[j]);
        if (p < 0 || p >= n) {
            bad++;
            continue;
        }
        unsigned bit = 1u << (p & 31);
        unsigned old = atomicOr(&bitmap[p >> 5], bit);
        if (old & bit) bad++;                      // repeated index: not a permutation
        if (in_k[p] != out_k[j]) bad++;            // key does not belong to that index
        if (j > 0) {
            uint64_t pk = ord_key<KK>(out_k[j - 1]);
            if (ok < pk) bad++;                                           // not sorted
            if (ok == pk && (int64_t)idx[j] <= (int64_t)idx[j - 1]) bad++;  // not stable
        }
    }
    bad = warp_sum(bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(viol, bad);
}

int injected_setup(Ctx &ctx, const void *d_keys, int32_t kd, const void *d_payload, int32_t pb, int64_t n,
                          const double *params, int64_t k, void *d_out_keys, void *d_out_payload, void *d_workspace,
                          size_t workspace_bytes, void *stream) {
    int rc = check_common(d_keys, kd, pb, n);
    if (rc) return rc;
    if (n < 1 || k < 2 || k > K_LEVEL1_MAX || !params)
        return fail(ZSB_ERR_ARG, "need n >= 1, 2 <= k <= 2048 and params");
    if (!(params[1] > 0.0) || !(params[3] > 0.0)) return fail(ZSB_ERR_ARG, "std and scale must be positive");
    ctx.n = n;
    ctx.P.k = k;
    ctx.P.cap = finish_cap(pb);
    ctx.P.half = fin_window(ctx.P.cap);
    int64_t target = (int64_t)num_sms() * 2;
    int64_t tl = std::max<int64_t>(std::max<int64_t>(4 * k, 2048), (n + target - 1) / target);
    ctx.P.tile_len = (tl + 255) & ~(int64_t)255;
    ctx.P.ntiles = (n + ctx.P.tile_len - 1) / ctx.P.tile_len;
    ctx.L = make_layout(n, pb, ctx.P, false);
    if (!d_workspace || workspace_bytes < ctx.L.total) return fail(ZSB_ERR_WORKSPACE, "workspace too small");
    ctx.ws = (unsigned char *)d_workspace;
    ctx.st = (cudaStream_t)stream;
    ctx.B.in_k = (const uint64_t *)d_keys;
    ctx.B.in_p = d_payload;
    ctx.B.tmp_k = nullptr;
    ctx.B.tmp_p = nullptr;
    ctx.B.out_k = (uint64_t *)d_out_keys;
    ctx.B.out_p = d_out_payload;
    ctx.B.cuts = nullptr;
    ctx.B.cdf = nullptr;
    ctx.B.status = nullptr;
    ctx.B.n = n;
    ctx.B.peers = nullptr;
    SegParams *seg = (SegParams *)(ctx.ws + ctx.L.seg_a);
    int64_t *kfirst = (int64_t *)(ctx.ws + ctx.L.kfirst);
    k_init_level1<<<1, 1, 0, ctx.st>>>(seg, kfirst, nullptr, 0, n, k, ctx.P.tile_len, ctx.P.ntiles, 0, params[0],
                                       params[1], params[2], params[3], MODE_ZSCORE);
    ZSB_LAUNCH("k_init_level1");
    return ZSB_OK;
}

template <int KK, int PB>
struct ScatterOp {
    static int run(Ctx &c) {
        SegParams *seg = (SegParams *)(c.ws + c.L.seg_a);
        unsigned long long *ctrl = (unsigned long long *)(c.ws + c.L.ctrl);
        cudaMemsetAsync(ctrl, 0, C_SLOTS * 8, c.st);
        int rc = launch_partition<KK, PB>(c, seg, 1, c.P.ntiles, c.P.k * c.P.ntiles, (int)c.P.k, 2);
        if (rc) return rc;
        ZSB_CUDA(cudaStreamSynchronize(c.st));
        return ZSB_OK;
    }
};


Plan1 plan_partition(int64_t n, int pb, int nparts) {
    Plan1 P;
    P.cap = finish_cap(pb);
    P.half = fin_window(P.cap);
    P.k = nparts;
    int64_t target = (int64_t)num_sms() * 2;
    int64_t tl = std::max<int64_t>(4096, (n + target - 1) / target);
    P.tile_len = (tl + 255) & ~(int64_t)255;
    P.ntiles = (n + P.tile_len - 1) / P.tile_len;
    return P;
}

template <int KK, int PB>
struct PartitionOp {
    static int run(Ctx &c, int phases) {
        SegParams *seg = (SegParams *)(c.ws + c.L.seg_a);
        unsigned long long *ctrl = (unsigned long long *)(c.ws + c.L.ctrl);
        if (phases & 1) ZSB_CUDA(cudaMemsetAsync(ctrl, 0, C_SLOTS * 8, c.st));
        if (phases & 1) g_t.records[PH_HIST] += c.n;     // the shard's records pass through each phase once
        if (phases & 2) g_t.records[PH_SCATTER] += c.n;
        return launch_partition_l<KK, PB, 0>(c, seg, 1, c.P.ntiles, c.P.k * c.P.ntiles, (int)c.P.k, 2, false, nullptr,
                                             phases);
    }
};

}  // namespace

// ================================================================== C ABI

extern "C" {

const char *zsb_last_error(void) { return g_err.c_str(); }

int64_t zsb_check_violations(int32_t reset) {
#ifdef ZSB_CHECKS
    unsigned long long h = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&h, zsb_check_count, sizeof(h));
    if (reset) {
        const unsigned long long z = 0;
        cudaMemcpyToSymbol(zsb_check_count, &z, sizeof(z));
    }
    return (int64_t)h;
#else
    (void)reset;
    return -1;  // not a bounds-check build
#endif
}

void zsb_timing_enable(int32_t on) {
    g_t.on = on != 0;
    g_t.slot_of.clear();
    g_t.used = 0;
}

int32_t zsb_timing_read(double *ms, int64_t *launches, int32_t nslots, int32_t reset) {
    int k = nslots < PH_SLOTS ? nslots : PH_SLOTS;
    for (int i = 0; i < k; i++) {
        if (ms) ms[i] = g_t.ms[i];
        if (launches) launches[i] = g_t.launches[i];
    }
    if (reset) {
        for (int i = 0; i < PH_SLOTS; i++) {
            g_t.ms[i] = 0;
            g_t.launches[i] = 0;
            g_t.records[i] = 0;
        }
        g_t.launch_total = 0;
    }
    return PH_SLOTS;
}

int32_t zsb_timing_records(int64_t *records, int32_t nslots) {
    int k = nslots < PH_SLOTS ? nslots : PH_SLOTS;
    for (int i = 0; i < k; i++)
        if (records) records[i] = g_t.records[i];
    return PH_SLOTS;
}

const char *zsb_version(void) {
    return "zsort_b200 0.2 (sm_100a; level-1 sampled CDF map, K2 TMA-ring histogram, K3 look-back scan, "
           "K4 shared-memory ranked stable scatter, K5 shared-memory finish, K5t team finish, K8 checker)";
}

size_t zsb_workspace_bytes(int64_t n, int32_t key_dtype, int32_t payload_bytes, const zsb_config *cfg) {
    (void)key_dtype;
    zsb_config c = cfg ? *cfg : default_cfg();
    if (n < 1) n = 1;
    Plan1 P = plan_level1(n, payload_bytes, c);
    return make_layout(n, payload_bytes, P, true).total;
}

}  // extern "C"

namespace {
int sort_entry(const void *d_keys, int32_t key_dtype, const void *d_payload, int32_t payload_bytes, void *d_out_keys,
               void *d_out_payload, int64_t n, const zsb_config *cfg, void *d_workspace, size_t workspace_bytes,
               int64_t *h_stats, void *stream, const RecStart *rec) {
    int rc = check_common(d_keys, key_dtype, payload_bytes, n);
    if (rc) return rc;
    zsb_config c = cfg ? *cfg : default_cfg();
    rc = check_cfg(c);
    if (rc) return rc;
    if (h_stats) memset(h_stats, 0, sizeof(int64_t) * ZSB_STAT_SLOTS);
    if (n == 0) return ZSB_OK;
    if (!d_out_keys || (payload_bytes && (!d_payload || !d_out_payload)))
        return fail(ZSB_ERR_ARG, "null output or payload pointer");
    Ctx ctx;
    ctx.n = n;
    ctx.P = rec ? plan_rec(n, payload_bytes, rec->k) : plan_level1(n, payload_bytes, c);
    ctx.L = make_layout(n, payload_bytes, ctx.P, true);
    if (!d_workspace || workspace_bytes < ctx.L.total) return fail(ZSB_ERR_WORKSPACE, "workspace too small");
    ctx.ws = (unsigned char *)d_workspace;
    ctx.st = (cudaStream_t)stream;
    ctx.B.in_k = (const uint64_t *)d_keys;
    ctx.B.in_p = d_payload;
    ctx.B.tmp_k = (uint64_t *)(ctx.ws + ctx.L.tmp_k);
    ctx.B.tmp_p = ctx.ws + ctx.L.tmp_p;
    ctx.B.out_k = (uint64_t *)d_out_keys;
    ctx.B.out_p = d_out_payload;
    ctx.B.cuts = nullptr;
    ctx.B.cdf = (const float2 *)(ctx.ws + ctx.L.lut);
    ctx.B.status = (unsigned long long *)(ctx.ws + ctx.L.ctrl) + C_STATUS;
    ctx.B.n = n;
    ctx.B.peers = nullptr;
    return dispatch<SortOp>(key_dtype, payload_bytes, ctx, c, h_stats, rec);
}
}  // namespace

extern "C" {

int zsb_sort(const void *d_keys, int32_t key_dtype, const void *d_payload, int32_t payload_bytes, void *d_out_keys,
             void *d_out_payload, int64_t n, const zsb_config *cfg, void *d_workspace, size_t workspace_bytes,
             int64_t *h_stats, void *stream) {
    return sort_entry(d_keys, key_dtype, d_payload, payload_bytes, d_out_keys, d_out_payload, n, cfg, d_workspace,
                      workspace_bytes, h_stats, stream, nullptr);
}

size_t zsb_rec_workspace_bytes(int64_t n, int32_t key_dtype, int32_t payload_bytes, int64_t k) {
    (void)key_dtype;
    if (n < 1) n = 1;
    return make_layout(n, payload_bytes, plan_rec(n, payload_bytes, k), true).total;
}

int zsb_sort_rec(const void *d_keys, int32_t key_dtype, const void *d_payload, int32_t payload_bytes,
                 void *d_out_keys, void *d_out_payload, int64_t n, int64_t k, double scale, double mean_est,
                 int64_t depth, const zsb_config *cfg, void *d_workspace, size_t workspace_bytes, int64_t *h_stats,
                 void *stream) {
    // core.py:416-424 validation
    if (depth < 1) return fail(ZSB_ERR_ARG, "depth must be >= 1");
    if (k < 2) return fail(ZSB_ERR_ARG, "k must be >= 2");
    if (!(scale > 0.0)) return fail(ZSB_ERR_ARG, "scale must be positive");
    if (!std::isfinite(mean_est)) return fail(ZSB_ERR_ARG, "mean_est must be finite");
    zsb_config c = cfg ? *cfg : default_cfg();
    if (n <= c.insertion_threshold && n > 0)
        return fail(ZSB_ERR_ARG, "zsort_rec requires a segment larger than the insertion threshold");
    if (depth + 1 > (int64_t)1 << 30) return fail(ZSB_ERR_ARG, "depth too large");
    RecStart r{mean_est, scale, std::min<int64_t>(k, K_LEVEL1_MAX), (int32_t)(depth + 1)};
    return sort_entry(d_keys, key_dtype, d_payload, payload_bytes, d_out_keys, d_out_payload, n, &c, d_workspace,
                      workspace_bytes, h_stats, stream, &r);
}

int zsb_moments(const void *d_keys, int32_t key_dtype, int64_t n, void *d_workspace, size_t workspace_bytes,
                double *h_out, int64_t *h_limbs, uint64_t *h_min_max_bits, void *stream) {
    int rc = check_common(d_keys, key_dtype, 0, n);
    if (rc) return rc;
    if (n < 1) return fail(ZSB_ERR_ARG, "moments require a nonempty segment");
    size_t need = align_up((size_t)num_sms() * MOM_GRID_PER_SM * sizeof(MomPartial)) + align_up(sizeof(SegParams)) +
                  align_up(C_SLOTS * 8) + align_up(16 * 8);
    if (!d_workspace || workspace_bytes < need) return fail(ZSB_ERR_WORKSPACE, "workspace too small");
    unsigned char *ws = (unsigned char *)d_workspace;
    MomPartial *parts = (MomPartial *)ws;
    SegParams *seg = (SegParams *)(ws + align_up((size_t)num_sms() * MOM_GRID_PER_SM * sizeof(MomPartial)));
    unsigned long long *ctrl = (unsigned long long *)((unsigned char *)seg + align_up(sizeof(SegParams)));
    double *dbg = (double *)((unsigned char *)ctrl + align_up(C_SLOTS * 8));
    cudaStream_t st = (cudaStream_t)stream;
    ZSB_CUDA(cudaMemsetAsync(ctrl, 0, C_SLOTS * 8, st));
    ZSB_CUDA(cudaMemsetAsync(seg, 0, sizeof(SegParams), st));
    int grid = std::max(1, std::min<int>(num_sms() * MOM_GRID_PER_SM, (int)((n + NT - 1) / NT)));
    MapCfg mc{ZSB_MAP_FITTED, 32};
    if (key_dtype == ZSB_KEY_I64)
        k_moments<0><<<grid, NT, 0, st>>>((const uint64_t *)d_keys, n, parts, ctrl, seg, mc, dbg);
    else
        k_moments<1><<<grid, NT, 0, st>>>((const uint64_t *)d_keys, n, parts, ctrl, seg, mc, dbg);
    ZSB_LAUNCH("k_moments");
    double h[16];
    ZSB_CUDA(cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, st));
    ZSB_CUDA(cudaStreamSynchronize(st));
    if (h_out) {
        for (int i = 0; i < 8; i++) h_out[i] = h[i];
        h_out[5] = h_out[6] = 0.0;
    }
    if (h_limbs) memcpy(h_limbs, &h[8], 16);
    if (h_min_max_bits) memcpy(h_min_max_bits, &h[10], 16);
    return ZSB_OK;
}

int zsb_histogram(const void *d_keys, int32_t key_dtype, int64_t n, const double *params, int64_t k,
                  int64_t *d_counts, void *d_workspace, size_t workspace_bytes, void *stream) {
    Ctx ctx;
    int rc = injected_setup(ctx, d_keys, key_dtype, nullptr, 0, n, params, k, nullptr, nullptr, d_workspace,
                            workspace_bytes, stream);
    if (rc) return rc;
    SegParams *seg = (SegParams *)(ctx.ws + ctx.L.seg_a);
    uint32_t *mat = (uint32_t *)(ctx.ws + ctx.L.mat);
    size_t kb = (size_t)k * 4;
    if (key_dtype == ZSB_KEY_I64) {
        smem_optin(k_hist<0, 0>, kb);
        k_hist<0, 0><<<(unsigned)ctx.P.ntiles, HT, kb, ctx.st>>>(ctx.B, seg, 1, mat,
                                                           (unsigned long long *)(ctx.ws + ctx.L.ctrl) + C_STATUS, 0,
                                                           nullptr, 0, nullptr);
    } else {
        smem_optin(k_hist<1, 0>, kb);
        k_hist<1, 0><<<(unsigned)ctx.P.ntiles, HT, kb, ctx.st>>>(ctx.B, seg, 1, mat,
                                                           (unsigned long long *)(ctx.ws + ctx.L.ctrl) + C_STATUS, 0,
                                                           nullptr, 0, nullptr);
    }
    ZSB_LAUNCH("k_hist");
    k_bucket_totals<<<(unsigned)((k + 255) / 256), 256, 0, ctx.st>>>(mat, k, ctx.P.ntiles, d_counts);
    ZSB_LAUNCH("k_bucket_totals");
    ZSB_CUDA(cudaStreamSynchronize(ctx.st));
    return ZSB_OK;
}

int zsb_scatter(const void *d_keys, int32_t key_dtype, const void *d_payload, int32_t payload_bytes, int64_t n,
                const double *params, int64_t k, void *d_out_keys, void *d_out_payload, void *d_workspace,
                size_t workspace_bytes, void *stream) {
    Ctx ctx;
    int rc = injected_setup(ctx, d_keys, key_dtype, d_payload, payload_bytes, n, params, k, d_out_keys,
                            d_out_payload, d_workspace, workspace_bytes, stream);
    if (rc) return rc;
    return dispatch<ScatterOp>(key_dtype, payload_bytes, ctx);
}

size_t zsb_check_workspace_bytes(int64_t n) { return align_up((size_t)((n + 31) / 32) * 4) + 256; }

int zsb_check_sorted(const void *d_in_keys, const void *d_out_keys, const void *d_index, int32_t index_bytes,
                     int32_t key_dtype, int64_t n, int64_t index_base, void *d_workspace, int64_t *h_result,
                     void *stream) {
    int rc = check_common(d_in_keys, key_dtype, 0, n);
    if (rc) return rc;
    if (index_bytes != 4 && index_bytes != 8) return fail(ZSB_ERR_DTYPE, "index must be int32 or int64");
    if (n == 0) {
        if (h_result) *h_result = 0;
        return ZSB_OK;
    }
    cudaStream_t st = (cudaStream_t)stream;
    unsigned int *bitmap = (unsigned int *)d_workspace;
    size_t bm = align_up((size_t)((n + 31) / 32) * 4);
    unsigned long long *viol = (unsigned long long *)((unsigned char *)d_workspace + bm);
    ZSB_CUDA(cudaMemsetAsync(d_workspace, 0, bm + 8, st));
    int grid = num_sms() * 8;
    if (key_dtype == ZSB_KEY_I64) {
        if (index_bytes == 8)
            k_check<0, long long><<<grid, 256, 0, st>>>((const uint64_t *)d_in_keys, (const uint64_t *)d_out_keys,
                                                      (const long long *)d_index, n, index_base, bitmap, viol);
        else
            k_check<0, int><<<grid, 256, 0, st>>>((const uint64_t *)d_in_keys, (const uint64_t *)d_out_keys,
                                                (const int *)d_index, n, index_base, bitmap, viol);
    } else {
        if (index_bytes == 8)
            k_check<1, long long><<<grid, 256, 0, st>>>((const uint64_t *)d_in_keys, (const uint64_t *)d_out_keys,
                                                      (const long long *)d_index, n, index_base, bitmap, viol);
        else
            k_check<1, int><<<grid, 256, 0, st>>>((const uint64_t *)d_in_keys, (const uint64_t *)d_out_keys,
                                                (const int *)d_index, n, index_base, bitmap, viol);
    }
    ZSB_LAUNCH("k_check");
    unsigned long long h = 0;
    ZSB_CUDA(cudaMemcpyAsync(&h, viol, 8, cudaMemcpyDeviceToHost, st));
    ZSB_CUDA(cudaStreamSynchronize(st));
    if (h_result) *h_result = (int64_t)h;
    return ZSB_OK;
}


int zsb_local_moments(const void *d_keys, int32_t key_dtype, int64_t n, double shift, double *d_out4,
                      uint64_t *d_out_bits2, void *stream) {
    int rc = check_common(d_keys, key_dtype, 0, n);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    count_launches(1);
    k_dist_init<<<1, 32, 0, st>>>(d_out4, (unsigned long long *)d_out_bits2);
    ZSB_LAUNCH("k_dist_init");
    if (n == 0) return ZSB_OK;
    const int grid = std::max(1, std::min<int>(num_sms() * 4, (int)((n + NT - 1) / NT)));
    const int self = std::isnan(shift) ? 1 : 0;  // NaN: shift by the shard's first key
    count_launches(1);
    if (key_dtype == ZSB_KEY_I64)
        k_local_moments<0><<<grid, NT, 0, st>>>((const uint64_t *)d_keys, n, shift, self, d_out4,
                                                (unsigned long long *)d_out_bits2);
    else
        k_local_moments<1><<<grid, NT, 0, st>>>((const uint64_t *)d_keys, n, shift, self, d_out4,
                                                (unsigned long long *)d_out_bits2);
    ZSB_LAUNCH("k_local_moments");
    return ZSB_OK;
}

int zsb_occurrence_index(const void *d_keys, int32_t key_dtype, int64_t n, uint64_t key_bits, int64_t occurrence,
                         void *d_workspace, int64_t *h_index, void *stream) {
    int rc = check_common(d_keys, key_dtype, 0, n);
    if (rc) return rc;
    if (!h_index || !d_workspace) return fail(ZSB_ERR_ARG, "null workspace or result pointer");
    *h_index = -1;
    if (n == 0 || occurrence < 0) return ZSB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int nch = std::max(1, std::min<int>(OCC_CHUNKS, (int)((n + 4095) / 4096)));
    const int64_t chunk = (n + nch - 1) / nch;
    unsigned long long *cnt = (unsigned long long *)d_workspace;
    long long *out = (long long *)(cnt + OCC_CHUNKS);
    uint64_t target = key_bits ^ SIGN;  // ordered image (host copy of ord_key)
    if (key_dtype == ZSB_KEY_F64) {
        const uint64_t b = key_bits == SIGN ? 0ull : key_bits;
        target = (b & SIGN) ? ~b : (b | SIGN);
    }
    count_launches(2);
    if (key_dtype == ZSB_KEY_I64) {
        k_occ_count<0><<<nch, NT, 0, st>>>((const uint64_t *)d_keys, n, chunk, target, cnt);
        k_occ_find<0><<<1, OCC_T, 0, st>>>((const uint64_t *)d_keys, n, chunk, nch, target, occurrence, cnt, out);
    } else {
        k_occ_count<1><<<nch, NT, 0, st>>>((const uint64_t *)d_keys, n, chunk, target, cnt);
        k_occ_find<1><<<1, OCC_T, 0, st>>>((const uint64_t *)d_keys, n, chunk, nch, target, occurrence, cnt, out);
    }
    ZSB_LAUNCH("k_occ_count/find");
    long long h = -1;
    ZSB_CUDA(cudaMemcpyAsync(&h, out, 8, cudaMemcpyDeviceToHost, st));
    ZSB_CUDA(cudaStreamSynchronize(st));
    *h_index = h;
    return ZSB_OK;
}

size_t zsb_occurrence_workspace_bytes(void) { return (size_t)(OCC_CHUNKS + 1) * 8; }

int zsb_generate(int32_t family, int64_t offset, int64_t n, int64_t n_total, uint64_t seed, const double *params,
                 int64_t *d_out, void *stream) {
    if (family < GEN_UNIFORM || family > GEN_HIGH_DUP) return fail(ZSB_ERR_ARG, "unknown family");
    if (n < 0 || offset < 0 || offset + n > n_total) return fail(ZSB_ERR_ARG, "need 0 <= offset <= offset + n <= n_total");
    if (n == 0) return ZSB_OK;
    if (!d_out) return fail(ZSB_ERR_ARG, "null output pointer");
    GenParams gp{0.0, 1e9, 1.5, 1.0, 0.01, 1000};  // the reference's DistributionSpec defaults (datagen.py:48-59)
    if (params) {
        gp.normal_mu = params[0];
        gp.normal_sigma = params[1];
        gp.pareto_alpha = params[2];
        gp.pareto_xm = params[3];
        gp.swap_fraction = params[4];
        gp.dup_range = (uint64_t)params[5];
    }
    if (!(gp.normal_sigma > 0) || !(gp.pareto_alpha > 0) || !(gp.pareto_xm > 0) || !(gp.swap_fraction >= 0) ||
        !(gp.swap_fraction <= 0.5) || gp.dup_range < 1)
        return fail(ZSB_ERR_ARG, "bad family parameters");
    const uint64_t base = splitmix64_u(seed ^ ((uint64_t)(family + 1) << 56));
    const int grid = std::max(1, std::min<int>(num_sms() * 8, (int)((n + NT - 1) / NT)));
    count_launches(1);
    k_generate<<<grid, NT, 0, (cudaStream_t)stream>>>(family, base, offset, n, n_total, gp, d_out);
    ZSB_LAUNCH("k_generate");
    return ZSB_OK;
}

int zsb_bucket_histogram(const void *d_keys, int32_t key_dtype, int64_t n, const double *params, int64_t k,
                         int64_t *d_counts, void *stream) {
    int rc = check_common(d_keys, key_dtype, 0, n);
    if (rc) return rc;
    if (k < 2 || k > 16384 || !params) return fail(ZSB_ERR_ARG, "need 2 <= k <= 16384 and params");
    cudaStream_t st = (cudaStream_t)stream;
    ZSB_CUDA(cudaMemsetAsync(d_counts, 0, (size_t)k * 8, st));
    if (n == 0) return ZSB_OK;
    const int grid = std::max(1, std::min<int>(num_sms() * 2, (int)((n + NT - 1) / NT)));
    const size_t sm = (size_t)k * 4;
    if (key_dtype == ZSB_KEY_I64) {
        smem_optin(k_bucket_hist<0>, sm);
        count_launches(1);
        k_bucket_hist<0><<<grid, NT, sm, st>>>((const uint64_t *)d_keys, n, params[0], params[1], params[2], params[3],
                                               (int)k, (unsigned long long *)d_counts);
    } else {
        smem_optin(k_bucket_hist<1>, sm);
        count_launches(1);
        k_bucket_hist<1><<<grid, NT, sm, st>>>((const uint64_t *)d_keys, n, params[0], params[1], params[2], params[3],
                                               (int)k, (unsigned long long *)d_counts);
    }
    ZSB_LAUNCH("k_bucket_hist");
    return ZSB_OK;
}

int zsb_bucket_minmax(const void *d_keys, int32_t key_dtype, int64_t n, const double *params, int64_t k, int32_t nb,
                      const int32_t *d_buckets, uint64_t *d_omin, uint64_t *d_omax, void *stream) {
    int rc = check_common(d_keys, key_dtype, 0, n);
    if (rc) return rc;
    if (nb < 0 || nb > 32 || !params) return fail(ZSB_ERR_ARG, "need 0 <= nb <= 32 and params");
    cudaStream_t st = (cudaStream_t)stream;
    count_launches(1);
    k_minmax_init<<<1, 32, 0, st>>>(nb, (unsigned long long *)d_omin, (unsigned long long *)d_omax);
    ZSB_LAUNCH("k_minmax_init");
    if (n == 0 || nb == 0) return ZSB_OK;
    const int grid = std::max(1, std::min<int>(num_sms() * 4, (int)((n + NT - 1) / NT)));
    count_launches(1);
    if (key_dtype == ZSB_KEY_I64)
        k_bucket_minmax<0><<<grid, NT, 0, st>>>((const uint64_t *)d_keys, n, params[0], params[1], params[2],
                                                params[3], (int)k, nb, d_buckets, (unsigned long long *)d_omin,
                                                (unsigned long long *)d_omax);
    else
        k_bucket_minmax<1><<<grid, NT, 0, st>>>((const uint64_t *)d_keys, n, params[0], params[1], params[2],
                                                params[3], (int)k, nb, d_buckets, (unsigned long long *)d_omin,
                                                (unsigned long long *)d_omax);
    ZSB_LAUNCH("k_bucket_minmax");
    return ZSB_OK;
}

int zsb_range_histogram(const void *d_keys, int32_t key_dtype, int64_t n, const double *params, int64_t k, int32_t nq,
                        const int32_t *d_qbucket, const uint64_t *d_qlo, const uint64_t *d_qhi, const int32_t *d_qshift,
                        int32_t nbins, int64_t *d_counts, void *stream) {
    int rc = check_common(d_keys, key_dtype, 0, n);
    if (rc) return rc;
    if (nq < 0 || nq > 32 || nbins < 1 || nbins > 65536 || !params) return fail(ZSB_ERR_ARG, "bad range query");
    cudaStream_t st = (cudaStream_t)stream;
    ZSB_CUDA(cudaMemsetAsync(d_counts, 0, (size_t)nq * nbins * 8, st));
    if (n == 0 || nq == 0) return ZSB_OK;
    const int grid = std::max(1, std::min<int>(num_sms() * 4, (int)((n + NT - 1) / NT)));
    // counters in shared memory when they fit (<= 96 KB: two CTAs per SM)
    const size_t sm = (size_t)nq * nbins * 4;
    const int use_smem = sm <= (size_t)96 * 1024 ? 1 : 0;
    const size_t dyn = use_smem ? sm : 0;
    count_launches(1);
    if (key_dtype == ZSB_KEY_I64) {
        smem_optin(k_range_hist<0>, dyn);
        k_range_hist<0><<<grid, NT, dyn, st>>>((const uint64_t *)d_keys, n, params[0], params[1], params[2], params[3],
                                               (int)k, nq, d_qbucket, d_qlo, d_qhi, d_qshift, nbins,
                                               (unsigned long long *)d_counts, use_smem);
    } else {
        smem_optin(k_range_hist<1>, dyn);
        k_range_hist<1><<<grid, NT, dyn, st>>>((const uint64_t *)d_keys, n, params[0], params[1], params[2], params[3],
                                               (int)k, nq, d_qbucket, d_qlo, d_qhi, d_qshift, nbins,
                                               (unsigned long long *)d_counts, use_smem);
    }
    ZSB_LAUNCH("k_range_hist");
    return ZSB_OK;
}

size_t zsb_partition_workspace_bytes(int64_t n, int32_t payload_bytes, int32_t nparts) {
    if (n < 1) n = 1;
    Plan1 P = plan_partition(n, payload_bytes, nparts);
    return make_layout(n, payload_bytes, P, false).total + align_up(sizeof(DestCuts)) + align_up(sizeof(PeerDest));
}

int zsb_partition_to_ranks(const void *d_keys, int32_t key_dtype, const void *d_payload, int32_t payload_bytes,
                           int64_t n, const double *params, int64_t k, int64_t gidx_base, int32_t ncuts,
                           const int32_t *h_cut_bucket, const uint64_t *h_cut_ord, const int64_t *h_cut_gidx,
                           void *d_out_keys, void *d_out_payload, int64_t *h_part_counts, void *d_workspace,
                           size_t workspace_bytes, void *stream) {
    int rc = check_common(d_keys, key_dtype, payload_bytes, n);
    if (rc) return rc;
    if (ncuts < 0 || ncuts > MAX_CUTS || !params || k < 2 || k > 16384)
        return fail(ZSB_ERR_ARG, "need 0 <= ncuts <= 15, 2 <= k <= 16384 and params");
    const int nparts = ncuts + 1;
    for (int j = 0; j < nparts; j++) h_part_counts[j] = 0;
    if (n == 0) return ZSB_OK;
    Ctx ctx;
    ctx.n = n;
    ctx.P = plan_partition(n, payload_bytes, nparts);
    ctx.L = make_layout(n, payload_bytes, ctx.P, false);
    const size_t need = ctx.L.total + align_up(sizeof(DestCuts)) + align_up(sizeof(PeerDest));
    if (!d_workspace || workspace_bytes < need) return fail(ZSB_ERR_WORKSPACE, "workspace too small");
    ctx.ws = (unsigned char *)d_workspace;
    ctx.st = (cudaStream_t)stream;
    DestCuts hc{};
    hc.center = params[0];
    hc.std = params[1];
    hc.zmin = params[2];
    hc.scale = params[3];
    hc.k = (int32_t)k;
    hc.ncuts = ncuts;
    hc.gidx_base = gidx_base;
    for (int j = 0; j < ncuts; j++) {
        hc.bucket[j] = h_cut_bucket[j];
        hc.ord[j] = h_cut_ord[j];
        hc.gidx[j] = h_cut_gidx[j];
    }
    DestCuts *dc = (DestCuts *)(ctx.ws + ctx.L.total);
    ZSB_CUDA(cudaMemcpyAsync(dc, &hc, sizeof(hc), cudaMemcpyHostToDevice, ctx.st));
    ctx.B.in_k = (const uint64_t *)d_keys;
    ctx.B.in_p = d_payload;
    ctx.B.tmp_k = nullptr;
    ctx.B.tmp_p = nullptr;
    ctx.B.out_k = (uint64_t *)d_out_keys;
    ctx.B.out_p = d_out_payload;
    ctx.B.cuts = dc;
    ctx.B.cdf = nullptr;
    ctx.B.status = nullptr;
    ctx.B.n = n;
    ctx.B.peers = nullptr;
    SegParams *seg = (SegParams *)(ctx.ws + ctx.L.seg_a);
    int64_t *kfirst = (int64_t *)(ctx.ws + ctx.L.kfirst);
    count_launches(1);
    k_init_level1<<<1, 1, 0, ctx.st>>>(seg, kfirst, nullptr, 0, n, nparts, ctx.P.tile_len, ctx.P.ntiles, 0, 0.0, 1.0,
                                       0.0, 1.0, MODE_DEST);
    ZSB_LAUNCH("k_init_level1");
    rc = dispatch<PartitionOp>(key_dtype, payload_bytes, ctx, d_out_keys ? 3 : 1);
    if (rc) return rc;
    // per-destination totals from the scanned matrix: starts at tile 0 of each part
    std::vector<uint32_t> starts(nparts);
    const uint32_t *mat = (const uint32_t *)(ctx.ws + ctx.L.mat);
    ZSB_CUDA(cudaMemcpy2DAsync(starts.data(), sizeof(uint32_t), mat, (size_t)ctx.P.ntiles * 4, sizeof(uint32_t),
                               nparts, cudaMemcpyDeviceToHost, ctx.st));
    ZSB_CUDA(cudaStreamSynchronize(ctx.st));
    for (int j = 0; j < nparts; j++)
        h_part_counts[j] = (int64_t)((j + 1 < nparts) ? starts[j + 1] : (uint32_t)n) - (int64_t)starts[j];
    return ZSB_OK;
}


int zsb_partition_send(const void *d_keys, int32_t key_dtype, const void *d_payload, int32_t payload_bytes, int64_t n,
                       int32_t nparts, const uint64_t *h_dest_keys, const uint64_t *h_dest_payload,
                       const int64_t *h_dest_offset, void *d_workspace, size_t workspace_bytes, void *stream) {
    int rc = check_common(d_keys, key_dtype, payload_bytes, n);
    if (rc) return rc;
    if (nparts < 1 || nparts > MAX_PEERS || !h_dest_keys || !h_dest_offset || (payload_bytes && !h_dest_payload))
        return fail(ZSB_ERR_ARG, "need 1 <= nparts <= 16 and destination tables");
    if (n == 0) return ZSB_OK;
    Ctx ctx;  // the plan and layout of the zsb_partition_to_ranks call (counts only) on this workspace
    ctx.n = n;
    ctx.P = plan_partition(n, payload_bytes, nparts);
    ctx.L = make_layout(n, payload_bytes, ctx.P, false);
    const size_t need = ctx.L.total + align_up(sizeof(DestCuts)) + align_up(sizeof(PeerDest));
    if (!d_workspace || workspace_bytes < need) return fail(ZSB_ERR_WORKSPACE, "workspace too small");
    ctx.ws = (unsigned char *)d_workspace;
    ctx.st = (cudaStream_t)stream;
    // local starts of the destinations (the scanned matrix at tile 0), then delta = offset - start
    std::vector<uint32_t> starts(nparts);
    const uint32_t *mat = (const uint32_t *)(ctx.ws + ctx.L.mat);
    ZSB_CUDA(cudaMemcpy2DAsync(starts.data(), sizeof(uint32_t), mat, (size_t)ctx.P.ntiles * 4, sizeof(uint32_t),
                               nparts, cudaMemcpyDeviceToHost, ctx.st));
    ZSB_CUDA(cudaStreamSynchronize(ctx.st));
    PeerDest hp{};
    for (int j = 0; j < nparts; j++) {
        hp.k[j] = h_dest_keys[j];
        hp.p[j] = payload_bytes ? h_dest_payload[j] : 0;
        hp.delta[j] = h_dest_offset[j] - (int64_t)starts[j];
    }
    PeerDest *pd = (PeerDest *)(ctx.ws + ctx.L.total + align_up(sizeof(DestCuts)));
    ZSB_CUDA(cudaMemcpyAsync(pd, &hp, sizeof(hp), cudaMemcpyHostToDevice, ctx.st));
    ctx.B.in_k = (const uint64_t *)d_keys;
    ctx.B.in_p = d_payload;
    ctx.B.tmp_k = nullptr;
    ctx.B.tmp_p = nullptr;
    ctx.B.out_k = nullptr;
    ctx.B.out_p = nullptr;
    ctx.B.cuts = (const DestCuts *)(ctx.ws + ctx.L.total);
    ctx.B.cdf = nullptr;
    ctx.B.status = nullptr;
    ctx.B.n = n;
    ctx.B.peers = pd;
    rc = dispatch<PartitionOp>(key_dtype, payload_bytes, ctx, 2);
    if (rc) return rc;
    ZSB_CUDA(cudaStreamSynchronize(ctx.st));  // every record stored (peers read after the caller's barrier)
    return ZSB_OK;
}

}  // extern "C"
