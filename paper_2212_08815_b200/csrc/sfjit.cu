// Per-layer specialised sparse-filter convolution ("sfjit"): the filter bank's
// nonzero pattern and values are compiled into the kernel.
//
// Same computation as sf3x3_kernel (sf_conv.cu; reference _conv_all_filters_kernel,
// layers.py:170-180, over _window_acc, kernels.py:78-97, 3x3/s1/p1) and the same
// per-output accumulation order -- channels ascending, then the filter's taps
// (kh, kw) ascending, one fp32 FMA each, + bias, ReLU, fused 2x2 max-pool -- so the
// two kernels give bit-identical outputs.  What changes is how the sparsity is
// walked: instead of dispatching every nonzero through a jump table at run time,
// each group of KT filters gets its own straight-line code, one FFMA2 (with the weight
// as an immediate) per nonzero.  No weight loads, no index decoding, no indirect
// branches: per input channel a lane loads its 3x4 input patch (6 LDS.64) and issues one
// FFMA2 per nonzero of the group at that channel.
//
//   lane   = one 1x2 output tile (acc: KT filters as column pairs, KT b64); the smallest
//            tile that keeps FFMA2, so the code -- which must stay L2-resident, see
//            below -- is one 16-byte instruction per nonzero
//   tiles  = ordered per image by row pair, then blocks of BW columns, then row parity,
//            then column: the lanes of a 2x2 pooling window are lane ^ BW (shuffle)
//   CTA    = one filter group over TI consecutive tiles of that order: a 1/M part of an
//            image (large images) or Q whole images (small ones), WARPS = ceil(TI/32)
//            warps -- as many as the registers allow, since every warp of the CTA shares
//            the one instruction stream; grid = N*M or ceil(N/Q) per group
//
// Input channels stream through a shared-memory ring (S stages of CC channels): one
// TMA box per image the CTA's tile range touches (full padded row width, BH rows,
// CC channels; the TMA zero fill provides the conv padding), completed on one
// mbarrier per stage; a CTA barrier before each restage keeps the warps of a CTA in
// lockstep, which is what makes this fast: every warp of an SM executes the same
// instruction stream, so one instruction fetch serves all of them (measured: the
// straight-line code is fetch-bound at ~0.17 instructions/clock/SM, shared by every
// warp in lockstep -- tools/jit_proto).
//
// The PTX of each group is generated here (C++), compiled with nvJitLink on a pool of
// host threads (cached on disk by content hash), and loaded with the driver API.
#include <cuda.h>
#include <nvJitLink.h>
#include <stdarg.h>
#include <stdlib.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <fstream>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace fscnn {
namespace {

// ------------------------------------------------------------------------------------
// driver API (through the runtime's entry-point query: no libcuda link dependency)
// ------------------------------------------------------------------------------------
struct Driver {
    CUresult (*moduleLoadData)(CUmodule *, const void *) = nullptr;
    CUresult (*moduleUnload)(CUmodule) = nullptr;
    CUresult (*moduleGetFunction)(CUfunction *, CUmodule, const char *) = nullptr;
    CUresult (*funcSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
    CUresult (*funcGetAttribute)(int *, CUfunction_attribute, CUfunction) = nullptr;
    CUresult (*launchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                             CUstream, void **, void **) = nullptr;
    CUresult (*encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                            const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill) = nullptr;
    CUresult (*getErrorString)(CUresult, const char **) = nullptr;
    bool ok = false;
};

template <typename F>
bool entry(const char *name, F &fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        return false;
    fn = reinterpret_cast<F>(p);
    return true;
}

const Driver &driver() {
    static Driver d;
    static std::once_flag once;
    std::call_once(once, [] {
        d.ok = entry("cuModuleLoadData", d.moduleLoadData) && entry("cuModuleUnload", d.moduleUnload) &&
               entry("cuModuleGetFunction", d.moduleGetFunction) &&
               entry("cuFuncSetAttribute", d.funcSetAttribute) && entry("cuFuncGetAttribute", d.funcGetAttribute) &&
               entry("cuLaunchKernel", d.launchKernel) && entry("cuTensorMapEncodeTiled", d.encodeTiled) &&
               entry("cuGetErrorString", d.getErrorString);
    });
    return d;
}

const char *cu_err(CUresult r) {
    const char *s = "unknown";
    if (driver().getErrorString) driver().getErrorString(r, &s);
    return s;
}

// ------------------------------------------------------------------------------------
// host thread pool for the compile jobs
// ------------------------------------------------------------------------------------
class Pool {
  public:
    static Pool &get() {
        // never destroyed: the workers are detached and block on cv_ until the process
        // exits; a static destructor would tear the cv down under them (hang at exit)
        static Pool *p = new Pool;
        return *p;
    }
    void submit(std::function<void()> job) {
        {
            std::lock_guard<std::mutex> g(mu_);
            q_.push_back(std::move(job));
        }
        cv_.notify_one();
    }

  private:
    Pool() {
        unsigned n = std::thread::hardware_concurrency();
        if (const char *e = getenv("FSCNN_JIT_THREADS")) n = (unsigned)atoi(e);
        if (n == 0) n = 4;
        for (unsigned i = 0; i < n; ++i) std::thread([this] { run(); }).detach();
    }
    void run() {
        for (;;) {
            std::function<void()> job;
            {
                std::unique_lock<std::mutex> g(mu_);
                cv_.wait(g, [this] { return !q_.empty(); });
                job = std::move(q_.front());
                q_.pop_front();
            }
            job();
        }
    }
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> q_;
};

// ------------------------------------------------------------------------------------
// plan
// ------------------------------------------------------------------------------------
struct Plan {
    int C, K, H, W, relu, pool;
    int KT, WARPS, T;   // filters per group, warps per CTA, threads per CTA (32*WARPS)
    int MODE;           // 0: M CTAs per image (TI tiles each), 1: Q whole images per CTA
    int M, Q, TI;
    int TPR, TPI;       // tiles per row (w/2, padded to a multiple of 8 when odd), per image
    int TPRR;           // real tiles per row (w/2): lanes past it compute nothing they store
    int BW;             // column block of the lane order (pool partner = lane ^ BW)
    int P;              // smem row pitch (floats) == TMA box width
    int BH;             // TMA box rows
    int NB;             // max images (boxes) per CTA
    int CC, S;          // channels per chunk, ring stages
    int64_t box_bytes;  // one box (CC channels), 128-byte multiple
    int64_t stage_bytes;
    int64_t smem_bytes;
    int n_groups, n_chunks;
    int fused;     // 1: one kernel for all groups (grid.y = group), one compile job
    int odd_mode;  // kw = 1 pair: 0 = two 4-byte loads, 1 = moves from the even pairs
    int tma_hint;  // 1: input boxes loaded L2 evict-first
    int store_cs;  // 1: outputs stored streaming (evict-first)
    int nobar;     // 1: per-stage empty mbarriers instead of a CTA barrier per chunk
    int tma_split; // TMA operations per box (each CC / tma_split channels; they run concurrently)
    int uni;       // 1: chunk-boundary control flow without divergent regions (warp-uniform polls, predicated restage)
    int tma_merge; // 1: whole-image mode loads a chunk's Q image boxes as ONE operation (box image extent Q)
};

int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// Rows (BH) of the CTA's TMA box: part mode covers the row pairs of its TI tiles (+ the
// halo rows), multi-image mode whole padded images.
void box_geometry(Plan &p) {
    const int U = 2 * p.TPR;
    if (p.MODE == 1) {
        p.BH = p.H + 2;
        p.NB = p.Q;
        return;
    }
    int bh = 0;
    for (int part = 0; part < p.M; ++part) {
        const int a = part * p.TI, e = std::min(a + p.TI, p.TPI) - 1;
        bh = std::max(bh, 2 * (e / U - a / U + 1) + 2);
    }
    p.BH = std::min(bh, p.H + 2);
    p.NB = 1;
}

bool make_plan(Plan &p, int c, int k, int h, int w, int relu, int pool, int flags, char *why, size_t why_n) {
    p.C = c, p.K = k, p.H = h, p.W = w, p.relu = relu, p.pool = pool;
    if (h % 2 || w % 2) {
        snprintf(why, why_n, "extents must be even (1x2 lane tiles, 2x2 pooling windows)");
        return false;
    }
    // kw = 1 pair: two 4-byte loads (their half-warps collide on odd banks: 2 wavefronts
    // each) or moves from the even pairs (more code).  Shared-memory-bound shallow layers
    // (C <= 64: few channels, the code stays cached) take the moves: VGG16 L1 -10 %,
    // L2 -5 %; the fetch-bound deep layers keep the loads (L3/L4 +3-7 % with moves)
    p.odd_mode = getenv("FSCNN_SFJIT_ODD") ? atoi(getenv("FSCNN_SFJIT_ODD")) : (c > 16 && c <= 64 ? 1 : 0);
    p.tma_hint = getenv("FSCNN_SFJIT_TMA_HINT") ? atoi(getenv("FSCNN_SFJIT_TMA_HINT")) : 1;
    p.store_cs = getenv("FSCNN_SFJIT_STORE_CS") ? atoi(getenv("FSCNN_SFJIT_STORE_CS")) : 1;
    p.nobar = getenv("FSCNN_SFJIT_NOBAR") ? atoi(getenv("FSCNN_SFJIT_NOBAR")) : 1;
    // chunk-boundary control flow without divergent regions: the stage polls vote to a
    // warp-uniform result and branch .uni, warp 0 as a whole polls the empty barrier and
    // lane 0 issues the (predicated) TMA -- no BSSY/BSYNC reconvergence points, whose
    // fetch restarts held ~10 % of an L10 group's stall samples (every layer -0.4..-2.8 %,
    // C3 step +1.1 %, bit-identical; FSCNN_SFJIT_UNI=0 restores the thread-0 branches)
    p.uni = getenv("FSCNN_SFJIT_UNI") ? atoi(getenv("FSCNN_SFJIT_UNI")) : 1;
    // 48 filters per group: measured best on the VGG16 stack (32: -6 %, 64: -20 %; more
    // filters per group = less code per FMA, fewer warps per CTA sharing its fetch)
    p.KT = std::min(48, k);
    if (getenv("FSCNN_SFJIT_KT")) p.KT = std::min(atoi(getenv("FSCNN_SFJIT_KT")), k);
    if (flags & 0xff) p.KT = std::min(flags & 0xff, k);
    // an odd tile-row length (w = 14: 7 tiles) would pair rows of a pooling window in a
    // column block of 1, whose 8-byte patch loads collide on banks at every row-pair
    // wrap (ncu: 55 % excessive wavefronts); pad the row to 8 tiles instead -- the extra
    // lanes cost no time on these fetch-bound layers and store nothing
    p.TPRR = w / 2;
    p.TPR = (p.TPRR % 2) ? (int)align_up(p.TPRR, 8) : p.TPRR;
    // a 9..15-tile row (w = 28: 14 tiles) has BW = 2 and wraps a warp across row pairs:
    // the second half-warp's 8-byte patch loads then collide on 8 of 32 banks (ncu: 44 %
    // excessive wavefronts, the warm-code bound of these layers); padding the row to 16
    // tiles (BW = 16, 12.5 % idle lanes) measured VGG16 L7 -16 %, L8 -18 %.  Wider rows
    // (56 -> 64, 28 -> 32 tiles) measured neutral to slower and keep their width
    if (p.TPRR > 8 && p.TPRR < 16) p.TPR = 16;
    if (getenv("FSCNN_SFJIT_PADTPR")) p.TPR = (int)align_up(p.TPRR, atoi(getenv("FSCNN_SFJIT_PADTPR")));
    p.TPI = p.TPR * h;
    p.BW = 16;
    while (p.TPR % p.BW) p.BW >>= 1;
    // warps per CTA: the register file shared by one CTA (~2*KT accumulator registers +
    // patch/addressing); flags bits 8-15 cap it
    const int wcap = getenv("FSCNN_SFJIT_WMAX") ? atoi(getenv("FSCNN_SFJIT_WMAX")) : 20;
    int wmax = std::min(wcap, 65536 / (32 * (2 * p.KT + 36)));
    if ((flags >> 8) & 0xff) wmax = std::min(wmax, (flags >> 8) & 0xff);
    // very shallow inputs (the first layer, c = 3): the code is a few hundred
    // instructions and each CTA mostly waits for its one TMA stage and stores -- several
    // smaller CTAs per SM overlap those waits
    if (c <= 16) wmax = std::min(wmax, 8);
    wmax = std::max(wmax, 1);
    const int cap = 32 * wmax;
    const int unit = 2 * p.BW;  // part boundaries keep pooling partners (lane ^ BW) together
    if (p.TPI > cap) {
        p.MODE = 0, p.Q = 1;
        p.M = (p.TPI + cap - 1) / cap;
        p.TI = (int)align_up((p.TPI + p.M - 1) / p.M, unit);
        while (p.TI > cap) {
            ++p.M;
            p.TI = (int)align_up((p.TPI + p.M - 1) / p.M, unit);
        }
    } else {
        p.MODE = 1, p.M = 1;
        p.Q = std::max(1, cap / p.TPI);
        p.TI = p.Q * p.TPI;
    }
    p.WARPS = (p.TI + 31) / 32;
    p.T = 32 * p.WARPS;
    // row pitch: >= 2 TPR + 2 (the padded tile row's patches; w + 2 would cover every real
    // lane -- padded lanes then read into the next row and store nothing -- and shrinks
    // the 14x14 boxes 3x, but measured -1..-2 % at 90 % zeros and +2..4 % at 50 % on
    // L10/L11: FSCNN_SFJIT_REALP=1), 16-byte multiple (TMA box width).  With BW < 16 a
    // half-warp covers both rows of a row pair, whose 8-byte patch loads stay on distinct
    // banks when pitch/2 == 8 (mod 16)
    p.P = (int)align_up((getenv("FSCNN_SFJIT_REALP") ? w : 2 * p.TPR) + 2, 4);
    if (p.BW < 16)
        while (p.P % 32 != 16) p.P += 4;
    if (p.P > 256) {
        snprintf(why, why_n, "row width %d exceeds the TMA box limit", w);
        return false;
    }
    box_geometry(p);
    if (p.BH > 256) {
        snprintf(why, why_n, "box height %d exceeds the TMA limit", p.BH);
        return false;
    }
    // one CTA per SM by default; FSCNN_SFJIT_SMEM_KB (with FSCNN_SFJIT_MINB) packs more
    const int64_t budget = (getenv("FSCNN_SFJIT_SMEM_KB") ? atoi(getenv("FSCNN_SFJIT_SMEM_KB")) : 215) * 1024;
    const int64_t per_ch = (int64_t)p.BH * p.P * 4;
    p.S = 4;
    for (;;) {
        int64_t cc = budget / (p.S * p.NB * per_ch + 1);
        // keep a 128-byte multiple per box
        while (cc > 0 && p.S * p.NB * align_up(cc * per_ch, 128) > budget) --cc;
        if (cc >= 1 || p.S == 2) {
            p.CC = (int)std::max<int64_t>(1, std::min<int64_t>(cc, 16));
            break;
        }
        --p.S;
    }
    p.CC = std::min(p.CC, c);
    p.S = std::min<int>(p.S, (c + p.CC - 1) / p.CC);  // no stages beyond the chunks
    // one box as tma_split TMA operations of CC / tma_split channels each (same bytes, same
    // layout: the channel is the box's outermost extent); FSCNN_SFJIT_TMA_SPLIT requests it,
    // the largest divisor of CC not above the request is taken
    p.tma_split = getenv("FSCNN_SFJIT_TMA_SPLIT") ? std::max(1, atoi(getenv("FSCNN_SFJIT_TMA_SPLIT"))) : 1;
    p.tma_split = std::min(p.tma_split, p.CC);
    while (p.tma_split > 1 && (p.CC % p.tma_split || (((int64_t)p.CC / p.tma_split) * per_ch) % 128)) --p.tma_split;
    p.box_bytes = align_up((int64_t)p.CC * per_ch, 128);
    // whole-image CTAs: the Q images' boxes of a chunk as one TMA operation (the image is
    // the box's outermost extent, images past the batch are zero-filled and counted)
    // (one operation instead of Q per chunk: VGG16 14x14 layers -3..-10 %, C3 step +0.7 %,
    // bit-identical; FSCNN_SFJIT_TMA_MERGE=0 keeps one operation per image)
    p.tma_merge = !(getenv("FSCNN_SFJIT_TMA_MERGE") && !atoi(getenv("FSCNN_SFJIT_TMA_MERGE"))) && p.MODE == 1 && p.NB > 1 &&
                  p.tma_split == 1 && p.box_bytes == (int64_t)p.CC * per_ch;
    p.stage_bytes = p.NB * p.box_bytes;
    p.smem_bytes = p.S * p.stage_bytes + 16 * p.S;  // full[S] + empty[S] mbarriers
    if (p.smem_bytes > 227 * 1024) {
        snprintf(why, why_n, "shared memory %lld bytes exceeds the limit", (long long)p.smem_bytes);
        return false;
    }
    p.n_groups = (k + p.KT - 1) / p.KT;
    p.fused = (flags >> 16) & 1;
    p.n_chunks = (c + p.CC - 1) / p.CC;
    return true;
}

// ------------------------------------------------------------------------------------
// PTX generation
// ------------------------------------------------------------------------------------
struct Out {
    std::string s;
    void operator()(const char *fmt, ...) __attribute__((format(printf, 2, 3))) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        int n = vsnprintf(buf, sizeof(buf), fmt, ap);
        va_end(ap);
        s.append(buf, (size_t)std::min(n, (int)sizeof(buf) - 1));
        s.push_back('\n');
    }
};

uint32_t fbits(float v) {
    uint32_t u;
    memcpy(&u, &v, 4);
    return u;
}

// wt: dense [K][C][3][3] fp32 (host), bias [K] (host, may be null)
// gen_group: one group's standalone kernel; gen_fused: one kernel for every group of
// the layer (blockIdx.y = group, a jump table to the group's code) -- small layers,
// where one launch beats a fork over per-group launches.
std::string gen_kernel(const Plan &p, const float *wt, const float *bias, int g_first, int g_count) {
    Out o;
    o.s.reserve(1 << 20);
    const int KT = p.KT;
    const bool fused = g_count > 1;
    int kn = 0;
    for (int g = g_first; g < g_first + g_count; ++g) kn = std::max(kn, std::min(KT, p.K - g * KT));
    const int U = 2 * p.TPR;  // tiles per row pair
    o(".version 8.7");
    o(".target sm_100a");
    o(".address_size 64");
    o(".extern .shared .align 1024 .b8 smem[];");
    o(".visible .entry sfjit(.param .align 64 .b8 tmap[128], .param .u64 py, .param .u32 pldo, .param .u32 pn)");
    o(".maxntid %d, 1, 1", p.T);
    o(".minnctapersm %d", getenv("FSCNN_SFJIT_MINB") ? atoi(getenv("FSCNN_SFJIT_MINB")) : 1);
    o("{");
    o(".reg .pred pv, pt0, pw, pl, pp0, pw0;");
    o(".reg .b32 tid, cta, nimg, i0, ulo, tt, img, r2, qq, par, col, row, bi, rb, ldo, nbox, y0f;");
    o(".reg .b32 q0, q1, q2, q3, q4, qdst, qimg, qy, qc, qbi, rbar;");
    o(".reg .b64 tm, yp, yb, ks, w64;");
    o(".reg .b64 a<%d>;", kn);
    o(".reg .b64 e<6>;");
    o(".reg .b64 od<3>;");
    o(".reg .f32 fw, f0, f1, g0, g1, fm;");
    o(".reg .b64 dw, pol;");
    // ---- prologue: this CTA's images / tile range and the lane's tile
    o("mov.b64 tm, tmap;");
    o("cvta.param.u64 tm, tm;");
    o("ld.param.u64 yp, [py];");
    o("ld.param.u32 ldo, [pldo];");
    o("ld.param.u32 nimg, [pn];");
    o("mov.u32 tid, %%tid.x;");
    o("mov.u32 cta, %%ctaid.x;");
    if (p.MODE == 0) {
        // CTA = part (cta % M) of image cta / M: tiles part*TI .. min(part*TI + TI, TPI) - 1
        o("div.u32 i0, cta, %d;", p.M);
        o("rem.u32 q0, cta, %d;", p.M);
        o("mul.lo.u32 q0, q0, %d;", p.TI);      // first tile of the part
        o("div.u32 ulo, q0, %d;", U);           // its row pair
        o("add.u32 tt, q0, tid;");
        o("add.u32 q1, q0, %d;", p.TI);
        o("min.u32 q1, q1, %d;", p.TPI);        // end of the part
        o("setp.lt.u32 pv, tt, q1;");
        o("sub.u32 q1, q1, 1;");
        o("min.u32 tt, tt, q1;");
        o("mov.u32 img, i0;");
        o("mov.u32 nbox, 1;");
        o("shl.b32 y0f, ulo, 1;");
        o("sub.u32 y0f, y0f, 1;");              // the box starts at row 2*ulo - 1
    } else {
        // CTA = images cta*Q .. cta*Q + Q - 1 (clipped to the batch), whole padded images
        o("mul.lo.u32 i0, cta, %d;", p.Q);
        o("div.u32 q0, tid, %d;", p.TPI);
        o("rem.u32 tt, tid, %d;", p.TPI);
        o("add.u32 img, i0, q0;");
        o("setp.lt.u32 pv, img, nimg;");
        o("setp.lt.u32 pw, tid, %d;", p.TI);
        o("and.pred pv, pv, pw;");
        o("selp.b32 img, img, i0, pv;");        // idle lanes address the first image
        o("selp.b32 tt, tt, 0, pv;");
        o("sub.u32 nbox, nimg, i0;");
        o("min.u32 nbox, nbox, %d;", p.Q);
        o("mov.u32 ulo, 0;");
        o("mov.u32 y0f, -1;");
    }
    o("div.u32 r2, tt, %d;", U);
    o("rem.u32 qq, tt, %d;", U);
    // qq = block * 2BW + parity * BW + column in block
    o("and.b32 q0, qq, %d;", p.BW - 1);
    o("shr.u32 q1, qq, %d;", __builtin_ctz(2 * p.BW));
    o("mad.lo.u32 col, q1, %d, q0;", p.BW);
    o("shr.u32 par, qq, %d;", __builtin_ctz(p.BW));
    o("and.b32 par, par, 1;");
    o("shl.b32 row, r2, 1;");
    o("add.u32 row, row, par;");
    o("setp.eq.u32 pp0, par, 0;");
    if (p.TPR != p.TPRR) {  // padded tile row: the columns past the image store nothing
        o("setp.lt.u32 pl, col, %d;", p.TPRR);
        o("and.pred pv, pv, pl;");
    }
    o("sub.u32 bi, img, i0;");
    // smem row of the patch's first row (image row - 1): the first box starts at row
    // 2*ulo - 1, later boxes at -1
    o("setp.eq.u32 pw, bi, 0;");
    o("selp.b32 q0, ulo, 0, pw;");
    o("shl.b32 q0, q0, 1;");
    o("sub.u32 q1, row, q0;");
    o("mov.u32 rb, smem;");
    o("mad.lo.u32 rb, bi, %lld, rb;", (long long)p.box_bytes);
    o("mad.lo.u32 rb, q1, %d, rb;", p.P * 4);
    o("shl.b32 q2, col, 3;");
    o("add.u32 rb, rb, q2;");
    o("mov.u32 rbar, smem;");
    o("add.u32 rbar, rbar, %lld;", (long long)(p.S * p.stage_bytes));
    o("setp.eq.u32 pt0, tid, 0;");
    o("setp.lt.u32 pw0, tid, 32;");
    // activations stream through L2 evict-first: the layer's code (fetched by every CTA)
    // must stay L2-resident -- instruction fetch from HBM halves the issue rate
    // (measured, tools/jit_proto)
    o("createpolicy.fractional.L2::evict_first.b64 pol, 1.0;");
    o("@!pt0 bra PRO_DONE;");
    for (int s = 0; s < p.S; ++s) o("mbarrier.init.shared::cta.b64 [rbar+%d], 1;", 8 * s);
    if (p.nobar)  // empty[s]: one arrival per warp when it is done reading stage s
        for (int s = 0; s < p.S; ++s) o("mbarrier.init.shared::cta.b64 [rbar+%d], %d;", 8 * (p.S + s), p.WARPS);
    o("fence.mbarrier_init.release.cluster;");
    o("prefetch.tensormap [tm];");
    std::string lp = "p_";  // label prefix: prologue, then one per group
    auto issue = [&](int j) {
        const int s = j % p.S;
        const int c0 = j * p.CC;
        // the transaction count is the bytes the boxes deliver (boxes sit at 128-byte
        // aligned strides, but only CC*BH*P floats of each are written)
        if (p.tma_merge)
            o("mov.u32 q0, %lld;", (long long)p.NB * p.CC * p.BH * p.P * 4);
        else
            o("mul.lo.u32 q0, nbox, %lld;", (long long)p.CC * p.BH * p.P * 4);
        o("@pt0 mbarrier.arrive.expect_tx.shared::cta.b64 _, [rbar+%d], q0;", 8 * s);
        o("mov.u32 qdst, smem;");
        o("add.u32 qdst, qdst, %lld;", (long long)(s * p.stage_bytes));
        o("mov.u32 qimg, i0;");
        o("mov.u32 qy, y0f;");
        o("mov.u32 qc, %d;", c0);
        o("mov.u32 qbi, 0;");
        o("add.u32 q2, rbar, %d;", 8 * s);
        o("mov.u32 q3, 0;");
        o("%sISS%d:", lp.c_str(), j);
        const int cs = p.CC / p.tma_split;
        const long long sub_bytes = (long long)cs * p.BH * p.P * 4;
        for (int sub = 0; sub < p.tma_split; ++sub) {
            if (sub) {
                o("add.u32 qc, qc, %d;", cs);
                o("add.u32 qdst, qdst, %lld;", sub_bytes);
            }
            if (p.tma_hint)
                o("@pt0 cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [qdst], "
                  "[tm, {q3, qy, qc, qimg}], [q2], pol;");
            else
                o("@pt0 cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [qdst], [tm, "
                  "{q3, qy, qc, qimg}], [q2];");
        }
        if (p.tma_split > 1) o("mov.u32 qc, %d;", c0);
        o("add.u32 qdst, qdst, %lld;", (long long)p.box_bytes - (p.tma_split - 1) * sub_bytes);
        o("add.u32 qimg, qimg, 1;");
        o("mov.u32 qy, -1;");
        o("add.u32 qbi, qbi, 1;");
        if (p.tma_merge)
            o("setp.lt.u32 pl, qbi, 1;");
        else
            o("setp.lt.u32 pl, qbi, nbox;");
        if (p.uni && (p.tma_merge || p.NB == 1))
            ;  // one operation per chunk: no loop
        else if (p.uni)
            o("@pl bra.uni %sISS%d;", lp.c_str(), j);  // nbox is CTA-uniform
        else
            o("@pl bra %sISS%d;", lp.c_str(), j);
    };
    for (int j = 0; j < std::min(p.S, p.n_chunks); ++j) issue(j);
    o("PRO_DONE:");
    o("barrier.sync 0;");
    for (int i = 0; i < kn; ++i) o("mov.b64 a%d, 0;", i);
    if (fused) {
        std::string t = "GTBL: .branchtargets ";
        for (int g = g_first; g < g_first + g_count; ++g) t += (g > g_first ? ", G" : "G") + std::to_string(g);
        o.s += t + ";\n";
        o("{ .reg .b32 gy; mov.u32 gy, %%ctaid.y; brx.idx.uni gy, GTBL; }");
    }
    struct Nz {
        int kl, kh, kw;
        uint32_t w;
    };
    std::vector<Nz> nz;
    nz.reserve(9 * 64);
  for (int g = g_first; g < g_first + g_count; ++g) {
    const int k0 = g * KT;
    const int kn = std::min(KT, p.K - k0);
    lp = "g" + std::to_string(g) + "_";
    if (fused) o("G%d:", g);
    // ---- channel chunks
    for (int j = 0; j < p.n_chunks; ++j) {
        const int s = j % p.S;
        const int par_bit = (j / p.S) & 1;
        // bounded wait: a stage that never completes traps instead of hanging the GPU
        o("mov.u32 q4, %d;", par_bit);
        o("mov.u32 q3, 0;");
        o("%sWT%d:", lp.c_str(), j);
        o("mbarrier.try_wait.parity.shared::cta.b64 pw, [rbar+%d], q4;", 8 * s);
        if (p.uni) {
            o("vote.sync.all.pred pw, pw, 0xffffffff;");
            o("@pw bra.uni %sWD%d;", lp.c_str(), j);
        } else
            o("@pw bra %sWD%d;", lp.c_str(), j);
        o("add.u32 q3, q3, 1;");
        o("setp.gt.u32 pl, q3, 4000000;");
        o("@pl trap;");
        o("bra.uni %sWT%d;", lp.c_str(), j);
        o("%sWD%d:", lp.c_str(), j);
        // debug (FSCNN_SFJIT_REPEAT=R): run the chunk's code R times on the same stage
        // (wrong results) -- measures the cost of a warm re-execution of the code
        const int rep = getenv("FSCNN_SFJIT_REPEAT") ? atoi(getenv("FSCNN_SFJIT_REPEAT")) : 1;
        if (rep > 1) {
            o("mov.u32 q3, 0;");
            o("%sRP%d:", lp.c_str(), j);
        }
        const int cend = std::min(p.C, (j + 1) * p.CC);
        for (int c = j * p.CC; c < cend; ++c) {
            const int cl = c - j * p.CC;
            // nonzeros of the group at channel c: filter, then tap (kh*3+kw) ascending --
            // per accumulator the same order as sf3x3_kernel's packed stream
            nz.clear();
            bool row_needed[3] = {false, false, false}, odd_row[3] = {false, false, false};
            for (int kl = 0; kl < kn; ++kl) {
                const float *wk = wt + ((int64_t)(k0 + kl) * p.C + c) * 9;
                for (int tap = 0; tap < 9; ++tap) {
                    if (wk[tap] == 0.0f) continue;  // +-0.0 are not stored (sparsify drops them)
                    Nz z{kl, tap / 3, tap % 3, fbits(wk[tap])};
                    nz.push_back(z);
                    row_needed[z.kh] = true;
                    if (z.kw == 1) odd_row[z.kh] = true;
                }
            }
            if (nz.empty()) continue;
            const int64_t off0 = (int64_t)s * p.stage_bytes + (int64_t)cl * p.BH * p.P * 4;
            for (int r = 0; r < 3; ++r) {
                if (!row_needed[r]) continue;
                o("ld.shared.b64 e%d, [rb+%lld];", 2 * r, (long long)(off0 + (int64_t)r * p.P * 4));
                o("ld.shared.b64 e%d, [rb+%lld];", 2 * r + 1, (long long)(off0 + (int64_t)r * p.P * 4 + 8));
            }
            // the odd pair (columns 1, 2) for kw = 1 taps: two 4-byte loads straight into an
            // aligned register pair (building it from the even pairs costs ptxas ~2.7x the
            // two moves it needs: it rematerialises the pair per use)
            for (int r = 0; r < 3; ++r) {
                if (!odd_row[r] || p.odd_mode == 2) continue;
                if (p.odd_mode == 3)  // debug: one aligned 8-byte load (wrong values) -- the cost of a shifted plane
                    o("ld.shared.b64 od%d, [rb+%lld];", r, (long long)(off0 + (int64_t)r * p.P * 4 + 16));
                else if (p.odd_mode == 0)
                    o("{ .reg .f32 x1, x2; ld.shared.f32 x1, [rb+%lld]; ld.shared.f32 x2, [rb+%lld]; mov.b64 od%d, "
                      "{x1, x2}; }",
                      (long long)(off0 + (int64_t)r * p.P * 4 + 4), (long long)(off0 + (int64_t)r * p.P * 4 + 8), r);
                else
                    o("{ .reg .f32 x0, x1, x2, x3; mov.b64 {x0, x1}, e%d; mov.b64 {x2, x3}, e%d; mov.b64 od%d, {x1, "
                      "x2}; }",
                      2 * r, 2 * r + 1, r);
            }
            for (const Nz &z : nz) {
                o("mov.b32 fw, 0f%08X;", z.w);
                o("mov.b64 dw, {fw, fw};");
                if (z.kw == 1 && p.odd_mode == 2)
                    // two scalar FMAs on the halves (columns 1 and 2 of the patch row)
                    o("{ .reg .f32 x0, x1, x2, x3, s0, s1; mov.b64 {x0, x1}, e%d; mov.b64 {x2, x3}, e%d; "
                      "mov.b64 {s0, s1}, a%d; fma.rn.f32 s0, x1, fw, s0; fma.rn.f32 s1, x2, fw, s1; "
                      "mov.b64 a%d, {s0, s1}; }",
                      2 * z.kh, 2 * z.kh + 1, z.kl, z.kl);
                else if (z.kw == 1)
                    o("fma.rn.f32x2 a%d, od%d, dw, a%d;", z.kl, z.kh, z.kl);
                else
                    o("fma.rn.f32x2 a%d, e%d, dw, a%d;", z.kl, 2 * z.kh + z.kw / 2, z.kl);
            }
        }
        if (rep > 1) {
            o("add.u32 q3, q3, 1;");
            o("setp.lt.u32 pl, q3, %d;", rep);
            o("@pl bra %sRP%d;", lp.c_str(), j);
        }
        if (j + p.S < p.n_chunks) {
            if (!p.nobar) {
                // every warp is done with stage s: thread 0 restages it with chunk j+S
                o("barrier.sync 0;");
                o("@!pt0 bra %sRS%d;", lp.c_str(), j);
                issue(j + p.S);
                o("%sRS%d:", lp.c_str(), j);
            } else {
                // no CTA barrier: each warp arrives on empty[s]; thread 0 waits for all of
                // them before restaging, the other warps run on (up to S-1 chunks ahead)
                o("{ .reg .b32 ln; .reg .pred pz; and.b32 ln, tid, 31; setp.eq.u32 pz, ln, 0;");
                o("@pz mbarrier.arrive.shared::cta.b64 _, [rbar+%d]; }", 8 * (p.S + s));
                if (p.uni)
                    o("@!pw0 bra.uni %sRS%d;", lp.c_str(), j);  // warp 0 as a whole polls, lane 0 issues
                else
                    o("@!pt0 bra %sRS%d;", lp.c_str(), j);
                o("mov.u32 q4, %d;", (j / p.S) & 1);
                o("%sEW%d:", lp.c_str(), j);
                o("mbarrier.try_wait.parity.shared::cta.b64 pw, [rbar+%d], q4;", 8 * (p.S + s));
                if (p.uni) {
                    o("vote.sync.all.pred pw, pw, 0xffffffff;");
                    o("@!pw bra.uni %sEW%d;", lp.c_str(), j);
                } else
                    o("@!pw bra %sEW%d;", lp.c_str(), j);
                issue(j + p.S);
                o("%sRS%d:", lp.c_str(), j);
            }
        }
    }

    // ---- epilogue: + bias, ReLU (np.maximum semantics), [2x2 max-pool], store into the
    // next layer's halo-column buffer (logical column x at memory column x+1)
    const int HO = p.pool ? p.H / 2 : p.H;
    // yb = y + ((img*K + k0)*HO + orow)*ldo + ocol + 1   (floats)
    o("mad.lo.u32 q0, img, %d, %d;", p.K, k0);
    o("mul.wide.u32 yb, q0, %d;", HO);
    o("cvt.u64.u32 w64, %s;", p.pool ? "r2" : "row");
    o("add.u64 yb, yb, w64;");
    o("cvt.u64.u32 w64, ldo;");
    o("mul.lo.u64 yb, yb, w64;");
    if (p.pool) {
        o("add.u32 q1, col, 1;");
    } else {
        o("shl.b32 q1, col, 1;");
        o("add.u32 q1, q1, 1;");
    }
    o("cvt.u64.u32 w64, q1;");
    o("add.u64 yb, yb, w64;");
    o("shl.b64 yb, yb, 2;");
    o("add.u64 yb, yb, yp;");
    o("mul.wide.u32 ks, ldo, %d;", HO * 4);  // bytes between filter planes
    // pooled results are stored by the row-0 lane of each window
    if (p.pool) o("and.pred pv, pv, pp0;");
    // (aligned 8-byte pair stores -- the left lane's f1 shuffled in -- measured slower on
    // the store-bound first layer, 0.140 -> 0.157 ms, and neutral elsewhere)
    auto relu_np = [&](const char *f) {
        // keep v if its bits are > 0 as int (positive, not -0.0) or it is a NaN
        o("{ .reg .b32 u, m; .reg .pred k1, k2; mov.b32 u, %s; setp.gt.s32 k1, u, 0; and.b32 m, u, 2147483647; "
          "setp.gt.u32 k2, m, 2139095040; or.pred k1, k1, k2; selp.b32 u, u, 0, k1; mov.b32 %s, u; }",
          f, f);
    };
    for (int kl = 0; kl < kn; ++kl) {
        const uint32_t b = bias ? fbits(bias[k0 + kl]) : 0u;
        o("mov.b64 {f0, f1}, a%d;", kl);
        o("add.rn.f32 f0, f0, 0f%08X;", b);
        o("add.rn.f32 f1, f1, 0f%08X;", b);
        if (p.relu) {
            relu_np("f0");
            relu_np("f1");
        }
        if (p.pool) {
            // the other row of the window lives in lane ^ BW; every lane exchanges, the
            // row-0 lane reduces in the reference order: -inf start, '>' compare, (ph, pw)
            // row-major (_pool_dense_kernel, layers.py:250-271)
            o("shfl.sync.bfly.b32 g0, f0, %d, 31, -1;", p.BW);
            o("shfl.sync.bfly.b32 g1, f1, %d, 31, -1;", p.BW);
            o("mov.b32 fm, 0fFF800000;");
            for (const char *v : {"f0", "f1", "g0", "g1"})
                o("{ .reg .pred g; setp.gt.f32 g, %s, fm; selp.f32 fm, %s, fm, g; }", v, v);
            o(p.store_cs ? "@pv st.global.cs.f32 [yb], fm;" : "@pv st.global.f32 [yb], fm;");
        } else {
            o(p.store_cs ? "@pv st.global.cs.f32 [yb], f0;" : "@pv st.global.f32 [yb], f0;");
            o(p.store_cs ? "@pv st.global.cs.f32 [yb+4], f1;" : "@pv st.global.f32 [yb+4], f1;");
        }
        if (kl + 1 < kn) o("add.u64 yb, yb, ks;");
    }
    o("ret;");
  }
    o("}");
    return o.s;
}

std::string gen_group(const Plan &p, const float *wt, const float *bias, int g) {
    return gen_kernel(p, wt, bias, g, 1);
}

uint64_t fnv1a(const std::string &s, uint64_t h = 1469598103934665603ull) {
    for (unsigned char ch : s) h = (h ^ ch) * 1099511628211ull;
    return h;
}

std::string cache_dir() {
    if (const char *e = getenv("FSCNN_JIT_CACHE")) return e;
    const char *home = getenv("HOME");
    return std::string(home ? home : "/tmp") + "/.cache/fscnn_b200/sfjit";
}

void mkdirs(const std::string &path) {
    std::string cur;
    for (size_t i = 0; i < path.size(); ++i) {
        cur.push_back(path[i]);
        if (path[i] == '/' && cur.size() > 1) mkdir(cur.c_str(), 0755);
    }
    mkdir(path.c_str(), 0755);
}

// PTX -> cubin through nvJitLink (ptxas -O3 inside).  Returns "" on success or the log.
std::string compile_ptx(const std::string &ptx, std::vector<char> &cubin) {
    nvJitLinkHandle h;
    const char *opts[] = {"-arch=sm_100a", "-O3"};
    if (nvJitLinkCreate(&h, 2, opts) != NVJITLINK_SUCCESS) return "nvJitLinkCreate failed";
    std::string err;
    if (nvJitLinkAddData(h, NVJITLINK_INPUT_PTX, ptx.data(), ptx.size(), "sfjit.ptx") != NVJITLINK_SUCCESS ||
        nvJitLinkComplete(h) != NVJITLINK_SUCCESS) {
        size_t n = 0;
        nvJitLinkGetErrorLogSize(h, &n);
        err.resize(n + 1);
        nvJitLinkGetErrorLog(h, &err[0]);
        if (err.empty() || err[0] == 0) err = "nvJitLink failed";
    } else {
        size_t n = 0;
        nvJitLinkGetLinkedCubinSize(h, &n);
        cubin.resize(n);
        nvJitLinkGetLinkedCubin(h, cubin.data());
    }
    nvJitLinkDestroy(&h);
    return err;
}

struct Group {
    std::vector<char> cubin;
    std::string err;
    bool cached = false;
    double seconds = 0;
    CUmodule mod = nullptr;
    CUfunction fn = nullptr;
    int regs = 0;
};

// Filters per group from the bank's density: 48 (measured best at 90 % zeros on the
// VGG16 stack), 64 for banks at <= 7 % density when that plan still runs >= 10 warps per
// CTA -- at 95 % zeros a 48-filter channel block is ~21 FFMA2 against the same 12 patch
// loads, and 64 filters measured L1/L3 -21 %, L5 -9 %, L10 -8 % (L7-L9 fall to 7 warps
// and keep 48).  An explicit KT (flags, FSCNN_SFJIT_KT) wins.
int pick_flags(const float *wt, int c, int k, int h, int w, int relu, int pool, int flags) {
    if ((flags & 0xff) || getenv("FSCNN_SFJIT_KT")) return flags;
    const int64_t n = (int64_t)k * c * 9;
    int64_t nnz = 0;
    for (int64_t i = 0; i < n; ++i) nnz += wt[i] != 0.0f;
    if (nnz * 100 > n * 7 || k <= 48) return flags;
    Plan p;
    char why[160];
    if (make_plan(p, c, k, h, w, relu, pool, flags | 64, why, sizeof(why)) && p.WARPS >= 10) return flags | 64;
    return flags;
}

}  // namespace
}  // namespace fscnn

struct fscnn_sfjit {
    fscnn::Plan plan;
    // side streams + events for the concurrent group launches (created at first launch,
    // on the launching device)
    // per caller stream: that stream's own side streams + events (callers on different
    // streams -- the engine's batch parts -- must not share side streams, or their group
    // launches would serialise behind each other, in a captured graph too)
    struct Side {
        std::vector<cudaStream_t> streams;
        std::vector<cudaEvent_t> done;
        cudaEvent_t fork = nullptr;
    };
    std::vector<std::pair<cudaStream_t, Side>> sides;
    // the last input's tensor map (encoding one costs ~1 us of host time per launch)
    const float *map_x = nullptr;
    int map_n = 0, map_ldi = 0;
    CUtensorMap map;
    std::vector<fscnn::Group> groups;
    std::mutex mu;
    std::condition_variable cv;
    int pending = 0;
    bool loaded = false;
    std::string err;
    double gen_seconds = 0;
};

using namespace fscnn;

extern "C" {

int fscnn_sfjit_create(const float *w_kc33, const float *bias, int k, int c, int h, int w, int relu, int pool,
                       int flags, fscnn_sfjit **out) {
    FSCNN_REQUIRE(out && w_kc33, "null argument");
    FSCNN_REQUIRE(k > 0 && c > 0 && h > 0 && w > 0, "bad extents");
    auto j = std::make_unique<fscnn_sfjit>();
    char why[160];
    flags = pick_flags(w_kc33, c, k, h, w, relu, pool, flags);
    if (!make_plan(j->plan, c, k, h, w, relu, pool, flags, why, sizeof(why))) {
        set_error("sfjit: %s", why);
        return FSCNN_ERR_UNSUPPORTED;
    }
    const Plan &p = j->plan;
    const int n_jobs = p.fused ? 1 : p.n_groups;
    j->groups.resize(n_jobs);
    j->pending = n_jobs;
    const auto t0 = std::chrono::steady_clock::now();
    // weights are copied for the background generators (the caller's buffers may go away)
    auto wt = std::make_shared<std::vector<float>>(w_kc33, w_kc33 + (int64_t)k * c * 9);
    auto bs = std::make_shared<std::vector<float>>();
    if (bias) bs->assign(bias, bias + k);
    const std::string dir = cache_dir();
    const bool use_cache = !(getenv("FSCNN_JIT_CACHE") && std::string(getenv("FSCNN_JIT_CACHE")) == "off");
    fscnn_sfjit *raw = j.get();
    for (int g = 0; g < n_jobs; ++g) {
        Pool::get().submit([raw, g, wt, bs, dir, use_cache] {
            Group &G = raw->groups[g];
            const auto s0 = std::chrono::steady_clock::now();
            const Plan &pl = raw->plan;
            const std::string ptx = pl.fused ? gen_kernel(pl, wt->data(), bs->empty() ? nullptr : bs->data(), 0,
                                                          pl.n_groups)
                                             : gen_group(pl, wt->data(), bs->empty() ? nullptr : bs->data(), g);
            char name[64];
            snprintf(name, sizeof(name), "/%016llx.cubin", (unsigned long long)fnv1a(ptx));
            const std::string path = dir + name;
            bool hit = false;
            if (use_cache) {
                std::ifstream f(path, std::ios::binary);
                if (f) {
                    G.cubin.assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
                    hit = G.cubin.size() > 64;
                }
            }
            if (!hit) {
                G.err = compile_ptx(ptx, G.cubin);
                if (G.err.empty() && use_cache) {
                    mkdirs(dir);
                    const std::string tmp = path + ".tmp" + std::to_string(getpid()) + "_" + std::to_string(g);
                    std::ofstream f(tmp, std::ios::binary);
                    f.write(G.cubin.data(), (std::streamsize)G.cubin.size());
                    f.close();
                    rename(tmp.c_str(), path.c_str());
                }
            }
            G.cached = hit;
            G.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - s0).count();
            std::lock_guard<std::mutex> lk(raw->mu);
            if (--raw->pending == 0) raw->cv.notify_all();
        });
    }
    j->gen_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = j.release();
    return FSCNN_OK;
}

// Join the compile jobs (no GPU needed): FSCNN_OK when every group compiled.
int fscnn_sfjit_compiled(fscnn_sfjit *j) {
    FSCNN_REQUIRE(j, "null handle");
    {
        std::unique_lock<std::mutex> lk(j->mu);
        j->cv.wait(lk, [j] { return j->pending == 0; });
    }
    for (size_t g = 0; g < j->groups.size() && j->err.empty(); ++g)
        if (!j->groups[g].err.empty())
            j->err = "sfjit compile (group " + std::to_string(g) + "): " + j->groups[g].err.substr(0, 400);
    if (!j->err.empty()) {
        set_error("%s", j->err.c_str());
        return FSCNN_ERR_CUDA;
    }
    return FSCNN_OK;
}

// Wait for the compile jobs and load the modules into the current context.
int fscnn_sfjit_wait(fscnn_sfjit *j) {
    int st = fscnn_sfjit_compiled(j);
    if (st != FSCNN_OK || j->loaded) return st;
    const Driver &d = driver();
    if (!d.ok) {
        set_error("sfjit: CUDA driver entry points unavailable (no GPU?)");
        return FSCNN_ERR_CUDA;
    }
    cudaFree(0);  // make the runtime's primary context current for the module loads
    for (size_t g = 0; g < j->groups.size(); ++g) {
        Group &G = j->groups[g];
        CUresult r = d.moduleLoadData(&G.mod, G.cubin.data());
        if (r == CUDA_SUCCESS) r = d.moduleGetFunction(&G.fn, G.mod, "sfjit");
        if (r == CUDA_SUCCESS)
            r = d.funcSetAttribute(G.fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)j->plan.smem_bytes);
        if (r == CUDA_SUCCESS) d.funcGetAttribute(&G.regs, CU_FUNC_ATTRIBUTE_NUM_REGS, G.fn);
        if (r != CUDA_SUCCESS) {
            j->err = std::string("sfjit module load: ") + cu_err(r);
            set_error("%s", j->err.c_str());
            return FSCNN_ERR_CUDA;
        }
        std::vector<char>().swap(G.cubin);
    }
    j->loaded = true;
    return FSCNN_OK;
}

// x: halo-column input [n][c][h][ldi] (logical column j at memory column j+1, column 0
// zero, ldi >= w+1 and a multiple of 4, 16-byte aligned); y: halo-column output
// [n][k][h'][ldo] (h' = h/2, w' = w/2 with the fused pool; columns 0 and > w' untouched).
int fscnn_sfjit_launch(fscnn_sfjit *j, const float *x, int n, int ldi, float *y, int ldo, void *stream) {
    FSCNN_REQUIRE(j && x && y, "null argument");
    int st = fscnn_sfjit_wait(j);
    if (st != FSCNN_OK) return st;
    const Plan &p = j->plan;
    FSCNN_REQUIRE(n > 0, "bad batch");
    FSCNN_REQUIRE(ldi >= p.W + 1 && ldi % 4 == 0, "input row pitch must be >= w + 1 and a multiple of 4");
    FSCNN_REQUIRE(ldo >= (p.pool ? p.W / 2 : p.W) + 1, "output row pitch too small");
    FSCNN_REQUIRE((reinterpret_cast<uintptr_t>(x) & 15) == 0, "input must be 16-byte aligned");
    FSCNN_REQUIRE((int64_t)n * p.M < (1ll << 31), "batch too large");
    const Driver &d = driver();
    CUresult r = CUDA_SUCCESS;
    if (x != j->map_x || n != j->map_n || ldi != j->map_ldi) {
        cuuint64_t gdim[4] = {(cuuint64_t)p.W + 1, (cuuint64_t)p.H, (cuuint64_t)p.C, (cuuint64_t)n};
        cuuint64_t gstride[3] = {(cuuint64_t)ldi * 4, (cuuint64_t)ldi * p.H * 4, (cuuint64_t)ldi * p.H * p.C * 4};
        cuuint32_t box[4] = {(cuuint32_t)p.P, (cuuint32_t)p.BH, (cuuint32_t)(p.CC / p.tma_split), (cuuint32_t)(p.tma_merge ? p.NB : 1)};
        cuuint32_t es[4] = {1, 1, 1, 1};
        r = d.encodeTiled(&j->map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(x), gdim, gstride, box,
                          es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            j->map_x = nullptr;
            set_error("sfjit: cuTensorMapEncodeTiled failed (%s)", cu_err(r));
            return FSCNN_ERR_CUDA;
        }
        j->map_x = x, j->map_n = n, j->map_ldi = ldi;
    }
    CUtensorMap &map = j->map;
    const unsigned grid = p.MODE == 0 ? (unsigned)(n * p.M) : (unsigned)((n + p.Q - 1) / p.Q);
    uint32_t ldo_u = (uint32_t)ldo, nt_u = (uint32_t)n;
    // The groups are independent kernels over the same input: fork them over side
    // streams so they share the GPU (one group's grid alone leaves SMs idle on the deep
    // layers), join back on the caller's stream.  Stream-ordered and graph-capturable.
    cudaStream_t cs = as_stream(stream);
    if (p.fused) {
        float *yg = y;
        void *args[] = {&map, &yg, &ldo_u, &nt_u};
        r = d.launchKernel(j->groups[0].fn, grid, (unsigned)p.n_groups, 1, (unsigned)p.T, 1, 1,
                           (unsigned)p.smem_bytes, reinterpret_cast<CUstream>(stream), args, nullptr);
        if (r != CUDA_SUCCESS) {
            set_error("sfjit launch: %s", cu_err(r));
            return FSCNN_ERR_CUDA;
        }
        note_launch(1);
        return FSCNN_OK;
    }
    static const int max_side = getenv("FSCNN_SFJIT_STREAMS") ? atoi(getenv("FSCNN_SFJIT_STREAMS")) : 16;
    const int n_side = (int)std::min<size_t>(j->groups.size(), (size_t)std::max(1, max_side));
    fscnn_sfjit::Side *sd = nullptr;
    for (auto &e : j->sides)
        if (e.first == cs) sd = &e.second;
    if (!sd) {
        j->sides.emplace_back(cs, fscnn_sfjit::Side());
        sd = &j->sides.back().second;
    }
    if (n_side > 1 && (int)sd->streams.size() < n_side) {
        if (!sd->fork && cudaEventCreateWithFlags(&sd->fork, cudaEventDisableTiming) != cudaSuccess) {
            set_error("sfjit: event creation failed");
            return FSCNN_ERR_CUDA;
        }
        while ((int)sd->streams.size() < n_side) {
            cudaStream_t s2;
            cudaEvent_t e2;
            // highest priority: the groups of a layer go before other queued work
            int lo_pri = 0, hi_pri = 0;
            cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri);
            if (cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, hi_pri) != cudaSuccess ||
                cudaEventCreateWithFlags(&e2, cudaEventDisableTiming) != cudaSuccess) {
                set_error("sfjit: stream creation failed");
                return FSCNN_ERR_CUDA;
            }
            sd->streams.push_back(s2);
            sd->done.push_back(e2);
        }
    }
    if (n_side > 1) {
        cudaEventRecord(sd->fork, cs);
        for (int i = 0; i < n_side; ++i) cudaStreamWaitEvent(sd->streams[i], sd->fork, 0);
    }
    // FSCNN_SFJIT_DEBUG=d > 0 (wrong results): launch g runs group g % d's code --
    // isolates the cost of the per-layer code footprint
    static const int dbg = getenv("FSCNN_SFJIT_DEBUG") ? atoi(getenv("FSCNN_SFJIT_DEBUG")) : 0;
    for (size_t g = 0; g < j->groups.size(); ++g) {
        float *yg = y;  // each group's kernel offsets by its first filter itself
        void *args[] = {&map, &yg, &ldo_u, &nt_u};
        cudaStream_t sg = n_side > 1 ? sd->streams[g % n_side] : cs;
        r = d.launchKernel(j->groups[dbg > 0 ? g % dbg : g].fn, grid, 1, 1, (unsigned)p.T, 1, 1, (unsigned)p.smem_bytes,
                           reinterpret_cast<CUstream>(sg), args, nullptr);
        if (r != CUDA_SUCCESS) {
            set_error("sfjit launch: %s", cu_err(r));
            return FSCNN_ERR_CUDA;
        }
        note_launch(1);
    }
    if (n_side > 1) {
        for (int i = 0; i < n_side; ++i) {
            cudaEventRecord(sd->done[i], sd->streams[i]);
            cudaStreamWaitEvent(cs, sd->done[i], 0);
        }
    }
    return FSCNN_OK;
}

// info[0..11]: groups, CTAs per image (part mode) or -images per CTA, warps,
// filters per group, channels per chunk, stages, smem bytes, box rows, row pitch,
// boxes per CTA, max registers, cached groups (filled after wait);
// secs[0..1]: generation seconds (submit), summed compile seconds over groups.
int fscnn_sfjit_info(fscnn_sfjit *j, int64_t *info, double *secs) {
    FSCNN_REQUIRE(j && info, "null argument");
    int st = fscnn_sfjit_compiled(j);
    if (st != FSCNN_OK) return st;
    const Plan &p = j->plan;
    int regs = 0, cached = 0;
    double cs = 0;
    for (auto &G : j->groups) {
        regs = std::max(regs, G.regs);
        cached += G.cached;
        cs += G.seconds;
    }
    int64_t v[12] = {p.n_groups, p.MODE == 0 ? p.M : -p.Q, p.WARPS, p.KT, p.CC, p.S, p.smem_bytes,
                     p.BH, p.P, p.NB, regs, cached};
    memcpy(info, v, sizeof(v));
    if (secs) {
        secs[0] = j->gen_seconds;
        secs[1] = cs;
    }
    return FSCNN_OK;
}

// The generated PTX of one group (for inspection and the CPU tests): returns its length
// (without the terminator); copies it into buf when cap > length.
int64_t fscnn_sfjit_ptx(const float *w_kc33, const float *bias, int k, int c, int h, int w, int relu, int pool,
                        int flags, int group, char *buf, int64_t cap) {
    if (!w_kc33 || k <= 0 || c <= 0) return -1;
    Plan p;
    char why[160];
    flags = pick_flags(w_kc33, c, k, h, w, relu, pool, flags);
    if (!make_plan(p, c, k, h, w, relu, pool, flags, why, sizeof(why))) {
        set_error("sfjit: %s", why);
        return -1;
    }
    if (group < 0 || group >= p.n_groups) return -1;
    const std::string s = gen_group(p, w_kc33, bias, group);
    if (buf && cap > (int64_t)s.size()) memcpy(buf, s.c_str(), s.size() + 1);
    return (int64_t)s.size();
}

void fscnn_sfjit_destroy(fscnn_sfjit *j) {
    if (!j) return;
    {
        std::unique_lock<std::mutex> lk(j->mu);
        j->cv.wait(lk, [j] { return j->pending == 0; });
    }
    for (auto &G : j->groups)
        if (G.mod && driver().moduleUnload) driver().moduleUnload(G.mod);
    for (auto &e : j->sides) {
        for (auto s2 : e.second.streams) cudaStreamDestroy(s2);
        for (auto e2 : e.second.done) cudaEventDestroy(e2);
        if (e.second.fork) cudaEventDestroy(e.second.fork);
    }
    delete j;
}

}  // extern "C"
