// api.cu -- the C ABI (include/fvv_b200.h): validation with the reference's
// error classes, workspace planning, recursion-stage scheduling.  No host
// synchronisation and no allocation after fvv_engine_create.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "fvv_device.cuh"
#include "conv_tc.h"
#include "vinet.h"
#include "refine.h"
#include "encode.h"
#include "deflate.h"
#include "literal.h"

namespace fvv {
extern thread_local int g_failed_class;
cudaError_t run_interp_stage(const Geometry& g, const PairTable& pt, uint8_t* ws, const Planes& P,
                             const int16_t* const* rank_of, const int16_t* const* cand_of_rank,
                             int npairs, double* mask_out, Prof* prof, cudaStream_t st);
cudaError_t run_diag(const Geometry& g, const PairTable& pt, uint8_t* ws, const Planes& P, int pair,
                     float* flow_lr, float* flow_rl, double* mask, cudaStream_t st);
cudaError_t run_level_diag(const Geometry& g, uint8_t* ws, const Planes& P, int pair, int level,
                           float* flow_lr, float* flow_rl, double* err_lr, double* err_rl,
                           cudaStream_t st);
size_t level_mask_scratch_bytes(const Geometry& g, int level);
cudaError_t run_direct_state(const Geometry& g, uint8_t* ws, const Planes& P, int pair, const double* mask,
                             float* state, cudaStream_t st);
cudaError_t run_level_mask(const Geometry& g, uint8_t* ws, const Planes& P, int pair, int level, void* scratch,
                           double* mask, double* blend, const LDiagSrc& src, cudaStream_t st);
cudaError_t launch_downscale(int W, int H, int fmt, const uint8_t* frames, int n, int f,
                             uint8_t* out, cudaStream_t st);
cudaError_t launch_assemble(int W, int H, int fmt, const uint8_t* anchor,
                            const uint8_t* const* smalls, int nsmall, int sw, uint8_t* out,
                            cudaStream_t st);
cudaError_t launch_rig_clusters(int W, int H, int fmt, const ClusterJob* jobs, int njobs,
                                long max_cluster_bytes, const uint8_t* views, uint8_t* out,
                                cudaStream_t st, int skip_period = 0);
cudaError_t launch_rig_clusters_src(int W, int H, int fmt, const ClusterJob* jobs, int njobs,
                                    long max_cluster_bytes, const ViewSrc& vs, uint8_t* out,
                                    cudaStream_t st, int skip_period);
}  // namespace fvv

using namespace fvv;

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* where) {
    return fail(FVV_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

size_t align_up(size_t v, size_t a = 256) { return (v + a - 1) / a * a; }

bool pow2_block(int b) { return b == 2 || b == 4 || b == 8; }

int check_desc(const fvv_frame_desc* d) {
    if (!d) return fail(FVV_EINVAL, "null frame descriptor");
    if (d->width <= 0 || d->height <= 0)
        return fail(FVV_EINVAL, "bad frame size " + std::to_string(d->width) + "x" +
                                    std::to_string(d->height));
    if (d->format < FVV_GRAY8 || d->format > FVV_RGB8)
        return fail(FVV_EINVAL, "unknown pixel format " + std::to_string(d->format));
    return FVV_OK;
}

// Tie-rule order of flow.py:57-66: lexsort((dx, dy, |dy|, dx^2+dy^2))
void candidate_tables(int r, std::vector<int16_t>& rank_of, std::vector<int16_t>& cand_of_rank) {
    const int side = 2 * r + 1, n = side * side;
    std::vector<int> idx(n);
    for (int i = 0; i < n; i++) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
        int ady = a / side - r, adx = a % side - r, bdy = b / side - r, bdx = b % side - r;
        int da = adx * adx + ady * ady, db = bdx * bdx + bdy * bdy;
        if (da != db) return da < db;
        if (std::abs(ady) != std::abs(bdy)) return std::abs(ady) < std::abs(bdy);
        if (ady != bdy) return ady < bdy;
        return adx < bdx;
    });
    rank_of.assign(n, 0);
    cand_of_rank.assign(n, 0);
    for (int k = 0; k < n; k++) {
        cand_of_rank[k] = (int16_t)idx[k];
        rank_of[idx[k]] = (int16_t)k;
    }
}

void make_geometry(const fvv_frame_desc* d, const fvv_interp_params* p, Geometry* g) {
    g->W = d->width;
    g->H = d->height;
    g->fmt = d->format;
    g->cw = (d->width + 1) / 2;
    g->ch = (d->height + 1) / 2;
    fvv_frame_desc dd = *d;
    g->frame_bytes = (long)fvv_frame_bytes(&dd);
    for (int s = 0; s < 3; s++) {
        const int f = s == 0 ? 4 : (s == 1 ? 2 : 1);
        Level& L = g->lv[s];
        L.w = d->width / f;
        L.h = d->height / f;
        L.block = p->block_size[s];
        L.r = p->search_radius[s];
        L.nbx = (L.w + L.block - 1) / L.block;
        L.nby = (L.h + L.block - 1) / L.block;
    }
    g->eps = p->mask_epsilon;
    g->eps2 = 2.0 * p->mask_epsilon;
    g->fastdiv = p->mask_epsilon >= 1e-30 && p->mask_epsilon <= 1e30;
    // exact fixed-point units (fvv_device.cuh)
    for (int s = 0; s < 3; s++) {
        int lb = 0;
        while ((1 << lb) < 2 * p->block_size[s]) lb++;
        g->rb[s] = 2 * lb;
    }
    g->fb[0] = g->rb[0];
    g->fb[1] = std::max(g->fb[0] + 3, g->rb[1]);
    g->fb[2] = std::max(g->fb[1] + 3, g->rb[2]);
    g->qmargin[0] = 0;
    g->qmargin[1] = 2 * p->search_radius[0];
    g->qmargin[2] = 4 * p->search_radius[0] + 2 * p->search_radius[1];
    {
        const int span = 4 * p->search_radius[0] + 2 * p->search_radius[1] + p->search_radius[2];
        g->mmargin = (span + 1) / 2 + 1;
        g->cmargin = (span + 3) / 4 + 1;
    }
    g->scan_coop_min = kScanCoopMinDefault;
    g->sadw_rb_min_ctas = kSadwRbMinCtasDefault;
    g->mask_cols2 = FVV_MASK_COLS2;
    g->pdl = FVV_PDL;
    g->mh = 64;  // the mask walker band height; run_interp picks it per launch
}

// workspace = [header: candidate tables][pair slot 0][pair slot 1]...
struct Layout {
    size_t header;
    size_t tab_off[3][2];
    Planes P;
};

Layout make_layout(const Geometry& g) {
    Layout lay{};
    size_t off = 0;
    for (int s = 0; s < 3; s++) {
        const int side = 2 * g.lv[s].r + 1;
        for (int k = 0; k < 2; k++) {
            lay.tab_off[s][k] = off;
            off = align_up(off + (size_t)side * side * 2);
        }
    }
    lay.header = off;
    Planes& P = lay.P;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes); return r; };
    const size_t W = g.W, H = g.H;
    const size_t n0 = (size_t)g.lv[0].w * g.lv[0].h, n1 = (size_t)g.lv[1].w * g.lv[1].h;
    const size_t n2 = W * H;
    for (int s = 0; s < 2; s++) {
        P.luma[s] = g.fmt == FVV_RGB8 ? take(n2) : 0;
        P.s4[s] = take(n1 * 2);
        P.s16[s] = take(n0 * 2);
        P.q0[s] = take(n0 * 2);
    }
    for (int d = 0; d < 2; d++) {
        for (int s = 0; s < 3; s++)
            P.hit[s][d] = take((size_t)g.lv[s].nbx * g.lv[s].nby * sizeof(BlockHit));
        P.flow0[d] = take(n0 * 8);
        P.flow1[d] = take(n1 * 8);
        P.tq1[d] = take(n1 * 2);
        P.tq2[d] = take(n2 * 2);
    }
    P.sd = take(n2 * 2);
    P.occ_l = take(n2 * 4);
    P.occ_r = take(n2 * 4);
    P.wl = take(n2);
    P.wr = take(n2);
    P.wc = g.fmt == FVV_YUV420 ? take((size_t)g.cw * g.ch * 4) : 0;
    P.wrgb = g.fmt == FVV_RGB8 ? take(n2 * 6) : 0;
    P.carry = take((size_t)H * ((W + 7) / 8) * 8);
    P.stride = align_up(o, 4096);
    return lay;
}
}  // namespace

struct fvv_engine {
    Geometry g;
    bool literal = false;  // outside the fixed-point domain: literal_kernels.cu, one pair at a time
    LitLayout lit{};
    int block[3], radius[3];
    Layout lay;
    Planes P;  // plane offsets relative to the first pair slot
    uint8_t* ws;
    uint8_t* slots;
    int max_pairs;
    const int16_t* rank_of[3];
    const int16_t* cand_of_rank[3];
    PairTable last;  // frame pointers of the most recent batch (diagnostics)
    int last_npairs;
    Prof prof;
    bool profiling = false;
    ~fvv_engine() { free_prof(); }
    void free_prof() {
        for (int i = 0; i < 2 * prof.capacity; i++) cudaEventDestroy(prof.ev[i]);
        delete[] prof.ev;
        delete[] prof.cls;
        prof = Prof();
        profiling = false;
    }
};

extern "C" {

const char* fvv_last_error(void) { return g_err.c_str(); }

const char* fvv_build_info(void) {
    return "fvv_b200: sm_100a, integer SAD (u16x2 VIMNMX), literal-f64 warps, "
           "scipy running-sum replay";
}

size_t fvv_frame_bytes(const fvv_frame_desc* d) {
    if (!d || d->width <= 0 || d->height <= 0) return 0;
    const size_t w = d->width, h = d->height;
    if (d->format == FVV_GRAY8) return w * h;
    if (d->format == FVV_RGB8) return w * h * 3;
    return w * h + 2 * ((w + 1) / 2) * ((h + 1) / 2);
}

int fvv_validate_params(const fvv_interp_params* p) {
    if (!p) return fail(FVV_EINVAL, "null params");
    int mb = std::min(std::min(p->block_size[0], p->block_size[1]), p->block_size[2]);
    int mr = std::min(std::min(p->search_radius[0], p->search_radius[1]), p->search_radius[2]);
    if (mb < 2 || mr < 1) return fail(FVV_EINVAL, "degenerate block size or search radius");
    if (!(p->mask_epsilon > 0.0))
        return fail(FVV_EUNSUPPORTED, "mask_epsilon must be positive on the B200 path");
    return FVV_OK;
}

// The fixed-point fast path's domain: power-of-two blocks make
// every flow value a dyadic rational; max_span <= 120 keeps the 32-bit
// coordinates.  Anything else the reference accepts runs the literal path
// (literal_kernels.cu), same results, no speed claim.
static bool fast_domain(const fvv_interp_params* p) {
    for (int s = 0; s < 3; s++)
        if (!pow2_block(p->block_size[s])) return false;
    return 4 * p->search_radius[0] + 2 * p->search_radius[1] + p->search_radius[2] <= 120;
}

static int check_interp_desc(const fvv_frame_desc* d) {
    int rc = check_desc(d);
    if (rc) return rc;
    if (d->width % 4 || d->height % 4)
        return fail(FVV_EINVAL, "frame dimensions must be divisible by 4 for the 3-scale pyramid");
    if (d->width > 8192 || d->height > 8192)
        return fail(FVV_EUNSUPPORTED, "frames wider or taller than 8192 px are outside the B200 path "
                                      "(32-bit fixed-point coordinates)");
    return FVV_OK;
}

size_t fvv_engine_workspace_size(const fvv_frame_desc* d, const fvv_interp_params* p,
                                 int max_pairs) {
    if (check_interp_desc(d) || fvv_validate_params(p) || max_pairs < 1) return 0;
    Geometry g;
    make_geometry(d, p, &g);
    Layout lay = make_layout(g);
    if (!fast_domain(p)) return lay.header + lit_layout(d->width, d->height, d->format, p->block_size).bytes;
    return lay.header + lay.P.stride * (size_t)max_pairs;
}

int fvv_engine_create(const fvv_frame_desc* d, const fvv_interp_params* p, int max_pairs,
                      void* workspace, size_t workspace_bytes, fvv_engine** out) {
    int rc;
    if ((rc = check_interp_desc(d))) return rc;
    if ((rc = fvv_validate_params(p))) return rc;
    if (max_pairs < 1) return fail(FVV_EINVAL, "max_pairs must be >= 1");
    if (!out) return fail(FVV_EINVAL, "null engine out-pointer");
    const size_t need = fvv_engine_workspace_size(d, p, max_pairs);
    if (!workspace || workspace_bytes < need)
        return fail(FVV_EINVAL, "workspace too small: need " + std::to_string(need) + " bytes");
    fvv_engine* e = new fvv_engine();
    make_geometry(d, p, &e->g);
    e->lay = make_layout(e->g);
    e->P = e->lay.P;
    e->ws = static_cast<uint8_t*>(workspace);
    e->slots = e->ws + e->lay.header;
    e->max_pairs = max_pairs;
    e->last_npairs = 0;
    e->literal = !fast_domain(p);
    for (int s = 0; s < 3; s++) { e->block[s] = p->block_size[s]; e->radius[s] = p->search_radius[s]; }
    if (e->literal) e->lit = lit_layout(d->width, d->height, d->format, p->block_size);
    for (int s = 0; s < 3; s++) {
        std::vector<int16_t> ro, cr;
        candidate_tables(e->g.lv[s].r, ro, cr);
        cudaError_t ce = cudaMemcpy(e->ws + e->lay.tab_off[s][0], ro.data(), ro.size() * 2,
                                    cudaMemcpyHostToDevice);
        if (ce == cudaSuccess)
            ce = cudaMemcpy(e->ws + e->lay.tab_off[s][1], cr.data(), cr.size() * 2,
                            cudaMemcpyHostToDevice);
        if (ce != cudaSuccess) {
            delete e;
            return cuda_fail(ce, "fvv_engine_create: table upload");
        }
        e->rank_of[s] = reinterpret_cast<const int16_t*>(e->ws + e->lay.tab_off[s][0]);
        e->cand_of_rank[s] = reinterpret_cast<const int16_t*>(e->ws + e->lay.tab_off[s][1]);
    }
    *out = e;
    return FVV_OK;
}

void fvv_engine_destroy(fvv_engine* e) { delete e; }

int fvv_engine_max_pairs(const fvv_engine* e) { return e ? e->max_pairs : 0; }

int fvv_engine_set_tuning(fvv_engine* e, int key, int value) {
    if (!e) return fail(FVV_EINVAL, "null engine");
    switch (key) {
        case FVV_TUNE_SCAN_COOP_MIN: e->g.scan_coop_min = value < 0 ? kScanCoopMinDefault : value; break;
        case FVV_TUNE_SADW_RB_MIN_CTAS: e->g.sadw_rb_min_ctas = value < 0 ? kSadwRbMinCtasDefault : value; break;
        case FVV_TUNE_MASK_COLS2: e->g.mask_cols2 = value < 0 ? FVV_MASK_COLS2 : (value != 0); break;
        case FVV_TUNE_PDL: e->g.pdl = value < 0 ? FVV_PDL : (value != 0); break;
        default: return fail(FVV_EINVAL, "unknown tuning key " + std::to_string(key));
    }
    return FVV_OK;
}

static int run_pairs(fvv_engine* e, const uint8_t* const* L, const uint8_t* const* R,
                     uint8_t* const* O, int npairs, cudaStream_t st) {
    if (e->literal) {
        for (int i = 0; i < npairs; i++) {
            cudaError_t ce = lit_interpolate(e->lit, e->slots, e->g.W, e->g.H, e->g.fmt, e->block, e->radius,
                                             e->cand_of_rank, e->g.eps, L[i], R[i], O[i], st);
            if (ce != cudaSuccess) return cuda_fail(ce, "interpolate (literal path)");
        }
        if (npairs > 0) {
            e->last.left[0] = L[npairs - 1];
            e->last.right[0] = R[npairs - 1];
            e->last.out[0] = O[npairs - 1];
            e->last_npairs = npairs;
        }
        return FVV_OK;
    }
    for (int b = 0; b < npairs; b += std::min(e->max_pairs, kMaxPairsPerLaunch)) {
        const int n = std::min(std::min(e->max_pairs, kMaxPairsPerLaunch), npairs - b);
        PairTable pt;
        for (int i = 0; i < n; i++) {
            pt.left[i] = L[b + i];
            pt.right[i] = R[b + i];
            pt.out[i] = O[b + i];
        }
        cudaError_t ce = run_interp_stage(e->g, pt, e->slots, e->P, e->rank_of, e->cand_of_rank, n,
                                          nullptr, e->profiling ? &e->prof : nullptr, st);
        if (ce != cudaSuccess) {
            const int c = g_failed_class;
            g_failed_class = -1;
            return cuda_fail(ce, c >= 0 ? (std::string("interpolate (") + fvv_kernel_class_name(c) + ")").c_str()
                                        : "interpolate");
        }
        e->last = pt;
        e->last_npairs = n;
    }
    return FVV_OK;
}

int fvv_profile_enable(fvv_engine* e, int capacity) {
    if (!e) return fail(FVV_EINVAL, "null engine");
    e->free_prof();
    if (capacity <= 0) return FVV_OK;
    e->prof.ev = new cudaEvent_t[2 * capacity];
    e->prof.cls = new int[capacity];
    for (int i = 0; i < 2 * capacity; i++) {
        cudaError_t ce = cudaEventCreate(&e->prof.ev[i]);
        if (ce != cudaSuccess) {
            e->prof.capacity = i / 2;
            e->free_prof();
            return cuda_fail(ce, "fvv_profile_enable");
        }
    }
    e->prof.capacity = capacity;
    e->prof.n = 0;
    e->profiling = true;
    return FVV_OK;
}

int fvv_profile_read(fvv_engine* e, double* ms, int* launches, int nclasses) {
    if (!e || !ms || !launches) return fail(FVV_EINVAL, "null argument");
    for (int c = 0; c < nclasses; c++) { ms[c] = 0.0; launches[c] = 0; }
    for (int i = 0; i < e->prof.n; i++) {
        cudaError_t ce = cudaEventSynchronize(e->prof.ev[2 * i + 1]);
        if (ce != cudaSuccess) return cuda_fail(ce, "fvv_profile_read");
        float t = 0.f;
        ce = cudaEventElapsedTime(&t, e->prof.ev[2 * i], e->prof.ev[2 * i + 1]);
        if (ce != cudaSuccess) return cuda_fail(ce, "fvv_profile_read");
        const int c = e->prof.cls[i];
        if (c < nclasses) { ms[c] += t; launches[c] += 1; }
    }
    e->prof.n = 0;
    return FVV_OK;
}

const char* fvv_kernel_class_name(int c) {
    static const char* names[KC_COUNT] = {"k_pyramid", "k_sad<0>", "k_flow<0>", "k_warpq<1>",
                                          "k_sad<1>", "k_flow<1>", "k_warpq<2>", "k_sad<2>",
                                          "k_mask_cols", "k_scan_carry", "k_blend"};
    return c >= 0 && c < KC_COUNT ? names[c] : "";
}

int fvv_interpolate_pairs(fvv_engine* e, const uint8_t* const* left, const uint8_t* const* right,
                          uint8_t* const* out, int npairs, void* stream) {
    if (!e) return fail(FVV_EINVAL, "null engine");
    if (npairs < 0) return fail(FVV_EINVAL, "npairs < 0");
    if (npairs == 0) return FVV_OK;
    if (!left || !right || !out) return fail(FVV_EINVAL, "null pointer table");
    return run_pairs(e, left, right, out, npairs, static_cast<cudaStream_t>(stream));
}

static int lit_pair_check(const fvv_engine* e, int pair) {
    if (pair != e->last_npairs - 1)
        return fail(FVV_EINVAL, "the literal path (non power-of-two blocks / max_span > 120) keeps the diagnostics "
                                "of the last pair of a batch only");
    return FVV_OK;
}

int fvv_interp_diagnostics(fvv_engine* e, int pair, float* flow_lr, float* flow_rl, double* mask,
                           void* stream) {
    if (!e) return fail(FVV_EINVAL, "null engine");
    if (pair < 0 || pair >= e->last_npairs)
        return fail(FVV_EINVAL, "no such pair in the most recent batch");
    if (e->literal) {
        int rc = lit_pair_check(e, pair);
        if (rc) return rc;
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const size_t n = (size_t)e->g.W * e->g.H;
        cudaError_t ce = cudaSuccess;
        if (flow_lr) ce = cudaMemcpyAsync(flow_lr, e->slots + e->lit.flow[2][0], n * 8, cudaMemcpyDeviceToDevice, st);
        if (ce == cudaSuccess && flow_rl)
            ce = cudaMemcpyAsync(flow_rl, e->slots + e->lit.flow[2][1], n * 8, cudaMemcpyDeviceToDevice, st);
        if (ce == cudaSuccess && mask) ce = cudaMemcpyAsync(mask, e->slots + e->lit.mask, n * 8, cudaMemcpyDeviceToDevice, st);
        return ce == cudaSuccess ? FVV_OK : cuda_fail(ce, "diagnostics (literal path)");
    }
    cudaError_t ce = run_diag(e->g, e->last, e->slots, e->P, pair, flow_lr, flow_rl, mask,
                              static_cast<cudaStream_t>(stream));
    if (ce != cudaSuccess) return cuda_fail(ce, "diagnostics");
    return FVV_OK;
}

int fvv_interp_level_diagnostics(fvv_engine* e, int pair, int level, float* flow_lr, float* flow_rl,
                                 double* err_lr, double* err_rl, void* stream) {
    if (!e) return fail(FVV_EINVAL, "null engine");
    if (pair < 0 || pair >= e->last_npairs)
        return fail(FVV_EINVAL, "no such pair in the most recent batch");
    if (level < 0 || level > 2) return fail(FVV_EINVAL, "level must be 0, 1 or 2");
    if (e->literal) {
        int rc = lit_pair_check(e, pair);
        if (rc) return rc;
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const Level& L = e->g.lv[level];
        const size_t n = (size_t)L.w * L.h;
        cudaError_t ce = cudaSuccess;
        if (flow_lr) ce = cudaMemcpyAsync(flow_lr, e->slots + e->lit.flow[level][0], n * 8, cudaMemcpyDeviceToDevice, st);
        if (ce == cudaSuccess && flow_rl)
            ce = cudaMemcpyAsync(flow_rl, e->slots + e->lit.flow[level][1], n * 8, cudaMemcpyDeviceToDevice, st);
        if (ce == cudaSuccess && err_lr) ce = lit_level_err(e->lit, e->slots, e->g.W, e->g.H, e->block, level, 0, err_lr, st);
        if (ce == cudaSuccess && err_rl) ce = lit_level_err(e->lit, e->slots, e->g.W, e->g.H, e->block, level, 1, err_rl, st);
        return ce == cudaSuccess ? FVV_OK : cuda_fail(ce, "level diagnostics (literal path)");
    }
    cudaError_t ce = run_level_diag(e->g, e->slots, e->P, pair, level, flow_lr, flow_rl, err_lr, err_rl,
                                    static_cast<cudaStream_t>(stream));
    if (ce != cudaSuccess) return cuda_fail(ce, "level diagnostics");
    return FVV_OK;
}

size_t fvv_interp_level_mask_scratch(const fvv_engine* e, int level) {
    if (!e || level < 0 || level > 1) return 0;
    return level_mask_scratch_bytes(e->g, level);
}

int fvv_interp_level_mask(fvv_engine* e, int pair, int level, void* scratch, size_t scratch_bytes, double* mask,
                          double* blend_luma, void* stream) {
    if (!e) return fail(FVV_EINVAL, "null engine");
    if (pair < 0 || pair >= e->last_npairs) return fail(FVV_EINVAL, "no such pair in the most recent batch");
    if (level < 0 || level > 1) return fail(FVV_EINVAL, "coarse-scale masks exist for levels 0 and 1");
    if (!scratch || scratch_bytes < level_mask_scratch_bytes(e->g, level) || !mask || !blend_luma)
        return fail(FVV_EINVAL, "scratch too small or null output");
    LDiagSrc src{};
    if (e->literal) {
        int rc = lit_pair_check(e, pair);
        if (rc) return rc;
        for (int side = 0; side < 2; side++) {
            src.lum[side] = reinterpret_cast<const float*>(e->slots + e->lit.lum[level][side]);
            src.flow[side] = reinterpret_cast<const float2*>(e->slots + e->lit.flow[level][side]);
        }
    }
    cudaError_t ce = run_level_mask(e->g, e->slots, e->P, e->literal ? 0 : pair, level, scratch, mask, blend_luma,
                                    src, static_cast<cudaStream_t>(stream));
    if (ce != cudaSuccess) return cuda_fail(ce, "level mask diagnostics");
    return FVV_OK;
}

// Recursive midpoints over a views array whose slot k holds position k:
// stage s interpolates between positions a and a+step for every a, writing
// a+step/2 (interp.py:163-169).  `base` points at slot 0; `nslots` = last+1.
static int run_recursion(fvv_engine* e, uint8_t* base, long stride, int nslots, int stages,
                         cudaStream_t st) {
    std::vector<const uint8_t*> L, R;
    std::vector<uint8_t*> O;
    for (int k = 1; k <= stages; k++) {
        const int step = 1 << (stages - k + 1);
        L.clear(); R.clear(); O.clear();
        for (int a = 0; a + step < nslots; a += step) {
            L.push_back(base + (long)a * stride);
            R.push_back(base + (long)(a + step) * stride);
            O.push_back(base + (long)(a + step / 2) * stride);
        }
        int rc = run_pairs(e, L.data(), R.data(), O.data(), (int)L.size(), st);
        if (rc) return rc;
    }
    return FVV_OK;
}

size_t fvv_dense_views_scratch(const fvv_engine* e, int mode) {
    if (!e) return 0;
    if (mode == FVV_DENSE_RECURSIVE) return 0;
    const size_t n = (size_t)e->g.W * e->g.H;
    return align_up(n * 5 * sizeof(float)) + align_up(n * sizeof(double)) + align_up((size_t)e->g.frame_bytes);
}

// direct-t (mode 1): ONE interpolation of (left, right) -- its output is the
// t = 1/2 view, bit-exact with interp.py:131-132 -- then every other view
// t = j / 2^stages from the same flows and mask in one synthesis pass (the
// VINet direct-t kernel: F_t->l = 2t F_m->l, F_t->r = 2(1-t) F_m->r,
// w_t = (1-t) M / ((1-t) M + t (1-M)); fp32, oracle vinet_ref.synth)
static int dense_direct(fvv_engine* e, const uint8_t* left, const uint8_t* right, int stages, uint8_t* views,
                        void* scratch, size_t scratch_bytes, cudaStream_t st) {
    if (e->literal) return fail(FVV_EUNSUPPORTED, "direct-t runs on the fixed-point path (power-of-two blocks)");
    if (!scratch || scratch_bytes < fvv_dense_views_scratch(e, FVV_DENSE_DIRECT))
        return fail(FVV_EINVAL, "direct-t needs fvv_dense_views_scratch(engine, 1) bytes of scratch");
    const size_t n = (size_t)e->g.W * e->g.H;
    float* state = static_cast<float*>(scratch);
    double* mask = reinterpret_cast<double*>(static_cast<uint8_t*>(scratch) + align_up(n * 5 * sizeof(float)));
    uint8_t* mid = static_cast<uint8_t*>(scratch) + align_up(n * 5 * sizeof(float)) + align_up(n * sizeof(double));
    PairTable pt;
    pt.left[0] = left;
    pt.right[0] = right;
    pt.out[0] = mid;
    cudaError_t ce = run_interp_stage(e->g, pt, e->slots, e->P, e->rank_of, e->cand_of_rank, 1, mask,
                                      e->profiling ? &e->prof : nullptr, st);
    if (ce != cudaSuccess) return cuda_fail(ce, "dense_views (direct-t): interpolate");
    e->last = pt;
    e->last_npairs = 1;
    if ((ce = run_direct_state(e->g, e->slots, e->P, 0, mask, state, st)) != cudaSuccess)
        return cuda_fail(ce, "dense_views (direct-t): state");
    const int nv = (1 << stages) - 1;
    VinPairs pp{};
    pp.left[0] = left;
    pp.right[0] = right;
    const size_t fb = (size_t)e->g.frame_bytes;
    if ((ce = vin_synth(pp, 1, state, e->g.fmt, e->g.W, e->g.H, nv, views, fb, (size_t)nv * fb, st)) != cudaSuccess)
        return cuda_fail(ce, "dense_views (direct-t): synthesis");
    ce = cudaMemcpyAsync(views + (size_t)(nv / 2) * fb, mid, fb, cudaMemcpyDeviceToDevice, st);
    if (ce != cudaSuccess) return cuda_fail(ce, "dense_views (direct-t): midpoint");
    return FVV_OK;
}

int fvv_dense_views(fvv_engine* e, const uint8_t* left, const uint8_t* right, int stages, int mode,
                    uint8_t* views, void* scratch, size_t scratch_bytes, void* stream) {
    if (!e) return fail(FVV_EINVAL, "null engine");
    if (stages < 1) return fail(FVV_EINVAL, "stages must be >= 1");
    if (stages > 6) return fail(FVV_EINVAL, "stages > 6 refused: 2**n - 1 views grows too fast");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (mode == FVV_DENSE_DIRECT) return dense_direct(e, left, right, stages, views, scratch, scratch_bytes, st);
    if (mode != FVV_DENSE_RECURSIVE) return fail(FVV_EINVAL, "mode must be 0 (recursive) or 1 (direct-t)");
    const long fb = e->g.frame_bytes;
    const int n = (1 << stages) - 1;
    // the recursion reads the endpoints from their own buffers: build a
    // pointer table over [left, views..., right]
    std::vector<const uint8_t*> slot(n + 2);
    slot[0] = left;
    for (int i = 0; i < n; i++) slot[i + 1] = views + (long)i * fb;
    slot[n + 1] = right;
    std::vector<const uint8_t*> L, R;
    std::vector<uint8_t*> O;
    for (int k = 1; k <= stages; k++) {
        const int step = 1 << (stages - k + 1);
        L.clear(); R.clear(); O.clear();
        for (int a = 0; a + step <= n + 1; a += step) {
            L.push_back(slot[a]);
            R.push_back(slot[a + step]);
            O.push_back(const_cast<uint8_t*>(slot[a + step / 2]));
        }
        int rc = run_pairs(e, L.data(), R.data(), O.data(), (int)L.size(), st);
        if (rc) return rc;
    }
    return FVV_OK;
}

int fvv_rig_views(fvv_engine* e, const uint8_t* cams, int ncams, int stages, uint8_t* views,
                  void* stream) {
    if (!e) return fail(FVV_EINVAL, "null engine");
    if (ncams < 2) return fail(FVV_EINVAL, "need at least 2 cameras");
    if (stages < 1 || stages > 6) return fail(FVV_EINVAL, "stages must be in 1..6");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long fb = e->g.frame_bytes;
    const int step = 1 << stages;
    for (int c = 0; c < ncams; c++) {
        cudaError_t ce = cudaMemcpyAsync(views + (long)c * step * fb, cams + (long)c * fb, fb,
                                         cudaMemcpyDeviceToDevice, st);
        if (ce != cudaSuccess) return cuda_fail(ce, "rig_views: camera copy");
    }
    return run_recursion(e, views, fb, (ncams - 1) * step + 1, stages, st);
}

size_t fvv_rig_views_scratch(const fvv_engine* e, int ncams, int mode) {
    if (!e || ncams < 2 || mode == FVV_DENSE_RECURSIVE) return 0;
    const size_t n = (size_t)e->g.W * e->g.H, np = (size_t)(ncams - 1);
    return align_up(np * n * 5 * sizeof(float)) + align_up(np * n * sizeof(double)) +
           np * align_up((size_t)e->g.frame_bytes);
}

int fvv_rig_views_mode(fvv_engine* e, const uint8_t* cams, int ncams, int stages, int mode, uint8_t* views,
                       void* scratch, size_t scratch_bytes, void* stream) {
    if (mode == FVV_DENSE_RECURSIVE) return fvv_rig_views(e, cams, ncams, stages, views, stream);
    if (!e) return fail(FVV_EINVAL, "null engine");
    if (mode != FVV_DENSE_DIRECT) return fail(FVV_EINVAL, "mode must be 0 (recursive) or 1 (direct-t)");
    if (e->literal) return fail(FVV_EUNSUPPORTED, "direct-t runs on the fixed-point path (power-of-two blocks)");
    if (ncams < 2) return fail(FVV_EINVAL, "need at least 2 cameras");
    if (stages < 1 || stages > 6) return fail(FVV_EINVAL, "stages must be in 1..6");
    const int npairs = ncams - 1;
    if (npairs > e->max_pairs || npairs > kVinMaxPairs)
        return fail(FVV_EINVAL, "direct-t rig needs max_pairs >= ncams - 1 (at most 64)");
    if (!scratch || scratch_bytes < fvv_rig_views_scratch(e, ncams, mode))
        return fail(FVV_EINVAL, "direct-t rig needs fvv_rig_views_scratch(engine, ncams, 1) bytes of scratch");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t n = (size_t)e->g.W * e->g.H, fb = (size_t)e->g.frame_bytes;
    const int step = 1 << stages, nv = step - 1;
    uint8_t* sp = static_cast<uint8_t*>(scratch);
    float* state = reinterpret_cast<float*>(sp);  // (npairs, 5, H, W): the layout vin_synth reads
    double* mask = reinterpret_cast<double*>(sp + align_up((size_t)npairs * n * 5 * sizeof(float)));
    uint8_t* mids = sp + align_up((size_t)npairs * n * 5 * sizeof(float)) + align_up((size_t)npairs * n * sizeof(double));
    const size_t sstride = 5 * n;
    for (int c = 0; c < ncams; c++) {
        cudaError_t ce = cudaMemcpyAsync(views + (size_t)c * step * fb, cams + (size_t)c * fb, fb,
                                         cudaMemcpyDeviceToDevice, st);
        if (ce != cudaSuccess) return cuda_fail(ce, "rig_views (direct-t): camera copy");
    }
    // one interpolation per gap, all gaps in one launch: the t = 1/2 views and the masks
    PairTable pt;
    for (int c = 0; c < npairs; c++) {
        pt.left[c] = cams + (size_t)c * fb;
        pt.right[c] = cams + (size_t)(c + 1) * fb;
        pt.out[c] = mids + (size_t)c * align_up(fb);
    }
    cudaError_t ce = run_interp_stage(e->g, pt, e->slots, e->P, e->rank_of, e->cand_of_rank, npairs, mask,
                                      e->profiling ? &e->prof : nullptr, st);
    if (ce != cudaSuccess) return cuda_fail(ce, "rig_views (direct-t): interpolate");
    e->last = pt;
    e->last_npairs = npairs;
    VinPairs pp{};
    for (int c = 0; c < npairs && ce == cudaSuccess; c++) {
        pp.left[c] = pt.left[c];
        pp.right[c] = pt.right[c];
        ce = run_direct_state(e->g, e->slots, e->P, c, mask + (size_t)c * n, state + (size_t)c * sstride, st);
    }
    if (ce != cudaSuccess) return cuda_fail(ce, "rig_views (direct-t): state");
    ce = vin_synth(pp, npairs, state, e->g.fmt, e->g.W, e->g.H, nv, views + fb, fb, (size_t)step * fb, st);
    for (int c = 0; c < npairs && ce == cudaSuccess; c++)
        ce = cudaMemcpyAsync(views + ((size_t)c * step + step / 2) * fb, mids + (size_t)c * align_up(fb), fb,
                             cudaMemcpyDeviceToDevice, st);
    if (ce != cudaSuccess) return cuda_fail(ce, "rig_views (direct-t): synthesis");
    return FVV_OK;
}

int fvv_downscale(const fvv_frame_desc* d, const uint8_t* frames, int nframes, int factor,
                  uint8_t* out, void* stream) {
    int rc = check_desc(d);
    if (rc) return rc;
    if (factor < 1) return fail(FVV_EINVAL, "factor must be >= 1");
    if (d->width % factor || d->height % factor)
        return fail(FVV_EINVAL, std::to_string(d->width) + "x" + std::to_string(d->height) +
                                    " not divisible by " + std::to_string(factor));
    if (d->format == FVV_YUV420) {
        const int cw = (d->width + 1) / 2, ch = (d->height + 1) / 2;
        if (cw % factor || ch % factor)
            return fail(FVV_EINVAL, std::to_string(ch) + "x" + std::to_string(cw) +
                                        " not divisible by " + std::to_string(factor));
    }
    cudaError_t ce = launch_downscale(d->width, d->height, d->format, frames, nframes, factor, out,
                                      static_cast<cudaStream_t>(stream));
    if (ce != cudaSuccess) return cuda_fail(ce, "downscale");
    return FVV_OK;
}

int fvv_cluster_width(int base_width, int nsmall) {
    const int cols = (nsmall + 3) / 4;
    return base_width + cols * (base_width / 4);
}

int fvv_assemble_cluster(const fvv_frame_desc* d, const uint8_t* anchor,
                         const uint8_t* const* smalls, int nsmall, uint8_t* stitched,
                         void* stream) {
    int rc = check_desc(d);
    if (rc) return rc;
    if (d->format == FVV_RGB8) return fail(FVV_ELAYOUT, "cluster frames are gray or 4:2:0");
    if (d->width % 8 || d->height % 8)
        return fail(FVV_ELAYOUT, "anchor dimensions must be divisible by 8");
    if (nsmall < 0 || nsmall > 256) return fail(FVV_ELAYOUT, "too many small tiles");
    cudaError_t ce = launch_assemble(d->width, d->height, d->format, anchor, smalls, nsmall,
                                     fvv_cluster_width(d->width, nsmall), stitched,
                                     static_cast<cudaStream_t>(stream));
    if (ce != cudaSuccess) return cuda_fail(ce, "assemble");
    return FVV_OK;
}

// cluster.py:58-74 build_layouts for camera c
static void layout_of(int ncams, int stages, int vps, int c, int* lo, int* hi) {
    const int total = (ncams - 1) * (1 << stages) + 1;
    const int anchor = c << stages;
    *lo = std::max(0, anchor - vps);
    *hi = std::min(total - 1, anchor + vps);
}

size_t fvv_rig_cluster_bytes(const fvv_frame_desc* d, int ncams, int stages, int vps,
                             int cluster) {
    if (check_desc(d) || cluster < 0 || cluster >= ncams) return 0;
    int lo, hi;
    layout_of(ncams, stages, vps, cluster, &lo, &hi);
    const int nsmall = hi - lo;  // tiles minus the anchor
    fvv_frame_desc s = *d;
    s.width = fvv_cluster_width(d->width, nsmall);
    return fvv_frame_bytes(&s);
}

}  // extern "C"

// Validates a rig clustering request (PipelineHandle._stitch, server/pipeline.py:273-292)
// and, when `jobs` is given, lays out one ClusterJob per camera.
static int cluster_jobs_of(const fvv_frame_desc* d, int ncams, int stages, int vps, std::vector<ClusterJob>* jobs,
                           long* maxb) {
    int rc = check_desc(d);
    if (rc) return rc;
    if (ncams < 2) return fail(FVV_EINVAL, "need at least 2 cameras");
    if (stages < 1 || stages > 6) return fail(FVV_EINVAL, "stages must be in 1..6");
    if (vps < 1) return fail(FVV_ELAYOUT, "views_per_side must be >= 1");
    if (vps > (1 << stages))
        return fail(FVV_ELAYOUT, "views_per_side " + std::to_string(vps) + " exceeds the " +
                                     std::to_string((1 << stages) - 1) +
                                     " interpolated views available per gap");
    if (d->format == FVV_RGB8) return fail(FVV_ELAYOUT, "cluster frames are gray or 4:2:0");
    if (d->width % 8 || d->height % 8)
        return fail(FVV_ELAYOUT, "anchor dimensions must be divisible by 8");
    if (!jobs) return FVV_OK;
    jobs->assign(ncams, ClusterJob{});
    long off = 0;
    *maxb = 0;
    for (int c = 0; c < ncams; c++) {
        int lo, hi;
        layout_of(ncams, stages, vps, c, &lo, &hi);
        ClusterJob& j = (*jobs)[c];
        j.anchor_view = c << stages;
        j.first_small = lo;
        j.nsmall = hi - lo;
        j.skip = j.anchor_view;
        j.sw = fvv_cluster_width(d->width, j.nsmall);
        j.out_offset = off;
        const long b = (long)fvv_rig_cluster_bytes(d, ncams, stages, vps, c);
        off += b;
        *maxb = std::max(*maxb, b);
    }
    if (*maxb >= (1l << 31)) return fail(FVV_ELAYOUT, "a cluster frame of 2^31 bytes or more");  // 32-bit kernel indexing
    return FVV_OK;
}

extern "C" {

int fvv_rig_clusters(const fvv_frame_desc* d, int ncams, int stages, int vps,
                     const uint8_t* views, uint8_t* clusters, void* stream) {
    std::vector<ClusterJob> jobs;
    long maxb = 0;
    int rc = cluster_jobs_of(d, ncams, stages, vps, &jobs, &maxb);
    if (rc) return rc;
    cudaError_t ce = launch_rig_clusters(d->width, d->height, d->format, jobs.data(), ncams, maxb,
                                         views, clusters, static_cast<cudaStream_t>(stream));
    if (ce != cudaSuccess) return cuda_fail(ce, "rig_clusters");
    return FVV_OK;
}

int fvv_rig_clusters_shard(const fvv_frame_desc* d, int ncams, int stages, int vps, int first_cluster,
                           int ncluster, const uint8_t* views, int view_base, int nviews,
                           const uint8_t* halo, int halo_first, int halo_count, uint8_t* clusters,
                           void* stream) {
    std::vector<ClusterJob> all;
    long maxb = 0;
    int rc = cluster_jobs_of(d, ncams, stages, vps, &all, &maxb);
    if (rc) return rc;
    if (ncluster == 0) return FVV_OK;
    if (first_cluster < 0 || ncluster < 0 || first_cluster + ncluster > ncams)
        return fail(FVV_EINVAL, "cluster range outside the rig");
    if (!views || !clusters || nviews < 1 || view_base < 0)
        return fail(FVV_EINVAL, "null or empty local views");
    if (halo_count < 0 || (halo_count > 0 && !halo)) return fail(FVV_EINVAL, "bad halo tiles");
    auto local = [&](int vi) { return vi >= view_base && vi < view_base + nviews; };
    auto in_halo = [&](int vi) { return vi >= halo_first && vi < halo_first + halo_count; };
    std::vector<ClusterJob> jobs(all.begin() + first_cluster, all.begin() + first_cluster + ncluster);
    const long off0 = jobs[0].out_offset;
    maxb = 0;
    for (ClusterJob& j : jobs) {
        j.out_offset -= off0;
        if (!local(j.anchor_view))
            return fail(FVV_EINVAL, "anchor view " + std::to_string(j.anchor_view) + " is not in the local views");
        for (int i = 0; i < j.nsmall; i++) {
            int vi = j.first_small + i;
            if (vi >= j.skip) vi += 1;
            if (!local(vi) && !in_halo(vi))
                return fail(FVV_EINVAL, "view " + std::to_string(vi) + " of cluster " +
                                            std::to_string(&j - jobs.data() + first_cluster) +
                                            " is neither local nor in the halo");
        }
        maxb = std::max(maxb, (long)fvv_rig_cluster_bytes(d, ncams, stages, vps, (int)(&j - jobs.data()) + first_cluster));
    }
    ViewSrc vs{views, view_base, halo, halo_first, halo_count};
    cudaError_t ce = launch_rig_clusters_src(d->width, d->height, d->format, jobs.data(), ncluster, maxb, vs,
                                             clusters, static_cast<cudaStream_t>(stream), 0);
    if (ce != cudaSuccess) return cuda_fail(ce, "rig_clusters_shard");
    return FVV_OK;
}

}  // extern "C"

extern "C" int fvv_conv2d_bf16(const fvv_conv_desc* d, const void* x, const void* w, const float* bias,
                               void* out, void* stream) {
    if (!d || !x || !w || !bias || !out) return fail(FVV_EINVAL, "null argument");
    if (d->batch < 1 || d->in_h < 1 || d->in_w < 1 || d->out_h < 1 || d->out_w < 1 || d->out_channels < 1)
        return fail(FVV_EINVAL, "empty convolution");
    const int cp = d->in_cpad;
    if (!(cp == 16 || cp == 32 || (cp % 64 == 0 && cp <= 1024)))
        return fail(FVV_EUNSUPPORTED, "in_cpad must be 16, 32 or a multiple of 64");
    const int nt = d->ntile;
    if (!(nt == 16 || nt == 32 || nt == 64 || nt == 128 || nt == 256))
        return fail(FVV_EINVAL, "ntile must be 16, 32, 64, 128 or 256");
    if (d->out_coff < 0 || d->out_coff + d->out_channels > d->out_cstride)
        return fail(FVV_EINVAL, "output channels outside out_cstride");
    if (!d->out_f32 && (d->out_cstride % 8 || d->out_coff % 8) && d->out_channels % 8 == 0)
        ;  // scalar stores handle unaligned bf16 placement
    const int npad = (d->out_channels + nt - 1) / nt * nt;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ConvTCParams p{};
    p.Hout = d->out_h;
    p.Wout = d->out_w;
    p.ostride = d->out_cstride;
    p.ocoff = d->out_coff;
    p.N = d->out_channels;
    p.act = d->relu ? 1 : 0;
    p.out_f32 = d->out_f32 ? 1 : 0;
    cudaError_t e = cudaSuccess;
    if (!d->transposed) {
        const int k = d->kernel, s = d->stride;
        if (k < 1 || k * k > kConvMaxTaps || s < 1 || s > 2)
            return fail(FVV_EUNSUPPORTED, "kernel*kernel <= 16 and stride 1 or 2");
        if ((d->in_h + 2 * d->pad - k) / s + 1 != d->out_h || (d->in_w + 2 * d->pad - k) / s + 1 != d->out_w)
            return fail(FVV_EINVAL, "output size does not match the convolution");
        p.Hg = d->out_h;
        p.Wg = d->out_w;
        p.sy = p.sx = s;
        p.by0 = p.bx0 = -d->pad;
        p.ntaps = k * k;
        for (int t = 0; t < k * k; t++) { p.tdy[t] = t / k; p.tdx[t] = t % k; }
        p.omy = p.omx = 1;
        p.oay = p.oax = 0;
        e = conv_tc(x, d->batch, d->in_h, d->in_w, cp, w, npad, 0, nt, bias, out, p, st);
    } else if (d->transposed == 2) {
        // ConvTranspose2d(k4 s2 p1) as ONE 3x3 sub-pixel convolution on the input grid: N = 4 x
        // out_channels (row n = phase * out_channels + c, convtc.pack_convT_subpixel), the epilogue
        // scatters phase (oy&1, ox&1); every input row is read once for all four phases
        if (d->kernel != 4 || d->stride != 2 || d->pad != 1)
            return fail(FVV_EUNSUPPORTED, "transposed convolution: kernel 4, stride 2, pad 1 only");
        if (d->out_h != 2 * d->in_h || d->out_w != 2 * d->in_w)
            return fail(FVV_EINVAL, "transposed output must be twice the input size");
        p.Hg = d->in_h;
        p.Wg = d->in_w;
        p.sy = p.sx = 1;
        p.by0 = p.bx0 = -1;
        p.ntaps = 9;
        for (int t = 0; t < 9; t++) { p.tdy[t] = t / 3; p.tdx[t] = t % 3; }
        p.omy = p.omx = 1;
        p.oay = p.oax = 0;
        p.N = 4 * d->out_channels;
        p.shuffle_c = d->out_channels;
        const int npad4 = (p.N + nt - 1) / nt * nt;
        e = conv_tc(x, d->batch, d->in_h, d->in_w, cp, w, npad4, 0, nt, bias, out, p, st);
    } else {
        if (d->kernel != 4 || d->stride != 2 || d->pad != 1)
            return fail(FVV_EUNSUPPORTED, "transposed convolution: kernel 4, stride 2, pad 1 only");
        if (d->out_h != 2 * d->in_h || d->out_w != 2 * d->in_w)
            return fail(FVV_EINVAL, "transposed output must be twice the input size");
        p.Hg = d->in_h;
        p.Wg = d->in_w;
        p.sy = p.sx = 1;
        p.by0 = p.bx0 = 0;
        p.ntaps = 4;
        p.omy = p.omx = 2;
        static const int off[2][2] = {{0, -1}, {1, 0}};  // [parity][tap]
        for (int ph = 0; ph < 4 && e == cudaSuccess; ph++) {
            const int a = ph >> 1, b = ph & 1;
            for (int t = 0; t < 4; t++) { p.tdy[t] = off[a][t >> 1]; p.tdx[t] = off[b][t & 1]; }
            p.oay = a;
            p.oax = b;
            e = conv_tc(x, d->batch, d->in_h, d->in_w, cp, w, 4 * npad, ph * npad, nt, bias, out, p, st);
        }
    }
    if (e != cudaSuccess) return cuda_fail(e, "fvv_conv2d_bf16");
    return FVV_OK;
}

static int vin_check_desc(const fvv_frame_desc* d) {
    if (!d) return fail(FVV_EINVAL, "null frame descriptor");
    if (d->width < 64 || d->height < 64 || d->width % 4 || d->height % 4)
        return fail(FVV_EINVAL, "VINet frames need width, height >= 64 and multiples of 4");
    if (d->format != FVV_GRAY8 && d->format != FVV_YUV420 && d->format != FVV_RGB8)
        return fail(FVV_EINVAL, "unknown pixel format");
    return FVV_OK;
}

extern "C" size_t fvv_vinet_workspace_size(const fvv_frame_desc* d, int max_pairs) {
    if (vin_check_desc(d) || max_pairs < 1) return 0;
    return vin_layout(d->width, d->height, std::min(max_pairs, kVinMaxPairs)).bytes;
}

extern "C" int fvv_vinet_flow(const fvv_frame_desc* d, const fvv_vinet_weights* wts, const uint8_t* const* left,
                              const uint8_t* const* right, int npairs, float* flows, void* ws, size_t ws_bytes,
                              void* stream) {
    int rc;
    if ((rc = vin_check_desc(d))) return rc;
    if (!wts || !left || !right || !flows || !ws) return fail(FVV_EINVAL, "null argument");
    if (npairs < 1) return fail(FVV_EINVAL, "npairs must be >= 1");
    int B = std::min(npairs, kVinMaxPairs);
    while (B > 1 && vin_layout(d->width, d->height, B).bytes > ws_bytes) B--;
    const VinLayout L = vin_layout(d->width, d->height, B);
    if (L.bytes > ws_bytes) return fail(FVV_EINVAL, "workspace too small for one pair");
    VinWeights vw;
    for (int i = 0; i < 3; i++)
        for (int k = 0; k < 10; k++) {
            if (!wts->w[i][k] || !wts->b[i][k]) return fail(FVV_EINVAL, "null layer weights");
            vw.w[i][k] = wts->w[i][k];
            vw.b[i][k] = wts->b[i][k];
        }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t plane = (size_t)5 * d->width * d->height;
    for (int p0 = 0; p0 < npairs; p0 += B) {
        const int n = std::min(B, npairs - p0);
        VinLayout Ln = vin_layout(d->width, d->height, n);
        VinPairs pp{};
        for (int i = 0; i < n; i++) {
            if (!left[p0 + i] || !right[p0 + i]) return fail(FVV_EINVAL, "null frame pointer");
            pp.left[i] = left[p0 + i];
            pp.right[i] = right[p0 + i];
        }
        cudaError_t e = vin_flows(Ln, vw, pp, d->format, static_cast<uint8_t*>(ws), flows + plane * p0, nullptr, st);
        if (e != cudaSuccess) return cuda_fail(e, "fvv_vinet_flow");
    }
    return FVV_OK;
}

extern "C" int fvv_vinet_synth(const fvv_frame_desc* d, const uint8_t* const* left, const uint8_t* const* right,
                               const float* flows, int npairs, int nviews, uint8_t* views, void* stream) {
    int rc;
    if ((rc = vin_check_desc(d))) return rc;
    if (!left || !right || !flows || !views) return fail(FVV_EINVAL, "null argument");
    if (npairs < 1 || nviews < 1) return fail(FVV_EINVAL, "npairs and nviews must be >= 1");
    fvv_frame_desc dd = *d;
    const size_t fb = fvv_frame_bytes(&dd);
    const size_t plane = (size_t)5 * d->width * d->height;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    for (int p0 = 0; p0 < npairs; p0 += kVinMaxPairs) {
        const int n = std::min(kVinMaxPairs, npairs - p0);
        VinPairs pp{};
        for (int i = 0; i < n; i++) {
            if (!left[p0 + i] || !right[p0 + i]) return fail(FVV_EINVAL, "null frame pointer");
            pp.left[i] = left[p0 + i];
            pp.right[i] = right[p0 + i];
        }
        cudaError_t e = vin_synth(pp, n, flows + plane * p0, d->format, d->width, d->height, nviews,
                                  views + (size_t)p0 * nviews * fb, fb, (size_t)nviews * fb, st);
        if (e != cudaSuccess) return cuda_fail(e, "fvv_vinet_synth");
    }
    return FVV_OK;
}

// camera anchors + per-chunk flows and direct-t views of a rig frame; with
// `tab` the synthesis also writes the views' quarter tiles into `clusters`.
static int vin_rig_run(const fvv_frame_desc* d, const fvv_vinet_weights* wts, const uint8_t* cams, int ncams,
                       int stages, uint8_t* views, void* ws, size_t ws_bytes, cudaStream_t st, const char* who,
                       const VinTileDst* tab, uint8_t* clusters) {
    fvv_frame_desc dd = *d;
    const size_t fb = fvv_frame_bytes(&dd);
    const int nv = (1 << stages) - 1, npairs = ncams - 1;
    // anchors: camera c lands at global view index c * 2^stages (ViewIndexModel, viewmodel.py:23-71)
    for (int c = 0; c < ncams; c++) {
        cudaError_t e = cudaMemcpyAsync(views + (size_t)c * (nv + 1) * fb, cams + (size_t)c * fb, fb,
                                        cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return cuda_fail(e, who);
    }
    int B = std::min(npairs, kVinMaxPairs);
    while (B > 1 && vin_layout(d->width, d->height, B).bytes > ws_bytes) B--;
    if (vin_layout(d->width, d->height, B).bytes > ws_bytes) return fail(FVV_EINVAL, "workspace too small for one pair");
    VinWeights vw;
    for (int i = 0; i < 3; i++)
        for (int k = 0; k < 10; k++) {
            if (!wts->w[i][k] || !wts->b[i][k]) return fail(FVV_EINVAL, "null layer weights");
            vw.w[i][k] = wts->w[i][k];
            vw.b[i][k] = wts->b[i][k];
        }
    for (int p0 = 0; p0 < npairs; p0 += B) {
        const int n = std::min(B, npairs - p0);
        const VinLayout L = vin_layout(d->width, d->height, n);
        VinPairs pp{};
        for (int i = 0; i < n; i++) {
            pp.left[i] = cams + (size_t)(p0 + i) * fb;
            pp.right[i] = cams + (size_t)(p0 + i + 1) * fb;
        }
        float* fl = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + L.flows);
        uint8_t* vout = views + ((size_t)p0 * (nv + 1) + 1) * fb;
        cudaError_t e = vin_flows(L, vw, pp, d->format, static_cast<uint8_t*>(ws), fl, nullptr, st);
        if (e == cudaSuccess) {
            if (tab)
                e = vin_synth_tiled(pp, n, fl, d->format, d->width, d->height, nv, vout, fb, (size_t)(nv + 1) * fb,
                                    tab, p0 * (nv + 1), nv + 1, clusters, st);
            else
                e = vin_synth(pp, n, fl, d->format, d->width, d->height, nv, vout, fb, (size_t)(nv + 1) * fb, st);
        }
        if (e != cudaSuccess) return cuda_fail(e, who);
    }
    return FVV_OK;
}

extern "C" int fvv_vinet_rig(const fvv_frame_desc* d, const fvv_vinet_weights* wts, const uint8_t* cams, int ncams,
                             int stages, uint8_t* views, void* ws, size_t ws_bytes, void* stream) {
    int rc;
    if ((rc = vin_check_desc(d))) return rc;
    if (!wts || !cams || !views || !ws) return fail(FVV_EINVAL, "null argument");
    if (ncams < 2) return fail(FVV_EINVAL, "a rig needs at least two cameras");
    if (stages < 1 || stages > 6) return fail(FVV_EINVAL, "stages must be in [1, 6]");
    return vin_rig_run(d, wts, cams, ncams, stages, views, ws, ws_bytes, static_cast<cudaStream_t>(stream),
                       "fvv_vinet_rig", nullptr, nullptr);
}

extern "C" int fvv_vinet_rig_clusters(const fvv_frame_desc* d, const fvv_vinet_weights* wts, const uint8_t* cams,
                                      int ncams, int stages, int vps, uint8_t* views, uint8_t* clusters, void* ws,
                                      size_t ws_bytes, void* stream) {
    int rc;
    if ((rc = vin_check_desc(d))) return rc;
    if (!wts || !cams || !views || !clusters || !ws) return fail(FVV_EINVAL, "null argument");
    if (ncams < 2) return fail(FVV_EINVAL, "a rig needs at least two cameras");
    if (stages < 1 || stages > 6) return fail(FVV_EINVAL, "stages must be in [1, 6]");
    if ((rc = cluster_jobs_of(d, ncams, stages, vps, nullptr, nullptr))) return rc;
    const int total = ((ncams - 1) << stages) + 1;
    if (total > kVinMaxViews)
        return fail(FVV_EINVAL, "fused tiling supports at most " + std::to_string(kVinMaxViews) + " views per rig frame");
    std::vector<ClusterJob> jobs;
    long maxb = 0;
    cluster_jobs_of(d, ncams, stages, vps, &jobs, &maxb);
    // the tile table lives in the workspace: size it for the largest chunk that fits
    int B = std::min(ncams - 1, kVinMaxPairs);
    while (B > 1 && vin_layout(d->width, d->height, B).bytes > ws_bytes) B--;
    const VinLayout L = vin_layout(d->width, d->height, B);
    if (L.bytes > ws_bytes) return fail(FVV_EINVAL, "workspace too small for one pair");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    VinTileDst* tab = reinterpret_cast<VinTileDst*>(static_cast<uint8_t*>(ws) + L.tiles);
    cudaError_t e = cudaMemsetAsync(tab, 0xFF, (size_t)2 * total * sizeof(VinTileDst), st);
    for (size_t b = 0; b < jobs.size() && e == cudaSuccess; b += kMaxClusters) {
        ClusterJobs cj;
        const int n = (int)std::min<size_t>(kMaxClusters, jobs.size() - b);
        for (int k = 0; k < n; k++) cj.job[k] = jobs[b + k];
        e = vin_tile_table(cj, n, total, tab, st);
    }
    if (e != cudaSuccess) return cuda_fail(e, "fvv_vinet_rig_clusters");
    if ((rc = vin_rig_run(d, wts, cams, ncams, stages, views, ws, ws_bytes, st, "fvv_vinet_rig_clusters", tab,
                          clusters)))
        return rc;
    e = launch_rig_clusters(d->width, d->height, d->format, jobs.data(), ncams, maxb, views, clusters, st,
                            1 << stages);
    if (e != cudaSuccess) return cuda_fail(e, "fvv_vinet_rig_clusters");
    return FVV_OK;
}

// ---------------------------------------------------------------------------
// RefineNet + ContextNet (refine_kernels.cu; orchestration in refine.py)
// ---------------------------------------------------------------------------
static int ref_check(const fvv_frame_desc* d, int n, int cap) {
    int rc = vin_check_desc(d);
    if (rc) return rc;
    if (n < 1 || n > cap) return fail(FVV_EINVAL, "batch must hold 1.." + std::to_string(cap) + " entries");
    return FVV_OK;
}

extern "C" int fvv_refine_image(const fvv_frame_desc* d, const uint8_t* const* frames, int nsrc, void* out,
                                void* stream) {
    int rc = ref_check(d, nsrc, 2 * kRefMaxViews);
    if (rc) return rc;
    if (!frames || !out) return fail(FVV_EINVAL, "null argument");
    RefSrc s{};
    for (int i = 0; i < nsrc; i++) s.frame[i] = frames[i];
    const int Wp = (d->width + 63) / 64 * 64, Hp = (d->height + 63) / 64 * 64;
    cudaError_t e = ref_img(s, nsrc, d->format, d->width, d->height, Wp, Hp, out, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? FVV_OK : cuda_fail(e, "fvv_refine_image");
}

extern "C" int fvv_refine_inputs(const fvv_frame_desc* d, const uint8_t* const* left, const uint8_t* const* right,
                                 const float* const* state, const float* t, int nviews, void* x0, float* merged,
                                 float* flow0, void* stream) {
    int rc = ref_check(d, nviews, kRefMaxViews);
    if (rc) return rc;
    if (!left || !right || !state || !t || !x0 || !merged || !flow0) return fail(FVV_EINVAL, "null argument");
    RefViews rv{};
    for (int i = 0; i < nviews; i++) {
        if (!(t[i] > 0.0f && t[i] < 1.0f)) return fail(FVV_EINVAL, "view positions must lie in (0, 1)");
        rv.left[i] = left[i];
        rv.right[i] = right[i];
        rv.state[i] = state[i];
        rv.t[i] = t[i];
    }
    const int Wp = (d->width + 63) / 64 * 64, Hp = (d->height + 63) / 64 * 64;
    cudaError_t e = ref_inputs(rv, nviews, d->format, d->width, d->height, Wp, Hp, x0, merged, flow0,
                               static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? FVV_OK : cuda_fail(e, "fvv_refine_inputs");
}

extern "C" int fvv_refine_flow_pool(const float* in, float* out, int w, int h, int nb, void* stream) {
    if (!in || !out || w < 2 || h < 2 || (w & 1) || (h & 1) || nb < 1) return fail(FVV_EINVAL, "bad flow pyramid level");
    cudaError_t e = ref_flow_pool(in, out, w, h, nb, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? FVV_OK : cuda_fail(e, "fvv_refine_flow_pool");
}

extern "C" int fvv_refine_warp_features(const void* feat, int fs, int channels, int w, int h, const float* flow,
                                        int comp, int src_mul, int src_add, void* dst, int ds, int coff, int nb,
                                        void* stream) {
    if (!feat || !flow || !dst || channels % 8 || fs % 8 || ds % 8 || coff % 8 || coff + channels > ds ||
        channels > fs || w < 2 || h < 2 || nb < 1 || (comp != 0 && comp != 2))
        return fail(FVV_EINVAL, "bad feature warp");
    cudaError_t e = ref_warp_feat(feat, fs, channels, w, h, flow, comp, src_mul, src_add, dst, ds, coff, nb,
                                  static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? FVV_OK : cuda_fail(e, "fvv_refine_warp_features");
}

extern "C" int fvv_nhwc_copy(const void* src, int ss, int channels, void* dst, int ds, int coff, long long npix,
                             void* stream) {
    if (!src || !dst || channels % 8 || ss % 8 || ds % 8 || coff % 8 || coff + channels > ds || channels > ss ||
        npix < 0)
        return fail(FVV_EINVAL, "bad channel copy");
    if (npix == 0) return FVV_OK;
    cudaError_t e = nhwc_copy(src, ss, channels, dst, ds, coff, npix, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? FVV_OK : cuda_fail(e, "fvv_nhwc_copy");
}

extern "C" int fvv_refine_output(const fvv_frame_desc* d, uint8_t* const* out, int nviews, const float* r, int rs,
                                 const float* merged, void* stream) {
    int rc = ref_check(d, nviews, kRefMaxViews);
    if (rc) return rc;
    if (!out || !r || !merged || rs < 3) return fail(FVV_EINVAL, "null argument");
    RefViews rv{};
    for (int i = 0; i < nviews; i++) rv.out[i] = out[i];
    const int Wp = (d->width + 63) / 64 * 64, Hp = (d->height + 63) / 64 * 64;
    cudaError_t e = ref_out(rv, nviews, d->format, d->width, d->height, Wp, Hp, r, rs, merged,
                            static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? FVV_OK : cuda_fail(e, "fvv_refine_output");
}

// ---------------------------------------------------------------------------
// FVT1 tile encoder, device stage (encode_kernels.cu; host framing in encoder.py)
// ---------------------------------------------------------------------------
static_assert(sizeof(EncJob) == sizeof(fvv_enc_job), "fvv_enc_job mirrors fvv::EncJob");

extern "C" int fvv_encode_set_tables(const double* dct64, const uint8_t* zigzag64) {
    if (!dct64 || !zigzag64) return fail(FVV_EINVAL, "null table");
    for (int i = 0; i < 64; i++)
        if (zigzag64[i] > 63) return fail(FVV_EINVAL, "zigzag index out of range");
    cudaError_t e = enc_set_constants(dct64, zigzag64);
    return e == cudaSuccess ? FVV_OK : cuda_fail(e, "fvv_encode_set_tables");
}

extern "C" int fvv_encode_blocks(const fvv_enc_job* jobs_dev, int njobs, long long total_blocks, int lossless,
                                 int16_t* zz, int* ntok, void* stream) {
    if (!jobs_dev || njobs < 1 || total_blocks < 0 || !zz || !ntok) return fail(FVV_EINVAL, "bad encode batch");
    cudaError_t e = enc_blocks(reinterpret_cast<const EncJob*>(jobs_dev), njobs, total_blocks, lossless ? 1 : 0, zz,
                               ntok, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? FVV_OK : cuda_fail(e, "fvv_encode_blocks");
}

extern "C" int fvv_encode_tokens(const int16_t* zz, const long long* tok_off, long long nblocks, uint8_t* out,
                                 void* stream) {
    if (!zz || !tok_off || !out || nblocks < 0) return fail(FVV_EINVAL, "bad token batch");
    cudaError_t e = enc_tokens(zz, tok_off, nblocks, out, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? FVV_OK : cuda_fail(e, "fvv_encode_tokens");
}

// ---------------------------------------------------------------------------
// DEFLATE of many byte streams (deflate_kernels.cu): zlib.compress(x, 6)[2:-4]
// ---------------------------------------------------------------------------
static int deflate_lengths(const long long* offsets, int nstreams, std::vector<int64_t>& len) {
    if (!offsets || nstreams < 1) return fail(FVV_EINVAL, "bad stream offsets");
    len.resize(nstreams);
    for (int s = 0; s < nstreams; s++) {
        if (offsets[s + 1] < offsets[s] || offsets[s] < 0) return fail(FVV_EINVAL, "stream offsets must ascend");
        len[s] = offsets[s + 1] - offsets[s];
    }
    return FVV_OK;
}

extern "C" int fvv_deflate_scratch_bytes(const long long* offsets, int nstreams, size_t* scratch_bytes,
                                         size_t* out_capacity) {
    std::vector<int64_t> len;
    if (int r = deflate_lengths(offsets, nstreams, len)) return r;
    if (scratch_bytes) *scratch_bytes = zd_scratch_bytes(len.data(), nstreams);
    if (out_capacity) *out_capacity = zd_out_capacity(len.data(), nstreams);
    return FVV_OK;
}

extern "C" int fvv_deflate(const uint8_t* data, const long long* offsets, int nstreams, uint8_t* out,
                           long long* out_offsets, void* scratch, size_t scratch_bytes, void* stream) {
    std::vector<int64_t> len;
    if (int r = deflate_lengths(offsets, nstreams, len)) return r;
    if (!data || !out || !out_offsets || !scratch) return fail(FVV_EINVAL, "null deflate buffer");
    if (reinterpret_cast<uintptr_t>(out) % 8) return fail(FVV_EINVAL, "deflate output must be 8-byte aligned");
    if (scratch_bytes < zd_scratch_bytes(len.data(), nstreams)) return fail(FVV_EINVAL, "deflate scratch too small");
    static_assert(sizeof(long long) == sizeof(int64_t), "offsets are int64");
    cudaError_t e = zd_deflate(data, reinterpret_cast<const int64_t*>(offsets), nstreams, out,
                               reinterpret_cast<int64_t*>(out_offsets), scratch, scratch_bytes,
                               static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? FVV_OK : cuda_fail(e, "fvv_deflate");
}
