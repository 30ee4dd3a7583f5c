// abi.cu — the C-ABI of include/ubqp.h: handle, Q residency, workspace, pointer-kind
// detection, launch order and error mapping.  All arithmetic of the method runs in the
// kernels of gen.cu / eval_tc.cu / screen.cu / ascend.cu; the host only forms T(lambda)
// in binary64 and marshals arguments.
#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "ubqp_internal.cuh"

using ubqp::Ctx;

struct ubqp_ctx : public Ctx {};

namespace {

const char *kNullHandleMsg = "ubqp: null handle";

int fail(ubqp_t h, int code, const char *msg) {
    if (h) h->err = msg;
    return code;
}

int fail_cuda(ubqp_t h, cudaError_t e, const char *where) {
    if (h) {
        h->sticky_cuda = true;
        h->err = std::string("ubqp: CUDA error in ") + where + ": " + cudaGetErrorString(e);
    }
    return UBQP_E_CUDA;
}

#define CK(expr)                                                       \
    do {                                                               \
        cudaError_t e_ = (expr);                                       \
        if (e_ != cudaSuccess) return fail_cuda(h, e_, #expr);         \
    } while (0)

#define CK_LAUNCH(where)                                               \
    do {                                                               \
        cudaError_t e_ = cudaGetLastError();                           \
        if (e_ != cudaSuccess) return fail_cuda(h, e_, where);         \
    } while (0)

#define GUARD(h)                                                       \
    do {                                                               \
        if (!(h)) return UBQP_E_INVALID;                               \
        if ((h)->sticky_cuda) return UBQP_E_CUDA;                      \
        cudaError_t e_ = cudaSetDevice((h)->device);                   \
        if (e_ != cudaSuccess) return fail_cuda(h, e_, "cudaSetDevice"); \
    } while (0)

bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

template <typename T>
void dfree(T *&p) {
    if (p) cudaFree(p);
    p = nullptr;
}

void free_batch(Ctx &c) {
    dfree(c.Xb); dfree(c.X8); dfree(c.f); dfree(c.gains); dfree(c.surv); dfree(c.blk_count);
    dfree(c.asc_f); dfree(c.asc_flips); dfree(c.asc_bits); dfree(c.asc_slots); dfree(c.asc_aux);
    dfree(c.part); dfree(c.grp_cnt); dfree(c.grp_res); dfree(c.X8r);
    dfree(c.part_poll); dfree(c.grp_poll);
    c.part_cap = c.grp_cap = 0;
    c.asc_cap = 0;
    c.k_max = 0; c.k_cap_pad = 0; c.k_local = -1;
    c.f_valid = c.gains_valid = c.gains64_valid = false;
}

void free_all(Ctx &c) {
    free_batch(c);
    dfree(c.Q8); dfree(c.Q8L); dfree(c.diag); dfree(c.seed); dfree(c.parents); dfree(c.guides);
    dfree(c.ell);
    c.nnz = 0;
    c.ell_stride = 0;
    c.parents_cap = c.guides_cap = 0; dfree(c.scratch64);
    for (int s = 0; s < ubqp::kSlices; ++s) dfree(c.Qs[s]);
    for (int s = 0; s < ubqp::kMaxLimbs; ++s) { dfree(c.Qw[s]); dfree(c.QwL[s]); }
    dfree(c.wdiag); dfree(c.zdiag);
    dfree(c.fs); dfree(c.fint); dfree(c.freal); dfree(c.Qt); dfree(c.diagt); dfree(c.gains64);
    c.op_full = c.op_tri = c.op_wide = ubqp::Operand{};
    for (auto &o : c.op_walk) o = ubqp::Operand{};
    c.qt_ld = 0;
    c.real = false;
    c.freal_valid = false;
    c.q_exp = c.w_exp = c.w_limbs = 0;
    c.n = 0;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                             &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2-D int8 tensor map: inner dim `cols` bytes (contiguous), outer `rows`, box 128 x box_rows,
// 128-byte swizzle (the UMMA K-major SW128 canonical layout).
bool encode_map(CUtensorMap *m, void *base, uint64_t cols, uint64_t rows, uint32_t box_rows,
                uint64_t ld = 0) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {ld ? ld : cols};
    cuuint32_t box[2] = {128u, box_rows};
    cuuint32_t estr[2] = {1u, 1u};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// B operand from int8 planes [rows][ld] (plane s weighs 128^s): 256-row and 128-row boxes
bool set_operand(ubqp::Operand &op, int8_t *const *planes, int count, uint64_t ld, bool tri,
                 const int32_t *const *diag, int n_pad, int q_rows) {
    op = ubqp::Operand{};
    op.planes = count;
    op.tri = tri;
    for (int s = 0; s < count; ++s) {
        if (!encode_map(&op.full[s], planes[s], n_pad, q_rows, ubqp::kBN, ld) ||
            !encode_map(&op.half[s], planes[s], n_pad, q_rows, ubqp::kBN / 2, ld))
            return false;
        op.diag[s] = diag[s];
    }
    return true;
}

// grow the in-kernel fold buffers for a launch of this shape (synchronises when growing;
// new counters start at zero and reset themselves after every launch)
int ensure_fold(ubqp_t h, const ubqp::EvalShape &s) {
    if (s.part_elems > h->part_cap) {
        CK(cudaStreamSynchronize(h->stream));
        dfree(h->part);
        dfree(h->part_poll);
        h->part_cap = 0;
        if (cudaMalloc(&h->part, s.part_elems * sizeof(int32_t)) != cudaSuccess ||
            cudaMalloc(&h->part_poll, s.part_elems * sizeof(int32_t)) != cudaSuccess) {
            cudaGetLastError();
            return fail(h, UBQP_E_NOMEM, "ubqp: cannot allocate the evaluation partials");
        }
        CK(cudaMemsetAsync(h->part_poll, 0x80, s.part_elems * sizeof(int32_t), h->stream));
        h->part_cap = s.part_elems;
    }
    if (s.num_groups + 1 > h->grp_cap) {
        CK(cudaStreamSynchronize(h->stream));
        dfree(h->grp_cnt);
        dfree(h->grp_res);
        dfree(h->grp_poll);
        h->grp_cap = 0;
        const int64_t cap = s.num_groups + 1;
        if (cudaMalloc(&h->grp_cnt, cap * sizeof(unsigned)) != cudaSuccess ||
            cudaMalloc(&h->grp_res, cap * 4 * sizeof(int64_t)) != cudaSuccess ||
            cudaMalloc(&h->grp_poll, cap * 2 * sizeof(int64_t)) != cudaSuccess) {
            cudaGetLastError();
            return fail(h, UBQP_E_NOMEM, "ubqp: cannot allocate the evaluation counters");
        }
        CK(cudaMemsetAsync(h->grp_cnt, 0, cap * sizeof(unsigned), h->stream));
        CK(cudaMemsetAsync(h->grp_poll, 0x80, cap * 2 * sizeof(int64_t), h->stream));
        h->grp_cap = cap;
    }
    return UBQP_OK;
}

// one evaluation launch (sizes the fold buffers first)
int eval_launch(ubqp_t h, const ubqp::EvalLaunch &L) {
    if (L.k <= 0) return UBQP_OK;
    const ubqp::EvalShape s = ubqp::eval_shape(*h, L.k, L.op->planes, L.emit_gains, L.op->tri && !L.emit_gains);
    int rc = ensure_fold(h, s);
    if (rc) return rc;
    if (ubqp::launch_eval(*h, L)) return fail(h, UBQP_E_CUDA, "ubqp: evaluation fold buffers too small");
    CK_LAUNCH("eval_tc kernel");
    return UBQP_OK;
}

// Fixed-stride rows of Q without the diagonal for the sparse ascent (NEXT-3), built when the
// off-diagonal density is at most kSparseBuildDensity: entries (j << 8) | (Q_kj & 0xFF), j
// ascending, padded with 0xFFFFFFFF to the longest row rounded up to 32 entries
constexpr double kSparseBuildDensity = 0.25;
int build_sparse(ubqp_t h, const int32_t *Qh) {
    const int n = h->n;
    int64_t nnz = 0;
    int maxrow = 0;
    for (int i = 0; i < n; ++i) {
        int r = 0;
        for (int j = 0; j < n; ++j) r += (j != i && Qh[static_cast<int64_t>(i) * n + j] != 0);
        nnz += r;
        maxrow = std::max(maxrow, r);
    }
    h->nnz = nnz;
    if (n < 2 || static_cast<double>(nnz) > kSparseBuildDensity * n * (n - 1.0)) return UBQP_OK;
    const int stride = std::max(32, (maxrow + 31) / 32 * 32);
    std::vector<uint32_t> ent(static_cast<size_t>(n) * stride, 0xFFFFFFFFu);
    for (int i = 0; i < n; ++i) {
        int at = 0;
        for (int j = 0; j < n; ++j) {
            const int32_t v = Qh[static_cast<int64_t>(i) * n + j];
            if (j != i && v != 0)
                ent[static_cast<size_t>(i) * stride + at++] = (static_cast<uint32_t>(j) << 8) | (static_cast<uint32_t>(v) & 0xFFu);
        }
    }
    if (cudaMalloc(&h->ell, ent.size() * sizeof(uint32_t)) != cudaSuccess) {
        cudaGetLastError();
        free_all(*h);
        return fail(h, UBQP_E_NOMEM, "ubqp: cannot allocate the sparse rows of Q");
    }
    h->ell_stride = stride;
    CK(cudaMemcpy(h->ell, ent.data(), ent.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    return UBQP_OK;
}

int ensure_gains(ubqp_t h) {
    if (h->gains) return UBQP_OK;
    size_t bytes = static_cast<size_t>(h->k_max) * h->n_pad * sizeof(int32_t);
    cudaError_t e = cudaMalloc(&h->gains, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        h->gains = nullptr;
        return fail(h, UBQP_E_NOMEM, "ubqp: cannot allocate the gains buffer");
    }
    return UBQP_OK;
}

int ensure_asc(ubqp_t h, int64_t m) {
    if (m <= h->asc_cap) return UBQP_OK;
    dfree(h->asc_f); dfree(h->asc_flips); dfree(h->asc_bits); dfree(h->asc_slots); dfree(h->asc_aux);
    int64_t cap = m;
    if (cudaMalloc(&h->asc_f, cap * sizeof(int64_t)) != cudaSuccess ||
        cudaMalloc(&h->asc_flips, cap * sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&h->asc_aux, cap * sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&h->asc_bits, cap * h->W64 * sizeof(uint64_t)) != cudaSuccess ||
        cudaMalloc(&h->asc_slots, cap * sizeof(int32_t)) != cudaSuccess) {
        cudaGetLastError();
        h->asc_cap = 0;
        return fail(h, UBQP_E_NOMEM, "ubqp: cannot allocate ascent buffers");
    }
    h->asc_cap = cap;
    return UBQP_OK;
}

// host -> device copy on the handle's stream, then wait: a pinned source copies truly
// asynchronously, and include/ubqp.h promises that the call synchronises when it reads a
// host array, so the caller may reuse or free it as soon as the call returns.
int h2d_sync(ubqp_t h, void *dst, const void *src, size_t bytes) {
    if (!bytes) return UBQP_OK;
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return UBQP_OK;
}

// stage rows*W64 packed words on the device (device pointers pass through)
int stage_rows(ubqp_t h, const uint64_t *src, int64_t rows, uint64_t *&buf, int64_t &cap, const uint64_t *&out) {
    if (is_device_ptr(src)) {
        out = src;
        return UBQP_OK;
    }
    if (rows > cap) {
        CK(cudaStreamSynchronize(h->stream));
        dfree(buf);
        cap = 0;
        if (cudaMalloc(&buf, rows * h->W64 * sizeof(uint64_t)) != cudaSuccess) {
            cudaGetLastError();
            return fail(h, UBQP_E_NOMEM, "ubqp: cannot allocate a staging buffer");
        }
        cap = rows;
    }
    const int rc = h2d_sync(h, buf, src, rows * h->W64 * sizeof(uint64_t));
    if (rc) return rc;
    out = buf;
    return UBQP_OK;
}

// run the evaluation GEMM on the current batch: f (+ gains) and the stats {sum, K, max_key, 0}
// folded in-kernel into h->f / scratch64[0..3] and, when given, device copies f_dev / stats_dev
int run_eval(ubqp_t h, bool emit_gains, int64_t *f_dev = nullptr, int64_t *stats_dev = nullptr) {
    if (emit_gains) {
        int rc = ensure_gains(h);
        if (rc) return rc;
    }
    const int64_t k = h->k_local;
    if (k == 0) {   // empty batch: the stats of nothing
        const int64_t z[4] = {0, 0, -1, 0};
        CK(cudaMemcpyAsync(h->scratch64, z, sizeof z, cudaMemcpyHostToDevice, h->stream));
        if (stats_dev) CK(cudaMemcpyAsync(stats_dev, z, sizeof z, cudaMemcpyHostToDevice, h->stream));
        CK(cudaStreamSynchronize(h->stream));   // z is a stack array
    } else {
        ubqp::EvalLaunch L;
        L.tmX = &h->tmap_X8;
        L.Xb = h->Xb;
        L.k = k;
        L.op = (h->sym_eval && !emit_gains) ? &h->op_tri : &h->op_full;
        L.emit_gains = emit_gains;
        L.mode = ubqp::kFoldInt;
        L.f = h->f;
        L.f2 = f_dev;
        L.stats = h->scratch64;
        L.stats2 = stats_dev;
        L.rank = h->rank;
        L.world = h->world;
        L.shard_b = h->shard_b;
        const int rc = eval_launch(h, L);
        if (rc) return rc;
    }
    h->f_valid = true;
    h->gains_valid = emit_gains;
    return UBQP_OK;
}

int check_batch_args(ubqp_t h, int64_t k_local, int32_t rank, int32_t world) {
    if (h->n <= 0) return fail(h, UBQP_E_STATE, "ubqp: no Q loaded");
    if (k_local < 0 || k_local > h->k_max) return fail(h, UBQP_E_INVALID, "ubqp: k_local out of [0, k_max]");
    if (world < 1 || rank < 0 || rank >= world) return fail(h, UBQP_E_INVALID, "ubqp: bad rank/world");
    if (k_local > 0 && ubqp::global_index(k_local - 1, rank, world, h->shard_b) >= (1ll << 22))
        return fail(h, UBQP_E_INVALID, "ubqp: global index g exceeds 2^22");
    return UBQP_OK;
}

}  // namespace

extern "C" {

int ubqp_version(void) { return 200; }   // 2.00: int128 real-Q stats of the evaluation image, ubqp_set_option

int ubqp_create(int device, void *cuda_stream, ubqp_t *out) {
    if (!out) return UBQP_E_INVALID;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) {
        cudaGetLastError();
        return UBQP_E_INVALID;
    }
    ubqp_t h = new (std::nothrow) ubqp_ctx();
    if (!h) return UBQP_E_NOMEM;
    h->device = device;
    if (cudaSetDevice(device) != cudaSuccess) { delete h; return UBQP_E_CUDA; }
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
    if (major != 10 || minor != 0) {
        delete h;
        return UBQP_E_INVALID;   // built for sm_100a (B200) only
    }
    if (const char *env = getenv("UBQP_FULL_EVAL")) h->sym_eval = env[0] == '0';
    if (const char *env = getenv("UBQP_EVAL_2SM")) h->eval_pair = env[0] != '0';
    if (cuda_stream) {
        h->stream = static_cast<cudaStream_t>(cuda_stream);
    } else {
        if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess) {
            delete h;
            return UBQP_E_CUDA;
        }
        h->own_stream = true;
    }
    if (cudaMalloc(&h->scratch64, 32 * sizeof(int64_t)) != cudaSuccess) {
        if (h->own_stream) cudaStreamDestroy(h->stream);
        delete h;
        return UBQP_E_NOMEM;
    }
    *out = h;
    return UBQP_OK;
}

int ubqp_destroy(ubqp_t h) {
    if (!h) return UBQP_E_INVALID;
    cudaSetDevice(h->device);
    cudaStreamSynchronize(h->stream);
    free_all(*h);
    if (h->own_stream) cudaStreamDestroy(h->stream);
    delete h;
    return UBQP_OK;
}

const char *ubqp_last_error(ubqp_t h) {
    if (!h) return kNullHandleMsg;
    return h->err.c_str();
}

int ubqp_load_Q(ubqp_t h, int32_t n, const int32_t *Q, int64_t k_max) {
    GUARD(h);
    if (!Q || n < 1 || n > 16384) return fail(h, UBQP_E_INVALID, "ubqp: n must be in [1, 16384]");
    if (k_max < 1 || k_max > (1ll << 22)) return fail(h, UBQP_E_INVALID, "ubqp: k_max must be in [1, 2^22]");
    const int64_t nn = static_cast<int64_t>(n) * n;
    std::vector<int32_t> hq;
    const int32_t *Qh = Q;
    if (is_device_ptr(Q)) {
        // ordered after the caller's work on the handle's stream (Q may have just been written there)
        hq.resize(nn);
        CK(cudaMemcpyAsync(hq.data(), Q, nn * sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        Qh = hq.data();
    }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const int32_t v = Qh[static_cast<int64_t>(i) * n + j];
            if (v < -127 || v > 127) return fail(h, UBQP_E_RANGE, "ubqp: |Q_ij| > 127 (int8 tensor-core path)");
            if (j > i && v != Qh[static_cast<int64_t>(j) * n + i])
                return fail(h, UBQP_E_NOT_SYMMETRIC, "ubqp: Q is not symmetric");
        }
    CK(cudaStreamSynchronize(h->stream));
    free_all(*h);
    CK(cudaMalloc(&h->scratch64, 32 * sizeof(int64_t)));
    h->n = n;
    h->n_pad = (n + ubqp::kNPadAlign - 1) / ubqp::kNPadAlign * ubqp::kNPadAlign;
    h->q_rows = (n + ubqp::kQRowAlign - 1) / ubqp::kQRowAlign * ubqp::kQRowAlign;
    h->W64 = (n + 63) / 64;
    h->q_ld = ubqp::ascend_capacity(h->n_pad);
    std::vector<int8_t> q8(static_cast<size_t>(h->q_rows) * h->q_ld, 0);
    std::vector<int32_t> dg(h->q_rows, 0);
    std::vector<int8_t> q8l(static_cast<size_t>(h->q_rows) * h->n_pad, 0);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j <= i; ++j)
            q8l[static_cast<size_t>(i) * h->n_pad + j] = static_cast<int8_t>(Qh[static_cast<int64_t>(i) * n + j]);
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j)
            q8[static_cast<size_t>(i) * h->q_ld + j] = static_cast<int8_t>(Qh[static_cast<int64_t>(i) * n + j]);
        dg[i] = Qh[static_cast<int64_t>(i) * n + i];
    }
    int qmax = 0;
    for (int64_t e = 0; e < nn; ++e) qmax = std::max(qmax, std::abs(Qh[e]));
    if (cudaMalloc(&h->Q8, q8.size()) != cudaSuccess || cudaMalloc(&h->diag, dg.size() * 4) != cudaSuccess ||
        cudaMalloc(&h->Q8L, q8l.size()) != cudaSuccess ||
        cudaMalloc(&h->seed, h->W64 * sizeof(uint64_t)) != cudaSuccess) {
        cudaGetLastError();
        free_all(*h);
        return fail(h, UBQP_E_NOMEM, "ubqp: cannot allocate Q");
    }
    CK(cudaMemcpy(h->Q8, q8.data(), q8.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->Q8L, q8l.data(), q8l.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->diag, dg.data(), dg.size() * 4, cudaMemcpyHostToDevice));
    // batch workspace
    h->qmax = qmax;
    h->k_max = k_max;
    h->k_cap_pad = (k_max + ubqp::kBM - 1) / ubqp::kBM * ubqp::kBM;
    const int64_t nblk = (k_max + 4095) / 4096 + 1;
    if (cudaMalloc(&h->Xb, k_max * h->W64 * sizeof(uint64_t)) != cudaSuccess ||
        cudaMalloc(&h->X8, h->k_cap_pad * h->n_pad) != cudaSuccess ||
        cudaMalloc(&h->f, k_max * sizeof(int64_t)) != cudaSuccess ||
        cudaMalloc(&h->surv, k_max * sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&h->blk_count, nblk * sizeof(int32_t)) != cudaSuccess) {
        cudaGetLastError();
        free_all(*h);
        return fail(h, UBQP_E_NOMEM, "ubqp: cannot allocate the batch workspace");
    }
    CK(cudaMemset(h->X8, 0, h->k_cap_pad * h->n_pad));
    int8_t *full_pl[1] = {h->Q8}, *tri_pl[1] = {h->Q8L};
    const int32_t *dg_pl[1] = {h->diag};
    if (!encode_map(&h->tmap_X8, h->X8, h->n_pad, h->k_cap_pad, ubqp::kBM) ||
        !set_operand(h->op_full, full_pl, 1, h->q_ld, false, dg_pl, h->n_pad, h->q_rows) ||
        !set_operand(h->op_tri, tri_pl, 1, h->n_pad, true, dg_pl, h->n_pad, h->q_rows)) {
        free_all(*h);
        return fail(h, UBQP_E_CUDA, "ubqp: cuTensorMapEncodeTiled failed");
    }
    {
        int rc2 = build_sparse(h, Qh);
        if (rc2) return rc2;
    }
    h->k_local = -1;
    CK(cudaDeviceSynchronize());
    return UBQP_OK;
}

int ubqp_diversify(ubqp_t h, const uint64_t *seed_bits, int64_t t0, int64_t k_local, int32_t rank,
                   int32_t world) {
    GUARD(h);
    int rc = check_batch_args(h, k_local, rank, world);
    if (rc) return rc;
    if (!seed_bits) return fail(h, UBQP_E_INVALID, "ubqp: seed_bits is NULL");
    if (t0 < 0 || t0 > (1ll << 62)) return fail(h, UBQP_E_INVALID, "ubqp: t0 must be in [0, 2^62]");
    const uint64_t *seed_dev = seed_bits;
    if (!is_device_ptr(seed_bits)) {
        const int rc2 = h2d_sync(h, h->seed, seed_bits, h->W64 * sizeof(uint64_t));
        if (rc2) return rc2;
        seed_dev = h->seed;
    }
    h->rank = rank;
    h->world = world;
    h->k_local = k_local;
    h->f_valid = h->gains_valid = h->gains64_valid = false;
    ubqp::launch_glover(*h, seed_dev, t0, k_local);
    CK_LAUNCH("glover_kernel");
    return UBQP_OK;
}

int ubqp_blend(ubqp_t h, const uint64_t *seed_bits, const uint64_t *parents, int64_t n_parents, int64_t t0,
               int64_t k_local, int32_t rank, int32_t world) {
    GUARD(h);
    int rc = check_batch_args(h, k_local, rank, world);
    if (rc) return rc;
    if (!seed_bits || !parents) return fail(h, UBQP_E_INVALID, "ubqp: seed_bits or parents is NULL");
    if (n_parents < 1 || n_parents > (1ll << 22)) return fail(h, UBQP_E_INVALID, "ubqp: n_parents must be in [1, 2^22]");
    if (t0 < 0 || t0 > (1ll << 62)) return fail(h, UBQP_E_INVALID, "ubqp: t0 must be in [0, 2^62]");
    const uint64_t *seed_dev = seed_bits;
    if (!is_device_ptr(seed_bits)) {
        const int rc2 = h2d_sync(h, h->seed, seed_bits, h->W64 * sizeof(uint64_t));
        if (rc2) return rc2;
        seed_dev = h->seed;
    }
    const uint64_t *par_dev = nullptr;
    rc = stage_rows(h, parents, n_parents, h->parents, h->parents_cap, par_dev);
    if (rc) return rc;
    h->rank = rank;
    h->world = world;
    h->k_local = k_local;
    h->f_valid = h->gains_valid = h->gains64_valid = false;
    ubqp::launch_glover(*h, seed_dev, t0, k_local, par_dev, n_parents);
    CK_LAUNCH("glover_kernel");
    return UBQP_OK;
}

int ubqp_random(ubqp_t h, uint64_t seed, int64_t k_local, int32_t rank, int32_t world) {
    GUARD(h);
    int rc = check_batch_args(h, k_local, rank, world);
    if (rc) return rc;
    h->rank = rank;
    h->world = world;
    h->k_local = k_local;
    h->f_valid = h->gains_valid = h->gains64_valid = false;
    ubqp::launch_random(*h, seed, k_local);
    CK_LAUNCH("random_kernel");
    return UBQP_OK;
}

int ubqp_set_batch(ubqp_t h, const uint64_t *bits, int64_t k_local, int32_t rank, int32_t world) {
    GUARD(h);
    int rc = check_batch_args(h, k_local, rank, world);
    if (rc) return rc;
    if (!bits && k_local > 0) return fail(h, UBQP_E_INVALID, "ubqp: bits is NULL");
    const size_t bytes = static_cast<size_t>(k_local) * h->W64 * sizeof(uint64_t);
    if (bytes) {
        if (is_device_ptr(bits)) {
            CK(cudaMemcpyAsync(h->Xb, bits, bytes, cudaMemcpyDeviceToDevice, h->stream));
        } else {
            rc = h2d_sync(h, h->Xb, bits, bytes);
            if (rc) return rc;
        }
    }
    h->rank = rank;
    h->world = world;
    h->k_local = k_local;
    h->f_valid = h->gains_valid = h->gains64_valid = false;
    ubqp::launch_expand(*h, k_local);
    CK_LAUNCH("expand_kernel");
    return UBQP_OK;
}

int ubqp_first_derivative(ubqp_t h, uint64_t *bits_out) {
    GUARD(h);
    if (h->n <= 0) return fail(h, UBQP_E_STATE, "ubqp: no Q loaded");
    if (!bits_out) return fail(h, UBQP_E_INVALID, "ubqp: bits_out is NULL");
    const bool dev = is_device_ptr(bits_out);
    uint64_t *dst = dev ? bits_out : h->seed;
    ubqp::launch_first_derivative(*h, dst);
    CK_LAUNCH("first_derivative_kernel");
    if (!dev) {
        CK(cudaMemcpyAsync(bits_out, dst, h->W64 * sizeof(uint64_t), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    }
    return UBQP_OK;
}

int ubqp_get_batch(ubqp_t h, uint64_t *bits_out) {
    GUARD(h);
    if (h->k_local < 0) return fail(h, UBQP_E_STATE, "ubqp: no batch");
    if (!bits_out) return fail(h, UBQP_E_INVALID, "ubqp: bits_out is NULL");
    const size_t bytes = static_cast<size_t>(h->k_local) * h->W64 * sizeof(uint64_t);
    if (!bytes) return UBQP_OK;
    if (is_device_ptr(bits_out)) {
        CK(cudaMemcpyAsync(bits_out, h->Xb, bytes, cudaMemcpyDeviceToDevice, h->stream));
    } else {
        CK(cudaMemcpyAsync(bits_out, h->Xb, bytes, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    }
    return UBQP_OK;
}

int ubqp_eval_batch(ubqp_t h, int flags, int64_t *f_out, ubqp_stats *stats_out) {
    GUARD(h);
    if (h->real) return fail(h, UBQP_E_STATE, "ubqp: real-valued Q loaded: use ubqp_eval_batch_real");
    if (h->k_local < 0) return fail(h, UBQP_E_STATE, "ubqp: no batch to evaluate");
    if (flags & ~UBQP_EMIT_GAINS) return fail(h, UBQP_E_INVALID, "ubqp: unknown flags");
    const int64_t k = h->k_local;
    // device outputs are written by the kernel itself (one launch); host outputs are copied
    const bool f_dev = f_out && is_device_ptr(f_out);
    const bool s_dev = stats_out && is_device_ptr(stats_out);
    int rc = run_eval(h, (flags & UBQP_EMIT_GAINS) != 0, f_dev ? f_out : nullptr,
                      s_dev ? reinterpret_cast<int64_t *>(stats_out) : nullptr);
    if (rc) return rc;
    bool sync = false;
    if (f_out && !f_dev && k > 0) {
        CK(cudaMemcpyAsync(f_out, h->f, k * sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
        sync = true;
    }
    if (stats_out && !s_dev) {
        CK(cudaMemcpyAsync(stats_out, h->scratch64, sizeof(ubqp_stats), cudaMemcpyDeviceToHost, h->stream));
        sync = true;
    }
    if (sync) CK(cudaStreamSynchronize(h->stream));
    return UBQP_OK;
}

int ubqp_get_gains(ubqp_t h, int64_t slot0, int64_t count, int32_t *gains_out) {
    GUARD(h);
    if (!h->gains_valid) return fail(h, UBQP_E_STATE, "ubqp: last eval did not emit gains");
    if (slot0 < 0 || count < 0 || slot0 + count > h->k_local || (!gains_out && count))
        return fail(h, UBQP_E_INVALID, "ubqp: bad gains range");
    if (!count) return UBQP_OK;
    const bool dev = is_device_ptr(gains_out);
    CK(cudaMemcpy2DAsync(gains_out, h->n * sizeof(int32_t), h->gains + slot0 * h->n_pad, h->n_pad * sizeof(int32_t),
                         h->n * sizeof(int32_t), count, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                         h->stream));
    if (!dev) CK(cudaStreamSynchronize(h->stream));
    return UBQP_OK;
}

int ubqp_screen(ubqp_t h, double lambda, int64_t mean_sum, int64_t mean_count, int64_t max_value,
                int32_t *surv_out, int64_t *m_out, double *T_out) {
    GUARD(h);
    if (h->real) return fail(h, UBQP_E_STATE, "ubqp: real-valued Q loaded: use ubqp_screen_real");
    if (!std::isfinite(lambda)) return fail(h, UBQP_E_INVALID, "ubqp: lambda is not finite");
    if (mean_count <= 0) return fail(h, UBQP_E_STATE, "ubqp: mean_count <= 0");
    if (!h->f_valid) return fail(h, UBQP_E_STATE, "ubqp: no evaluated batch");
    if (!m_out || (!surv_out && h->k_local > 0)) return fail(h, UBQP_E_INVALID, "ubqp: null output");
    // T(lambda) = Mean + lambda (Max - Mean), binary64, one rounding per operation
    volatile double mean = static_cast<double>(mean_sum) / static_cast<double>(mean_count);
    volatile double diff = static_cast<double>(max_value) - mean;
    volatile double scaled = lambda * diff;
    const double T = mean + scaled;
    if (T_out) *T_out = T;
    // f > T  <=>  f > floor(T) for integer f; clamp to the int64 range
    int64_t t_floor;
    const double fl = std::floor(T);
    if (std::isnan(T)) return fail(h, UBQP_E_INVALID, "ubqp: T is NaN");
    if (fl >= 9.2233720368547758e18) t_floor = INT64_MAX;
    else if (fl < -9.2233720368547758e18) t_floor = INT64_MIN;
    else t_floor = static_cast<int64_t>(fl);
    const int64_t k = h->k_local;
    CK(ubqp::launch_screen(*h, k, t_floor, h->scratch64 + 4));
    CK_LAUNCH("screen kernels");
    int64_t m = 0;
    CK(cudaMemcpyAsync(&m, h->scratch64 + 4, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (m > 0) {
        const bool dev = is_device_ptr(surv_out);
        if (!dev || surv_out != h->surv) {
            CK(cudaMemcpyAsync(surv_out, h->surv, m * sizeof(int32_t), dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                               h->stream));
            if (!dev) CK(cudaStreamSynchronize(h->stream));
        }
    }
    *m_out = m;
    return UBQP_OK;
}

int ubqp_ascend(ubqp_t h, const int32_t *slots, int64_t m, int32_t max_flips, int64_t *f_out,
                int32_t *flips_out, uint64_t *bits_out, int64_t *best_key_out) {
    GUARD(h);
    if (h->real) return fail(h, UBQP_E_STATE, "ubqp: the ascent runs on integer Q only");
    if (!h->f_valid) return fail(h, UBQP_E_STATE, "ubqp: no evaluated batch");
    if (m < 0 || m > h->k_local || max_flips < 0 || (!slots && m > 0))
        return fail(h, UBQP_E_INVALID, "ubqp: bad ascend arguments");
    if (!h->gains_valid) {
        int rc = run_eval(h, true);     // gains of the whole batch (K-GAIN)
        if (rc) return rc;
    }
    int rc = ensure_asc(h, m > 0 ? m : 1);
    if (rc) return rc;
    // slots
    const int32_t *slots_dev = slots;
    if (m > 0 && !is_device_ptr(slots)) {
        for (int64_t i = 0; i < m; ++i)
            if (slots[i] < 0 || slots[i] >= h->k_local) return fail(h, UBQP_E_INVALID, "ubqp: slot out of range");
        const int rc2 = h2d_sync(h, h->asc_slots, slots, m * sizeof(int32_t));
        if (rc2) return rc2;
        slots_dev = h->asc_slots;
    }
    const bool f_dev = f_out && is_device_ptr(f_out);
    const bool fl_dev = flips_out && is_device_ptr(flips_out);
    const bool b_dev = bits_out && is_device_ptr(bits_out);
    const bool k_dev = best_key_out && is_device_ptr(best_key_out);
    int64_t *f_d = f_dev ? f_out : h->asc_f;
    int32_t *fl_d = fl_dev ? flips_out : h->asc_flips;
    uint64_t *b_d = b_dev ? bits_out : (bits_out ? h->asc_bits : nullptr);
    int64_t *k_d = k_dev ? best_key_out : h->scratch64 + 5;
    CK(cudaMemsetAsync(k_d, 0xFF, sizeof(int64_t), h->stream));     // -1 = none
    if (h->asc_kernel == 2 && !h->ell)
        return fail(h, UBQP_E_STATE, "ubqp: sparse ascent requested but the sparse rows were not built (density > 0.25)");
    if (ubqp::launch_ascend(*h, slots_dev, m, max_flips, f_d, fl_d, b_d, k_d))
        return fail(h, UBQP_E_RANGE, "ubqp: n outside the ascent kernel range");
    CK_LAUNCH("ascend_kernel");
    bool sync = false;
    if (f_out && !f_dev && m) { CK(cudaMemcpyAsync(f_out, f_d, m * 8, cudaMemcpyDeviceToHost, h->stream)); sync = true; }
    if (flips_out && !fl_dev && m) { CK(cudaMemcpyAsync(flips_out, fl_d, m * 4, cudaMemcpyDeviceToHost, h->stream)); sync = true; }
    if (bits_out && !b_dev && m) {
        CK(cudaMemcpyAsync(bits_out, b_d, m * h->W64 * 8, cudaMemcpyDeviceToHost, h->stream));
        sync = true;
    }
    if (best_key_out && !k_dev) { CK(cudaMemcpyAsync(best_key_out, k_d, 8, cudaMemcpyDeviceToHost, h->stream)); sync = true; }
    if (sync) CK(cudaStreamSynchronize(h->stream));
    if (!fl_dev && flips_out) {
        for (int64_t i = 0; i < m; ++i)
            if (flips_out[i] < 0) return fail(h, UBQP_E_INVALID, "ubqp: slot out of range");
    }
    return UBQP_OK;
}

int ubqp_relink(ubqp_t h, const uint64_t *guides, int64_t n_guides, const int32_t *slots, int64_t m,
                int64_t *f_out, int32_t *step_out, int32_t *len_out, uint64_t *bits_out, int64_t *best_key_out) {
    GUARD(h);
    if (h->real) return fail(h, UBQP_E_STATE, "ubqp: path relinking runs on integer Q only");
    if (!h->f_valid) return fail(h, UBQP_E_STATE, "ubqp: no evaluated batch");
    if (m < 0 || m > h->k_local || (!slots && m > 0) || !guides || n_guides < 1 || n_guides > (1ll << 22))
        return fail(h, UBQP_E_INVALID, "ubqp: bad relink arguments");
    if ((2ll * h->n - 1) * h->qmax >= (1ll << 21))
        return fail(h, UBQP_E_RANGE, "ubqp: relinking needs (2n-1)*qmax < 2^21");
    if (!h->gains_valid) {
        int rc = run_eval(h, true);
        if (rc) return rc;
    }
    int rc = ensure_asc(h, m > 0 ? m : 1);
    if (rc) return rc;
    const uint64_t *g_dev = nullptr;
    rc = stage_rows(h, guides, n_guides, h->guides, h->guides_cap, g_dev);
    if (rc) return rc;
    const int32_t *slots_dev = slots;
    if (m > 0 && !is_device_ptr(slots)) {
        for (int64_t i = 0; i < m; ++i)
            if (slots[i] < 0 || slots[i] >= h->k_local) return fail(h, UBQP_E_INVALID, "ubqp: slot out of range");
        const int rc2 = h2d_sync(h, h->asc_slots, slots, m * sizeof(int32_t));
        if (rc2) return rc2;
        slots_dev = h->asc_slots;
    }
    const bool f_dev = f_out && is_device_ptr(f_out);
    const bool s_dev = step_out && is_device_ptr(step_out);
    const bool l_dev = len_out && is_device_ptr(len_out);
    const bool b_dev = bits_out && is_device_ptr(bits_out);
    const bool k_dev = best_key_out && is_device_ptr(best_key_out);
    int64_t *f_d = f_dev ? f_out : h->asc_f;
    int32_t *s_d = s_dev ? step_out : h->asc_aux;
    int32_t *l_d = l_dev ? len_out : h->asc_flips;
    uint64_t *b_d = b_dev ? bits_out : (bits_out ? h->asc_bits : nullptr);
    int64_t *k_d = k_dev ? best_key_out : h->scratch64 + 5;
    CK(cudaMemsetAsync(k_d, 0xFF, sizeof(int64_t), h->stream));     // -1 = none
    if (ubqp::launch_relink(*h, slots_dev, m, g_dev, n_guides, f_d, nullptr, s_d, l_d, b_d, k_d))
        return fail(h, UBQP_E_RANGE, "ubqp: n outside the ascent kernel range");
    CK_LAUNCH("ascend_kernel<relink>");
    bool sync = false;
    if (f_out && !f_dev && m) { CK(cudaMemcpyAsync(f_out, f_d, m * 8, cudaMemcpyDeviceToHost, h->stream)); sync = true; }
    if (step_out && !s_dev && m) { CK(cudaMemcpyAsync(step_out, s_d, m * 4, cudaMemcpyDeviceToHost, h->stream)); sync = true; }
    if (len_out && !l_dev && m) { CK(cudaMemcpyAsync(len_out, l_d, m * 4, cudaMemcpyDeviceToHost, h->stream)); sync = true; }
    if (bits_out && !b_dev && m) {
        CK(cudaMemcpyAsync(bits_out, b_d, m * h->W64 * 8, cudaMemcpyDeviceToHost, h->stream));
        sync = true;
    }
    if (best_key_out && !k_dev) { CK(cudaMemcpyAsync(best_key_out, k_d, 8, cudaMemcpyDeviceToHost, h->stream)); sync = true; }
    if (sync) CK(cudaStreamSynchronize(h->stream));
    if (!l_dev && len_out) {
        for (int64_t i = 0; i < m; ++i)
            if (len_out[i] < 0) return fail(h, UBQP_E_INVALID, "ubqp: slot out of range");
    }
    return UBQP_OK;
}

// ---------------------------------------------------------------- real-valued Q (a4')
}  // extern "C"

namespace {

// R22: exponent of one nonzero coefficient v, |v| = fr 2^ex (fr in [1/2, 1)): the least e
// making v 2^e an integer, capped at 32 - ex, where |v| 2^e >= 2^31 so rounding costs at most
// 2^-32 of |v|.  A float32 coefficient never reaches the cap (24-bit significand): exact.
int coeff_exp(double v, int &ex_out) {
    int ex = 0;
    const double fr = std::frexp(std::fabs(v), &ex);
    const uint64_t M = static_cast<uint64_t>(std::ldexp(fr, 53));   // exact 53-bit integer
    const int tz = __builtin_ctzll(M);
    ex_out = ex;
    return std::min(53 - ex - tz, 32 - ex);
}

// rint(v 2^e) (half to even), exact, for |v 2^e| < 2^100
__int128 scaled_int(double v, int e) {
    if (v == 0.0) return 0;
    int ex = 0;
    const double fr = std::frexp(std::fabs(v), &ex);
    const uint64_t M = static_cast<uint64_t>(std::ldexp(fr, 53));
    const int sh = ex - 53 + e;
    unsigned __int128 r;
    if (sh >= 0) {
        r = static_cast<unsigned __int128>(M) << sh;
    } else {
        const int d = -sh;
        if (d > 63) {
            r = 0;   // |v 2^e| < 2^-10: rounds to 0 (cannot happen for e >= e_v, kept for safety)
        } else {
            const uint64_t q = M >> d, rem = M & ((1ull << d) - 1ull), half = 1ull << (d - 1);
            r = q + ((rem > half || (rem == half && (q & 1ull))) ? 1u : 0u);
        }
    }
    return v < 0 ? -static_cast<__int128>(r) : static_cast<__int128>(r);
}

}  // namespace

extern "C" {

int ubqp_load_Q_real(ubqp_t h, int32_t n, int dtype, const void *Q, int64_t k_max) {
    GUARD(h);
    if (!Q || n < 1 || n > 16384) return fail(h, UBQP_E_INVALID, "ubqp: n must be in [1, 16384]");
    if (dtype != UBQP_F32 && dtype != UBQP_F64) return fail(h, UBQP_E_INVALID, "ubqp: dtype must be UBQP_F32 or UBQP_F64");
    if (k_max < 1 || k_max > (1ll << 22)) return fail(h, UBQP_E_INVALID, "ubqp: k_max must be in [1, 2^22]");
    const int64_t nn = static_cast<int64_t>(n) * n;
    const size_t esz = dtype == UBQP_F32 ? 4 : 8;
    std::vector<unsigned char> raw;
    const void *Qh = Q;
    if (is_device_ptr(Q)) {
        raw.resize(nn * esz);
        CK(cudaMemcpyAsync(raw.data(), Q, nn * esz, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        Qh = raw.data();
    }
    auto at = [&](int64_t idx) -> double {
        return dtype == UBQP_F32 ? static_cast<double>(static_cast<const float *>(Qh)[idx])
                                 : static_cast<const double *>(Qh)[idx];
    };
    double amax = 0.0;
    int e_w = INT_MIN, ex_max = INT_MIN;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const double v = at(static_cast<int64_t>(i) * n + j);
            if (!std::isfinite(v)) return fail(h, UBQP_E_RANGE, "ubqp: non-finite coefficient");
            if (j > i && v != at(static_cast<int64_t>(j) * n + i))
                return fail(h, UBQP_E_NOT_SYMMETRIC, "ubqp: Q is not symmetric");
            if (v != 0.0) {
                int ex = 0;
                e_w = std::max(e_w, coeff_exp(v, ex));
                ex_max = std::max(ex_max, ex);
            }
            amax = std::fabs(v) > amax ? std::fabs(v) : amax;
        }
    // walk image (R20): 28-bit fixed point, |rint(Q 2^e)| <= 2^27 - 1 (four balanced base-128 limbs)
    int e = 0;
    if (amax > 0) {
        e = static_cast<int>(std::floor(std::log2((134217727.0) / amax)));
        while (e > -1000 && std::ldexp(amax, e) > 134217727.0) --e;
        while (std::ldexp(amax, e + 1) <= 134217727.0 && e < 1000) ++e;
    }
    if (e < -900 || e > 900) return fail(h, UBQP_E_RANGE, "ubqp: coefficient scale out of range");
    // evaluation image (R22): exponent e_w, limbs L with max|rint(Q 2^e_w)| <= 126 * 128^(L-1)
    if (e_w == INT_MIN) e_w = 0;   // Q = 0
    int limbs = 1;
    if (ex_max != INT_MIN && ex_max + e_w > 7 * ubqp::kMaxLimbs) {
        limbs = ubqp::kMaxLimbs + 1;   // |V| >= 2^70: beyond any admissible limb count
    } else if (amax > 0) {
        // balanced digits: the lower L-1 digits lie in [-64, 63], so the top one stays within
        // int8 when max|V| <= 126 * 128^(L-1) (L = 1: the value itself, <= 127)
        const __int128 vmax = scaled_int(amax, e_w);
        __int128 cap = 127;
        while (limbs <= ubqp::kMaxLimbs && vmax > cap) {
            ++limbs;
            cap = static_cast<__int128>(126) << (7 * (limbs - 1));
        }
    }
    if (limbs > ubqp::kMaxLimbs || e_w < -900 || e_w > 900)
        return fail(h, UBQP_E_RANGE,
                    "ubqp: coefficient dynamic range too wide: the evaluation image would need more than 10 int8 "
                    "limb planes (70 bits; DESIGN.md R22)");
    CK(cudaStreamSynchronize(h->stream));
    free_all(*h);
    CK(cudaMalloc(&h->scratch64, 32 * sizeof(int64_t)));
    h->n = n;
    h->n_pad = (n + ubqp::kNPadAlign - 1) / ubqp::kNPadAlign * ubqp::kNPadAlign;
    h->q_rows = (n + ubqp::kQRowAlign - 1) / ubqp::kQRowAlign * ubqp::kQRowAlign;
    h->W64 = (n + 63) / 64;
    h->real = true;
    h->q_exp = e;
    h->w_exp = e_w;
    h->w_limbs = limbs;
    h->q_ld = ubqp::ascend_capacity(h->n_pad);
    const size_t plane = static_cast<size_t>(h->q_rows) * h->q_ld;
    const size_t tplane = static_cast<size_t>(h->q_rows) * h->n_pad;
    std::vector<int8_t> L(plane * ubqp::kSlices, 0);
    std::vector<int8_t> W(plane * limbs, 0), WL(tplane * limbs, 0);
    std::vector<int32_t> wdg(static_cast<size_t>(ubqp::kMaxLimbs) * h->q_rows, 0);
    h->qt_ld = ubqp::real_qt_ld(h->n_pad);
    std::vector<int32_t> qt(static_cast<size_t>(h->q_rows) * h->qt_ld, 0), dgt(h->n_pad, 0);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const double q = at(static_cast<int64_t>(i) * n + j);
            long long v = std::llrint(std::ldexp(q, e));
            qt[static_cast<size_t>(i) * h->qt_ld + j] = static_cast<int32_t>(v);
            if (i == j) dgt[i] = static_cast<int32_t>(v);
            for (int sl = 0; sl < ubqp::kSlices; ++sl) {
                const long long r = ((v % 128) + 128) % 128;
                // balanced digits in [-64, 63]; the top digit takes the remainder, which is
                // round(v / 2^21) in [-64, 64] for |v| <= 2^27 - 1 (64 fits int8)
                const long long d = sl == ubqp::kSlices - 1 ? v : (r >= 64 ? r - 128 : r);
                L[sl * plane + static_cast<size_t>(i) * h->q_ld + j] = static_cast<int8_t>(d);
                v = (v - d) / 128;
            }
            // evaluation image: exact balanced base-128 digits of rint(Q 2^e_w), top digit |d| <= 127
            __int128 V = scaled_int(q, e_w);
            for (int sl = 0; sl < limbs; ++sl) {
                const int r = static_cast<int>(((V % 128) + 128) % 128);
                const int d = sl == limbs - 1 ? static_cast<int>(V) : (r >= 64 ? r - 128 : r);
                W[sl * plane + static_cast<size_t>(i) * h->q_ld + j] = static_cast<int8_t>(d);
                if (j <= i) WL[sl * tplane + static_cast<size_t>(i) * h->n_pad + j] = static_cast<int8_t>(d);
                if (i == j) wdg[static_cast<size_t>(sl) * h->q_rows + i] = d;
                V = (V - d) / 128;
            }
        }
    const int64_t nblk = (k_max + 4095) / 4096 + 1;
    h->k_max = k_max;
    h->k_cap_pad = (k_max + ubqp::kBM - 1) / ubqp::kBM * ubqp::kBM;
    bool ok = cudaMalloc(&h->seed, h->W64 * sizeof(uint64_t)) == cudaSuccess &&
              cudaMalloc(&h->zdiag, h->q_rows * sizeof(int32_t)) == cudaSuccess &&
              cudaMalloc(&h->wdiag, wdg.size() * sizeof(int32_t)) == cudaSuccess &&
              cudaMalloc(&h->Xb, k_max * h->W64 * sizeof(uint64_t)) == cudaSuccess &&
              cudaMalloc(&h->X8, h->k_cap_pad * h->n_pad) == cudaSuccess &&
              cudaMalloc(&h->f, k_max * sizeof(int64_t)) == cudaSuccess &&
              cudaMalloc(&h->fs, ubqp::kSlices * k_max * sizeof(int64_t)) == cudaSuccess &&
              cudaMalloc(&h->fint, k_max * sizeof(int64_t)) == cudaSuccess &&
              cudaMalloc(&h->freal, k_max * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&h->surv, k_max * sizeof(int32_t)) == cudaSuccess &&
              cudaMalloc(&h->blk_count, nblk * sizeof(int32_t)) == cudaSuccess;
    for (int sl = 0; ok && sl < ubqp::kSlices; ++sl) ok = cudaMalloc(&h->Qs[sl], plane) == cudaSuccess;
    for (int sl = 0; ok && sl < limbs; ++sl)
        ok = cudaMalloc(&h->Qw[sl], plane) == cudaSuccess && cudaMalloc(&h->QwL[sl], tplane) == cudaSuccess;
    ok = ok && cudaMalloc(&h->Qt, qt.size() * sizeof(int32_t)) == cudaSuccess &&
         cudaMalloc(&h->diagt, dgt.size() * sizeof(int32_t)) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        free_all(*h);
        return fail(h, UBQP_E_NOMEM, "ubqp: cannot allocate the real-Q workspace");
    }
    CK(cudaMemset(h->zdiag, 0, h->q_rows * sizeof(int32_t)));   // walk-plane gains carry no diagonal (R20)
    CK(cudaMemcpy(h->wdiag, wdg.data(), wdg.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->Qt, qt.data(), qt.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->diagt, dgt.data(), dgt.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    const int32_t *zd[1] = {h->zdiag};
    for (int sl = 0; sl < ubqp::kSlices; ++sl) {
        CK(cudaMemcpy(h->Qs[sl], L.data() + sl * plane, plane, cudaMemcpyHostToDevice));
        int8_t *pl[1] = {h->Qs[sl]};
        if (!set_operand(h->op_walk[sl], pl, 1, h->q_ld, false, zd, h->n_pad, h->q_rows)) {
            free_all(*h);
            return fail(h, UBQP_E_CUDA, "ubqp: cuTensorMapEncodeTiled failed");
        }
    }
    const int32_t *wd[ubqp::kMaxLimbs];
    for (int sl = 0; sl < limbs; ++sl) {
        CK(cudaMemcpy(h->Qw[sl], W.data() + sl * plane, plane, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(h->QwL[sl], WL.data() + sl * tplane, tplane, cudaMemcpyHostToDevice));
        wd[sl] = h->wdiag + static_cast<size_t>(sl) * h->q_rows;
    }
    if (!set_operand(h->op_wide, h->QwL, limbs, h->n_pad, true, wd, h->n_pad, h->q_rows)) {
        free_all(*h);
        return fail(h, UBQP_E_CUDA, "ubqp: cuTensorMapEncodeTiled failed");
    }
    CK(cudaMemset(h->X8, 0, h->k_cap_pad * h->n_pad));
    if (!encode_map(&h->tmap_X8, h->X8, h->n_pad, h->k_cap_pad, ubqp::kBM)) {
        free_all(*h);
        return fail(h, UBQP_E_CUDA, "ubqp: cuTensorMapEncodeTiled failed");
    }
    h->k_local = -1;
    CK(cudaDeviceSynchronize());
    return UBQP_OK;
}

int ubqp_eval_batch_real(ubqp_t h, double *f_out, ubqp_stats_real *stats_out) {
    GUARD(h);
    if (!h->real) return fail(h, UBQP_E_STATE, "ubqp: no real-valued Q loaded");
    if (h->k_local < 0) return fail(h, UBQP_E_STATE, "ubqp: no batch to evaluate");
    static_assert(sizeof(ubqp_stats_real) == 6 * sizeof(int64_t), "ubqp_stats_real layout");
    const int64_t k = h->k_local;
    const bool f_dev = f_out && is_device_ptr(f_out);
    const bool s_dev = stats_out && is_device_ptr(stats_out);
    int64_t *st = h->scratch64 + 8;
    if (k == 0) {
        const int64_t z[6] = {0, 0, 0, INT64_MIN, 0, static_cast<int64_t>(static_cast<uint32_t>(h->w_exp))};
        CK(cudaMemcpyAsync(st, z, sizeof z, cudaMemcpyHostToDevice, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    } else {
        // one launch: every limb plane of the evaluation image, f and int128 stats folded in-kernel
        ubqp::EvalLaunch L;
        L.tmX = &h->tmap_X8;
        L.Xb = h->Xb;
        L.k = k;
        L.op = &h->op_wide;
        L.mode = ubqp::kFoldReal;
        L.fr = h->freal;
        L.fr2 = f_dev ? f_out : nullptr;
        L.stats = st;
        L.stats2 = s_dev ? reinterpret_cast<int64_t *>(stats_out) : nullptr;
        L.rank = h->rank;
        L.world = h->world;
        L.shard_b = h->shard_b;
        L.q_exp = h->w_exp;
        const int rc = eval_launch(h, L);
        if (rc) return rc;
    }
    h->freal_valid = true;
    h->gains64_valid = false;
    bool sync = false;
    if (f_out && !f_dev && k > 0) {
        CK(cudaMemcpyAsync(f_out, h->freal, k * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        sync = true;
    }
    if (stats_out && (!s_dev || k == 0)) {
        CK(cudaMemcpyAsync(stats_out, st, sizeof(ubqp_stats_real), s_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                           h->stream));
        sync |= !s_dev;
    }
    if (sync) CK(cudaStreamSynchronize(h->stream));
    return UBQP_OK;
}

int ubqp_screen_real(ubqp_t h, double lambda, double mean, double max_value, int32_t *surv_out,
                     int64_t *m_out, double *T_out) {
    GUARD(h);
    if (!h->real || !h->freal_valid) return fail(h, UBQP_E_STATE, "ubqp: no evaluated real-Q batch");
    if (!std::isfinite(lambda) || !std::isfinite(mean) || !std::isfinite(max_value))
        return fail(h, UBQP_E_INVALID, "ubqp: non-finite screen argument");
    if (!m_out || (!surv_out && h->k_local > 0)) return fail(h, UBQP_E_INVALID, "ubqp: null output");
    volatile double diff = max_value - mean;
    volatile double scaled = lambda * diff;
    const double T = mean + scaled;
    if (T_out) *T_out = T;
    CK(ubqp::launch_screen_real(*h, h->k_local, T, h->scratch64 + 4));
    CK_LAUNCH("screen kernels (real)");
    int64_t m = 0;
    CK(cudaMemcpyAsync(&m, h->scratch64 + 4, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (m > 0) {
        const bool dev = is_device_ptr(surv_out);
        CK(cudaMemcpyAsync(surv_out, h->surv, m * sizeof(int32_t), dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                           h->stream));
        if (!dev) CK(cudaStreamSynchronize(h->stream));
    }
    *m_out = m;
    return UBQP_OK;
}

int ubqp_sync(ubqp_t h) {
    GUARD(h);
    CK(cudaStreamSynchronize(h->stream));
    return UBQP_OK;
}

int ubqp_query(ubqp_t h, int what, int64_t *value) {
    if (!h || !value) return UBQP_E_INVALID;
    switch (what) {
        case UBQP_Q_N: *value = h->n; break;
        case UBQP_Q_NPAD: *value = h->n_pad; break;
        case UBQP_Q_W64: *value = h->W64; break;
        case UBQP_Q_KMAX: *value = h->k_max; break;
        case UBQP_Q_KLOCAL: *value = h->k_local; break;
        case UBQP_Q_LAUNCHES: *value = h->launches; break;
        case UBQP_Q_STREAM: *value = reinterpret_cast<int64_t>(h->stream); break;
        case UBQP_Q_REAL_EXP: *value = h->real ? h->q_exp : 0; break;
        case UBQP_Q_IS_REAL: *value = h->real ? 1 : 0; break;
        case UBQP_Q_EVAL_EXP: *value = h->real ? h->w_exp : 0; break;
        case UBQP_Q_EVAL_LIMBS: *value = h->real ? h->w_limbs : 1; break;
        case UBQP_Q_NNZ: *value = h->nnz; break;
        case UBQP_Q_SPARSE_ROWS: *value = h->ell ? 1 : 0; break;
        case UBQP_Q_SHARD_BLOCK: *value = h->shard_b; break;
        case UBQP_Q_ASCENT_LAST: *value = h->asc_last; break;
        default: return UBQP_E_INVALID;
    }
    return UBQP_OK;
}

int ubqp_set_option(ubqp_t h, int what, int64_t value) {
    GUARD(h);
    switch (what) {
        case UBQP_OPT_ASCENT:
            if (value < 0 || value > 4) return fail(h, UBQP_E_INVALID, "ubqp: UBQP_OPT_ASCENT must be in [0, 4]");
            h->asc_kernel = static_cast<int>(value);
            break;
        case UBQP_OPT_EVAL_PAIR:
            if (value != 0 && value != 1) return fail(h, UBQP_E_INVALID, "ubqp: UBQP_OPT_EVAL_PAIR must be 0 or 1");
            h->eval_pair = value == 1;
            break;
        case UBQP_OPT_SHARD_BLOCK:
            if (value < 1 || value > 4096) return fail(h, UBQP_E_INVALID, "ubqp: UBQP_OPT_SHARD_BLOCK must be in [1, 4096]");
            h->shard_b = static_cast<int>(value);
            break;
        case UBQP_OPT_EVAL_TRI:
            if (value != 0 && value != 1) return fail(h, UBQP_E_INVALID, "ubqp: UBQP_OPT_EVAL_TRI must be 0 or 1");
            h->sym_eval = value == 1;
            break;
        default:
            return fail(h, UBQP_E_INVALID, "ubqp: unknown option");
    }
    return UBQP_OK;
}

int ubqp_ascend_real(ubqp_t h, const int32_t *slots, int64_t m, int32_t max_flips, double *f_out,
                     int64_t *fint_out, int32_t *flips_out, uint64_t *bits_out) {
    GUARD(h);
    if (!h->real) return fail(h, UBQP_E_STATE, "ubqp: no real-valued Q loaded");
    if (!h->freal_valid) return fail(h, UBQP_E_STATE, "ubqp: no evaluated real-Q batch");
    if (m < 0 || m > h->k_local || max_flips < 0 || (!slots && m > 0))
        return fail(h, UBQP_E_INVALID, "ubqp: bad ascend arguments");
    const int64_t k = h->k_local;
    if (!h->gains64_valid && k > 0) {
        int rc = ensure_gains(h);
        if (rc) return rc;
        if (!h->gains64) {
            if (cudaMalloc(&h->gains64, static_cast<size_t>(h->k_max) * h->n_pad * sizeof(int64_t)) != cudaSuccess) {
                cudaGetLastError();
                h->gains64 = nullptr;
                return fail(h, UBQP_E_NOMEM, "ubqp: cannot allocate the int64 gains buffer");
            }
        }
        // walk image (R20): Delta~ = Qt_jj + sum_s 128^s 2 (1 - 2x) Y_s from the four walk planes
        // (zero diagonal) and f~28 = sum_s 128^s x^t L_s x, combined exactly
        for (int sl = 0; sl < ubqp::kSlices; ++sl) {
            ubqp::EvalLaunch L;
            L.tmX = &h->tmap_X8;
            L.Xb = h->Xb;
            L.k = k;
            L.op = &h->op_walk[sl];
            L.emit_gains = true;
            L.mode = ubqp::kFoldPlane;
            L.f = h->fs + sl * h->k_max;
            rc = eval_launch(h, L);
            if (rc) return rc;
            ubqp::launch_gains_combine(*h, k, sl);
            CK_LAUNCH("gains_combine_kernel");
        }
        h->gains64_valid = true;
    }
    int rc = ensure_asc(h, m > 0 ? m : 1);
    if (rc) return rc;
    const int32_t *slots_dev = slots;
    if (m > 0 && !is_device_ptr(slots)) {
        for (int64_t i = 0; i < m; ++i)
            if (slots[i] < 0 || slots[i] >= h->k_local) return fail(h, UBQP_E_INVALID, "ubqp: slot out of range");
        const int rc2 = h2d_sync(h, h->asc_slots, slots, m * sizeof(int32_t));
        if (rc2) return rc2;
        slots_dev = h->asc_slots;
    }
    if (m == 0) return UBQP_OK;
    // device outputs pass through; host outputs go through scratch.  The final bits always land
    // in device memory: f of each local optimum is re-evaluated on the evaluation image (R22).
    const bool f_dev = f_out && is_device_ptr(f_out);
    const bool i_dev = fint_out && is_device_ptr(fint_out);
    const bool fl_dev = flips_out && is_device_ptr(flips_out);
    const bool b_dev = bits_out && is_device_ptr(bits_out);
    double *fr_d = f_dev ? f_out : (f_out ? reinterpret_cast<double *>(h->asc_f) : nullptr);
    int64_t *fi_d = i_dev ? fint_out : nullptr;
    int64_t *fi_host_tmp = nullptr;
    if (fint_out && !i_dev) {
        // second scratch: the per-walk-plane values (fs has kSlices * k_max; fint is already formed)
        fi_d = h->fs;
        fi_host_tmp = fint_out;
    }
    int32_t *fl_d = fl_dev ? flips_out : h->asc_flips;
    uint64_t *b_d = b_dev ? bits_out : h->asc_bits;
    if (ubqp::launch_ascend_real(*h, slots_dev, m, max_flips, nullptr, fi_d, fl_d, b_d))
        return fail(h, UBQP_E_RANGE, "ubqp: n outside the real ascent kernel range");
    CK_LAUNCH("ascend_real_kernel");
    if (fr_d) {
        if (!h->X8r) {
            if (cudaMalloc(&h->X8r, ubqp::kReevalRows * h->n_pad) != cudaSuccess) {
                cudaGetLastError();
                h->X8r = nullptr;
                return fail(h, UBQP_E_NOMEM, "ubqp: cannot allocate the re-evaluation workspace");
            }
            if (!encode_map(&h->tmap_X8r, h->X8r, h->n_pad, ubqp::kReevalRows, ubqp::kBM))
                return fail(h, UBQP_E_CUDA, "ubqp: cuTensorMapEncodeTiled failed");
        }
        for (int64_t c0 = 0; c0 < m; c0 += ubqp::kReevalRows) {
            const int64_t cm = std::min<int64_t>(ubqp::kReevalRows, m - c0);
            ubqp::launch_expand_to(*h, b_d + c0 * h->W64, cm, h->X8r);
            CK_LAUNCH("expand_kernel (re-evaluation)");
            ubqp::EvalLaunch L;
            L.tmX = &h->tmap_X8r;
            L.Xb = b_d + c0 * h->W64;
            L.k = cm;
            L.op = &h->op_wide;
            L.mode = ubqp::kFoldReal;
            L.fr = fr_d + c0;
            L.stats = h->scratch64 + 16;   // not reported
            L.q_exp = h->w_exp;
            rc = eval_launch(h, L);
            if (rc) return rc;
        }
    }
    bool sync = false;
    if (f_out && !f_dev) { CK(cudaMemcpyAsync(f_out, fr_d, m * 8, cudaMemcpyDeviceToHost, h->stream)); sync = true; }
    if (fi_host_tmp) { CK(cudaMemcpyAsync(fi_host_tmp, fi_d, m * 8, cudaMemcpyDeviceToHost, h->stream)); sync = true; }
    if (flips_out && !fl_dev) { CK(cudaMemcpyAsync(flips_out, fl_d, m * 4, cudaMemcpyDeviceToHost, h->stream)); sync = true; }
    if (bits_out && !b_dev) {
        CK(cudaMemcpyAsync(bits_out, b_d, m * h->W64 * 8, cudaMemcpyDeviceToHost, h->stream));
        sync = true;
    }
    if (sync) CK(cudaStreamSynchronize(h->stream));
    if (!fl_dev && flips_out) {
        for (int64_t i = 0; i < m; ++i)
            if (flips_out[i] < 0) return fail(h, UBQP_E_INVALID, "ubqp: slot out of range");
    }
    return UBQP_OK;
}

}  // extern "C"
