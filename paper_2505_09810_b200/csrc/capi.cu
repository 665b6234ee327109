// capi.cu -- extern "C" boundary of liblmc_b200.so (include/lmc_b200.h) and
// the host orchestration of the compress / decompress kernel pipelines.
//
// Single translation unit: the kernels live in compress.cu / decompress.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/lmc_b200.h"
#include "compress.cu"
#include "decompress.cu"

using namespace lmcg;

struct lmcg_ctx {
    int device = 0;
    std::string err;
    CrcTables* d_crc = nullptr;
    // device workspace (grow-only)
    uint8_t* ws = nullptr;
    size_t ws_cap = 0;
    // pinned staging for descriptors
    uint8_t* pin = nullptr;
    size_t pin_cap = 0;
    cudaEvent_t pin_done = nullptr;
    cudaStream_t side = nullptr;          // second stream for kernels that overlap the main chain
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    cudaEvent_t dfork_ev = nullptr, djoin_ev = nullptr;   // decompress: large-record k_decrec on the side stream
    cudaEvent_t dec_done = nullptr;       // end of the last eager decompress (lmcg_decompress_result waits on it)
    int sms = 148;                        // multiprocessors of the device
    // last compress (block_info)
    uint64_t last_nb = 0;
    const BlockMeta* last_meta = nullptr;
    const uint8_t* last_wire = nullptr;
    // host convenience buffers
    uint8_t* d_in = nullptr;
    size_t d_in_cap = 0;
    uint8_t* d_out = nullptr;
    size_t d_out_cap = 0;
    // decompress
    uint8_t* dws = nullptr;   // decompress workspace
    size_t dws_cap = 0;
    uint8_t* hws = nullptr;   // probe workspace
    size_t hws_cap = 0;
    int dn = -1;
    const void* d_sout = nullptr;
    const uint32_t* d_dstatus = nullptr;
    bool dec_attr = false;
    int scandec_occ = 1;
    bool crc_attr = false;
    int ung_occ = 0;                      // resident k_ungroup CTAs (persistent grid)
    bool serial = false;                  // LMCG_SERIAL=1: no side stream (per-kernel timing experiments)
    bool cb_attr = false;
    int crc_fork = 0;                     // LMCG_CRC_FORK: k_crc forks before (0) or after (1) the histogram
    uint8_t* part_ws = nullptr;
    size_t part_ws_cap = 0;
    bool res_attr = false;
    int pair_grid = 0;                    // persistent k_decpair CTAs (each owns a kPairRing slot)
    bool fuse = true;                     // fused decode + ungroup + CRC (k_decpair) for eligible windows
    uint64_t fuse_from = 16384;           // ... in decodes of at least this many record slots (LMCG_FUSE_FROM)
    uint32_t* d_sh992 = nullptr;
    int crc_occ = 1;
    bool enc_attr = false;
    bool hist_attr = false;
    // per-kernel event timing (lmcg_profile)
    bool prof = false;
    std::vector<std::pair<const char*, std::pair<cudaEvent_t, cudaEvent_t>>> prof_pending;
    std::vector<cudaEvent_t> prof_pool;
    std::vector<std::pair<std::string, std::pair<double, uint64_t>>> prof_acc;
};

namespace {

int fail(lmcg_ctx* c, int code, const char* fmt, ...) {
    if (c) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        c->err = buf;
    }
    return code;
}

#define CK(call)                                                                       \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess) return fail(ctx, LMCG_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

int width_of(int et) { return et == 0 ? 1 : (et == 3 ? 4 : 2); }

// ---- host CRC tables
uint32_t h_multmodp(uint32_t a, uint32_t b) {
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = b & 1 ? (b >> 1) ^ 0xEDB88320u : b >> 1;
    }
    return p;
}

static int occupancy(lmcg_ctx* ctx, const void* fn, int threads, size_t smem) {
    int per = 0, dev = ctx->device, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return std::max(1, per) * std::max(1, sms);
}

void build_crc_tables(CrcTables& t) {
    for (uint32_t i = 0; i < 256; i++) {
        uint32_t c = i;
        for (int k = 0; k < 8; k++) c = (c & 1) ? (c >> 1) ^ 0xEDB88320u : c >> 1;
        t.slice[0][i] = c;
    }
    for (int k = 1; k < 4; k++)
        for (int i = 0; i < 256; i++) t.slice[k][i] = (t.slice[k - 1][i] >> 8) ^ t.slice[0][t.slice[k - 1][i] & 0xFF];
    for (int i = 0; i < 256; i++)
        for (int tt = 0; tt < 4; tt++)
            for (int c = 0; c < 8; c++) t.rep4x8[32 * i + 8 * tt + c] = t.slice[tt][i];
    auto shift_table = [&](uint64_t nbytes, uint32_t (*out)[256]) {   // [k][b] = (b << 8k) * x^(8 nbytes)
        uint32_t p = 1u << 31;
        for (uint64_t nn = nbytes, k = 3; nn; nn >>= 1, k++)
            if (nn & 1) p = h_multmodp(t.x2n[k & 63], p);
        for (int k = 0; k < 4; k++)
            for (uint32_t b = 0; b < 256; b++) out[k][b] = b ? h_multmodp(p, b << (8 * k)) : 0;
    };
    t.x2n[0] = 1u << 30;  // x^1
    for (int k = 1; k < 64; k++) t.x2n[k] = h_multmodp(t.x2n[k - 1], t.x2n[k - 1]);
    for (int lvl = 0; lvl < 11; lvl++) {
        const uint64_t nbytes = 16ull << lvl;
        // x^(8 nbytes)
        uint32_t p = 1u << 31;
        uint64_t n = nbytes;
        int k = 3;
        while (n) {
            if (n & 1) p = h_multmodp(t.x2n[k & 63], p);
            n >>= 1;
            k++;
        }
        for (int byte = 0; byte < 4; byte++)
            for (uint32_t b = 0; b < 256; b++) {
                const uint32_t c = b << (8 * byte);
                t.shift[lvl][byte][b] = c ? h_multmodp(p, c) : 0;
            }
    }
    for (int m = 0; m < kPow2Levels; m++) {
        const uint32_t p = t.x2n[m + 3];  // x^(8 * 2^m)
        for (int byte = 0; byte < 4; byte++)
            for (uint32_t b = 0; b < 256; b++) {
                const uint32_t c = b << (8 * byte);
                t.pow2[m][byte][b] = c ? h_multmodp(p, c) : 0;
            }
    }
    shift_table(512, t.sh512);
    shift_table(kHistTileGap, t.shtile);
    shift_table(1024, t.sh1024);
    shift_table(kHistTileGap32, t.shtile32);
}

int ensure_ctx(lmcg_ctx* ctx) {
    CK(cudaSetDevice(ctx->device));
    return LMCG_OK;
}

int grow(lmcg_ctx* ctx, uint8_t** buf, size_t* cap, size_t need) {
    if (need <= *cap) return LMCG_OK;
    if (*buf) {
        CK(cudaDeviceSynchronize());
        CK(cudaFree(*buf));
        *buf = nullptr;
        *cap = 0;
    }
    size_t n = std::max<size_t>(need, 1 << 20);
    n = n + n / 4;
    CK(cudaMalloc(buf, n));
    *cap = n;
    return LMCG_OK;
}

int grow_pinned(lmcg_ctx* ctx, size_t need) {
    if (ctx->pin_done) CK(cudaEventSynchronize(ctx->pin_done));
    if (need <= ctx->pin_cap) return LMCG_OK;
    if (ctx->pin) CK(cudaFreeHost(ctx->pin));
    size_t n = std::max<size_t>(need, 1 << 16);
    n = n + n / 4;
    CK(cudaMallocHost(&ctx->pin, n));
    ctx->pin_cap = n;
    return LMCG_OK;
}

struct Arena {
    size_t off = 0;
    template <class T>
    size_t take(size_t count) {
        off = (off + 255) & ~size_t(255);
        size_t o = off;
        off += count * sizeof(T);
        return o;
    }
};

cudaEvent_t prof_event(lmcg_ctx* ctx) {
    if (!ctx->prof_pool.empty()) {
        cudaEvent_t e = ctx->prof_pool.back();
        ctx->prof_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// Brackets one kernel launch with events when profiling is enabled.
struct ProfScope {
    lmcg_ctx* ctx;
    const char* name;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    ProfScope(lmcg_ctx* c, const char* n, cudaStream_t s) : ctx(c), name(n), st(s) {
        if (ctx->prof) {
            a = prof_event(ctx);
            cudaEventRecord(a, st);
        }
    }
    ~ProfScope() {
        if (ctx->prof) {
            cudaEvent_t b = prof_event(ctx);
            cudaEventRecord(b, st);
            ctx->prof_pending.push_back({name, {a, b}});
        }
    }
};
#define PROF(name) ProfScope prof_scope_##name(ctx, #name, st)

bool host_valid_block(uint64_t b) { return b >= 4096 && b <= (1u << 20) && (b & (b - 1)) == 0; }

// ---------------------------------------------------------------- compress plan
struct CPlan {
    std::vector<StreamDesc> streams;
    std::vector<WinDesc> wins;
    uint64_t nb = 0, nslots = 0, ncrc = 0;
    uint64_t ncrc_k = 0;   // CRC chunks k_crc computes (windows k_hist does not fold)
    uint32_t min_w = 4;
};

void make_plan(const lmcg_tensor* t, int n, const lmcg_options* o, CPlan& P) {
    const uint64_t B = o->block_size, buf = o->buffer_size;
    P.streams.resize(n);
    for (int i = 0; i < n; i++) {
        StreamDesc& sd = P.streams[i];
        const int width = width_of(t[i].element_type);
        const uint32_t w = o->byte_group ? width : 1;
        sd.nbytes = t[i].nbytes;
        sd.blk0 = P.nb;
        sd.win0 = (uint32_t)P.wins.size();
        sd.flags = (o->byte_group ? 1u : 0u) | ((t[i].delta || t[i].prev) ? 2u : 0u);
        sd.et = (uint32_t)t[i].element_type;
        uint32_t nw = 0;
        for (uint64_t woff = 0; woff < t[i].nbytes; woff += buf) {
            WinDesc wd;
            wd.src = static_cast<const uint8_t*>(t[i].data) + woff;
            wd.prev = t[i].prev ? static_cast<const uint8_t*>(t[i].prev) + woff : nullptr;
            wd.W = std::min<uint64_t>(buf, t[i].nbytes - woff);
            wd.w = w;
            wd.n = wd.W / w;
            wd.nblocks = (uint32_t)((wd.W + B - 1) / B);
            if (w == 1) {
                wd.nslots = wd.nblocks;
            } else {
                uint64_t mx = 0;
                for (uint32_t g = 0; g < w; g++) {
                    const uint64_t sg = (g * wd.n + B - 1) / B;
                    const uint64_t sg1 = (g + 1 == w) ? wd.nblocks : ((g + 1) * wd.n + B - 1) / B;
                    mx = std::max<uint64_t>(mx, sg1 - sg);
                }
                wd.nslots = (uint32_t)(mx * w);
            }
            wd.blk0 = P.nb;
            wd.slot0 = P.nslots;
            wd.stream = (uint32_t)i;
            wd.win_local = nw++;
            const bool al = ((uint64_t)wd.src % 16 == 0) && ((uint64_t)wd.prev % 16 == 0);
            wd.vec = al && (w == 1 || wd.W % 16 == 0);
            wd.al16 = al ? 1u : 0u;
            // k_hist folds the CRC when every plane-0 block is whole and on
            // the vector path (its tiles then hold every source byte of the
            // block's element range); k_crc takes the other windows
            wd.hcrc = (wd.vec && wd.W % ((uint64_t)w * B) == 0) ? 1u : 0u;
            wd.cunit = wd.hcrc ? (uint64_t)w * B : kCrcChunk;
            wd.crc0 = P.ncrc;
            P.ncrc += (wd.W + wd.cunit - 1) / wd.cunit;
            if (!wd.hcrc) P.ncrc_k += (wd.W + kCrcChunk - 1) / kCrcChunk;
            P.nb += wd.nblocks;
            P.nslots += wd.nslots;
            P.min_w = std::min(P.min_w, w);
            P.wins.push_back(wd);
        }
        sd.nwin = nw;
        sd.nblk = P.nb - sd.blk0;
    }
}

}  // namespace

extern "C" {

int lmcg_version(void) { return 1; }

lmcg_ctx* lmcg_create(int device) {
    lmcg_ctx* ctx = new lmcg_ctx();
    ctx->device = device;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device) {
        ctx->err = "no CUDA device";
        return ctx;  // compute calls will fail with LMCG_ERR_CUDA
    }
    cudaSetDevice(device);
    CrcTables* h = new CrcTables();
    build_crc_tables(*h);
    if (cudaMalloc(&ctx->d_crc, sizeof(CrcTables)) == cudaSuccess)
        cudaMemcpy(ctx->d_crc, h, sizeof(CrcTables), cudaMemcpyHostToDevice);
    {
        // k_crc's 992-byte shift table: [k][b] = (b << 8k) * x^(8 * 992) mod P
        uint32_t p = 1u << 31;
        for (uint64_t nn = 992, k = 3; nn; nn >>= 1, k++)
            if (nn & 1) p = h_multmodp(h->x2n[k & 63], p);
        std::vector<uint32_t> t(1024);
        for (int k = 0; k < 4; k++)
            for (uint32_t b = 0; b < 256; b++) t[k * 256 + b] = b ? h_multmodp(p, b << (8 * k)) : 0;
        if (ctx->d_crc && cudaMalloc(&ctx->d_sh992, 1024 * sizeof(uint32_t)) == cudaSuccess)
            cudaMemcpy(ctx->d_sh992, t.data(), 1024 * sizeof(uint32_t), cudaMemcpyHostToDevice);
    }
    delete h;
    cudaEventCreateWithFlags(&ctx->pin_done, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->dfork_ev, cudaEventDisableTiming);
    cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, ctx->device);
    cudaEventCreateWithFlags(&ctx->djoin_ev, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->dec_done, cudaEventDisableTiming);
    cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking);
    if (const char* e = getenv("LMCG_SERIAL")) ctx->serial = e[0] == '1';
    if (const char* e = getenv("LMCG_CRC_FORK")) ctx->crc_fork = atoi(e);
    if (const char* e = getenv("LMCG_NOFUSE")) ctx->fuse = e[0] != '1';
    if (const char* e = getenv("LMCG_FUSE_FROM")) ctx->fuse_from = strtoull(e, nullptr, 10);
    return ctx;
}

void lmcg_destroy(lmcg_ctx* ctx) {
    if (!ctx) return;
    if (ctx->d_crc) {
        cudaDeviceSynchronize();
        cudaFree(ctx->d_crc);
        if (ctx->d_sh992) cudaFree(ctx->d_sh992);
        if (ctx->part_ws) cudaFree(ctx->part_ws);
        if (ctx->ws) cudaFree(ctx->ws);
        if (ctx->dws) cudaFree(ctx->dws);
        if (ctx->hws) cudaFree(ctx->hws);
        if (ctx->d_in) cudaFree(ctx->d_in);
        if (ctx->d_out) cudaFree(ctx->d_out);
        if (ctx->pin) cudaFreeHost(ctx->pin);
        if (ctx->pin_done) cudaEventDestroy(ctx->pin_done);
        if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
        if (ctx->join_ev) cudaEventDestroy(ctx->join_ev);
        if (ctx->dfork_ev) cudaEventDestroy(ctx->dfork_ev);
        if (ctx->djoin_ev) cudaEventDestroy(ctx->djoin_ev);
        if (ctx->dec_done) cudaEventDestroy(ctx->dec_done);
        if (ctx->side) cudaStreamDestroy(ctx->side);
    }
    delete ctx;
}

const char* lmcg_last_error(lmcg_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int lmcg_validate_options(const lmcg_options* o, int et, uint64_t nbytes) {
    if (!o || et < 0 || et > 3) return LMCG_ERR_ARGUMENT;
    if (!host_valid_block(o->block_size)) return LMCG_ERR_CONFIG;
    if (o->segment_count < 1) return LMCG_ERR_CONFIG;
    if (o->buffer_size < o->block_size) return LMCG_ERR_CONFIG;
    if (o->buffer_size % (uint64_t)width_of(et)) return LMCG_ERR_CONFIG;
    if (nbytes % (uint64_t)width_of(et)) return LMCG_ERR_ALIGNMENT;
    return LMCG_OK;
}

uint64_t lmcg_compress_bound(const lmcg_tensor* t, int n, const lmcg_options* o) {
    if (!t || !o || n < 0 || !host_valid_block(o->block_size) || o->buffer_size < o->block_size || o->segment_count < 1)
        return 0;
    uint64_t tot = 0;
    const uint64_t B = o->block_size, buf = o->buffer_size;
    for (int i = 0; i < n; i++) {
        const uint64_t nb = t[i].nbytes;
        const uint64_t nwin = (nb + buf - 1) / buf;
        uint64_t blocks = 0;
        if (nwin) blocks = (nwin - 1) * ((buf + B - 1) / B) + ((nb - (nwin - 1) * buf) + B - 1) / B;
        tot += kHeader + nwin * kSegEntry * (uint64_t)o->segment_count + nb + 5 * blocks;
    }
    return tot;
}

static size_t compress_layout(const CPlan& P, int n, size_t* offs /* 16 */) {
    Arena a;
    const uint64_t nb = P.nb;
    const uint64_t ntiles = nb / kScanTile + 1;
    offs[0] = a.take<WinDesc>(P.wins.size() + 1);
    offs[1] = a.take<StreamDesc>(n + 1);
    offs[2] = a.take<uint32_t>(P.nslots + 1);
    offs[3] = a.take<uint32_t>(nb * 256 + 1);
    offs[4] = a.take<uint32_t>(P.ncrc + 1);
    offs[5] = a.take<BlockMeta>(nb + 1);
    offs[6] = a.take<uint8_t>(nb * 128 + 1);
    offs[7] = a.take<uint64_t>(nb + 1);
    offs[8] = a.take<uint64_t>(ntiles);
    offs[9] = a.take<uint32_t>(4);   // ticket, pm_count
    offs[10] = a.take<uint32_t>(nb + 1);
    offs[11] = a.take<uint64_t>(n + 1);
    offs[12] = a.take<uint64_t>(n + 1);
    offs[13] = a.take<uint32_t>(P.ncrc + 1);   // CRC chunk -> window
    return a.off + 256;
}

uint64_t lmcg_compress_workspace(const lmcg_tensor* t, int n, const lmcg_options* o) {
    if (!t || !o || n < 0) return 0;
    CPlan P;
    make_plan(t, n, o, P);
    size_t offs[16];
    return compress_layout(P, n, offs);
}

static int check_compress_args(lmcg_ctx* ctx, const lmcg_tensor* t, int n, const lmcg_options* o) {
    if (!ctx || !o || n < 0 || (n > 0 && !t)) return fail(ctx, LMCG_ERR_ARGUMENT, "bad arguments");
    if (!ctx->d_crc) return fail(ctx, LMCG_ERR_CUDA, "no CUDA device: the LMC B200 path has no CPU fallback");
    if (o->reserved) return fail(ctx, LMCG_ERR_ARGUMENT, "reserved option field must be 0");
    for (int i = 0; i < n; i++) {
        int r = lmcg_validate_options(o, t[i].element_type, t[i].nbytes);
        if (r == LMCG_ERR_CONFIG) return fail(ctx, r, "invalid options (block %u, segments %u, buffer %llu)", o->block_size, o->segment_count, (unsigned long long)o->buffer_size);
        if (r) return fail(ctx, r, "tensor %d: %llu bytes is not a multiple of the element width", i, (unsigned long long)t[i].nbytes);
        if (t[i].nbytes && !t[i].data) return fail(ctx, LMCG_ERR_ARGUMENT, "tensor %d: null data", i);
    }
    return ensure_ctx(ctx);
}

// Kernel sequence of one compress over descriptors already resident on the
// device (workspace laid out by compress_layout).  No host synchronisation:
// capturable in a CUDA graph.
// Part mode (part_out != null, lmcg_compress_part): only blocks [part_lo,
// part_hi) are compressed, their records land back to back in part_out and
// their sizes in d_rec_sizes; no header, segment tables or CRC.
static int compress_launch(lmcg_ctx* ctx, int n, int nwin, uint64_t nb, uint64_t nslots, uint64_t ncrc, uint64_t ncrc_k,
                           uint32_t min_w,
                           const lmcg_options* o, uint8_t* ws, const size_t* offs, void* d_out, uint64_t* d_offsets,
                           uint64_t* d_lengths, cudaStream_t st, uint64_t part_lo = 0, uint64_t part_hi = ~0ull,
                           uint8_t* part_out = nullptr, uint32_t* d_rec_sizes = nullptr) {
    const bool part = part_out != nullptr;
    WinDesc* d_wins = reinterpret_cast<WinDesc*>(ws + offs[0]);
    StreamDesc* d_streams = reinterpret_cast<StreamDesc*>(ws + offs[1]);
    uint32_t* d_slot2win = reinterpret_cast<uint32_t*>(ws + offs[2]);
    uint32_t* d_hist = reinterpret_cast<uint32_t*>(ws + offs[3]);
    uint32_t* d_crcp = reinterpret_cast<uint32_t*>(ws + offs[4]);
    BlockMeta* d_meta = reinterpret_cast<BlockMeta*>(ws + offs[5]);
    uint8_t* d_wire = ws + offs[6];
    uint64_t* d_scan = reinterpret_cast<uint64_t*>(ws + offs[7]);
    uint64_t* d_status = reinterpret_cast<uint64_t*>(ws + offs[8]);
    uint32_t* d_ctr = reinterpret_cast<uint32_t*>(ws + offs[9]);
    uint32_t* d_pmlist = reinterpret_cast<uint32_t*>(ws + offs[10]);
    uint64_t* d_soff = d_offsets ? d_offsets : reinterpret_cast<uint64_t*>(ws + offs[11]);
    uint64_t* d_slen = d_lengths ? d_lengths : reinterpret_cast<uint64_t*>(ws + offs[12]);
    const uint64_t ntiles = (nb + kScanTile - 1) / kScanTile;
    CK(cudaMemsetAsync(d_status, 0, (ntiles + 1) * sizeof(uint64_t), st));
    CK(cudaMemsetAsync(d_ctr, 0, 4 * sizeof(uint32_t), st));
    uint32_t* d_crc2win = reinterpret_cast<uint32_t*>(ws + offs[13]);
    if (nwin) { PROF(k_slotmap); k_slotmap<<<nwin, 256, 0, st>>>(d_wins, nwin, d_slot2win, ncrc ? d_crc2win : nullptr); }
    // k_crc only reads the tensors: it runs on the side stream, overlapping
    // the histogram / codebook / encode chain, and joins before k_frame
    const bool fork = ncrc_k && n && !part;   // (k_hist folds the CRC of the other windows)
    auto launch_crc = [&]() -> int {
        if (!ctx->crc_attr) {
            CK(cudaFuncSetAttribute(k_crc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCrcSmem));
            ctx->crc_occ = occupancy(ctx, (const void*)k_crc, kCrcThreads, kCrcSmem);
            ctx->crc_attr = true;
        }
        if (!ctx->serial) {
            CK(cudaEventRecord(ctx->fork_ev, st));
            CK(cudaStreamWaitEvent(ctx->side, ctx->fork_ev, 0));
        }
        const uint64_t need = ncrc;   // (chunks are dealt CTA-major)
        cudaStream_t sst = ctx->serial ? st : ctx->side;
        ProfScope prof_scope_k_crc(ctx, "k_crc", sst);
        k_crc<<<(unsigned)std::min<uint64_t>(need, (uint64_t)ctx->crc_occ), kCrcThreads, kCrcSmem, sst>>>(
            d_wins, d_crc2win, ncrc, ctx->d_crc, ctx->d_sh992, d_crcp);
        CK(cudaEventRecord(ctx->join_ev, sst));
        return LMCG_OK;
    };
    if (fork && ctx->crc_fork == 0)
        if (int r = launch_crc()) return r;

    if (nslots) {
        PROF(k_hist);
        if (!ctx->hist_attr) {   // (static + dynamic shared memory above 48 KiB)
            CK(cudaFuncSetAttribute(k_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kHistSmem));
            ctx->hist_attr = true;
        }
        k_hist<<<(unsigned)nslots, kThreads, kHistSmem, st>>>(d_wins, d_slot2win, nslots, o->block_size, d_hist, d_meta,
                                                          part ? part_lo : 0, part ? part_hi : ~0ull, ctx->d_crc,
                                                          part ? nullptr : d_crcp);
    }
    if (fork && ctx->crc_fork == 1)
        if (int r = launch_crc()) return r;
    if (nb) {
        if (!ctx->cb_attr) {
            CK(cudaFuncSetAttribute(k_codebook<kCbBlocksLarge>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCbColBytes));
            ctx->cb_attr = true;
        }
        if (nb >= kCbLargeFrom) {
            PROF(k_codebook);
            k_codebook<kCbBlocksLarge><<<(unsigned)((nb + kCbBlocksLarge - 1) / kCbBlocksLarge), kCbWarps * 32, kCbColBytes, st>>>(
                d_hist, nb, d_meta, d_wire, nullptr, nullptr, d_ctr + 1, d_pmlist, part ? part_lo : 0, part ? part_hi : ~0ull);
        } else {
            PROF(k_codebook);
            k_codebook<kCbBlocksSmall><<<(unsigned)((nb + kCbBlocksSmall - 1) / kCbBlocksSmall), kCbWarps * 32,
                                         512 * kCbBlocksSmall * sizeof(uint16_t), st>>>(
                d_hist, nb, d_meta, d_wire, nullptr, nullptr, d_ctr + 1, d_pmlist, part ? part_lo : 0, part ? part_hi : ~0ull);
        }
        { PROF(k_pkgmerge); k_pkgmerge<<<kPmGrid, 32, 0, st>>>(d_hist, d_ctr + 1, d_pmlist, d_meta, d_wire, nullptr); }
    }
    { PROF(k_scan); k_scan<<<(unsigned)std::max<uint64_t>(ntiles, 1), kScanThreads, 0, st>>>(d_meta, nb, d_scan, d_status, d_ctr); }
    if (n && !part) {
        { PROF(k_layout); k_layout<<<1, 1024, 0, st>>>(d_streams, n, o->segment_count, d_scan, d_soff, d_slen); }
    }
    if (nslots) {
        const size_t smem = kEncSmem;
        if (smem > 48 * 1024 && !ctx->enc_attr) {
            CK(cudaFuncSetAttribute(k_encode, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            ctx->enc_attr = true;
        }
        PROF(k_encode);
        k_encode<<<(unsigned)nslots, kThreads, smem, st>>>(d_wins, d_slot2win, nslots, o->block_size, o->segment_count,
                                                         d_streams, d_meta, d_wire, d_scan, d_soff,
                                                         part ? part_out : static_cast<uint8_t*>(d_out),
                                                         part ? part_lo : 0, part ? part_hi : ~0ull);
    }
    if (part) {
        if (part_hi > part_lo)
            k_recsizes<<<(unsigned)((part_hi - part_lo + 255) / 256), 256, 0, st>>>(d_meta, part_lo, part_hi, d_rec_sizes);
    } else if (n) {
        if (fork) CK(cudaStreamWaitEvent(st, ctx->join_ev, 0));
        PROF(k_frame);
        k_frame<<<n, kThreads, 0, st>>>(d_streams, d_wins, o->block_size, o->segment_count, d_scan, d_crcp, ctx->d_crc, d_soff,
                                        static_cast<uint8_t*>(d_out));
    }
    CK(cudaGetLastError());
    ctx->last_nb = nb;
    ctx->last_meta = d_meta;
    ctx->last_wire = d_wire;
    return LMCG_OK;
}

int lmcg_compress(lmcg_ctx* ctx, const lmcg_tensor* t, int n, const lmcg_options* o, void* d_out,
                  uint64_t out_capacity, uint64_t* d_offsets, uint64_t* d_lengths, void* d_workspace,
                  uint64_t workspace_bytes, void* cuda_stream) {
    if (int r = check_compress_args(ctx, t, n, o)) return r;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    if (out_capacity < lmcg_compress_bound(t, n, o)) return fail(ctx, LMCG_ERR_CAPACITY, "output capacity below lmcg_compress_bound");
    CPlan P;
    make_plan(t, n, o, P);
    size_t offs[16];
    const size_t need = compress_layout(P, n, offs);
    uint8_t* ws = static_cast<uint8_t*>(d_workspace);
    if (!ws) {
        if (int r = grow(ctx, &ctx->ws, &ctx->ws_cap, need)) return r;
        ws = ctx->ws;
    } else if (workspace_bytes < need) {
        return fail(ctx, LMCG_ERR_CAPACITY, "workspace of %llu bytes < %llu", (unsigned long long)workspace_bytes, (unsigned long long)need);
    }
    // descriptors -> device through pinned staging
    const size_t wbytes = P.wins.size() * sizeof(WinDesc), sbytes = P.streams.size() * sizeof(StreamDesc);
    if (int r = grow_pinned(ctx, wbytes + sbytes + 64)) return r;
    if (wbytes) memcpy(ctx->pin, P.wins.data(), wbytes);
    if (sbytes) memcpy(ctx->pin + wbytes, P.streams.data(), sbytes);
    if (wbytes) CK(cudaMemcpyAsync(ws + offs[0], ctx->pin, wbytes, cudaMemcpyHostToDevice, st));
    if (sbytes) CK(cudaMemcpyAsync(ws + offs[1], ctx->pin + wbytes, sbytes, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(ctx->pin_done, st));
    return compress_launch(ctx, n, (int)P.wins.size(), P.nb, P.nslots, P.ncrc, P.ncrc_k, P.min_w, o, ws, offs, d_out, d_offsets,
                           d_lengths, st);
}

int lmcg_compress_part(lmcg_ctx* ctx, const lmcg_tensor* t, const lmcg_options* o, uint64_t blk_begin,
                       uint64_t blk_end, void* d_out, uint64_t out_capacity, uint32_t* d_rec_sizes, uint64_t crc_begin,
                       uint64_t crc_end, uint32_t* d_crc, void* cuda_stream) {
    if (int r = check_compress_args(ctx, t, 1, o)) return r;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    CPlan P;
    make_plan(t, 1, o, P);
    if (blk_begin > blk_end || blk_end > P.nb || crc_begin > crc_end || crc_end > t->nbytes ||
        (blk_end > blk_begin && (!d_out || !d_rec_sizes)))
        return fail(ctx, LMCG_ERR_ARGUMENT, "bad part ranges");
    // capacity: the stored-record bound of the blocks in range
    uint64_t need_out = 0;
    for (const WinDesc& wd : P.wins)
        for (uint64_t k = 0; k < wd.nblocks; k++) {
            const uint64_t b = wd.blk0 + k;
            if (b >= blk_begin && b < blk_end) need_out += std::min<uint64_t>(o->block_size, wd.W - k * o->block_size) + 5;
        }
    if (need_out > out_capacity) return fail(ctx, LMCG_ERR_CAPACITY, "part output capacity below %llu", (unsigned long long)need_out);
    size_t offs[16];
    const size_t need = compress_layout(P, 1, offs);
    if (int r = grow(ctx, &ctx->ws, &ctx->ws_cap, need)) return r;
    uint8_t* ws = ctx->ws;
    const size_t wbytes = P.wins.size() * sizeof(WinDesc), sbytes = P.streams.size() * sizeof(StreamDesc);
    if (int r = grow_pinned(ctx, wbytes + sbytes + 64)) return r;
    if (wbytes) memcpy(ctx->pin, P.wins.data(), wbytes);
    if (sbytes) memcpy(ctx->pin + wbytes, P.streams.data(), sbytes);
    if (wbytes) CK(cudaMemcpyAsync(ws + offs[0], ctx->pin, wbytes, cudaMemcpyHostToDevice, st));
    if (sbytes) CK(cudaMemcpyAsync(ws + offs[1], ctx->pin + wbytes, sbytes, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(ctx->pin_done, st));
    if (blk_end > blk_begin) {
        if (int r = compress_launch(ctx, 1, (int)P.wins.size(), P.nb, P.nslots, P.ncrc, P.ncrc_k, P.min_w, o, ws, offs, nullptr,
                                    nullptr, nullptr, st, blk_begin, blk_end, static_cast<uint8_t*>(d_out), d_rec_sizes))
            return r;
    }
    if (!d_crc) return LMCG_OK;
    const uint64_t L = crc_end - crc_begin;
    if (!L) {
        CK(cudaMemsetAsync(d_crc, 0, sizeof(uint32_t), st));
        return LMCG_OK;
    }
    // raw CRC of the element bytes [crc_begin, crc_end): k_crc over one
    // pseudo-window, then one combine
    const uint64_t nchunk = (L + kCrcChunk - 1) / kCrcChunk;
    if (int r = grow(ctx, &ctx->part_ws, &ctx->part_ws_cap, 256 + 8 * (nchunk + 1))) return r;
    WinDesc cw{};
    cw.src = static_cast<const uint8_t*>(t->data) + crc_begin;
    cw.prev = t->prev ? static_cast<const uint8_t*>(t->prev) + crc_begin : nullptr;
    cw.W = L;
    cw.n = L;
    cw.w = 1;
    cw.crc0 = 0;
    cw.cunit = kCrcChunk;
    cw.al16 = ((uint64_t)cw.src % 16 == 0) && ((uint64_t)cw.prev % 16 == 0);
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(ctx->part_ws, &cw, sizeof(WinDesc), cudaMemcpyHostToDevice));
    if (!ctx->crc_attr) {
        CK(cudaFuncSetAttribute(k_crc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCrcSmem));
        ctx->crc_occ = occupancy(ctx, (const void*)k_crc, kCrcThreads, kCrcSmem);
        ctx->crc_attr = true;
    }
    uint32_t* parts = reinterpret_cast<uint32_t*>(ctx->part_ws + 256);
    uint32_t* one_win = parts + nchunk + 1;   // every chunk -> window 0
    CK(cudaMemsetAsync(one_win, 0, 4 * (nchunk + 1), st));
    k_crc<<<(unsigned)std::min<uint64_t>(nchunk, (uint64_t)ctx->crc_occ), kCrcThreads, kCrcSmem, st>>>(
        reinterpret_cast<const WinDesc*>(ctx->part_ws), one_win, nchunk, ctx->d_crc, ctx->d_sh992, parts);
    k_crc_join<<<1, kThreads, 0, st>>>(parts, L, ctx->d_crc, d_crc);
    CK(cudaGetLastError());
    return LMCG_OK;
}

// ---------------------------------------------------------------- plans
struct lmcg_plan {
    int kind = 0;  // 1 compress, 2 decompress
    int n = 0;
    uint8_t* ws = nullptr;
    size_t ws_bytes = 0;
    // compress
    lmcg_options opts{};
    int nwin = 0;
    uint64_t nb = 0, nslots = 0, ncrc = 0, ncrc_k = 0, bound = 0;
    uint32_t min_w = 4;
    size_t offs[16] = {};
    // decompress
    uint64_t dn_win = 0, dn_seg = 0, dn_rec = 0, dn_chunk = 0, dn_tile = 0, out_bytes = 0;
    size_t doffs[20] = {};
    int scandec_grid = 0, fallback_grid = 0;
};

lmcg_plan* lmcg_compress_plan_create(lmcg_ctx* ctx, const lmcg_tensor* t, int n, const lmcg_options* o) {
    if (check_compress_args(ctx, t, n, o)) return nullptr;
    lmcg_plan* pl = new lmcg_plan();
    pl->kind = 1;
    pl->n = n;
    pl->opts = *o;
    CPlan P;
    make_plan(t, n, o, P);
    pl->nwin = (int)P.wins.size();
    pl->nb = P.nb;
    pl->nslots = P.nslots;
    pl->ncrc = P.ncrc;
    pl->ncrc_k = P.ncrc_k;
    pl->min_w = P.min_w;
    pl->bound = lmcg_compress_bound(t, n, o);
    pl->ws_bytes = compress_layout(P, n, pl->offs);
    if (cudaMalloc(&pl->ws, pl->ws_bytes) != cudaSuccess) {
        fail(ctx, LMCG_ERR_CUDA, "cudaMalloc of %zu bytes for a compress plan failed", pl->ws_bytes);
        delete pl;
        return nullptr;
    }
    if (!P.wins.empty()) cudaMemcpy(pl->ws + pl->offs[0], P.wins.data(), P.wins.size() * sizeof(WinDesc), cudaMemcpyHostToDevice);
    if (!P.streams.empty()) cudaMemcpy(pl->ws + pl->offs[1], P.streams.data(), P.streams.size() * sizeof(StreamDesc), cudaMemcpyHostToDevice);
    if (cudaGetLastError() != cudaSuccess) {
        cudaFree(pl->ws);
        delete pl;
        fail(ctx, LMCG_ERR_CUDA, "uploading compress plan descriptors failed");
        return nullptr;
    }
    return pl;
}

int lmcg_copy_to_host(void* h_dst, const void* d_src, uint64_t bytes, void* cuda_stream) {
    if ((bytes && (!h_dst || !d_src)) || bytes > (1u << 20)) return LMCG_ERR_ARGUMENT;
    if (!bytes) return LMCG_OK;
    void* dptr = nullptr;
    if (cudaHostGetDevicePointer(&dptr, h_dst, 0) != cudaSuccess) return LMCG_ERR_ARGUMENT;
    k_small_copy<<<1, 256, 0, static_cast<cudaStream_t>(cuda_stream)>>>(static_cast<uint8_t*>(dptr),
                                                                        static_cast<const uint8_t*>(d_src), bytes);
    return cudaGetLastError() == cudaSuccess ? LMCG_OK : LMCG_ERR_CUDA;
}

uint64_t lmcg_fallback_segments(int reset) {
    unsigned long long v = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&v, lmcg::lmcg_fallback_segs, sizeof(v));
    if (reset) {
        const unsigned long long z = 0;
        cudaMemcpyToSymbol(lmcg::lmcg_fallback_segs, &z, sizeof(z));
    }
    return v;
}

uint64_t lmcg_plan_output_bytes(const lmcg_plan* pl) {
    if (!pl) return 0;
    return pl->kind == 1 ? pl->bound : pl->out_bytes;
}

int lmcg_compress_plan_run(lmcg_ctx* ctx, lmcg_plan* pl, void* d_out, uint64_t out_capacity, uint64_t* d_offsets,
                           uint64_t* d_lengths, void* cuda_stream) {
    if (!ctx || !pl || pl->kind != 1) return fail(ctx, LMCG_ERR_ARGUMENT, "not a compress plan");
    if (out_capacity < pl->bound) return fail(ctx, LMCG_ERR_CAPACITY, "output capacity below the plan's bound");
    if (int r = ensure_ctx(ctx)) return r;
    return compress_launch(ctx, pl->n, pl->nwin, pl->nb, pl->nslots, pl->ncrc, pl->ncrc_k, pl->min_w, &pl->opts, pl->ws, pl->offs, d_out,
                           d_offsets, d_lengths, static_cast<cudaStream_t>(cuda_stream));
}

void lmcg_plan_destroy(lmcg_plan* pl) {
    if (!pl) return;
    if (pl->ws) {
        cudaDeviceSynchronize();
        cudaFree(pl->ws);
    }
    delete pl;
}

int lmcg_set_decode_fusion(lmcg_ctx* ctx, int enable, uint64_t min_records) {
    if (!ctx) return LMCG_ERR_ARGUMENT;
    ctx->fuse = enable != 0;
    ctx->fuse_from = min_records;
    return LMCG_OK;
}

int lmcg_profile(lmcg_ctx* ctx, int enable) {
    if (!ctx) return LMCG_ERR_ARGUMENT;
    ctx->prof = enable != 0;
    return LMCG_OK;
}

int64_t lmcg_profile_report(lmcg_ctx* ctx, char* buf, uint64_t cap) {
    if (!ctx) return -LMCG_ERR_ARGUMENT;
    if (cudaDeviceSynchronize() != cudaSuccess) return -LMCG_ERR_CUDA;
    for (auto& pe : ctx->prof_pending) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, pe.second.first, pe.second.second);
        bool found = false;
        for (auto& a : ctx->prof_acc)
            if (a.first == pe.first) { a.second.first += ms; a.second.second++; found = true; break; }
        if (!found) ctx->prof_acc.push_back({pe.first, {ms, 1}});
        ctx->prof_pool.push_back(pe.second.first);
        ctx->prof_pool.push_back(pe.second.second);
    }
    ctx->prof_pending.clear();
    std::string out;
    for (auto& a : ctx->prof_acc) {
        char line[160];
        snprintf(line, sizeof line, "%s %llu %.6f\n", a.first.c_str(), (unsigned long long)a.second.second, a.second.first);
        out += line;
    }
    if (buf && cap) {
        const size_t k = std::min<size_t>(out.size(), cap - 1);
        memcpy(buf, out.data(), k);
        buf[k] = 0;
    }
    ctx->prof_acc.clear();
    return (int64_t)out.size();
}

int64_t lmcg_block_info(lmcg_ctx* ctx, int32_t* modes, uint32_t* bits, uint32_t* record_sizes, uint8_t* wire,
                        uint32_t* pm_flags, int64_t cap) {
    if (!ctx || !ctx->last_meta) return 0;
    if (cudaDeviceSynchronize() != cudaSuccess) return -LMCG_ERR_CUDA;
    const uint64_t nb = ctx->last_nb;
    std::vector<BlockMeta> m(nb);
    if (nb && cudaMemcpy(m.data(), ctx->last_meta, nb * sizeof(BlockMeta), cudaMemcpyDeviceToHost) != cudaSuccess)
        return -LMCG_ERR_CUDA;
    const uint64_t k = std::min<uint64_t>(nb, (uint64_t)std::max<int64_t>(cap, 0));
    for (uint64_t i = 0; i < k; i++) {
        if (modes) modes[i] = m[i].mode;
        if (bits) bits[i] = m[i].bits;
        if (record_sizes) record_sizes[i] = m[i].recsize;
        if (pm_flags) pm_flags[i] = m[i].pm;
    }
    if (wire && k) cudaMemcpy(wire, ctx->last_wire, k * 128, cudaMemcpyDeviceToHost);
    return (int64_t)nb;
}

int lmcg_build_codebooks(lmcg_ctx* ctx, const uint32_t* d_hists, int nhist, uint8_t* d_lengths, void* cuda_stream) {
    if (!ctx || nhist < 0 || (nhist && (!d_hists || !d_lengths))) return fail(ctx, LMCG_ERR_ARGUMENT, "bad arguments");
    if (!ctx->d_crc) return fail(ctx, LMCG_ERR_CUDA, "no CUDA device");
    if (int r = ensure_ctx(ctx)) return r;
    if (!nhist) return LMCG_OK;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    const size_t need = 256 + (size_t)nhist * 4 + 64;
    if (int r = grow(ctx, &ctx->ws, &ctx->ws_cap, need)) return r;
    uint32_t* d_ctr = reinterpret_cast<uint32_t*>(ctx->ws);
    uint32_t* d_list = reinterpret_cast<uint32_t*>(ctx->ws + 256);
    CK(cudaMemsetAsync(d_ctr, 0, 16, st));
    { PROF(k_codebook); k_codebook<kCbBlocksSmall><<<(nhist + kCbBlocksSmall - 1) / kCbBlocksSmall, kCbWarps * 32, 0, st>>>(d_hists, (uint64_t)nhist, nullptr, nullptr,
                                                                             d_lengths, d_ctr, d_ctr + 1, d_list); }
    { PROF(k_pkgmerge); k_pkgmerge<<<kPmGrid, 32, 0, st>>>(d_hists, d_ctr + 1, d_list, nullptr, nullptr, d_lengths); }
    CK(cudaGetLastError());
    uint32_t flag = 0;
    CK(cudaMemcpyAsync(&flag, d_ctr, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ctx->last_meta = nullptr;
    return (flag & 2u) ? LMCG_ERR_EMPTY : LMCG_OK;
}

// ------------------------------------------------------------------ decompress
namespace {

struct DPlan {
    std::vector<DecCaps> caps;
    uint64_t nwin = 0, nseg = 0, nrec = 0, nchunk = 0, ntile = 0, scratch = 0;
};

void make_dplan(const uint64_t* lens, int n, const lmcg_stream_hint* hints, const uint64_t* out_off,
                uint64_t out_capacity, DPlan& P) {
    P.caps.assign(n, DecCaps{});
    uint64_t packed = 0;
    for (int i = 0; i < n; i++) {
        const lmcg_stream_hint& h = hints[i];
        DecCaps& c = P.caps[i];
        const uint64_t body = lens[i] > kHeader ? lens[i] - kHeader : 0;
        const uint64_t S = std::min<uint64_t>(std::max<uint32_t>(h.segments, 1), body / kSegEntry + 1);
        const uint64_t B = host_valid_block(h.block) ? h.block : 4096;
        uint64_t nw = h.windows ? h.windows : (h.orig + (128ull << 20) - 1) / (128ull << 20);
        nw = std::min<uint64_t>(nw, body / (kSegEntry * S) + 1);
        c.win0 = P.nwin; c.nwin = nw;
        c.seg0 = P.nseg; c.nseg = nw * S;
        c.rec0 = P.nrec; c.nrec = (h.orig + B - 1) / B + c.nseg;
        c.chunk0 = P.nchunk; c.nchunk = (lens[i] + kChunk - 1) / kChunk + c.nseg;
        c.tile0 = P.ntile; c.ntile = (h.orig + kOutTile - 1) / kOutTile + nw;
        c.scratch0 = P.scratch; c.scratch = ((h.orig + 15) & ~15ull) + 16 * nw;
        if (out_off) {
            c.out0 = out_off[i];
            c.out = out_off[i] <= out_capacity ? std::min<uint64_t>(h.orig, out_capacity - out_off[i]) : 0;
        } else {
            c.out0 = packed;
            c.out = packed <= out_capacity ? std::min<uint64_t>(h.orig, out_capacity - packed) : 0;
            packed += (h.orig + 15) & ~15ull;
        }
        P.nwin += c.nwin; P.nseg += c.nseg; P.nrec += c.nrec; P.nchunk += c.nchunk; P.ntile += c.ntile;
        P.scratch += c.scratch;
    }
}

}  // namespace

int lmcg_read_hints(lmcg_ctx* ctx, const void* const* d_streams, const uint64_t* lens, int n, lmcg_stream_hint* hints,
                    void* cuda_stream) {
    if (!ctx || n < 0 || (n && (!d_streams || !lens || !hints))) return fail(ctx, LMCG_ERR_ARGUMENT, "bad arguments");
    if (!ctx->d_crc) return fail(ctx, LMCG_ERR_CUDA, "no CUDA device: the LMC B200 path has no CPU fallback");
    if (int r = ensure_ctx(ctx)) return r;
    if (!n) return LMCG_OK;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    // probe: the parse kernel with empty capacity regions validates headers and
    // tables and reports the exact structure without writing any descriptor
    Arena a;
    const size_t o_in = a.take<DecStreamIn>(n + 1);
    const size_t o_caps = a.take<DecCaps>(n + 1);
    const size_t o_out = a.take<DecStreamOut>(n + 1);
    if (int r = grow(ctx, &ctx->hws, &ctx->hws_cap, a.off + 256)) return r;
    auto* d_in = reinterpret_cast<DecStreamIn*>(ctx->hws + o_in);
    auto* d_caps = reinterpret_cast<DecCaps*>(ctx->hws + o_caps);
    auto* d_sout = reinterpret_cast<DecStreamOut*>(ctx->hws + o_out);
    std::vector<DecStreamIn> in(n);
    for (int i = 0; i < n; i++) in[i] = DecStreamIn{static_cast<const uint8_t*>(d_streams[i]), lens[i], nullptr, 0};
    CK(cudaMemcpyAsync(d_in, in.data(), n * sizeof(DecStreamIn), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(d_caps, 0, n * sizeof(DecCaps), st));
    k_parse<<<(n + 127) / 128, 128, 0, st>>>(d_in, d_caps, n, d_sout, nullptr, nullptr, nullptr, 0);
    CK(cudaGetLastError());
    std::vector<DecStreamOut> so(n);
    CK(cudaMemcpyAsync(so.data(), d_sout, n * sizeof(DecStreamOut), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int i = 0; i < n; i++) {
        lmcg_stream_hint h{};
        if (so[i].status == ST_RETRY || so[i].status == 0) {
            h.orig = so[i].orig;
            h.segments = so[i].segs;
            h.block = so[i].block;
            h.windows = so[i].nwin;
        }
        hints[i] = h;
    }
    return LMCG_OK;
}

namespace {
// Workspace layout of one decompress (offsets into the workspace).
enum { D_IN, D_CAPS, D_SOUT, D_ST, D_WIN, D_SEG, D_CAND, D_CCNT, D_CTOT, D_CPRE, D_SCNT, D_SFAIL, D_RPOS, D_RNEXT, D_LARGE, D_TC, D_MAPS, D_PAIRS, D_RING, D_SCR, D_NOFF };
size_t dec_layout(const DPlan& P, int n, size_t* o, uint64_t ring_bytes) {
    Arena a;
    o[D_IN] = a.take<DecStreamIn>(n + 1);
    o[D_CAPS] = a.take<DecCaps>(n + 1);
    o[D_SOUT] = a.take<DecStreamOut>(n + 1);
    o[D_ST] = a.take<uint32_t>(n + 1);
    o[D_WIN] = a.take<DecWin>(P.nwin + 1);
    o[D_SEG] = a.take<DecSeg>(P.nseg + 1);
    o[D_CAND] = a.take<uint32_t>((P.nchunk + 1) * kWarps * kSpanCap);
    o[D_CCNT] = a.take<uint32_t>((P.nchunk + 1) * kWarps);
    o[D_CTOT] = a.take<uint32_t>(P.nchunk + 1);
    o[D_CPRE] = a.take<uint32_t>(P.nchunk + 1);
    o[D_SCNT] = a.take<uint32_t>(P.nseg + 1);
    o[D_SFAIL] = a.take<uint32_t>(P.nseg + 1);
    o[D_RPOS] = a.take<uint64_t>(P.nrec + 1);
    o[D_RNEXT] = a.take<uint64_t>(P.nrec + 1);
    o[D_LARGE] = a.take<uint32_t>(P.nrec + 2);   // k_classify: count | record slots
    o[D_TC] = a.take<uint32_t>(P.ntile + 1);
    o[D_MAPS] = a.take<uint32_t>(P.nchunk + P.nrec + P.ntile + 3);   // chunk2seg | rec2seg | tile2win
    o[D_PAIRS] = a.take<uint32_t>(P.nrec + P.nrec / 2 + 8);   // k_pairs: ctl[4] | pairs | singles
    o[D_RING] = a.take<uint8_t>(ring_bytes + 256);
    o[D_SCR] = a.take<uint8_t>(P.scratch + 64);
    return a.off + 256;
}
}  // namespace

// Persistent k_decpair grid (resident CTAs; each owns a kPairRing slot of the workspace).
static int ensure_pair_grid(lmcg_ctx* ctx) {
    if (!ctx->pair_grid) {
        const size_t dsm = dec_smem_bytes(kStageSmall);
        CK(cudaFuncSetAttribute(k_decpair, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
        ctx->pair_grid = occupancy(ctx, (const void*)k_decpair, kThreads, dsm);
    }
    return LMCG_OK;
}

// Kernel sequence of one decompress; DecStreamIn and DecCaps are already on
// the device.  No host synchronisation: capturable in a CUDA graph.
static int decompress_launch(lmcg_ctx* ctx, int n, uint64_t nwin, uint64_t nseg, uint64_t nrec, uint64_t nchunk,
                             uint64_t ntile, uint8_t* ws, const size_t* o, void* d_out, int32_t* d_codes,
                             cudaStream_t st) {
    auto* d_in = reinterpret_cast<DecStreamIn*>(ws + o[D_IN]);
    auto* d_caps = reinterpret_cast<DecCaps*>(ws + o[D_CAPS]);
    auto* d_sout = reinterpret_cast<DecStreamOut*>(ws + o[D_SOUT]);
    auto* d_st = reinterpret_cast<uint32_t*>(ws + o[D_ST]);
    auto* d_win = reinterpret_cast<DecWin*>(ws + o[D_WIN]);
    auto* d_seg = reinterpret_cast<DecSeg*>(ws + o[D_SEG]);
    auto* d_cand = reinterpret_cast<uint32_t*>(ws + o[D_CAND]);
    auto* d_ccnt = reinterpret_cast<uint32_t*>(ws + o[D_CCNT]);
    auto* d_ctot = reinterpret_cast<uint32_t*>(ws + o[D_CTOT]);
    auto* d_cpre = reinterpret_cast<uint32_t*>(ws + o[D_CPRE]);
    auto* d_scnt = reinterpret_cast<uint32_t*>(ws + o[D_SCNT]);
    auto* d_sfail = reinterpret_cast<uint32_t*>(ws + o[D_SFAIL]);
    auto* d_rpos = reinterpret_cast<uint64_t*>(ws + o[D_RPOS]);
    auto* d_rnext = reinterpret_cast<uint64_t*>(ws + o[D_RNEXT]);
    auto* d_large = reinterpret_cast<uint32_t*>(ws + o[D_LARGE]);
    auto* d_tc = reinterpret_cast<uint32_t*>(ws + o[D_TC]);
    auto* d_c2s = reinterpret_cast<uint32_t*>(ws + o[D_MAPS]);
    uint32_t* d_r2s = d_c2s + nchunk + 1;
    uint32_t* d_t2w = d_r2s + nrec + 1;
    auto* d_pairs = reinterpret_cast<uint32_t*>(ws + o[D_PAIRS]);
    uint8_t* d_ring = ws + o[D_RING];
    uint8_t* d_scr = ws + o[D_SCR];
    ctx->d_sout = d_sout;
    ctx->d_dstatus = d_st;
    ctx->dn = n;
    CK(cudaMemsetAsync(d_st, 0, (n + 1) * sizeof(uint32_t), st));
    CK(cudaMemsetAsync(d_sfail, 0, (nseg + 1) * sizeof(uint32_t), st));
    if (!n) return LMCG_OK;
    const size_t dsm = dec_smem_bytes(kStageLarge), dsm_small = dec_smem_bytes(kStageSmall);
    constexpr uint64_t kDecSplitFrom = 1024;   // record slots: below, one k_decrec launch
    if (!ctx->dec_attr) {
        CK(cudaFuncSetAttribute(k_decrec, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
        CK(cudaFuncSetAttribute(k_decrec_large, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
        CK(cudaFuncSetAttribute(k_fallback, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
        ctx->dec_attr = true;
    }
    if (int r = ensure_pair_grid(ctx)) return r;
    // fusion pays off when the pairs fill the persistent grid many times over;
    // a small decode keeps more CTAs busy as record-per-CTA + k_ungroup
    const bool fuse = ctx->fuse && nrec >= ctx->fuse_from;
    { PROF(k_parse); k_parse<<<(n + 127) / 128, 128, 0, st>>>(d_in, d_caps, n, d_sout, d_win, d_seg,
                                                            static_cast<const uint8_t*>(d_out), fuse ? 1 : 0); }
    CK(cudaMemsetAsync(d_c2s, 0xFF, (nchunk + nrec + ntile + 3) * sizeof(uint32_t), st));
    if (nseg + nwin) { PROF(k_maps); k_maps<<<(unsigned)(nseg + nwin), 256, 0, st>>>(d_seg, nseg, d_win, nwin, d_c2s, d_r2s, d_t2w); }
    if (nchunk) { PROF(k_cand); k_cand<<<(unsigned)nchunk, kThreads, 0, st>>>(d_seg, d_c2s, nchunk, d_cand, d_ccnt, d_ctot); }
    if (nseg) {
        PROF(k_number);
        k_number<<<(unsigned)std::min<uint64_t>(nseg, 148 * 4), kThreads, 0, st>>>(d_seg, nseg, d_ctot, d_cpre, d_scnt, d_sfail);
    }
    if (nchunk) {
        PROF(k_assign);
        k_assign<<<(unsigned)((nchunk + kWarps - 1) / kWarps), kThreads, 0, st>>>(d_seg, d_c2s, nchunk, d_cand, d_ccnt, d_cpre, d_sfail, d_rpos, d_rnext);
    }
    if (nrec) {
        { PROF(k_verify); k_verify<<<(unsigned)((nrec + 255) / 256), 256, 0, st>>>(d_seg, d_r2s, nrec, d_scnt, d_sfail, d_rpos, d_rnext); }
        if (!ctx->res_attr) {
            CK(cudaFuncSetAttribute(k_resolve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kResSmem));
            ctx->res_attr = true;
        }
        { PROF(k_resolve); k_resolve<<<(unsigned)std::min<uint64_t>(nseg, 148 * 2), kThreads, kResSmem, st>>>(
            d_seg, nseg, d_cand, d_ccnt, d_cpre, d_scnt, d_sfail, d_rpos, d_rnext); }
        // the split pays off inside CUDA graphs (plans); launched eagerly the
        // two kernels overlap worse than one, so eager calls take one launch
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        CK(cudaStreamIsCapturing(st, &cap));
        if (fuse) {
            // k_decpair takes every record: fused pairs, then the records of the other windows
        } else if (nrec < kDecSplitFrom || cap != cudaStreamCaptureStatusActive) {
            PROF(k_decrec);
            k_decrec<<<(unsigned)nrec, kThreads, dsm, st>>>(d_seg, d_r2s, d_win, nrec, d_sfail, d_rpos, d_scr, 0);
        } else {
            PROF(k_decrec);
            // records whose payload does not stage in kStageSmall are listed and
            // decoded by persistent CTAs (3 per SM) on the side stream while the
            // rest run at 4 CTAs per SM
            CK(cudaMemsetAsync(d_large, 0, sizeof(uint32_t), st));
            k_classify<<<(unsigned)((nrec + 255) / 256), 256, 0, st>>>(d_seg, d_r2s, d_win, nrec, d_sfail, d_rpos, d_large + 1, d_large);
            cudaStream_t sst = ctx->serial ? st : ctx->side;
            if (!ctx->serial) {
                CK(cudaEventRecord(ctx->dfork_ev, st));
                CK(cudaStreamWaitEvent(sst, ctx->dfork_ev, 0));
            }
            k_decrec_large<<<(unsigned)std::min<uint64_t>(nrec, (uint64_t)ctx->sms * 3), kThreads, dsm, sst>>>(
                d_seg, d_r2s, d_win, d_large + 1, d_large, d_sfail, d_rpos, d_scr);
            k_decrec<<<(unsigned)nrec, kThreads, dsm_small, st>>>(d_seg, d_r2s, d_win, nrec, d_sfail, d_rpos, d_scr, 1);
            if (!ctx->serial) {
                CK(cudaEventRecord(ctx->djoin_ev, sst));
                CK(cudaStreamWaitEvent(st, ctx->djoin_ev, 0));
            }
        }
        if (fuse) {
            PROF(k_decpair);
            CK(cudaMemsetAsync(d_pairs, 0, 4 * sizeof(uint32_t), st));
            uint32_t* d_plist = d_pairs + 4;
            uint32_t* d_slist = d_plist + nrec / 2 + 2;
            k_pairs<<<(unsigned)((nrec + 255) / 256), 256, 0, st>>>(d_seg, d_r2s, nrec, d_win, d_sfail, d_plist, d_slist, d_pairs);
            k_decpair<<<(unsigned)ctx->pair_grid, kThreads, dsm_small, st>>>(d_seg, d_r2s, d_win, d_plist, d_slist, d_pairs,
                                                                            d_sfail, d_rpos, d_ring, static_cast<uint8_t*>(d_out),
                                                                            ctx->d_crc, ctx->d_sh992, d_tc, d_scr);
        }
    }
    if (nseg) {
        const int grid = (int)std::min<uint64_t>(nseg, 148 * 2);
        PROF(k_fallback);
        k_fallback<<<grid, kThreads, dsm, st>>>(d_seg, nseg, d_sfail, d_st, d_scr);
    }
    if (ntile) {
        if (!ctx->ung_occ) {
            CK(cudaFuncSetAttribute(k_ungroup, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUngSmem));
            ctx->ung_occ = occupancy(ctx, (const void*)k_ungroup, kUngThreads, kUngSmem);
        }
        PROF(k_ungroup);
        k_ungroup<<<(unsigned)std::min<uint64_t>(ntile, (uint64_t)ctx->ung_occ), kUngThreads, kUngSmem, st>>>(
            d_win, d_t2w, ntile, d_scr, static_cast<uint8_t*>(d_out), ctx->d_crc, ctx->d_sh992, d_tc, d_st, d_sfail);
    }
    { PROF(k_finalize); k_finalize<<<n, kThreads, 0, st>>>(d_sout, d_caps, d_win, n, d_tc, ctx->d_crc, d_st, d_in); }
    if (d_codes) k_status<<<(n + 255) / 256, 256, 0, st>>>(d_sout, d_st, n, d_codes);
    CK(cudaGetLastError());
    return LMCG_OK;
}

static int decompress_impl(lmcg_ctx* ctx, const void* const* d_streams, const uint64_t* lens, int n,
                           const lmcg_stream_hint* hints, const void* const* d_prev, const uint64_t* prev_lens,
                           void* d_out, uint64_t out_capacity, const uint64_t* h_out_offsets, void* cuda_stream) {
    if (!ctx || n < 0 || (n && (!d_streams || !lens || !hints))) return fail(ctx, LMCG_ERR_ARGUMENT, "bad arguments");
    if (d_prev && !prev_lens) return fail(ctx, LMCG_ERR_ARGUMENT, "d_prev without prev_lengths");
    if (!ctx->d_crc) return fail(ctx, LMCG_ERR_CUDA, "no CUDA device: the LMC B200 path has no CPU fallback");
    if (int r = ensure_ctx(ctx)) return r;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    DPlan P;
    make_dplan(lens, n, hints, h_out_offsets, out_capacity, P);
    size_t o[D_NOFF];
    if (int r = ensure_pair_grid(ctx)) return r;
    const size_t need = dec_layout(P, n, o, (uint64_t)ctx->pair_grid * kPairRing);
    if (int r = grow(ctx, &ctx->dws, &ctx->dws_cap, need)) return r;
    uint8_t* ws = ctx->dws;
    const size_t hb = (size_t)n * (sizeof(DecStreamIn) + sizeof(DecCaps)) + 64;
    if (int r = grow_pinned(ctx, hb)) return r;
    if (n) {
        DecStreamIn* pin_in = reinterpret_cast<DecStreamIn*>(ctx->pin);
        for (int i = 0; i < n; i++) {
            const uint8_t* pv = d_prev ? static_cast<const uint8_t*>(d_prev[i]) : nullptr;
            pin_in[i] = DecStreamIn{static_cast<const uint8_t*>(d_streams[i]), lens[i], pv, pv ? prev_lens[i] : 0};
        }
        memcpy(ctx->pin + (size_t)n * sizeof(DecStreamIn), P.caps.data(), (size_t)n * sizeof(DecCaps));
        CK(cudaMemcpyAsync(ws + o[D_IN], ctx->pin, (size_t)n * sizeof(DecStreamIn), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(ws + o[D_CAPS], ctx->pin + (size_t)n * sizeof(DecStreamIn), (size_t)n * sizeof(DecCaps),
                           cudaMemcpyHostToDevice, st));
        CK(cudaEventRecord(ctx->pin_done, st));
    }
    if (int r = decompress_launch(ctx, n, P.nwin, P.nseg, P.nrec, P.nchunk, P.ntile, ws, o, d_out, nullptr, st)) return r;
    // lmcg_decompress_result reads the per-stream results after this event: the
    // caller's stream may be a non-blocking one that the legacy default stream
    // (a plain cudaMemcpy) would not wait for
    CK(cudaEventRecord(ctx->dec_done, st));
    return LMCG_OK;
}

int lmcg_decompress(lmcg_ctx* ctx, const void* const* d_streams, const uint64_t* lens, int n,
                    const lmcg_stream_hint* hints, void* d_out, uint64_t out_capacity, const uint64_t* h_out_offsets,
                    void* cuda_stream) {
    return decompress_impl(ctx, d_streams, lens, n, hints, nullptr, nullptr, d_out, out_capacity, h_out_offsets,
                           cuda_stream);
}

int lmcg_decompress_apply(lmcg_ctx* ctx, const void* const* d_streams, const uint64_t* lens, int n,
                          const lmcg_stream_hint* hints, const void* const* d_prev, const uint64_t* prev_lengths,
                          void* d_out, uint64_t out_capacity, const uint64_t* h_out_offsets, void* cuda_stream) {
    if (n && (!d_prev || !prev_lengths)) return fail(ctx, LMCG_ERR_ARGUMENT, "lmcg_decompress_apply needs d_prev and prev_lengths");
    return decompress_impl(ctx, d_streams, lens, n, hints, d_prev, prev_lengths, d_out, out_capacity, h_out_offsets,
                           cuda_stream);
}

lmcg_plan* lmcg_decompress_plan_create(lmcg_ctx* ctx, int n, const lmcg_stream_hint* hints, const uint64_t* len_bounds) {
    if (!ctx || n < 0 || (n && (!hints || !len_bounds))) { fail(ctx, LMCG_ERR_ARGUMENT, "bad arguments"); return nullptr; }
    if (!ctx->d_crc) { fail(ctx, LMCG_ERR_CUDA, "no CUDA device: the LMC B200 path has no CPU fallback"); return nullptr; }
    if (ensure_ctx(ctx)) return nullptr;
    lmcg_plan* pl = new lmcg_plan();
    pl->kind = 2;
    pl->n = n;
    DPlan P;
    make_dplan(len_bounds, n, hints, nullptr, ~0ull, P);
    uint64_t out = 0;
    for (int i = 0; i < n; i++) out += (hints[i].orig + 15) & ~15ull;
    pl->out_bytes = out;
    pl->dn_win = P.nwin; pl->dn_seg = P.nseg; pl->dn_rec = P.nrec; pl->dn_chunk = P.nchunk; pl->dn_tile = P.ntile;
    if (ensure_pair_grid(ctx)) { delete pl; return nullptr; }
    pl->ws_bytes = dec_layout(P, n, pl->doffs, (uint64_t)ctx->pair_grid * kPairRing);
    if (cudaMalloc(&pl->ws, pl->ws_bytes) != cudaSuccess) {
        fail(ctx, LMCG_ERR_CUDA, "cudaMalloc of %zu bytes for a decompress plan failed", pl->ws_bytes);
        delete pl;
        return nullptr;
    }
    if (n) cudaMemcpy(pl->ws + pl->doffs[D_CAPS], P.caps.data(), n * sizeof(DecCaps), cudaMemcpyHostToDevice);
    return pl;
}

int lmcg_decompress_plan_run(lmcg_ctx* ctx, lmcg_plan* pl, const void* d_base, const uint64_t* d_offsets,
                             const uint64_t* d_lengths, void* d_out, int32_t* d_status, void* cuda_stream) {
    if (!ctx || !pl || pl->kind != 2 || (pl->n && (!d_base || !d_offsets || !d_lengths))) return fail(ctx, LMCG_ERR_ARGUMENT, "not a decompress plan");
    if (int r = ensure_ctx(ctx)) return r;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    if (pl->n)
        k_mkin<<<(pl->n + 255) / 256, 256, 0, st>>>(static_cast<const uint8_t*>(d_base), d_offsets, d_lengths, pl->n,
                                                  reinterpret_cast<DecStreamIn*>(pl->ws + pl->doffs[D_IN]));
    return decompress_launch(ctx, pl->n, pl->dn_win, pl->dn_seg, pl->dn_rec, pl->dn_chunk, pl->dn_tile, pl->ws,
                             pl->doffs, d_out, d_status, st);
}

int lmcg_decompress_result(lmcg_ctx* ctx, int n, int32_t* h_status, uint64_t* h_orig, int32_t* h_et, int32_t* h_flags,
                           uint64_t* h_windows) {
    if (!ctx || n != ctx->dn || !ctx->d_sout) return fail(ctx, LMCG_ERR_ARGUMENT, "no decompress to report on");
    if (int r = ensure_ctx(ctx)) return r;
    std::vector<DecStreamOut> so(n);
    std::vector<uint32_t> st(n);
    if (n) {
        CK(cudaEventSynchronize(ctx->dec_done));   // the decompress this reports on has finished
        CK(cudaMemcpy(so.data(), ctx->d_sout, n * sizeof(DecStreamOut), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(st.data(), ctx->d_dstatus, n * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    }
    for (int i = 0; i < n; i++) {
        const uint32_t s = so[i].status | st[i];
        int32_t code = LMCG_OK;
        if (s & ST_UNSUPPORTED) code = LMCG_ERR_UNSUPPORTED;
        else if (s & ST_CORRUPT) code = LMCG_ERR_CORRUPT;
        else if (s & ST_RETRY) code = LMCG_ERR_RETRY;
        else if (s & ST_CAPACITY) code = LMCG_ERR_CAPACITY;
        else if (s & ST_INTEGRITY) code = LMCG_ERR_INTEGRITY;
        else if (s & ST_SHAPE) code = LMCG_ERR_SHAPE;
        if (h_status) h_status[i] = code;
        if (h_orig) h_orig[i] = so[i].orig;
        if (h_et) h_et[i] = (int32_t)so[i].et;
        if (h_flags) h_flags[i] = (int32_t)so[i].flags;
        if (h_windows) h_windows[i] = so[i].nwin;
    }
    return LMCG_OK;
}

// ------------------------------------------------------------ host wrappers
int lmcg_compress_host(lmcg_ctx* ctx, const void* data, uint64_t nbytes, int et, int delta, const lmcg_options* o,
                       void* out, uint64_t out_capacity, uint64_t* out_len) {
    if (!ctx || !o || (nbytes && !data) || !out || !out_len) return fail(ctx, LMCG_ERR_ARGUMENT, "bad arguments");
    if (!ctx->d_crc) return fail(ctx, LMCG_ERR_CUDA, "no CUDA device: the LMC B200 path has no CPU fallback");
    if (int r = lmcg_validate_options(o, et, nbytes)) return fail(ctx, r, "invalid options or alignment");
    if (int r = ensure_ctx(ctx)) return r;
    if (int r = grow(ctx, &ctx->d_in, &ctx->d_in_cap, nbytes + 16)) return r;
    lmcg_tensor t{ctx->d_in, nullptr, nbytes, et, delta};
    const uint64_t bound = lmcg_compress_bound(&t, 1, o);
    if (int r = grow(ctx, &ctx->d_out, &ctx->d_out_cap, bound + 64)) return r;
    if (nbytes) CK(cudaMemcpy(ctx->d_in, data, nbytes, cudaMemcpyHostToDevice));
    if (int r = lmcg_compress(ctx, &t, 1, o, ctx->d_out, ctx->d_out_cap, nullptr, nullptr, nullptr, 0, nullptr)) return r;
    // lengths live in the workspace: recompute pointer by re-deriving the layout
    CPlan P;
    make_plan(&t, 1, o, P);
    size_t offs[16];
    compress_layout(P, 1, offs);
    uint64_t len = 0;
    CK(cudaMemcpy(&len, ctx->ws + offs[12], sizeof(uint64_t), cudaMemcpyDeviceToHost));
    if (len > out_capacity) return fail(ctx, LMCG_ERR_CAPACITY, "stream of %llu bytes exceeds capacity", (unsigned long long)len);
    CK(cudaMemcpy(out, ctx->d_out, len, cudaMemcpyDeviceToHost));
    *out_len = len;
    return LMCG_OK;
}

int lmcg_decompress_host(lmcg_ctx* ctx, const void* stream, uint64_t len, void* out, uint64_t out_capacity,
                         uint64_t* out_len, int32_t* et, int32_t* flags) {
    if (!ctx || (len && !stream) || !out_len) return fail(ctx, LMCG_ERR_ARGUMENT, "bad arguments");
    if (!ctx->d_crc) return fail(ctx, LMCG_ERR_CUDA, "no CUDA device: the LMC B200 path has no CPU fallback");
    if (int r = ensure_ctx(ctx)) return r;
    if (int r = grow(ctx, &ctx->d_in, &ctx->d_in_cap, len + 16)) return r;
    if (len) CK(cudaMemcpy(ctx->d_in, stream, len, cudaMemcpyHostToDevice));
    const void* p = ctx->d_in;
    lmcg_stream_hint h{};
    if (int r = lmcg_read_hints(ctx, &p, &len, 1, &h, nullptr)) return r;
    for (int attempt = 0; attempt < 3; attempt++) {
        if (int r = grow(ctx, &ctx->d_out, &ctx->d_out_cap, h.orig + 64)) return r;
        if (int r = lmcg_decompress(ctx, &p, &len, 1, &h, ctx->d_out, ctx->d_out_cap, nullptr, nullptr)) return r;
        int32_t s = 0, e = 0, f = 0;
        uint64_t orig = 0, nw = 0;
        if (int r = lmcg_decompress_result(ctx, 1, &s, &orig, &e, &f, &nw)) return r;
        if (s == LMCG_ERR_RETRY || s == LMCG_ERR_CAPACITY) {
            h.orig = orig;
            h.windows = nw;
            continue;
        }
        if (s) return fail(ctx, s, s == LMCG_ERR_INTEGRITY ? "payload CRC mismatch" : "stream rejected");
        *out_len = orig;
        if (et) *et = e;
        if (flags) *flags = f;
        if (orig > out_capacity) return fail(ctx, LMCG_ERR_CAPACITY, "payload of %llu bytes exceeds capacity", (unsigned long long)orig);
        if (orig) CK(cudaMemcpy(out, ctx->d_out, orig, cudaMemcpyDeviceToHost));
        return LMCG_OK;
    }
    return fail(ctx, LMCG_ERR_CORRUPT, "stream structure does not converge");
}

#ifdef LMCG_DEBUG
int lmcg_debug_events(unsigned long long* out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, lmcg::lmcg_dbg_ev, sizeof(unsigned long long) * 4096);
    return 0;
}
int lmcg_debug_counters(unsigned long long* out, int reset) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, lmcg::lmcg_dbg, sizeof(unsigned long long) * 32);
    if (reset) {
        unsigned long long z[32] = {0};
        cudaMemcpyToSymbol(lmcg::lmcg_dbg, z, sizeof z);
    }
    return 0;
}
#endif
}  // extern "C"
