// compress.cu -- B200 kernels of the LMC compress path.
//
//   k_slotmap    slot -> window map (planes interleaved per window)
//   k_crc        raw CRC-32 of every 32 KiB chunk of the windows k_hist does
//                not fold (XOR delta applied), on the side stream next to
//                k_hist / k_codebook (stream.py:329); k_frame combines the parts
//   k_hist       K1: fused XOR delta + byte-group gather + per-block 256-bin
//                histogram (entropy.py:53-59, bytegroup.py:39-50,
//                delta.py:18-26); the plane-0 block of a whole-block window
//                also folds the raw CRC of its element range
//   k_codebook   K2: per-block mode + canonical length-limited Huffman lengths
//                (stream.py:161-177, huffman.py:79-137), one warp per block
//   k_pkgmerge   K2b: package-merge for blocks whose Huffman tree exceeds 15
//                bits (huffman.py:140-180), backtracking formulation
//   k_scan       decoupled look-back exclusive scan of record sizes
//   k_layout     per-stream totals and stream offsets in the packed output
//   k_frame      header (with combined CRC) + segment tables (stream.py:100-111,
//                271-284, 344-355)
//   k_encode     K4: canonical codes + bit packing of every record straight
//                from the source tensor (huffman.py:213-255, stream.py:161-177)
#include "lmc_common.cuh"

namespace lmcg {

constexpr int kEncRun = 64;  // k_encode positions per thread per round

// Record sizes of blocks [lo, hi) (lmcg_compress_part).
__global__ void k_recsizes(const BlockMeta* __restrict__ meta, uint64_t lo, uint64_t hi, uint32_t* __restrict__ out) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (lo + i < hi) out[i] = meta[lo + i].recsize;
}

// Bytes from device memory into mapped page-locked host memory (by the SMs).
__global__ void k_small_copy(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, uint64_t n) {
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
    __threadfence_system();
}

constexpr uint32_t kCrcChunk = 32768;   // k_crc's unit

// ------------------------------------------------------------------ slotmap
// Owner maps: block slot -> window (k_hist, k_encode) and CRC chunk ->
// window (k_crc); one load per unit instead of a search.
__global__ void k_slotmap(const WinDesc* __restrict__ wins, int nwin, uint32_t* __restrict__ slot2win,
                          uint32_t* __restrict__ crc2win) {
    int wi = blockIdx.x;
    if (wi >= nwin) return;
    const WinDesc wd = wins[wi];
    for (uint32_t i = threadIdx.x; i < wd.nslots; i += blockDim.x) slot2win[wd.slot0 + i] = (uint32_t)wi;
    if (crc2win) {
        const uint64_t nc = (wd.W + wd.cunit - 1) / wd.cunit;
        for (uint64_t i = threadIdx.x; i < nc; i += blockDim.x) crc2win[wd.crc0 + i] = (uint32_t)wi;
    }
}

// ------------------------------------------------------------------ CRC
// Raw CRC-32 of every 32 KiB chunk of every window's element bytes (the
// payload in original byte order, XOR delta applied), one warp per chunk.
// The warp reads 1 KiB rows (lane l: the 32 bytes at 1024 r + 32 l, two
// 16-byte loads that together cover whole lines) and lane l folds its
// pieces in order: shift by the 992 bytes of the other lanes' pieces (4
// lookups), then the piece by slicing-by-4 through the 32 KiB conflict-free
// layout (CrcTables::rep4x8, Crc4x8Lane: the 32 lanes of every lookup read
// 32 different banks).  Lane l's value ends 32 (31 - l)
// bytes before the chunk end: shift and XOR-reduce.  A short last chunk is
// treated as left-padded with zero bytes, which leave a raw CRC unchanged.
// k_frame combines the chunks (stream.py:329).
constexpr int kCrcThreads = 512;   // up to two CTAs per SM (36 KiB of tables each), leaving
                                   // registers and threads for the histogram / encode CTAs it overlaps
constexpr int kCrcWarps = kCrcThreads / 32;
constexpr size_t kCrcSmem = (256 * 32 + 1024) * sizeof(uint32_t);

__global__ void __launch_bounds__(kCrcThreads, 2) k_crc(const WinDesc* __restrict__ wins, const uint32_t* __restrict__ crc2win, uint64_t nchunk,
                                                const CrcTables* __restrict__ ct, const uint32_t* __restrict__ sh992,
                                                uint32_t* __restrict__ out) {
    extern __shared__ uint32_t tab[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < 256 * 32 / 4; i += kCrcThreads)
        reinterpret_cast<uint4*>(tab)[i] = __ldg(reinterpret_cast<const uint4*>(ct->rep4x8) + i);
    uint32_t* st = tab + 256 * 32;
    for (int i = tid; i < 1024; i += kCrcThreads) st[i] = sh992[i];
    __syncthreads();
    Crc4x8Lane cl;
    cl.init(tab, lane);
    constexpr uint32_t kRows = kCrcChunk / 1024;
    // chunks dealt CTA-major (c = blockIdx.x + gridDim.x * j): small inputs still use every SM
    for (uint64_t j = warp, c = blockIdx.x + (uint64_t)warp * gridDim.x; c < nchunk;
         j += kCrcWarps, c = blockIdx.x + j * gridDim.x) {
        const WinDesc wd = wins[crc2win[c]];
        if (wd.hcrc) continue;   // (k_hist folds this window's CRC)
        const uint64_t off = (c - wd.crc0) * kCrcChunk;
        const uint32_t L = (uint32_t)min((uint64_t)kCrcChunk, wd.W - off);
        const uint32_t Z = kCrcChunk - L;   // leading zero bytes of the padded chunk
        const uint8_t* src = wd.src + off;
        const uint8_t* prv = wd.prev ? wd.prev + off : nullptr;
        const bool vec = wd.al16 && (Z & 15) == 0;
        // two independent Horner chains per lane (rows [0, 16) and [16, 32))
        // for instruction-level parallelism
        auto load_piece = [&](uint32_t r, uint4 a[2]) {
            const uint32_t pb = 1024 * r + 32 * lane;   // padded offset of this lane's piece
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const uint32_t q = pb + 16 * h;
                a[h] = make_uint4(0, 0, 0, 0);
                if (q + 16 <= Z) continue;
                if (vec && q >= Z) {
                    a[h] = __ldg(reinterpret_cast<const uint4*>(src + (q - Z)));
                    if (prv) {
                        const uint4 b = __ldg(reinterpret_cast<const uint4*>(prv + (q - Z)));
                        a[h].x ^= b.x; a[h].y ^= b.y; a[h].z ^= b.z; a[h].w ^= b.w;
                    }
                } else {
                    uint32_t v[4] = {0, 0, 0, 0};
                    for (int i = 0; i < 16; i++) {
                        if (q + i >= Z) {
                            uint32_t x = src[q + i - Z];
                            if (prv) x ^= prv[q + i - Z];
                            v[i >> 2] |= x << (8 * (i & 3));
                        }
                    }
                    a[h] = make_uint4(v[0], v[1], v[2], v[3]);
                }
            }
        };
        auto shift992 = [&](uint32_t x) {
            return st[x & 0xFF] ^ st[256 + ((x >> 8) & 0xFF)] ^ st[512 + ((x >> 16) & 0xFF)] ^ st[768 + (x >> 24)];
        };
        uint32_t ca = 0, cb = 0;
        constexpr uint32_t kHalf = kRows / 2;
        for (uint32_t i = 0; i < kHalf; i++) {
            uint4 a[2], b[2];
            load_piece(i, a);
            load_piece(i + kHalf, b);
            ca = shift992(ca);
            cb = shift992(cb);
            ca = cl.word(ca, a[0].x); cb = cl.word(cb, b[0].x);
            ca = cl.word(ca, a[0].y); cb = cl.word(cb, b[0].y);
            ca = cl.word(ca, a[0].z); cb = cl.word(cb, b[0].z);
            ca = cl.word(ca, a[0].w); cb = cl.word(cb, b[0].w);
            ca = cl.word(ca, a[1].x); cb = cl.word(cb, b[1].x);
            ca = cl.word(ca, a[1].y); cb = cl.word(cb, b[1].y);
            ca = cl.word(ca, a[1].z); cb = cl.word(cb, b[1].z);
            ca = cl.word(ca, a[1].w); cb = cl.word(cb, b[1].w);
        }
        // chain a ends 16 rows (16 KiB) before chain b
        uint32_t crc = crc_shift_tab(&ct->pow2[14][0][0], ca) ^ cb;
        crc = crc_shift_bytes(ct, crc, 32u * (31 - lane));
#pragma unroll
        for (int o = 16; o; o >>= 1) crc ^= __shfl_xor_sync(0xFFFFFFFFu, crc, o);
        if (lane == 0) out[c] = crc;
    }
}

// -------------------------------------------------------------- K1 hist+crc
// One CTA per block slot.  Each warp owns 2 KiB warp-tiles of source bytes,
// read as four fully coalesced 512-byte rows: lane l holds the 16-byte
// pieces at 512 q + 16 l (q = 0..3), i.e. 16/w consecutive grouped positions
// of one plane each.  Fast tiles (entirely inside one plane, 16-byte
// aligned) use vector loads; other tiles gather byte by byte.  Plane-0
// tiles also fold their full elements into the CRC (lane tree over 16-byte
// pieces, then the four rows in order).
// The warp-tiles of one block for element width W (compile-time: the plane
// gather and the per-piece symbol count are then static).
// CRC: (plane-0 blocks of hcrc windows) lane l folds its pieces -- 16 bytes
// at 512 q + 16 l of each of the warp's tiles -- into four chains, one per
// row q (independent table lookups in flight: one chain through all rows was
// bound by the latency of its dependent lookups), each shifted by
// kHistTileGap between the warp's tiles; the chains are merged with 512-byte
// shifts at the end; *last = the warp's last tile.  (One 64-byte run per
// lane and tile instead -- one shift per tile -- measured slower: the strided
// loads cost more than the shifts.)
template <int W, bool CRC, bool P32 = false>
__device__ __forceinline__ uint32_t hist_tiles(const WinDesc& wd, uint64_t p0, uint64_t p1, uint32_t* hist, int lane, int warp,
                                               const Crc4x8Lane& cl, const uint32_t* s512, const uint32_t* sgap,
                                               uint32_t* last) {
    uint32_t ch[4] = {0u, 0u, 0u, 0u};
    auto shift = [](const uint32_t* t, uint32_t x) {
        return t[x & 0xFF] ^ t[256 + ((x >> 8) & 0xFF)] ^ t[512 + ((x >> 16) & 0xFF)] ^ t[768 + (x >> 24)];
    };
    constexpr uint32_t lw = W == 1 ? 0 : (W == 2 ? 1 : 2);
    constexpr uint64_t T = kTileBytes >> lw;    // positions per warp-tile
    constexpr int per = 16 / W;                 // symbols per 16-byte piece
    const uint64_t ntiles = (p1 - p0 + T - 1) / T;
    const uint64_t g0 = plane_of(p0, wd.n, W);
    const bool one = p1 <= (g0 + 1) * wd.n;   // the block lies in one plane (the usual case)
    for (uint64_t t = warp; t < ntiles; t += kWarps) {
        const uint64_t tp = p0 + t * T;
        const uint64_t te = min(tp + T, p1);
        const uint64_t g = one ? g0 : plane_of(tp, wd.n, W);
        const bool fast = wd.vec && (te - tp == T) && (one || te <= (g + 1) * wd.n);
        if (fast) {
            uint4 a[4];
            if (P32) {
                // two 1 KiB rows, lane l holds bytes 32 l .. 32 l + 31 of each (one
                // 256-bit load): one chain per row, one shift per 32 bytes
                const uint64_t base = ((tp - g * wd.n) << lw) + 32ull * lane;
                ldg32x(wd.src, wd.prev, base, a[0], a[1]);
                ldg32x(wd.src, wd.prev, base + 1024, a[2], a[3]);
            } else {
                const uint64_t base = ((tp - g * wd.n) << lw) + 16ull * lane;
#pragma unroll
                for (int q = 0; q < 4; q++) a[q] = ldg16x(wd.src, wd.prev, base + 512ull * q);
            }
            if (CRC && P32) {
#pragma unroll
                for (int q = 0; q < 2; q++) ch[q] = shift(sgap, ch[q]);   // (no-op on the warp's first tile: ch == 0)
#pragma unroll
                for (int h = 0; h < 2; h++) {
#pragma unroll
                    for (int q = 0; q < 2; q++) ch[q] = cl.word(ch[q], a[2 * q + h].x);
#pragma unroll
                    for (int q = 0; q < 2; q++) ch[q] = cl.word(ch[q], a[2 * q + h].y);
#pragma unroll
                    for (int q = 0; q < 2; q++) ch[q] = cl.word(ch[q], a[2 * q + h].z);
#pragma unroll
                    for (int q = 0; q < 2; q++) ch[q] = cl.word(ch[q], a[2 * q + h].w);
                }
                *last = (uint32_t)t;
            } else if (CRC) {
                // four chains (one per row q): independent lookups in flight
#pragma unroll
                for (int q = 0; q < 4; q++) ch[q] = shift(sgap, ch[q]);   // (no-op on the warp's first tile: ch == 0)
#pragma unroll
                for (int q = 0; q < 4; q++) ch[q] = cl.word(ch[q], a[q].x);
#pragma unroll
                for (int q = 0; q < 4; q++) ch[q] = cl.word(ch[q], a[q].y);
#pragma unroll
                for (int q = 0; q < 4; q++) ch[q] = cl.word(ch[q], a[q].z);
#pragma unroll
                for (int q = 0; q < 4; q++) ch[q] = cl.word(ch[q], a[q].w);
                *last = (uint32_t)t;
            }
#pragma unroll
            for (int q = 0; q < 4; q++) {
                uint32_t sy[4];
                piece_symbols(a[q], W, (uint32_t)g, sy);
#pragma unroll
                for (int i = 0; i < per; i++) atomicAdd(&hist[((sy[i >> 2] >> (8 * (i & 3))) & 0xFF) << 5], 1u);
            }
        } else {
            // slow gather: lane owns positions [tp + lane*T/32, ...)
            constexpr uint64_t pl = T / 32;
            const uint64_t a = tp + lane * pl, bnd = min(a + pl, te);
            for (uint64_t p = a; p < bnd; p++) atomicAdd(&hist[gather_byte(wd, p) << 5], 1u);
        }
    }
    // row q + 1's piece lies 512 bytes after row q's (32-byte pieces: two rows, 1024 bytes; s512 is then sh1024)
    if (CRC && P32) return shift(s512, ch[0]) ^ ch[1];
    return CRC ? shift(s512, shift(s512, shift(s512, ch[0]) ^ ch[1]) ^ ch[2]) ^ ch[3] : 0u;
}

// k_hist's dynamic shared memory: rep4x8 | sh512 | shtile (CRC folding) |
// the CTA's bins.  Bin of symbol s for lane l (of any warp): word 32 s + l, so
// lane l only ever touches bank l: the shared atomics of a warp never
// conflict, whatever the symbols (warp-private 256-word bins took 3.1
// wavefronts per atomic on the near-uniform planes, 2 on the exponent planes
// whose symbols 52.. and 180.. share banks).
constexpr int kHistCrcWords = 256 * 32 + 2 * 1024;
constexpr int kHistBinWords = 256 * 32;
constexpr size_t kHistSmem = (size_t)(kHistCrcWords + kHistBinWords) * sizeof(uint32_t);

__global__ void __launch_bounds__(kThreads, 3) k_hist(
    const WinDesc* __restrict__ wins, const uint32_t* __restrict__ slot2win, uint64_t nslots, uint32_t B,
    uint32_t* __restrict__ hist_out, BlockMeta* __restrict__ meta, uint64_t part_lo, uint64_t part_hi,
    const CrcTables* __restrict__ ct, uint32_t* __restrict__ crcpart) {
    extern __shared__ __align__(16) uint32_t crc_tab[];
    uint32_t* const bins = crc_tab + kHistCrcWords;
    __shared__ uint32_t sh_crc;
    const uint64_t slot = blockIdx.x;
    if (slot >= nslots) return;
    const WinDesc wd = wins[slot2win[slot]];
    const int64_t kk = slot_to_block(wd, slot - wd.slot0, B);
    if (kk < 0) return;
    const uint64_t k = (uint64_t)kk;
    if (wd.blk0 + k < part_lo || wd.blk0 + k >= part_hi) return;   // outside the part (lmcg_compress_part)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < kHistBinWords / 4; i += kThreads) reinterpret_cast<uint4*>(bins)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();

    const uint64_t p0 = k * B;
    const uint64_t p1 = min(wd.W, p0 + B);
    if (tid == 32 && p1 <= (plane_of(p0, wd.n, wd.w) + 1) * wd.n) {
        // the block's source elements (one plane): on their way to L2 before the first loads
        const uint64_t e0 = p0 - plane_of(p0, wd.n, wd.w) * wd.n;
        prefetch_l2(wd.src + e0 * wd.w, (uint32_t)((p1 - p0) * wd.w));
        if (wd.prev) prefetch_l2(wd.prev + e0 * wd.w, (uint32_t)((p1 - p0) * wd.w));
    }
    // the plane-0 block of an hcrc window folds the raw CRC of its element
    // range (every source byte of it passes through its tiles); part runs
    // (lmcg_compress_part) take their CRC from k_crc
    const bool crc = wd.hcrc && p1 <= wd.n && crcpart != nullptr;
    // 16-bit elements at 32-byte aligned addresses: 32-byte lane pieces (256-bit loads, half the chain shifts)
    const bool p32 = crc && wd.w == 2 && (reinterpret_cast<uint64_t>(wd.src) & 31) == 0 &&
                     (!wd.prev || (reinterpret_cast<uint64_t>(wd.prev) & 31) == 0);
    Crc4x8Lane cl;
    uint32_t ch = 0, last = 0;
    if (crc) {
        for (int i = tid; i < kHistCrcWords / 4; i += kThreads)
            reinterpret_cast<uint4*>(crc_tab)[i] = i < 256 * 32 / 4 ? __ldg(reinterpret_cast<const uint4*>(ct->rep4x8) + i)
                                                                   : __ldg(reinterpret_cast<const uint4*>(p32 ? &ct->sh1024[0][0] : &ct->sh512[0][0]) + (i - 256 * 32 / 4));
        if (tid == 0) sh_crc = 0;
        __syncthreads();
        cl.init(crc_tab, lane);
        const uint32_t* s512 = crc_tab + 256 * 32;
        const uint32_t* sgap = s512 + 1024;
        if (wd.w == 1) ch = hist_tiles<1, true>(wd, p0, p1, bins + lane, lane, warp, cl, s512, sgap, &last);
        else if (wd.w == 2) ch = p32 ? hist_tiles<2, true, true>(wd, p0, p1, bins + lane, lane, warp, cl, s512, sgap, &last)
                                     : hist_tiles<2, true>(wd, p0, p1, bins + lane, lane, warp, cl, s512, sgap, &last);
        else ch = hist_tiles<4, true>(wd, p0, p1, bins + lane, lane, warp, cl, s512, sgap, &last);
        // lane l's chain ends 1536 + 16 (l + 1) (32-byte pieces: 1024 + 32 (l +
        // 1)) bytes into the warp's last tile: a Horner tree over the lanes
        // (fixed shifts of 16 << k or 32 << k bytes), then lane 31 shifts the
        // warp's value to the end of the block
        const uint32_t Lb = (uint32_t)((p1 - p0) * wd.w);
        uint32_t x = ch;
#pragma unroll
        for (int q = 0; q < 5; q++) {
            const uint32_t y = crc_shift_tab(&ct->shift[q + (p32 ? 1 : 0)][0][0], __shfl_xor_sync(0xFFFFFFFFu, x, 1 << q));
            if (lane & (1 << q)) x ^= y;
        }
        if (lane == 31) {
            x = crc_shift_bytes(ct, x, Lb - (last + 1) * kTileBytes);
            if (x) atomicXor(&sh_crc, x);
        }
    } else {
        if (wd.w == 1) hist_tiles<1, false>(wd, p0, p1, bins + lane, lane, warp, cl, nullptr, nullptr, &last);
        else if (wd.w == 2) hist_tiles<2, false>(wd, p0, p1, bins + lane, lane, warp, cl, nullptr, nullptr, &last);
        else hist_tiles<4, false>(wd, p0, p1, bins + lane, lane, warp, cl, nullptr, nullptr, &last);
    }
    __syncthreads();
    if (crc && tid == 0) crcpart[wd.crc0 + k] = sh_crc;
    // block histogram
    const uint64_t b = wd.blk0 + k;
    {
        uint32_t sum = 0;   // thread s sums symbol s's 32 lane counters, skewed across the banks
#pragma unroll
        for (int q = 0; q < 32; q++) sum += bins[32 * tid + ((q + tid) & 31)];
        hist_out[b * 256 + tid] = sum;
    }
    if (tid == 0) {
        BlockMeta m;
        m.len = (uint32_t)(p1 - p0);
        m.recsize = 0; m.bits = 0; m.mode = 0; m.sym = 0; m.pm = 0; m.pad = 0;
        meta[b] = m;
    }
}

// ------------------------------------------------------------ K2 codebook
// Warp-level bitonic sort of 32 K keys (K per lane, lane-major: element
// i = lane K + r), ascending.
template <int K, class T>
__device__ __forceinline__ void warp_bitonic_sort(T key[K], int lane) {
#pragma unroll
    for (int kk = 2; kk <= 32 * K; kk <<= 1) {
#pragma unroll
        for (int j = kk >> 1; j > 0; j >>= 1) {
            if (j >= K) {
                const int lj = j / K;
#pragma unroll
                for (int r = 0; r < K; r++) {
                    const int i = lane * K + r;
                    const T other = __shfl_xor_sync(0xFFFFFFFFu, key[r], lj);
                    const bool up = (i & kk) == 0;
                    const bool lower = (i & j) == 0;
                    // lower element keeps min when ascending
                    const T mn = min(key[r], other), mx = max(key[r], other);
                    key[r] = (lower == up) ? mn : mx;
                }
            } else {
#pragma unroll
                for (int r = 0; r < K; r++) {
                    const int partner = r ^ j;
                    if (partner > r) {
                        const int i = lane * K + r;
                        const bool up = (i & kk) == 0;
                        const T a = key[r], c = key[partner];
                        if ((a > c) == up) { key[r] = c; key[partner] = a; }
                    }
                }
            }
        }
    }
}

struct alignas(16) CbSmem {
    uint32_t wt[512];     // node weights (leaves sorted, then internal nodes)
    uint16_t par[512];    // parent / ancestor
    uint8_t dep[512];     // depth accumulator
    uint8_t sym[256];     // leaf -> symbol
    uint8_t lens[256];    // symbol -> code length
};

// Two-queue Huffman (huffman.py:106-137) on the sorted leaves in s.wt[0..n),
// then leaf depths by pointer jumping.  Returns the maximum leaf depth.
__device__ int huffman_depths_warp(CbSmem& s, int n, int lane) {
    if (lane == 0) {
        const int total = 2 * n - 1;
        int leaf = 0, node = n;
        for (int nxt = n; nxt < total; nxt++) {
            uint32_t acc = 0;
#pragma unroll
            for (int q = 0; q < 2; q++) {
                int child;
                if (leaf < n && (node >= nxt || s.wt[leaf] <= s.wt[node])) child = leaf++;
                else child = node++;
                s.par[child] = (uint16_t)nxt;
                acc += s.wt[child];
            }
            s.wt[nxt] = acc;
        }
        s.par[total - 1] = (uint16_t)(total - 1);
    }
    __syncwarp();
    const int total = 2 * n - 1;
    for (int i = lane; i < total; i += 32) s.dep[i] = (i == total - 1) ? 0 : 1;
    __syncwarp();
    // pointer jumping: depth(i) = hops to the root
    for (int it = 0; it < 9; it++) {
        uint16_t na[16]; uint8_t nd[16];
        int c = 0;
        for (int i = lane; i < total; i += 32, c++) {
            const int a = s.par[i];
            na[c] = s.par[a];
            nd[c] = (uint8_t)(s.dep[i] + s.dep[a]);
        }
        __syncwarp();
        c = 0;
        for (int i = lane; i < total; i += 32, c++) { s.par[i] = na[c]; s.dep[i] = nd[c]; }
        __syncwarp();
    }
    int mx = 0;
    for (int i = lane; i < n; i += 32) mx = max(mx, (int)s.dep[i]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    return mx;
}

// Mode, bit cost, record size and 128-byte wire codebook from s.lens
// (stream.py:170-177, huffman.py:369-377).
__device__ void finish_block(CbSmem& s, const uint32_t cnt[8], int lane, BlockMeta* __restrict__ meta,
                             uint8_t* __restrict__ wire, uint64_t b) {
    uint32_t cost = 0;
#pragma unroll
    for (int r = 0; r < 8; r++) cost += cnt[r] * s.lens[lane * 8 + r];
#pragma unroll
    for (int o = 16; o; o >>= 1) cost += __shfl_xor_sync(0xFFFFFFFFu, cost, o);
    const uint32_t len = meta[b].len;
    const uint32_t hsize = kHuffOverhead + (cost + 7) / 8;
    const bool huff = hsize <= len;
    if (huff) {
        uint32_t wv = 0;
#pragma unroll
        for (int q = 0; q < 4; q++)
            wv |= (uint32_t)(s.lens[lane * 8 + 2 * q] | (s.lens[lane * 8 + 2 * q + 1] << 4)) << (8 * q);
        reinterpret_cast<uint32_t*>(wire + b * 128)[lane] = wv;
    }
    if (lane == 0) {
        BlockMeta m = meta[b];
        m.mode = huff ? MODE_HUFFMAN : MODE_STORED;
        m.bits = cost;
        m.recsize = huff ? 5 + hsize : 5 + len;
        m.pm = 0;
        meta[b] = m;
    }
}

// Sorted (count, symbol) leaves of one histogram; returns n present.  Keys
// are (count << 8) | symbol: 32-bit while counts < 2^24 (every record block:
// at most 1 MiB), 64-bit otherwise (stage-level histograms).  Only the
// present symbols are sorted: they are compacted (in symbol order) into
// `keys` (>= 2 KiB of scratch), then sorted as 64 or 256 keys.
template <int K, class T>
__device__ __forceinline__ void sort_compact(const T* keys, int np, int lane, uint32_t* wt, uint8_t* sym) {
    T key[K];
#pragma unroll
    for (int r = 0; r < K; r++) key[r] = lane * K + r < np ? keys[lane * K + r] : ~(T)0;
    warp_bitonic_sort<K, T>(key, lane);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < K; r++) {
        const int i = lane * K + r;
        if (i < np) { wt[i] = (uint32_t)(key[r] >> 8); sym[i] = (uint8_t)(key[r] & 0xFF); }
    }
}

template <class T>
__device__ __forceinline__ void compact_sort(const uint32_t cnt[8], int lane, int pre, int np, uint32_t* wt, uint8_t* sym,
                                             T* keys) {
#pragma unroll
    for (int r = 0; r < 8; r++)
        if (cnt[r]) keys[pre++] = ((T)cnt[r] << 8) | (T)(lane * 8 + r);
    __syncwarp();
    if (np <= 64) sort_compact<2, T>(keys, np, lane, wt, sym);
    else sort_compact<8, T>(keys, np, lane, wt, sym);
}

__device__ __noinline__ int sorted_leaves(const uint32_t cnt[8], int lane, uint32_t* wt, uint8_t* sym, void* keys) {
    int c = 0;
    uint32_t mx = 0;
#pragma unroll
    for (int r = 0; r < 8; r++) { c += cnt[r] ? 1 : 0; mx = max(mx, cnt[r]); }
    int pre = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xFFFFFFFFu, pre, o);
        if (lane >= o) pre += y;
    }
    const int np = __shfl_sync(0xFFFFFFFFu, pre, 31);
    pre -= c;
    if (__any_sync(0xFFFFFFFFu, mx >= (1u << 24))) compact_sort<uint64_t>(cnt, lane, pre, np, wt, sym, static_cast<uint64_t*>(keys));
    else compact_sort<uint32_t>(cnt, lane, pre, np, wt, sym, static_cast<uint32_t*>(keys));
    __syncwarp();
    return np;
}

constexpr int kCbWarps = 8;
// Blocks per CTA: 8 (one per warp: the most blocks in flight, for small
// inputs) or 16 (large inputs: the deferred cost pass keeps 16 lanes busy)
constexpr int kCbBlocksSmall = 8, kCbBlocksLarge = 16;
constexpr uint64_t kCbLargeFrom = 65536;   // blocks
constexpr int kDeferMin = 96;   // blocks with this many symbols defer their mode decision
constexpr size_t kCbColBytes = 512 * kCbBlocksLarge * sizeof(uint16_t);

// Mode, code lengths and wire codebook of block b (stream.py:161-177,
// huffman.py:79-137), warp-wide.  With `col` (record path only), a block of
// >= kDeferMin symbols stops after sorting: its sorted weights go to column
// `col` (u16, stride NB) and the symbol count is returned, for the cost pass.
template <int NB>
__device__ int cb_block(CbSmem& s, uint64_t b, int lane, const uint32_t* __restrict__ hist, BlockMeta* __restrict__ meta,
                        uint8_t* __restrict__ wire, uint8_t* __restrict__ lens_out, uint32_t* __restrict__ pm_flag,
                        uint32_t* __restrict__ pm_count, uint32_t* __restrict__ pm_list, uint16_t* col) {
    uint32_t cnt[8];
    {
        const uint4* h4 = reinterpret_cast<const uint4*>(hist + b * 256 + lane * 8);
        uint4 a = h4[0], c = h4[1];
        cnt[0] = a.x; cnt[1] = a.y; cnt[2] = a.z; cnt[3] = a.w;
        cnt[4] = c.x; cnt[5] = c.y; cnt[6] = c.z; cnt[7] = c.w;
    }
    uint32_t mx = 0, total = 0;
    int arg = 0;
#pragma unroll
    for (int r = 0; r < 8; r++) {
        total += cnt[r];
        if (cnt[r] > mx) { mx = cnt[r]; arg = lane * 8 + r; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        total += __shfl_xor_sync(0xFFFFFFFFu, total, o);
        uint32_t om = __shfl_xor_sync(0xFFFFFFFFu, mx, o);
        int oa = __shfl_xor_sync(0xFFFFFFFFu, arg, o);
        if (om > mx || (om == mx && oa < arg)) { mx = om; arg = oa; }
    }
    if (lens_out == nullptr && mx == total) {
        // monosymbolic block -> RLE record of 6 bytes (stream.py:165-169)
        if (lane == 0) {
            BlockMeta m = meta[b];
            m.mode = MODE_RLE; m.sym = (uint8_t)arg; m.recsize = 6; m.bits = 0; m.pm = 0;
            meta[b] = m;
        }
        return 0;
    }
    for (int i = lane; i < 256; i += 32) s.lens[i] = 0;
    if (total == 0) {  // empty histogram (stage-level API only)
        __syncwarp();
        if (lens_out) reinterpret_cast<uint2*>(lens_out + b * 256)[lane] = make_uint2(0, 0);
        if (lane == 0 && pm_flag) atomicOr(pm_flag, 2u);
        return 0;
    }
    bool near_stored = false;
    if (lens_out == nullptr) {
        // entropy bound: every prefix code costs at least n H bits; when even
        // that cannot beat the stored record (stream.py:173) the block is
        // stored and its code is never built (incompressible planes)
        // (single precision, MUFU log2: <= 2 ulp per log2, so each c log2 c
        // term is off by < 0.3 bits and the 256-term sum by < 100 bits; the
        // 256-bit margin keeps the bound conservative)
        float ent = 0.f;   // sum c log2 c
#pragma unroll
        for (int r = 0; r < 8; r++)
            if (cnt[r] > 1) ent += (float)cnt[r] * __log2f((float)cnt[r]);
#pragma unroll
        for (int o = 16; o; o >>= 1) ent += __shfl_xor_sync(0xFFFFFFFFu, ent, o);
        const float nH = (float)total * __log2f((float)total) - ent;
        const uint32_t len = meta[b].len;
        // within 3% of incompressible: most likely stored (the deferred cost pass)
        near_stored = 8.f * kHuffOverhead + nH > 0.97f * 8.f * len;
        if (8.f * kHuffOverhead + nH - 256.f > 8.f * len) {
            if (lane == 0) {
                BlockMeta m = meta[b];
                m.mode = MODE_STORED; m.bits = 0; m.recsize = 5 + len; m.pm = 0;
                meta[b] = m;
            }
            return 0;
        }
    }
    const int n = sorted_leaves(cnt, lane, s.wt, s.sym, s.wt);   // (keys alias wt)
    if (col && n >= kDeferMin && near_stored && total <= 65536) {   // (column entries are u16)
        // many symbols (near-uniform planes, usually stored): hand the sorted
        // weights to the CTA's lane-per-block cost pass instead of building
        // the code on one lane here
        for (int i = lane; i < n; i += 32) col[i * NB] = (uint16_t)s.wt[i];
        return n;
    }
    if (n == 1) {
        if (lane == 0) s.lens[s.sym[0]] = 1;  // huffman.py:89-91
    } else {
        const int mdep = huffman_depths_warp(s, n, lane);
        if (mdep > kMaxLen) {
            // package-merge fallback (huffman.py:100-101) runs in k_pkgmerge
            if (lane == 0) {
                if (lens_out) { if (pm_flag) atomicOr(pm_flag, 1u); }
                else { BlockMeta m = meta[b]; m.pm = 1; meta[b] = m; }
                pm_list[atomicAdd(pm_count, 1u)] = (uint32_t)b;
            }
            return 0;
        }
        for (int i = lane; i < n; i += 32) s.lens[s.sym[i]] = s.dep[i];
    }
    __syncwarp();
    if (lens_out) {
        reinterpret_cast<uint2*>(lens_out + b * 256)[lane] = reinterpret_cast<const uint2*>(s.lens)[lane];
        return 0;
    }
    finish_block(s, cnt, lane, meta, wire, b);
    return 0;
}

// Cost of the unlimited Huffman code of one sorted column of n >= 2 weights
// (= the sum of the internal node weights; the two-queue merge with leaf-first
// ties, huffman.py:106-137), one lane per column, no parent pointers.  The
// queue heads and next entries live in registers; each pick loads the entry
// after the next (branch-free).  Internal weights other than the root are
// < 2^16 (all n >= 2 leaves are non-zero), so the u16 column holds them.
template <int NB>
__device__ __forceinline__ uint32_t huff_cost_lane(uint16_t* col, int n) {
    constexpr uint32_t kInf = 0xFFFFFFFFu;
    uint32_t cost = 0;
    int leaf = 0, node = n;
    uint32_t L0 = col[0], L1 = n > 1 ? col[NB] : kInf, N0 = kInf, N1 = kInf;
    for (int nxt = n; nxt < 2 * n - 1; nxt++) {
        uint32_t w = 0;
#pragma unroll
        for (int q = 0; q < 2; q++) {
            const bool tl = leaf < n && (node >= nxt || L0 <= N0);
            w += tl ? L0 : N0;
            const int idx = tl ? leaf + 2 : node + 2;
            const bool ok = tl ? idx < n : idx < nxt;
            const uint32_t v = ok ? (uint32_t)col[idx * NB] : kInf;
            leaf += tl ? 1 : 0;
            node += tl ? 0 : 1;
            L0 = tl ? L1 : L0;
            L1 = tl ? v : L1;
            N0 = tl ? N0 : N1;
            N1 = tl ? N1 : v;
        }
        cost += w;
        col[nxt * NB] = (uint16_t)w;
        if (node == nxt) N0 = w;
        else if (node + 1 == nxt) N1 = w;
    }
    return cost;
}

// mode_only: block-level path (stream records).  For the stage-level API
// (lmcg_build_codebooks) lens_out != null and RLE is not special-cased.
// CTA of kCbWarps warps per NB blocks: the warps prepare the blocks;
// blocks with many symbols are decided by one lane each (Huffman cost vs the
// stored record: stored needs no code); the rest build their code warp-wide.
template <int NB>
__global__ void __launch_bounds__(kCbWarps * 32) k_codebook(const uint32_t* __restrict__ hist, uint64_t nb,
                                                          BlockMeta* __restrict__ meta, uint8_t* __restrict__ wire,
                                                          uint8_t* __restrict__ lens_out, uint32_t* __restrict__ pm_flag,
                                                          uint32_t* __restrict__ pm_count, uint32_t* __restrict__ pm_list,
                                                          uint64_t part_lo = 0, uint64_t part_hi = ~0ull) {
    __shared__ CbSmem sm[kCbWarps];
    extern __shared__ uint16_t cols[];   // (record path only) 512 rows x NB columns
    __shared__ int dn[NB];
    __shared__ uint32_t dcost[NB];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t b0 = (uint64_t)blockIdx.x * NB;
    for (int j = warp; j < NB; j += kCbWarps) {
        const uint64_t b = b0 + j;
        int n = 0;
        if (b < nb) {
            if (b < part_lo || b >= part_hi) {   // outside the part: no record
                if (lane == 0) {
                    BlockMeta m{};
                    meta[b] = m;
                }
            } else {
                n = cb_block<NB>(sm[warp], b, lane, hist, meta, wire, lens_out, pm_flag, pm_count, pm_list,
                             lens_out ? nullptr : cols + j);
            }
        }
        if (lane == 0) dn[j] = n;
    }
    __syncthreads();
    if (warp == 0 && lane < NB) {
        const int n = dn[lane];
        dcost[lane] = n ? huff_cost_lane<NB>(cols + lane, n) : 0u;
    }
    __syncthreads();
    for (int j = warp; j < NB; j += kCbWarps) {
        if (!dn[j]) continue;
        const uint64_t b = b0 + j;
        const uint32_t len = meta[b].len, cost = dcost[j];
        // a length-limited (package-merge) code costs at least the Huffman
        // code, so a Huffman cost that loses to the stored record settles it
        if (kHuffOverhead + (cost + 7) / 8 > len) {
            if (lane == 0) {
                BlockMeta m = meta[b];
                m.mode = MODE_STORED; m.bits = cost; m.recsize = 5 + len; m.pm = 0;
                meta[b] = m;
            }
        } else {
            cb_block<NB>(sm[warp], b, lane, hist, meta, wire, lens_out, pm_flag, pm_count, pm_list, nullptr);
        }
    }
}

// ------------------------------------------------------ K2b package-merge
// Length-limited lengths by package-merge with the reference's tie rules
// (huffman.py:140-180): packages pair items (2k, 2k+1); merge(leaves,
// packages) puts a leaf before an equal-weight package; the code length of a
// leaf is its multiplicity among the first 2n-2 items after 14 rounds.
// Backtracking form: at the last level take c = 2n-2 items; the leaves among
// them are the first l leaves; the c-l packages are made of the first
// 2(c-l) items of the previous level; recurse to level 0.
struct PmSmem {
    uint64_t lw[256];        // sorted leaf weights (64-bit: packages can repeat leaves)
    uint32_t lw32[256];
    uint8_t sym[256];
    uint64_t prev[512];      // level t-1 item weights
    uint64_t cur[512];       // level t item weights
    uint64_t pk[256];        // packages
    uint16_t lpos[15][256];  // leaf positions per level
    uint8_t lens[256];
};

constexpr int kPmGrid = 148 * 8;   // persistent single-warp CTAs (8 per SM by shared memory)
__global__ void __launch_bounds__(32) k_pkgmerge(const uint32_t* __restrict__ hist, const uint32_t* __restrict__ pm_count,
                                                 const uint32_t* __restrict__ pm_list, BlockMeta* __restrict__ meta,
                                                 uint8_t* __restrict__ wire, uint8_t* __restrict__ lens_out) {
    __shared__ PmSmem s;
    __shared__ CbSmem cs;
    const int lane = threadIdx.x;
    const uint32_t npm = *pm_count;
    for (uint32_t idx = blockIdx.x; idx < npm; idx += gridDim.x) {
    const uint64_t b = pm_list[idx];
    uint32_t cnt[8];
#pragma unroll
    for (int r = 0; r < 8; r++) cnt[r] = hist[b * 256 + lane * 8 + r];
    const int n = sorted_leaves(cnt, lane, s.lw32, s.sym, s.cur);
    for (int i = lane; i < n; i += 32) { s.lw[i] = s.lw32[i]; s.prev[i] = s.lw32[i]; s.lpos[0][i] = (uint16_t)i; }
    __syncwarp();
    int m = n;
    for (int t = 1; t < kMaxLen; t++) {
        const int np = m / 2;
        for (int k = lane; k < np; k += 32) s.pk[k] = s.prev[2 * k] + s.prev[2 * k + 1];
        __syncwarp();
        // leaf i -> i + #{packages < w_i}
        for (int i = lane; i < n; i += 32) {
            const uint64_t wi = s.lw[i];
            int lo = 0, hi = np;
            while (lo < hi) { int mid = (lo + hi) >> 1; if (s.pk[mid] < wi) lo = mid + 1; else hi = mid; }
            const int pos = i + lo;
            s.cur[pos] = wi;
            s.lpos[t][i] = (uint16_t)pos;
        }
        // package k -> k + #{leaves <= p_k}
        for (int k = lane; k < np; k += 32) {
            const uint64_t pw = s.pk[k];
            int lo = 0, hi = n;
            while (lo < hi) { int mid = (lo + hi) >> 1; if (s.lw[mid] <= pw) lo = mid + 1; else hi = mid; }
            s.cur[k + lo] = pw;
        }
        __syncwarp();
        m = n + np;
        for (int i = lane; i < m; i += 32) s.prev[i] = s.cur[i];
        __syncwarp();
    }
    // backward pass (all lanes compute the same scalars)
    for (int i = lane; i < 256; i += 32) s.lens[i] = 0;
    __syncwarp();
    int c = min(2 * n - 2, m);
    uint8_t mylen[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int t = kMaxLen - 1; t >= 0; t--) {
        int l;
        if (t == 0) {
            l = min(c, n);
        } else {
            // leaves among the first c items: leaf positions increase with i
            int lo = 0, hi = n;
            while (lo < hi) { int mid = (lo + hi) >> 1; if (s.lpos[t][mid] < c) lo = mid + 1; else hi = mid; }
            l = lo;
        }
#pragma unroll
        for (int r = 0; r < 8; r++) if (lane + 32 * r < l) mylen[r]++;
        c = 2 * (c - l);
    }
#pragma unroll
    for (int r = 0; r < 8; r++) if (lane + 32 * r < n) s.lens[s.sym[lane + 32 * r]] = mylen[r];
    __syncwarp();
    if (lens_out) {
        reinterpret_cast<uint2*>(lens_out + b * 256)[lane] = reinterpret_cast<const uint2*>(s.lens)[lane];
    } else {
        for (int i = lane; i < 256; i += 32) cs.lens[i] = s.lens[i];
        __syncwarp();
        finish_block(cs, cnt, lane, meta, wire, b);
    }
    __syncwarp();
    }
}

// --------------------------------------------------------------- scan
// Decoupled look-back exclusive scan of meta[i].recsize -> out[i] (u64), with
// out[n] = total.  status[] (one u64 per tile) and *ticket must be zeroed.
constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;
constexpr uint64_t kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(kScanThreads) k_scan(const BlockMeta* __restrict__ meta, uint64_t n,
                                                       uint64_t* __restrict__ out, uint64_t* status,
                                                       uint32_t* ticket) {
    __shared__ uint32_t sh_tile;
    __shared__ uint64_t sh_warp[kScanThreads / 32];
    __shared__ uint64_t sh_prefix;
    if (threadIdx.x == 0) sh_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint64_t tile = sh_tile;
    const uint64_t base = tile * kScanTile + (uint64_t)threadIdx.x * kScanItems;
    uint64_t v[kScanItems], sum = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; i++) {
        v[i] = (base + i < n) ? meta[base + i].recsize : 0;
        sum += v[i];
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) sh_warp[warp] = incl;
    __syncthreads();
    uint64_t wpre = 0, agg = 0;
    for (int q = 0; q < kScanThreads / 32; q++) {
        if (q < warp) wpre += sh_warp[q];
        agg += sh_warp[q];
    }
    if (threadIdx.x == 0) {
        if (tile == 0) {
            st_release(&status[0], kFlagInc | agg);
            sh_prefix = 0;
        } else {
            st_release(&status[tile], kFlagAgg | agg);
            uint64_t pre = 0;
            int64_t j = (int64_t)tile - 1;
            while (j >= 0) {
                uint64_t st;
                do { st = ld_acquire(&status[j]); } while ((st >> 62) == 0);
                pre += st & kValMask;
                if ((st >> 62) == 2) break;
                j--;
            }
            st_release(&status[tile], kFlagInc | (pre + agg));
            sh_prefix = pre;
        }
    }
    __syncthreads();
    uint64_t run = sh_prefix + wpre + incl - sum;
#pragma unroll
    for (int i = 0; i < kScanItems; i++) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
    const uint64_t last_tile = (n == 0) ? 0 : (n - 1) / kScanTile;
    if (tile == last_tile && threadIdx.x == kScanThreads - 1) out[n] = sh_prefix + agg;
}

// -------------------------------------------------------------- layout
// Per-stream totals (28 + nwin*16*S + records) and their exclusive scan.
__global__ void k_layout(const StreamDesc* __restrict__ streams, int ns, uint32_t segs,
                         const uint64_t* __restrict__ scan, uint64_t* __restrict__ soff,
                         uint64_t* __restrict__ slen) {
    __shared__ uint64_t sh_carry, sh_w[32];
    if (threadIdx.x == 0) sh_carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int base = 0; base < ns; base += blockDim.x) {
        const int i = base + threadIdx.x;
        uint64_t tot = 0;
        if (i < ns) {
            const StreamDesc sd = streams[i];
            tot = kHeader + (uint64_t)sd.nwin * kSegEntry * segs + (scan[sd.blk0 + sd.nblk] - scan[sd.blk0]);
            slen[i] = tot;
        }
        uint64_t incl = tot;
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) sh_w[warp] = incl;
        __syncthreads();
        uint64_t pre = sh_carry, all = 0;
        for (int q = 0; q < nw; q++) { if (q < warp) pre += sh_w[q]; all += sh_w[q]; }
        if (i < ns) soff[i] = pre + incl - tot;
        __syncthreads();
        if (threadIdx.x == 0) sh_carry += all;
        __syncthreads();
    }
}

// --------------------------------------------------------------- frame
__device__ __forceinline__ void put_u64(uint8_t* p, uint64_t v) {
#pragma unroll
    for (int i = 0; i < 8; i++) p[i] = (uint8_t)(v >> (8 * i));
}
__device__ __forceinline__ void put_u32(uint8_t* p, uint32_t v) {
#pragma unroll
    for (int i = 0; i < 4; i++) p[i] = (uint8_t)(v >> (8 * i));
}

// One CTA per stream: combine the per-block raw CRCs into zlib.crc32 of the
// whole payload, write the 28-byte header and every window's segment table.
__global__ void __launch_bounds__(kThreads) k_frame(const StreamDesc* __restrict__ streams,
                                                  const WinDesc* __restrict__ wins, uint32_t B, uint32_t segs,
                                                  const uint64_t* __restrict__ scan, const uint32_t* __restrict__ crcpart,
                                                  const CrcTables* __restrict__ ct, const uint64_t* __restrict__ soff,
                                                  uint8_t* __restrict__ out) {
    __shared__ uint32_t sh_red[kThreads];
    const int s = blockIdx.x;
    const StreamDesc sd = streams[s];
    const uint64_t base = soff[s];
    // --- CRC: a window's parts are the raw CRCs of consecutive cunit-byte
    // ranges (the last one shorter; k_crc's 32 KiB chunks or k_hist's
    // plane-0 element ranges): fold them CTA-wide with byte-shift tables,
    // then chain the windows.
    uint32_t acc = 0;
    for (uint32_t wl = 0; wl < sd.nwin; wl++) {
        const WinDesc wd = wins[sd.win0 + wl];
        const uint64_t unit = wd.cunit;
        const uint64_t nfull = wd.W / unit, rem = wd.W % unit;
        const uint32_t* cp = crcpart + wd.crc0;
        uint32_t wc = crc_combine_uniform(ct, nfull, unit, [&](uint64_t i) { return cp[i]; }, sh_red);
        if (threadIdx.x == 0) {
            if (rem) wc = crc_shift_bytes(ct, wc, rem) ^ cp[nfull];
            acc = crc_shift_bytes(ct, acc, wd.W) ^ wc;
        }
    }
    if (threadIdx.x == 0) {
        uint32_t crc = acc ^ crc_shift_bytes(ct, 0xFFFFFFFFu, sd.nbytes) ^ 0xFFFFFFFFu;
        uint8_t* h = out + base;
        h[0] = 'L'; h[1] = 'M'; h[2] = 'C'; h[3] = '1';
        h[4] = 1; h[5] = (uint8_t)sd.flags; h[6] = (uint8_t)sd.et; h[7] = 0;
        put_u64(h + 8, sd.nbytes);
        put_u32(h + 16, B);
        put_u32(h + 20, segs);
        put_u32(h + 24, crc);
    }
    // --- segment tables (segment_bounds, stream.py:271-284)
    const uint64_t sb0 = scan[sd.blk0];
    const uint64_t total_entries = (uint64_t)sd.nwin * segs;
    for (uint64_t q = threadIdx.x; q < total_entries; q += blockDim.x) {
        const uint32_t wl = (uint32_t)(q / segs), i = (uint32_t)(q % segs);
        const WinDesc wd = wins[sd.win0 + wl];
        const uint64_t nblk = wd.nblocks;
        const uint64_t ea = min(wd.W, ((uint64_t)i * nblk / segs) * B);
        const uint64_t eb = (i + 1 == segs) ? wd.W : min(wd.W, ((uint64_t)(i + 1) * nblk / segs) * B);
        const uint64_t ba = ea / B, bb = (eb == ea) ? ba : (eb + B - 1) / B;
        const uint64_t comp = scan[wd.blk0 + bb] - scan[wd.blk0 + ba];
        const uint64_t toff = base + kHeader + (uint64_t)wl * kSegEntry * segs + (scan[wd.blk0] - sb0);
        put_u64(out + toff + (uint64_t)i * kSegEntry, eb - ea);
        put_u64(out + toff + (uint64_t)i * kSegEntry + 8, comp);
    }
}

// Raw CRC-32 of one byte range from its k_crc chunk CRCs (lmcg_compress_part).
__global__ void __launch_bounds__(kThreads) k_crc_join(const uint32_t* __restrict__ parts, uint64_t L,
                                                     const CrcTables* __restrict__ ct, uint32_t* __restrict__ out) {
    __shared__ uint32_t red[kThreads];
    const uint64_t nfull = L / kCrcChunk, rem = L % kCrcChunk;
    uint32_t c = crc_combine_uniform(ct, nfull, kCrcChunk, [&](uint64_t i) { return parts[i]; }, red);
    if (threadIdx.x == 0) {
        if (rem) c = crc_shift_bytes(ct, c, rem) ^ parts[nfull];
        *out = c;
    }
}

// --------------------------------------------------------------- K4 encode
// Symbols of piece (q, lane) of a warp-tile: the 16 source bytes at
// 512 q + 16 lane, i.e. grouped positions [tp + (512 q + 16 lane)/w, +16/w)
// clipped to [tp, te); vector loads on fast tiles, byte gathers otherwise.
__device__ __forceinline__ int tile_piece(const WinDesc& wd, uint64_t tp, uint64_t te, uint64_t g, bool fast, int q,
                                          int lane, uint32_t sy[4], uint64_t& pos) {
    const uint32_t w = wd.w, lw = lg2w(w);
    const uint32_t rel = (512u * q + 16u * lane) >> lw;
    pos = tp + rel;
    if (fast) {
        const uint4 a = ldg16x(wd.src, wd.prev, ((tp - g * wd.n) << lw) + 512u * q + 16u * lane);
        return piece_symbols(a, w, (uint32_t)g, sy);
    }
    sy[0] = sy[1] = sy[2] = sy[3] = 0;
    const int want = 16 / (int)w;
    int ns = 0;
    for (int i = 0; i < want && pos + i < te; i++, ns++) sy[i >> 2] |= gather_byte(wd, pos + i) << (8 * (i & 3));
    return ns;
}

// Huffman packing of positions [p0, p1) of a window plane, in rounds of
// kEncRun positions per thread.  Thread t packs its contiguous run
// [r0 + t kEncRun, +kEncRun) MSB-first into a private slot of whole words
// through a 64-bit accumulator (one pass, no branches); a CTA scan of the
// run bit counts places every run, whose words are then shifted into the
// round's staging area on the destination's 4-byte grid (the two edge words
// of a run, shared with its neighbours, merged with atomicOr) and leave with
// coalesced 32-bit stores.
constexpr int kSlot = (kEncRun * kMaxLen + 31) / 32 + 1;   // private words per run
constexpr int kStageWords = (kEncRun * kThreads * kMaxLen) / 32 + 8;
// k_encode's dynamic shared memory: code table (256 words: len << 16 | code) |
// staging | private slots.  The packing loops address the code table through
// this symbol, so a lookup is one [register + constant] shared-memory load
// (a pointer handed through the call costs a base add per lookup).
extern __shared__ __align__(1024) uint32_t g_enc_smem[];
// The code table is stored permuted: the entry of symbol s at enc_slot(s) = s
// with bit 4 flipped when bit 7 is set.  The high planes of weights hold the
// same exponents under both signs (symbols 52.. and 180.., 128 apart: the
// same bank), which cost every table lookup a second wavefront; the flip
// moves the negative half 16 banks away.  enc_slot4 maps the four symbols of
// a word at once (two instructions per four symbols).
__device__ __forceinline__ uint32_t enc_slot(uint32_t s) { return s ^ ((s >> 3) & 0x10u); }
__device__ __forceinline__ uint32_t enc_slot4(uint32_t w) { return w ^ ((w >> 3) & 0x10101010u); }
// Code table entry of byte `b` (0..3) of word `w`: the table is 1 KiB aligned,
// so base | (index * 4) is its shared-memory address -- one shift, one LOP3
// and the load per symbol.
__device__ __forceinline__ uint32_t code_at(uint32_t cb, uint32_t w, int b) {
    const uint32_t a = cb | ((b == 0 ? w << 2 : w >> (8 * b - 2)) & 0x3FCu);
    uint32_t e;
    asm("ld.shared.u32 %0, [%1];" : "=r"(e) : "r"(a));
    return e;
}
constexpr int kEncCodeWords = 256;
constexpr size_t kEncSmem = (size_t)(kEncCodeWords + kStageWords + kThreads * kSlot) * sizeof(uint32_t);

// RUN: the block's code has a 1-bit codeword, which canonical assignment
// makes '0' (huffman.py:213-225), for symbol `runsym`.  Each thread then only
// looks up the other symbols of a piece (XOR deltas: a few percent of the
// bytes) and appends the run symbols between them as zero bits, instead of a
// table lookup per symbol.
template <int W, bool RUN>
__device__ void encode_runs(const WinDesc& wd, uint64_t p0, uint64_t p1,
                            uint32_t* sh_wsum, uint32_t* stg, uint32_t* gw, uint32_t lead,
                            uint32_t& bitpos, uint64_t& base_word, uint32_t runsym) {
    constexpr uint32_t lw = W == 1 ? 0 : (W == 2 ? 1 : 2);
    constexpr int per = 16 >> lw;   // symbols per 16-byte piece
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t* priv = stg + kStageWords + tid * kSlot;
    for (uint64_t r0 = p0; r0 < p1; r0 += (uint64_t)kEncRun * kThreads) {
        const uint64_t q0 = r0 + (uint64_t)tid * kEncRun;
        const uint64_t q1 = min(q0 + kEncRun, p1);
        const uint64_t g = q0 < q1 ? plane_of(q0, wd.n, W) : 0;
        const bool fast = q0 < q1 && wd.vec && ((q1 - q0) % per == 0) && (q1 <= (g + 1) * wd.n);
        const uint8_t* srcp = wd.src + ((q0 - g * wd.n) << lw);
        const uint8_t* prvp = wd.prev ? wd.prev + ((q0 - g * wd.n) << lw) : nullptr;
        // pack the run into the private slot
        uint64_t acc = 0;
        uint32_t n = 0, wi = 0;
        uint32_t pend = 0;   // RUN: run symbols not yet appended (<= kEncRun)
        const uint32_t rep4 = runsym * 0x01010101u;
        auto put = [&](uint32_t l, uint32_t code) {
            acc = (acc << l) | code;
            n += l;
            const bool fl = n >= 32;
            n -= fl ? 32 : 0;
            if (fl) priv[wi] = (uint32_t)(acc >> n);
            wi += fl ? 1 : 0;
        };
        auto zeros = [&](uint32_t z) {   // z <= 64 zero bits, in two steps of <= 32
            const uint32_t t1 = min(z, 32u);
            put(t1, 0u);
            put(z - t1, 0u);
        };
        // W == 2: when every lane of the warp has a full run in one plane, the
        // warp's 4 KiB of source are read as eight fully coalesced 512-byte
        // rows, the plane's symbols (slot-mapped) transposed through the idle
        // staging area, and each lane reads its 64 symbols back as four
        // 16-byte pieces.  (Each lane loading its own 128-byte run touched 32
        // lines per load instruction: eight times the LSU wavefronts, and the
        // kernel's LSU data pipe ran at 78%.)
        bool warp_t = false;
        if constexpr (W == 2) {
            const uint64_t g_0 = __shfl_sync(0xFFFFFFFFu, g, 0);
            warp_t = __all_sync(0xFFFFFFFFu, fast && q1 - q0 == (uint64_t)kEncRun && g == g_0);
        }
        if (warp_t) {
            // staging word 0 carries the previous round's open word: the buffer starts 16 bytes in
            uint8_t* tb = reinterpret_cast<uint8_t*>(stg) + 16 + warp * 2048;
            const uint64_t wbase = (((r0 + (uint64_t)(warp * 32) * kEncRun) - g * wd.n) << lw);   // source byte of the warp's first run
#pragma unroll
            for (int hq = 0; hq < 2; hq++) {
                uint4 a[4];
#pragma unroll
                for (int q = 0; q < 4; q++) a[q] = ldg16x(wd.src, wd.prev, wbase + 512ull * (4 * hq + q) + 16ull * lane);
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    uint32_t sy[4];
                    piece_symbols(a[q], W, (uint32_t)g, sy);
                    // run and piece of source bytes 512 (4 hq + q) + 16 lane; 16-byte unit u of run r sits at unit u ^ ((r >> 1) & 3)
                    const uint32_t r = 4 * (4 * hq + q) + (lane >> 3), pc = lane & 7;
                    const uint32_t off = r * 64 + (((pc >> 1) ^ ((r >> 1) & 3)) << 4) + ((pc & 1) << 3);
                    // (run blocks compare the raw symbols with the run symbol and map the slot per lookup)
                    *reinterpret_cast<uint2*>(tb + off) = RUN ? make_uint2(sy[0], sy[1]) : make_uint2(enc_slot4(sy[0]), enc_slot4(sy[1]));
                }
            }
            __syncwarp();
            const uint32_t pw0 = (uint32_t)__cvta_generic_to_shared(priv);
            uint32_t pw = pw0;   // running shared-memory address in the private slot
            const uint32_t cb = (uint32_t)__cvta_generic_to_shared(g_enc_smem);
            const uint32_t sw = (lane >> 1) & 3;
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint4 c = *reinterpret_cast<const uint4*>(tb + lane * 64 + ((u ^ sw) << 4));
                const uint32_t sy[4] = {c.x, c.y, c.z, c.w};
                if (RUN) {
                    // bit i: symbol i of the 16 is not the run symbol
                    uint32_t m = 0;
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        const uint32_t r = __vcmpne4(sy[k], rep4) & 0x80808080u;
                        m |= ((r * 0x00204081u) >> 28) << (4 * k);
                    }
                    uint32_t last = 0;
                    while (m) {
                        const uint32_t i = __ffs(m) - 1;
                        m &= m - 1;
                        zeros(pend + i - last);
                        pend = 0;
                        last = i + 1;
                        uint32_t word = sy[0];
                        word = (i >> 2) == 1 ? sy[1] : word;
                        word = (i >> 2) == 2 ? sy[2] : word;
                        word = (i >> 2) == 3 ? sy[3] : word;
                        const uint32_t e = g_enc_smem[enc_slot((word >> (8 * (i & 3))) & 0xFF)];
                        put(e >> 16, e & 0xFFFF);
                    }
                    pend += 16 - last;
                }
#pragma unroll
                for (int i = 0; !RUN && i < 16; i += 2) {
                    const uint32_t e1 = code_at(cb, sy[i >> 2], i & 3);
                    const uint32_t e2 = code_at(cb, sy[(i + 1) >> 2], (i + 1) & 3);
                    const uint32_t l2 = e2 >> 16;
                    const uint32_t pl = (e1 >> 16) + l2;
                    acc = (acc << pl) | (((e1 & 0xFFFF) << l2) | (e2 & 0xFFFF));
                    n += pl;
                    if (n >= 32) {
                        n -= 32;
                        asm volatile("st.shared.u32 [%0], %1;" ::"r"(pw), "r"((uint32_t)(acc >> n)) : "memory");
                        pw += 4;
                    }
                }
            }
            if (!RUN) wi = (pw - pw0) >> 2;
            __syncwarp();   // (the staging area is rewritten after the CTA barrier below)
        } else if (!RUN && fast) {
            // lean run: whole pieces of one plane, 16-byte loads one piece
            // ahead, every symbol pair unconditional, the private slot
            // addressed by a running pointer
            const uint4* sp = reinterpret_cast<const uint4*>(srcp);
            const uint4* pp = reinterpret_cast<const uint4*>(prvp);
            const uint32_t npc = (uint32_t)((q1 - q0) / per);
            auto ld = [&](uint32_t j) {
                uint4 a = __ldg(sp + j);
                if (pp) {
                    const uint4 c = __ldg(pp + j);
                    a.x ^= c.x; a.y ^= c.y; a.z ^= c.z; a.w ^= c.w;
                }
                return a;
            };
            const uint32_t pw0 = (uint32_t)__cvta_generic_to_shared(priv);
            uint32_t pw = pw0;   // running shared-memory address in the private slot
            const uint32_t cb = (uint32_t)__cvta_generic_to_shared(g_enc_smem);
            uint4 cur = ld(0);
#pragma unroll 2
            for (uint32_t j = 0; j < npc; j++) {
                const uint4 nxt = j + 1 < npc ? ld(j + 1) : make_uint4(0, 0, 0, 0);
                uint32_t sy[4];
                piece_symbols(cur, W, (uint32_t)g, sy);
#pragma unroll
                for (int i = 0; i < (per + 3) / 4; i++) sy[i] = enc_slot4(sy[i]);
#pragma unroll
                for (int i = 0; i < per; i += 2) {
                    const uint32_t e1 = code_at(cb, sy[i >> 2], i & 3);
                    const uint32_t e2 = code_at(cb, sy[(i + 1) >> 2], (i + 1) & 3);
                    const uint32_t l2 = e2 >> 16;
                    const uint32_t pl = (e1 >> 16) + l2;
                    acc = (acc << pl) | (((e1 & 0xFFFF) << l2) | (e2 & 0xFFFF));
                    n += pl;
                    if (n >= 32) {
                        n -= 32;
                        asm volatile("st.shared.u32 [%0], %1;" ::"r"(pw), "r"((uint32_t)(acc >> n)) : "memory");
                        pw += 4;
                    }
                }
                cur = nxt;
            }
            wi = (pw - pw0) >> 2;
        } else {
        // fast runs: the loads run kAhead pieces ahead of the packing (the
        // kernel is otherwise bound by load latency at its occupancy)
        constexpr int kAhead = 2;
        uint4 la[kAhead], lc[kAhead];
#pragma unroll
        for (int u = 0; u < kAhead; u++) {
            la[u] = lc[u] = make_uint4(0, 0, 0, 0);
            if (fast && q0 + (uint64_t)u * per < q1) {
                la[u] = __ldg(reinterpret_cast<const uint4*>(srcp + ((uint64_t)u * per << lw)));
                if (prvp) lc[u] = __ldg(reinterpret_cast<const uint4*>(prvp + ((uint64_t)u * per << lw)));
            }
        }
        for (uint64_t pos = q0; pos < q1; pos += per) {
            uint32_t sy[4];
            int ns;
            if (fast) {
                uint4 a = la[0];
                const uint4 c = lc[0];
                a.x ^= c.x; a.y ^= c.y; a.z ^= c.z; a.w ^= c.w;
#pragma unroll
                for (int u = 0; u + 1 < kAhead; u++) { la[u] = la[u + 1]; lc[u] = lc[u + 1]; }
                const uint64_t nx = pos + (uint64_t)kAhead * per;
                if (nx < q1) {
                    la[kAhead - 1] = __ldg(reinterpret_cast<const uint4*>(srcp + ((nx - q0) << lw)));
                    if (prvp) lc[kAhead - 1] = __ldg(reinterpret_cast<const uint4*>(prvp + ((nx - q0) << lw)));
                }
                ns = piece_symbols(a, W, (uint32_t)g, sy);
            } else {
                sy[0] = sy[1] = sy[2] = sy[3] = 0;
                ns = 0;
                for (int i = 0; i < per && pos + i < q1; i++, ns++) sy[i >> 2] |= gather_byte(wd, pos + i) << (8 * (i & 3));
            }
            if (RUN) {
                // bit i of the piece's group: symbol i is not the run symbol
                uint32_t m = 0;
#pragma unroll
                for (int k = 0; k < (per + 3) / 4; k++) {
                    const uint32_t r = __vcmpne4(sy[k], rep4) & 0x80808080u;
                    m |= ((r * 0x00204081u) >> 28) << (4 * k);
                }
                m &= (1u << ns) - 1;   // ns <= 16
                uint32_t last = 0;
                while (m) {
                    const uint32_t i = __ffs(m) - 1;
                    m &= m - 1;
                    zeros(pend + i - last);
                    pend = 0;
                    last = i + 1;
                    uint32_t word = sy[0];
                    if (per > 4) word = (i >> 2) == 1 ? sy[1] : word;
                    if (per > 8) { word = (i >> 2) == 2 ? sy[2] : word; word = (i >> 2) == 3 ? sy[3] : word; }
                    const uint32_t e = g_enc_smem[enc_slot((word >> (8 * (i & 3))) & 0xFF)];
                    put(e >> 16, e & 0xFFFF);
                }
                pend += ns - last;
            }
            // symbol pairs: two codes (<= 30 bits) joined in 32 bits, one
            // accumulator update and at most one word flush per pair
#pragma unroll
            for (int i = 0; i < per; i += 2) {
                if (!RUN && i < ns) {
                    const uint32_t e1 = g_enc_smem[enc_slot((sy[i >> 2] >> (8 * (i & 3))) & 0xFF)];
                    const uint32_t e2 = (i + 1 < ns) ? g_enc_smem[enc_slot((sy[(i + 1) >> 2] >> (8 * ((i + 1) & 3))) & 0xFF)] : 0u;
                    const uint32_t l2 = e2 >> 16;
                    const uint32_t pl = (e1 >> 16) + l2;
                    acc = (acc << pl) | (((e1 & 0xFFFF) << l2) | (e2 & 0xFFFF));
                    n += pl;
                    const bool fl = n >= 32;
                    n -= fl ? 32 : 0;
                    if (fl) priv[wi] = (uint32_t)(acc >> n);
                    wi += fl ? 1 : 0;
                }
            }
        }
        }
        if (RUN) zeros(pend);
        const uint32_t nwp = wi + (n ? 1 : 0);
        if (n) priv[wi] = (uint32_t)(acc << (32 - n));
        const uint32_t nb = wi * 32 + n;
        // CTA exclusive scan of nb
        uint32_t incl = nb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) sh_wsum[warp] = incl;
        __syncthreads();
        uint32_t pre = 0, tot = 0;
#pragma unroll
        for (int q = 0; q < kWarps; q++) { if (q < warp) pre += sh_wsum[q]; tot += sh_wsum[q]; }
        const uint32_t start = bitpos + pre + incl - nb;
        const uint32_t fw = start >> 5, lwi = (start + nb - 1) >> 5;
        if (nb && fw) stg[fw] = 0;           // word 0 holds the carry of the previous round
        if (nb && lwi != fw) stg[lwi] = 0;
        __syncthreads();
        if (nb) {
            const uint32_t s0 = start & 31;
            const uint32_t nwo = lwi - fw + 1;
            for (uint32_t k = 0; k < nwo; k++) {
                const uint32_t cur = k < nwp ? priv[k] : 0u;
                const uint32_t v = s0 ? ((k ? priv[k - 1] << (32 - s0) : 0u) | (cur >> s0)) : cur;
                if (k == 0 || k + 1 == nwo) atomicOr(&stg[fw + k], v);
                else stg[fw + k] = v;
            }
        }
        __syncthreads();
        const uint32_t end = bitpos + tot;
        const uint32_t full = end >> 5;   // complete words in staging
        for (uint32_t j = tid; j < full; j += kThreads) {
            const uint64_t gwi = base_word + j;
            const uint32_t v = bswap32(stg[j]);
            if (gwi == 0 && lead) {
                uint8_t* bp = reinterpret_cast<uint8_t*>(gw);
                for (uint32_t q = lead / 8; q < 4; q++) bp[q] = (uint8_t)(v >> (8 * q));
            } else {
                gw[gwi] = v;
            }
        }
        const uint32_t carry = stg[full];
        __syncthreads();
        if (tid == 0) stg[0] = (end & 31) ? carry : 0u;
        base_word += full;
        bitpos = end & 31;
        __syncthreads();
    }
}

// Stored record payload: the plane's bytes of [p0, p1), gathered with
// coalesced 16-byte loads into the staging area on the destination's 4-byte
// grid, then written with coalesced 32-bit stores (the record's first and
// last words bytewise: they share bytes with the header / the next record).
__device__ void store_plane(const WinDesc& wd, uint64_t p0, uint64_t p1, uint32_t* stg, uint8_t* d0) {
    // The staging area holds each round's payload bytes at aligned offsets
    // (a piece of 16/w symbols is 1, 2 or 4 whole words).  Destination words
    // that lie entirely inside the round leave as 32-bit stores, shifted onto
    // the destination's 4-byte grid; the at most 3 + 3 bytes at the round's
    // edges go out bytewise (the record's first / last word shares bytes with
    // the header / the next record, and rounds meet inside words).
    const int tid = threadIdx.x;
    const uint32_t w = wd.w, lw = lg2w(w);
    const uint32_t per = 16u >> lw;
    const uint32_t lb = (uint32_t)(reinterpret_cast<uint64_t>(d0) & 3);
    uint32_t* gwd = reinterpret_cast<uint32_t*>(reinterpret_cast<uint64_t>(d0) & ~3ull);
    const uint8_t* sb = reinterpret_cast<const uint8_t*>(stg);
    const uint64_t round = (uint64_t)kThreads * 4 * per;   // positions (= payload bytes) per round
    for (uint64_t r0 = p0; r0 < p1; r0 += round) {
        const uint64_t r1 = min(r0 + round, p1);
        const uint64_t g0 = plane_of(r0, wd.n, w), gend = (g0 + 1) * wd.n;
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const uint64_t pos = r0 + (uint64_t)(q * kThreads + tid) * per;
            if (pos >= r1) continue;
            const uint64_t g = pos >= gend ? g0 + 1 : g0;
            uint32_t* dw = stg + ((pos - r0) >> 2);
            if (wd.vec && pos + per <= r1 && pos + per <= (g + 1) * wd.n) {
                const uint4 a = ldg16x(wd.src, wd.prev, (pos - g * wd.n) << lw);
                uint32_t sy[4];
                piece_symbols(a, w, (uint32_t)g, sy);
                if (per == 16) *reinterpret_cast<uint4*>(dw) = make_uint4(sy[0], sy[1], sy[2], sy[3]);
                else if (per == 8) *reinterpret_cast<uint2*>(dw) = make_uint2(sy[0], sy[1]);
                else *dw = sy[0];
            } else {
                uint8_t* dst = reinterpret_cast<uint8_t*>(dw);
                for (uint32_t i = 0; i < per && pos + i < r1; i++) dst[i] = (uint8_t)gather_byte(wd, pos + i);
            }
        }
        __syncthreads();
        // destination word j holds payload bytes [4j - lb, 4j - lb + 4)
        const uint64_t R0 = r0 - p0, R1 = r1 - p0;
        const uint64_t ja = (R0 + lb + 3) / 4, je = (R1 + lb) / 4;   // words inside [R0, R1)
        const uint32_t sh = 8 * ((4 - lb) & 3);                       // staging byte phase
        for (uint64_t j = ja + tid; j < je; j += kThreads) {
            const uint32_t i0 = (uint32_t)((4 * j - lb - R0) >> 2);
            gwd[j] = sh ? __funnelshift_r(stg[i0], stg[i0 + 1], sh) : stg[i0];
        }
        if (tid == 0)
            for (uint64_t pb = R0; pb < min(R1, 4 * ja - lb); pb++) d0[pb] = sb[pb - R0];
        if (tid == 32)
            for (uint64_t pb = max(R0, 4 * je - lb); pb < R1; pb++) d0[pb] = sb[pb - R0];
        __syncthreads();
    }
}

// Stored record payload, fast path: [p0, p1) inside one plane, a multiple of
// 16 bytes, 16-byte source loads allowed.  Thread t owns payload piece k (16
// bytes gathered from 16 W source bytes) and writes the 16-byte aligned
// destination chunk k, which holds the end of piece k-1 (from the lane below
// by shuffle; lane 0 takes the last piece of the warp's previous iteration)
// and the start of piece k: aligned 16-byte stores, no staging.  The record's first and last chunks share bytes
// with the header / the next record and are written bytewise.
template <int W>
__device__ __forceinline__ uint4 stored_piece(const WinDesc& wd, uint64_t sb, uint32_t g, uint32_t k) {
    constexpr uint32_t lw = W == 1 ? 0 : (W == 2 ? 1 : 2);
    const uint64_t s = sb + ((uint64_t)k << (4 + lw));
    if constexpr (W == 1) {
        return ldg16x(wd.src, wd.prev, s);
    } else {
        uint32_t o[4];
#pragma unroll
        for (int q = 0; q < W; q++) {
            uint32_t sy[4];
            piece_symbols(ldg16x(wd.src, wd.prev, s + 16 * q), W, g, sy);
#pragma unroll
            for (int i = 0; i < 4 / W; i++) o[q * (4 / W) + i] = sy[i];
        }
        return make_uint4(o[0], o[1], o[2], o[3]);
    }
}

__device__ __forceinline__ uint4 chunk_of(uint4 Q, uint4 P, uint32_t lb) {
    // bytes [16 - lb, 32 - lb) of Q ++ P (1 <= lb <= 15)
    const uint32_t s = 16 - lb, r = 8 * (s & 3);
    switch (s >> 2) {
    case 0: return make_uint4(__funnelshift_r(Q.x, Q.y, r), __funnelshift_r(Q.y, Q.z, r), __funnelshift_r(Q.z, Q.w, r), __funnelshift_r(Q.w, P.x, r));
    case 1: return make_uint4(__funnelshift_r(Q.y, Q.z, r), __funnelshift_r(Q.z, Q.w, r), __funnelshift_r(Q.w, P.x, r), __funnelshift_r(P.x, P.y, r));
    case 2: return make_uint4(__funnelshift_r(Q.z, Q.w, r), __funnelshift_r(Q.w, P.x, r), __funnelshift_r(P.x, P.y, r), __funnelshift_r(P.y, P.z, r));
    default: return make_uint4(__funnelshift_r(Q.w, P.x, r), __funnelshift_r(P.x, P.y, r), __funnelshift_r(P.y, P.z, r), __funnelshift_r(P.z, P.w, r));
    }
}

template <int W>
__device__ void store_plane_fast(const WinDesc& wd, uint64_t p0, uint64_t p1, uint8_t* d0) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t g = (uint32_t)plane_of(p0, wd.n, W);
    const uint64_t sb = (p0 - (uint64_t)g * wd.n) * W;   // source byte of payload byte 0
    const uint32_t K = (uint32_t)((p1 - p0) / 16);
    const uint32_t lb = (uint32_t)(reinterpret_cast<uint64_t>(d0) & 15);
    uint4* A = reinterpret_cast<uint4*>(reinterpret_cast<uint64_t>(d0) & ~15ull);
    // each warp owns a contiguous range of pieces, 32 per iteration: lane
    // 0's neighbour piece is lane 31's of the iteration before (carried by a
    // shuffle), gathered again only once per warp
    const uint32_t Kw = (K + kWarps - 1) / kWarps;
    const uint32_t ka = min(K, warp * Kw), kb = min(K, ka + Kw);
    uint4 carry = make_uint4(0, 0, 0, 0);
    if (lb && ka > 0 && ka < kb) carry = stored_piece<W>(wd, sb, g, ka - 1);   // (every lane: one broadcast gather)
    for (uint32_t k0 = ka; k0 < kb; k0 += 32) {
        const uint32_t k = k0 + lane;
        const bool have = k < kb;
        const uint4 P = have ? stored_piece<W>(wd, sb, g, k) : make_uint4(0, 0, 0, 0);
        if (lb == 0) {
            if (have) A[k] = P;
            continue;
        }
        uint4 Q;
        Q.x = __shfl_up_sync(0xFFFFFFFFu, P.x, 1);
        Q.y = __shfl_up_sync(0xFFFFFFFFu, P.y, 1);
        Q.z = __shfl_up_sync(0xFFFFFFFFu, P.z, 1);
        Q.w = __shfl_up_sync(0xFFFFFFFFu, P.w, 1);
        if (lane == 0) Q = carry;
        carry.x = __shfl_sync(0xFFFFFFFFu, P.x, 31);
        carry.y = __shfl_sync(0xFFFFFFFFu, P.y, 31);
        carry.z = __shfl_sync(0xFFFFFFFFu, P.z, 31);
        carry.w = __shfl_sync(0xFFFFFFFFu, P.w, 31);
        if (!have) continue;
        if (k > 0) A[k] = chunk_of(Q, P, lb);
        if (k == 0 || k + 1 == K) {   // the partial chunks: bytewise
            const uint64_t lo = (uint64_t)P.x | ((uint64_t)P.y << 32), hi = (uint64_t)P.z | ((uint64_t)P.w << 32);
            auto byte = [&](uint32_t i) { return (uint8_t)((i < 8 ? lo >> (8 * i) : hi >> (8 * (i - 8))) & 0xFF); };
            if (k == 0)
                for (uint32_t i = 0; i < 16 - lb; i++) d0[i] = byte(i);
            if (k + 1 == K)
                for (uint32_t i = 16 - lb; i < 16; i++) d0[16 * (uint64_t)k + i] = byte(i);
        }
    }
}

// One CTA per block slot.  Canonical codes (huffman.py:213-225) are built in
// shared memory from the wire codebook; each lane packs the codes of its four
// pieces MSB-first into a shared staging area laid out on the 4-byte grid of
// the destination, so complete words leave with plain 32-bit stores and only
// the two edge words of a record are written bytewise.  Stored records copy
// the symbols straight to the output.
__global__ void __launch_bounds__(kThreads) k_encode(
    const WinDesc* __restrict__ wins, const uint32_t* __restrict__ slot2win, uint64_t nslots, uint32_t B,
    uint32_t segs, const StreamDesc* __restrict__ streams, const BlockMeta* __restrict__ meta,
    const uint8_t* __restrict__ wire, const uint64_t* __restrict__ scan, const uint64_t* __restrict__ soff,
    uint8_t* __restrict__ out, uint64_t part_lo, uint64_t part_hi) {
    uint32_t* const sh_code = g_enc_smem;
    uint32_t* const stg = g_enc_smem + kEncCodeWords;
    __shared__ uint32_t sh_cnt[kWarps][16];
    __shared__ uint32_t sh_first[16];
    __shared__ uint32_t sh_wsum[kWarps];
    __shared__ uint32_t sh_run;   // symbol with the 1-bit code '0', or 256
    const uint64_t slot = blockIdx.x;
    if (slot >= nslots) return;
    const WinDesc wd = wins[slot2win[slot]];
    const int64_t kk = slot_to_block(wd, slot - wd.slot0, B);
    if (kk < 0) return;
    const uint64_t k = (uint64_t)kk;
    const uint64_t b = wd.blk0 + k;
    if (b < part_lo || b >= part_hi) return;
    const BlockMeta m = meta[b];
    const StreamDesc sd = streams[wd.stream];
    // a part (lmcg_compress_part) holds its records only, back to back
    const uint64_t rec = part_hi != ~0ull ? scan[b] - scan[part_lo]
                                          : soff[wd.stream] + kHeader + (uint64_t)(wd.win_local + 1) * kSegEntry * segs +
                                                (scan[b] - scan[sd.blk0]);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint8_t* rp = out + rec;
    if (m.mode == MODE_RLE) {
        if (tid == 0) { rp[0] = MODE_RLE; put_u32(rp + 1, m.len); rp[5] = m.sym; }
        return;
    }
    const bool huff = m.mode == MODE_HUFFMAN;
    const uint32_t hdr = huff ? 5 + kHuffOverhead : 5;
    // preamble: mode | len | [codebook | bit count]
    if (tid < (int)hdr) {
        uint8_t v;
        if (tid == 0) v = m.mode;
        else if (tid < 5) v = (uint8_t)(m.len >> (8 * (tid - 1)));
        else if (tid < 133) v = wire[b * 128 + (tid - 5)];
        else v = (uint8_t)(m.bits >> (8 * (tid - 133)));
        rp[tid] = v;
    }
    const uint32_t w = wd.w;
    const uint64_t p0 = k * B, p1 = min(wd.W, p0 + B);
    if (tid == 32 && p1 <= (plane_of(p0, wd.n, w) + 1) * wd.n) {
        // the block's source elements (one plane): in L2 before the first loads
        const uint64_t e0 = p0 - plane_of(p0, wd.n, w) * wd.n;
        prefetch_l2(wd.src + e0 * w, (uint32_t)((p1 - p0) * w));
        if (wd.prev) prefetch_l2(wd.prev + e0 * w, (uint32_t)((p1 - p0) * w));
    }
    if (!huff) {  // stored record: the block's bytes verbatim after the 5-byte header
        const uint64_t g0 = plane_of(p0, wd.n, w);
        if (wd.vec && ((p1 - p0) & 15) == 0 && p1 <= (g0 + 1) * wd.n) {
            if (w == 1) store_plane_fast<1>(wd, p0, p1, rp + 5);
            else if (w == 2) store_plane_fast<2>(wd, p0, p1, rp + 5);
            else store_plane_fast<4>(wd, p0, p1, rp + 5);
            return;
        }
        store_plane(wd, p0, p1, stg, rp + 5);
        return;
    }
    // canonical code table (huffman.py:213-225): thread t handles symbol t
    if (tid < kWarps * 16) (&sh_cnt[0][0])[tid] = 0;
    __syncthreads();
    uint32_t my_len, my_rank_w;
    {
        const uint8_t wb = wire[b * 128 + (tid >> 1)];
        my_len = (tid & 1) ? (wb >> 4) : (wb & 15);
        const uint32_t mm = __match_any_sync(0xFFFFFFFFu, my_len);
        my_rank_w = __popc(mm & ((1u << lane) - 1));
        if (lane == __ffs(mm) - 1) sh_cnt[warp][my_len] = __popc(mm);
    }
    __syncthreads();
    if (tid < 16) {
        uint32_t tot[16];
        for (int l = 0; l < 16; l++) {
            uint32_t c = 0;
            for (int q = 0; q < kWarps; q++) c += sh_cnt[q][l];
            tot[l] = c;
        }
        uint32_t start = 0;
        for (int l = 1; l < 16; l++) {
            if (l == tid) sh_first[tid] = start;
            start += tot[l] << (kMaxLen - l);
        }
        if (tid == 0) sh_first[0] = 0;
    }
    __syncthreads();
    if (my_len) {
        uint32_t r = my_rank_w;
        for (int q = 0; q < warp; q++) r += sh_cnt[q][my_len];
        sh_code[enc_slot(tid)] = (my_len << 16) | ((sh_first[my_len] >> (kMaxLen - my_len)) + r);
    } else {
        sh_code[enc_slot(tid)] = 0;
    }
    const uint64_t gaddr = (uint64_t)(rp + hdr);
    const uint32_t lead = (uint32_t)(gaddr & 3) * 8;
    uint32_t* gw = reinterpret_cast<uint32_t*>(gaddr & ~(uint64_t)3);
    uint32_t bitpos = lead;     // staging coordinate of the next bit (< 32 at a round start)
    uint64_t base_word = 0;     // global word index (relative to gw) of stg[0]
    if (tid == 0) stg[0] = 0;
    if (tid == 0) sh_run = 256;
    __syncthreads();
    if (sh_code[enc_slot(tid)] == (1u << 16)) sh_run = tid;
    __syncthreads();
    // the run path pays off only when most symbols are the run symbol
    // (<= 1.5 code bits per symbol on average: XOR deltas, sparse tensors)
    const uint32_t rs = ((uint64_t)m.bits * 2 <= (uint64_t)(p1 - p0) * 3) ? sh_run : 256u;
    if (rs < 256) {
        if (w == 1) encode_runs<1, true>(wd, p0, p1, sh_wsum, stg, gw, lead, bitpos, base_word, rs);
        else if (w == 2) encode_runs<2, true>(wd, p0, p1, sh_wsum, stg, gw, lead, bitpos, base_word, rs);
        else encode_runs<4, true>(wd, p0, p1, sh_wsum, stg, gw, lead, bitpos, base_word, rs);
    } else {
        if (w == 1) encode_runs<1, false>(wd, p0, p1, sh_wsum, stg, gw, lead, bitpos, base_word, 0);
        else if (w == 2) encode_runs<2, false>(wd, p0, p1, sh_wsum, stg, gw, lead, bitpos, base_word, 0);
        else encode_runs<4, false>(wd, p0, p1, sh_wsum, stg, gw, lead, bitpos, base_word, 0);
    }
    // trailing partial word: bytes up to the record end
    if (tid == 0 && bitpos) {
        const uint32_t v = bswap32(stg[0]);
        uint8_t* bp = reinterpret_cast<uint8_t*>(gw) + base_word * 4;
        const uint32_t q0 = (base_word == 0) ? lead / 8 : 0;
        const uint32_t q1 = (bitpos + 7) / 8;
        for (uint32_t q = q0; q < q1; q++) bp[q] = (uint8_t)(v >> (8 * q));
    }
}

}  // namespace lmcg
