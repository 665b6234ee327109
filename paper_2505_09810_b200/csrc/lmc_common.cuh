// lmc_common.cuh -- shared layout, CRC-32 machinery and byte gathers for the
// B200 LMC kernels.  See DESIGN.md for the HBM layout and the roofline of
// each kernel.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace lmcg {

constexpr int kMaxLen = 15;               // huffman.py:33
constexpr uint32_t kHeader = 28;          // stream.py:72,77
constexpr uint32_t kSegEntry = 16;        // stream.py:74
constexpr uint32_t kHuffOverhead = 132;   // 128-byte codebook + u32 bit count, stream.py:80
constexpr int kThreads = 256;             // CTA size of the block kernels
constexpr int kWarps = kThreads / 32;
constexpr int kLaneBytes = 64;            // contiguous source bytes per lane per warp-tile
constexpr int kTileBytes = 32 * kLaneBytes;  // source bytes per warp-tile (2 KiB)

enum : uint8_t { MODE_HUFFMAN = 0, MODE_RLE = 1, MODE_STORED = 2 };

// One buffer-size window of one stream (stream.py:332-340).  A window is
// byte-grouped into w planes of n bytes; its grouped bytes are cut into
// blocks of B bytes (the last may be short, and when n % B != 0 a block
// straddles two planes).
struct WinDesc {
    const uint8_t* src;   // window start in the (next) payload
    const uint8_t* prev;  // window start in the previous step (fused XOR) or null
    uint64_t W;           // window bytes
    uint64_t n;           // bytes per plane = W / w
    uint64_t blk0;        // global index of the window's first block
    uint64_t slot0;       // global index of the window's first CTA slot
    uint32_t w;           // planes (element width when byte-grouped, else 1)
    uint32_t nblocks;     // ceil(W / B)
    uint32_t nslots;      // CTA slots (planes interleaved, see slot_to_block)
    uint32_t stream;      // owning stream
    uint32_t win_local;   // window index inside the stream
    uint32_t vec;         // 16-byte vector loads allowed (alignment of src/prev/W)
    uint64_t crc0;        // global index of the window's first CRC part
    uint32_t al16;        // src / prev 16-byte aligned
    uint32_t hcrc;        // 1: k_hist folds the CRC (parts = plane-0 blocks' element ranges, cunit bytes)
    uint64_t cunit;       // bytes per CRC part (kCrcChunk for k_crc, w * B for k_hist)
};

// One stream of the batch.
struct StreamDesc {
    uint64_t nbytes;      // original_length
    uint64_t blk0;        // first global block
    uint64_t nblk;        // blocks in this stream
    uint32_t win0;        // first global window
    uint32_t nwin;
    uint32_t flags;       // FLAG_BYTE_GROUPED | FLAG_DELTA
    uint32_t et;          // element type wire code
};

// Per-block result of the codebook stage (stream.py:161-177).
struct BlockMeta {
    uint32_t len;      // block bytes
    uint32_t recsize;  // serialized record bytes (mode u8 | len u32 | payload)
    uint32_t bits;     // Huffman payload bit count
    uint8_t mode;      // MODE_*
    uint8_t sym;       // RLE symbol
    uint8_t pm;        // 1 = lengths need package-merge (set by k_codebook)
    uint8_t pad;
};

// ---------------------------------------------------------------- CRC-32
// IEEE reflected polynomial 0xEDB88320 (zlib.crc32, stream.py:329).  Kernels
// compute *raw* CRCs (zero initial register, no final xor) of contiguous
// pieces and merge them with shift operators: raw(A||B) = shift(raw(A),|B|) ^
// raw(B); leading zero bytes leave a raw CRC unchanged.  The zlib value of a
// message of N bytes is raw ^ shift(0xFFFFFFFF, N) ^ 0xFFFFFFFF.
//
// Global tables (built once per context, see capi.cu):
//   crc_slice[4][256]     slice-by-4 tables
//   crc_shift[k][4][256]  byte-sliced operators "append 16*2^k zero bytes",
//                         k = 0..10 (16 B .. 16 KiB)
//   x2n[64]               x^(2^k) mod P for the generic shift
constexpr int kPow2Levels = 61;            // shifts by 2^m bytes, m = 0..60
struct CrcTables {
    uint32_t slice[4][256];
    uint32_t shift[11][4][256];            // shift by (16 << lvl) bytes
    uint32_t x2n[64];
    uint32_t pow2[kPow2Levels][4][256];    // shift by 2^m bytes
    // slice-by-4 tables for shared memory without bank conflicts in 32 KiB:
    // slice[t][i] at rep4x8[32 i + 8 t + c] for c = 0..7.  Lane l = c + 8 g
    // takes table t = (s + g) & 3 at its s-th lookup of a word, so the 32
    // lanes of every lookup instruction read 32 different banks.
    uint32_t rep4x8[256 * 32];
    // byte-sliced shift operators for k_hist's lane chains: 512 bytes (from
    // one row's piece to the next row's) and kHistTileGap bytes (from the end
    // of a piece to the piece of the same row in the warp's next tile)
    uint32_t sh512[4][256];
    uint32_t shtile[4][256];
    // the same for 32-byte lane pieces (sources aligned to 32 bytes, 256-bit
    // loads): two 1 KiB rows per tile, 1024 bytes apart, gap kHistTileGap32
    uint32_t sh1024[4][256];
    uint32_t shtile32[4][256];
};
constexpr uint32_t kHistTileGap = kWarps * kTileBytes - 16;
constexpr uint32_t kHistTileGap32 = kWarps * kTileBytes - 32;

// Per-lane view of rep4x8 for one word: tab[s] = table base of lookup s
// (column 8 t + c), sel[s] = byte-perm selector of the byte that pairs with
// table t (byte 3 - t, zero-extended).
struct Crc4x8Lane {
    const uint32_t* tab[4];
    uint32_t sel[4];
    __device__ __forceinline__ void init(const uint32_t* smem_rep4x8, int lane) {
        const int c = lane & 7, g = lane >> 3;
#pragma unroll
        for (int s = 0; s < 4; s++) {
            const int t = (s + g) & 3;
            tab[s] = smem_rep4x8 + 8 * t + c;
            sel[s] = 0x4440u | (uint32_t)(3 - t);
        }
    }
    // raw CRC after one little-endian word
    __device__ __forceinline__ uint32_t word(uint32_t crc, uint32_t w) const {
        const uint32_t x = crc ^ w;
        return tab[0][__byte_perm(x, 0, sel[0]) * 32] ^ tab[1][__byte_perm(x, 0, sel[1]) * 32] ^
               tab[2][__byte_perm(x, 0, sel[2]) * 32] ^ tab[3][__byte_perm(x, 0, sel[3]) * 32];
    }
};

__device__ __forceinline__ uint32_t crc_word(const uint32_t* __restrict__ sl, uint32_t crc, uint32_t word) {
    crc ^= word;
    return sl[768 + (crc & 0xFF)] ^ sl[512 + ((crc >> 8) & 0xFF)] ^ sl[256 + ((crc >> 16) & 0xFF)] ^
           sl[crc >> 24];
}
// Slicing-by-4 through 32-fold replicated tables: tl = table base + lane,
// entry (k, i) of slice k at tl[(256 k + i) * 32], so every lane reads its own
// bank (no conflicts) and one 32-bit word costs four lookups and no shifts of
// the running CRC between them.
constexpr size_t kRep4Words = 4 * 256 * 32;
__device__ __forceinline__ void load_rep4(uint32_t* tab, const CrcTables* __restrict__ ct) {
    const uint32_t* flat = &ct->slice[0][0];
    for (int i = threadIdx.x; i < (int)kRep4Words; i += blockDim.x) tab[i] = __ldg(flat + (i >> 5));
}
__device__ __forceinline__ uint32_t crc4_rep(const uint32_t* __restrict__ tl, uint32_t crc, uint32_t w) {
    const uint32_t x = crc ^ w;
    return tl[(768 + (x & 0xFF)) * 32] ^ tl[(512 + ((x >> 8) & 0xFF)) * 32] ^ tl[(256 + ((x >> 16) & 0xFF)) * 32] ^
           tl[(x >> 24) * 32];
}
__device__ __forceinline__ uint32_t crc_byte(const uint32_t* __restrict__ sl, uint32_t crc, uint32_t b) {
    return (crc >> 8) ^ sl[(crc ^ b) & 0xFF];
}
// shift by 64*2^k bytes through a byte-sliced operator table
__device__ __forceinline__ uint32_t crc_shift_tab(const uint32_t* __restrict__ t, uint32_t c) {
    return __ldg(&t[c & 0xFF]) ^ __ldg(&t[256 + ((c >> 8) & 0xFF)]) ^ __ldg(&t[512 + ((c >> 16) & 0xFF)]) ^
           __ldg(&t[768 + (c >> 24)]);
}
// a*b mod P in the reflected representation (zlib multmodp)
__device__ __forceinline__ uint32_t multmodp(uint32_t a, uint32_t b) {
    if (a == 0 || b == 0) return 0;
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
// x^(8*nbytes) mod P
__device__ __forceinline__ uint32_t x8nmodp(const uint32_t* __restrict__ x2n, uint64_t nbytes) {
    uint32_t p = 1u << 31;  // x^0
    int k = 3;
    uint64_t n = nbytes;
    while (n) {
        if (n & 1) p = multmodp(__ldg(&x2n[k & 63]), p);
        n >>= 1;
        k++;
    }
    return p;
}
__device__ __forceinline__ uint32_t crc_shift_generic(const uint32_t* __restrict__ x2n, uint32_t c, uint64_t nbytes) {
    if (c == 0 || nbytes == 0) return c;
    return multmodp(x8nmodp(x2n, nbytes), c);
}
// raw CRC shifted by n zero bytes: one table shift per set bit of n
__device__ __forceinline__ uint32_t crc_shift_bytes(const CrcTables* __restrict__ ct, uint32_t c, uint64_t n) {
    while (c && n) {
        const int m = __ffsll((long long)n) - 1;
        c = crc_shift_tab(&ct->pow2[m][0][0], c);
        n &= n - 1;
    }
    return c;
}

// Raw CRC of `count` consecutive parts of `unit` bytes each, part(i) given by
// get(i), combined by the whole CTA (blockDim.x threads, `red` = blockDim.x
// words of shared memory).  Missing leading parts are treated as zero bytes,
// which leave a raw CRC unchanged, so every thread folds the same number of
// parts.  Result valid on thread 0.
template <class F>
__device__ uint32_t crc_combine_uniform(const CrcTables* __restrict__ ct, uint64_t count, uint64_t unit, F get,
                                        uint32_t* red) {
    const int T = blockDim.x, tid = threadIdx.x;
    const uint64_t q = (count + T - 1) / T;
    const int64_t pad = (int64_t)(q * T) - (int64_t)count;
    uint32_t acc = 0;
    for (uint64_t v = (uint64_t)tid * q; v < (uint64_t)tid * q + q; v++) {
        const int64_t i = (int64_t)v - pad;
        acc = crc_shift_bytes(ct, acc, unit);
        if (i >= 0) acc ^= get((uint64_t)i);
    }
    red[tid] = acc;
    __syncthreads();
    for (int k = 1; k < T; k <<= 1) {
        if ((tid & (2 * k - 1)) == 0 && tid + k < T)
            red[tid] = crc_shift_bytes(ct, red[tid], unit * q * (uint64_t)k) ^ red[tid + k];
        __syncthreads();
    }
    const uint32_t r = red[0];
    __syncthreads();
    return r;
}

constexpr int kShift16 = 0, kShift512 = 5, kShift2K = 7, kShift16K = 10;  // crc_shift levels

// Warp tree over 32 lane parts of (16 << lvl0) bytes each (lane order = byte
// order): returns on lane 0 the raw CRC of the 32 parts.
__device__ __forceinline__ uint32_t crc_warp_tree(const CrcTables* __restrict__ ct, uint32_t c, int lane, int lvl0) {
#pragma unroll
    for (int k = 0; k < 5; k++) {
        uint32_t other = __shfl_down_sync(0xFFFFFFFFu, c, 1 << k);
        uint32_t shifted = crc_shift_tab(&ct->shift[lvl0 + k][0][0], c);
        if ((lane & ((2 << k) - 1)) == 0) c = shifted ^ other;
    }
    return c;
}

// raw CRC of 16 bytes held as 4 little-endian words
__device__ __forceinline__ uint32_t crc16(const uint32_t* __restrict__ sl, uint4 a) {
    uint32_t c = crc_word(sl, 0, a.x);
    c = crc_word(sl, c, a.y);
    c = crc_word(sl, c, a.z);
    return crc_word(sl, c, a.w);
}

// Plane-g symbols of the 16/w elements in one 16-byte piece, packed 4 per
// word in position order; returns the symbol count (16, 8 or 4).
__device__ __forceinline__ int piece_symbols(uint4 a, uint32_t w, uint32_t g, uint32_t s[4]) {
    if (w == 1) {
        s[0] = a.x; s[1] = a.y; s[2] = a.z; s[3] = a.w;
        return 16;
    }
    if (w == 2) {
        const uint32_t sel = g ? 0x7531 : 0x6420;
        s[0] = __byte_perm(a.x, a.y, sel);
        s[1] = __byte_perm(a.z, a.w, sel);
        return 8;
    }
    const uint32_t sel = g | ((4 + g) << 4);
    s[0] = __byte_perm(__byte_perm(a.x, a.y, sel), __byte_perm(a.z, a.w, sel), 0x5410);
    return 4;
}

__device__ __forceinline__ uint4 ldg16x(const uint8_t* src, const uint8_t* prev, uint64_t off) {
    uint4 a = __ldg(reinterpret_cast<const uint4*>(src + off));
    if (prev) {
        const uint4 b = __ldg(reinterpret_cast<const uint4*>(prev + off));
        a.x ^= b.x; a.y ^= b.y; a.z ^= b.z; a.w ^= b.w;
    }
    return a;
}

// 32 contiguous source bytes (32-byte aligned) XOR the previous step: one
// 256-bit load per operand (sm_100: LDG.E.ENL2.256)
__device__ __forceinline__ void ldg32x(const uint8_t* src, const uint8_t* prev, uint64_t off, uint4& a, uint4& b) {
    asm("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
        : "l"(src + off));
    if (prev) {
        uint4 c, d;
        asm("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w), "=r"(d.x), "=r"(d.y), "=r"(d.z), "=r"(d.w)
            : "l"(prev + off));
        a.x ^= c.x; a.y ^= c.y; a.z ^= c.z; a.w ^= c.w;
        b.x ^= d.x; b.y ^= d.y; b.z ^= d.z; b.w ^= d.w;
    }
}

// ------------------------------------------------------------- gathers
__device__ __forceinline__ uint4 ldg16(const uint8_t* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }

// 64 contiguous source bytes (16-byte aligned) XOR the previous step.
__device__ __forceinline__ void load64(const uint8_t* __restrict__ src, const uint8_t* __restrict__ prev,
                                       uint64_t off, uint32_t v[16]) {
#pragma unroll
    for (int q = 0; q < 4; q++) {
        uint4 a = ldg16(src + off + 16 * q);
        v[4 * q + 0] = a.x; v[4 * q + 1] = a.y; v[4 * q + 2] = a.z; v[4 * q + 3] = a.w;
    }
    if (prev) {
#pragma unroll
        for (int q = 0; q < 4; q++) {
            uint4 b = ldg16(prev + off + 16 * q);
            v[4 * q + 0] ^= b.x; v[4 * q + 1] ^= b.y; v[4 * q + 2] ^= b.z; v[4 * q + 3] ^= b.w;
        }
    }
}

// Plane-g symbols of the 64/w elements held in v (little-endian element
// bytes), packed 4 per word in position order.  Returns the symbol count.
__device__ __forceinline__ int extract_plane(const uint32_t v[16], uint32_t w, uint32_t g, uint32_t s[16]) {
    if (w == 1) {
#pragma unroll
        for (int k = 0; k < 16; k++) s[k] = v[k];
        return 64;
    }
    if (w == 2) {
        const uint32_t sel = g ? 0x7531 : 0x6420;
#pragma unroll
        for (int k = 0; k < 8; k++) s[k] = __byte_perm(v[2 * k], v[2 * k + 1], sel);
        return 32;
    }
    const uint32_t sel = g | ((4 + g) << 4);
#pragma unroll
    for (int k = 0; k < 4; k++) {
        uint32_t lo = __byte_perm(v[4 * k], v[4 * k + 1], sel);
        uint32_t hi = __byte_perm(v[4 * k + 2], v[4 * k + 3], sel);
        s[k] = __byte_perm(lo, hi, 0x5410);
    }
    return 16;
}

__device__ __forceinline__ uint32_t sym_at(const uint32_t s[16], int i) {
    return (s[i >> 2] >> (8 * (i & 3))) & 0xFF;
}

// Byte of grouped window position p (slow path).
__device__ __forceinline__ uint32_t gather_byte(const WinDesc& wd, uint64_t p) {
    uint64_t g = wd.w == 1 ? 0 : p / wd.n;
    uint64_t e = p - g * wd.n;
    uint64_t o = e * wd.w + g;
    uint32_t b = wd.src[o];
    if (wd.prev) b ^= wd.prev[o];
    return b;
}

// Map a CTA slot of a window to its block index, interleaving planes so that
// the CTAs reading the same source elements run back to back (the second read
// is then served from L2).  Returns -1 for idle slots.
__device__ __forceinline__ int64_t slot_to_block(const WinDesc& wd, uint64_t local, uint32_t B) {
    if (wd.w == 1) return local < wd.nblocks ? (int64_t)local : -1;
    uint64_t g = local % wd.w, j = local / wd.w;
    uint64_t sg = (g * wd.n + B - 1) / B;
    uint64_t sg1 = (g + 1 == wd.w) ? wd.nblocks : ((g + 1) * wd.n + B - 1) / B;
    uint64_t k = sg + j;
    return k < sg1 ? (int64_t)k : -1;
}

// log2 of an element width (1, 2 or 4)
__device__ __forceinline__ uint32_t lg2w(uint32_t w) { return w == 1 ? 0u : (w == 2 ? 1u : 2u); }
// plane of grouped position p (no 64-bit division)
__device__ __forceinline__ uint64_t plane_of(uint64_t p, uint64_t n, uint32_t w) {
    uint64_t g = 0;
    while (g + 1 < w && p >= (g + 1) * n) g++;
    return g;
}

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// TMA prefetch of [p, p + bytes) into L2 (16-byte aligned cover; nothing is
// written, a prefetch never faults the kernel)
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    const uint64_t a = reinterpret_cast<uint64_t>(p) & ~15ull;
    const uint64_t e = (reinterpret_cast<uint64_t>(p) + bytes + 15) & ~15ull;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(e - a)) : "memory");
}

}  // namespace lmcg
