// decompress.cu -- B200 kernels of the LMC decompress path.
//
// The host lays out, from per-stream hints (original length, segment count,
// window count: exact for streams this library produced, header-derived
// otherwise), fixed capacity regions for every stream's windows, segments,
// record slots, scan chunks and output tiles.  The whole pipeline then runs
// without a host round trip:
//
//   k_parse     one thread per stream: header + window/segment-table walk
//               with the reference's exact validation (stream.py:114-142,
//               358-389); window / segment descriptors (or RETRY when a
//               stream does not fit the hinted capacities); marks the windows
//               k_decpair decodes fused
//   k_maps      chunk -> segment, record slot -> segment, tile -> window
//   k_cand      record-header candidates "mode<=2|len==block" per 8 KiB span
//   k_number    per segment: exclusive scan of the chunk candidate counts
//   k_assign    record slot of every candidate (+ the tail record)
//   k_verify    one thread per record slot: candidates must chain exactly
//               (p -> p + record size) with the canonical record lengths
//   k_resolve   segments with false candidates: the path from the segment
//               start by pointer doubling
//   k_pairs +   (large decodes) persistent CTAs: low/high record pairs of
//   k_decpair   two-plane windows decoded into an L2 ring slot, interleaved
//               into the output with the tile CRCs in the same pass
//               (stream.py:190-215,392-403, huffman.py:258-349,
//               bytegroup.py:53-62); then the other windows' records into
//               the grouped scratch
//   k_decrec    (small decodes) CTA per record slot into the grouped scratch;
//               k_classify / k_decrec_large take the records whose payload
//               does not stage in kStageSmall
//   k_fallback  segments that failed discovery or decode are re-walked
//               serially, exactly like decompress_segment (stream.py:234-268)
//               -- the authoritative path for any stream
//   k_ungroup   inverse byte-grouping of the windows k_decpair did not write
//               (bytegroup.py:53-62) + raw CRC-32 of each 32 KiB output tile
//   k_finalize  per-stream CRC combine and status (stream.py:416-423)
#include <type_traits>

#include "lmc_common.cuh"

namespace lmcg {

constexpr int kChunk = 65536;        // segment payload bytes per k_scandec chunk
constexpr int kOutTile = 32768;      // output bytes per k_ungroup warp
constexpr int kLut = 11;             // LUT index bits
constexpr int kCntLut = 12;          // count-LUT index bits (no symbols: more codewords per lookup)

#ifdef LMCG_DEBUG
__device__ unsigned long long lmcg_dbg[32];
__device__ unsigned long long lmcg_dbg_ev[4096];   // 512 events x 8 words
#define DBG_ADD(i, v) atomicAdd(&lmcg_dbg[i], (unsigned long long)(v))
#define DBG_T0(var) unsigned long long var = clock64()
#define DBG_TADD(i, var) do { if (threadIdx.x == 0) atomicAdd(&lmcg_dbg[i], clock64() - var); } while (0)
#else
#define DBG_ADD(i, v) ((void)0)
#define DBG_T0(var) ((void)0)
#define DBG_TADD(i, var) ((void)0)
#endif

// segments the serial path (k_fallback) walked since the last reset
// (lmcg_fallback_segments): streams this library or the reference wrote
// decode on the parallel path; tests assert that it stays there.
__device__ unsigned long long lmcg_fallback_segs;

enum : uint32_t { ST_CORRUPT = 1, ST_INTEGRITY = 2, ST_UNSUPPORTED = 4, ST_RETRY = 8, ST_CAPACITY = 16, ST_SHAPE = 32 };

struct DecStreamIn {
    const uint8_t* p;
    uint64_t len;
    const uint8_t* prev;      // lmcg_decompress_apply: XOR the payload with prev (nullptr: plain decode)
    uint64_t prev_len;
};

// Per-stream capacity regions (host-computed from hints).
struct DecCaps {
    uint64_t win0, nwin;
    uint64_t seg0, nseg;
    uint64_t rec0, nrec;
    uint64_t chunk0, nchunk;
    uint64_t tile0, ntile;
    uint64_t scratch0, scratch;
    uint64_t out0, out;       // output offset and capacity
};

// Per-stream parse result (device; read back by the host with the status).
struct DecStreamOut {
    uint64_t orig;
    uint32_t status;
    uint32_t et, flags, crc;
    uint32_t nwin, nseg;       // actual counts (valid also on RETRY)
    uint64_t nrec, nchunk, ntile, scratch;
    uint32_t segs, block;
};

struct DecWin {
    uint64_t W, n;
    uint64_t goff;            // absolute scratch offset (16-aligned)
    uint64_t ooff;            // absolute output offset
    uint64_t soff;            // window start within the stream payload
    uint64_t tile0;           // global first tile
    uint32_t ntile, w, stream;
    uint32_t fuse;            // 1: k_decpair decodes the window straight into the output (see there)
    const uint8_t* prev;      // xor_apply source of this window's output (nullptr: none)
    uint64_t rec0, seg0;      // global first record slot / segment of the window
    uint32_t nseg, pad;
};

struct DecSeg {
    const uint8_t* base;      // segment payload start
    uint64_t comp, orig;      // compressed / original bytes
    uint64_t goff;            // absolute scratch offset of the segment's first byte
    uint64_t rec0, chunk0;    // global first record slot / chunk
    uint32_t nrec, nchunk;    // canonical records, scan chunks
    uint32_t block, stream;
    uint32_t win, pad;        // global window index
};

__device__ __forceinline__ uint32_t rd32(const uint8_t* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
__device__ __forceinline__ uint64_t rd64(const uint8_t* p) { return (uint64_t)rd32(p) | ((uint64_t)rd32(p + 4) << 32); }
__device__ __forceinline__ bool valid_block(uint32_t b) { return b >= 4096 && b <= (1u << 20) && (b & (b - 1)) == 0; }

// ---------------------------------------------------------------- k_parse
// Fused windows (DecWin.fuse, decoded by k_decpair): two byte planes (bf16 /
// fp16 byte-grouped), blocks of 16, 32 or 64 KiB, planes a whole number of
// blocks and every segment a whole number of blocks (so every record is a full
// block and low-plane record k pairs with high-plane record n / B + k), and
// 16-byte aligned output (and xor_apply source).
__global__ void k_parse(const DecStreamIn* __restrict__ in, const DecCaps* __restrict__ caps, int ns,
                        DecStreamOut* __restrict__ sout, DecWin* __restrict__ wins, DecSeg* __restrict__ segs,
                        const uint8_t* out, int fuse_ok) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ns) return;
    const uint8_t* p = in[s].p;
    const uint64_t len = in[s].len;
    const DecCaps cp = caps[s];
    DecStreamOut h = {};
    uint64_t nwin = 0, nseg = 0, nrec = 0, nchunk = 0, ntile = 0, scr = 0;
    bool bad = false;
    // parse_header (stream.py:114-142)
    if (len < kHeader || p[0] != 'L' || p[1] != 'M' || p[2] != 'C' || p[3] != '1' || p[4] != 1) {
        h.status = ST_UNSUPPORTED;
    } else {
        h.flags = p[5];
        h.et = p[6];
        h.orig = rd64(p + 8);
        const uint32_t B = rd32(p + 16), S = rd32(p + 20);
        h.block = B;
        h.segs = S;
        h.crc = rd32(p + 24);
        const uint32_t width = h.et == 0 ? 1 : (h.et == 3 ? 4 : 2);
        if ((h.flags & ~3u) || p[7] != 0 || h.et > 3 || !valid_block(B) || S < 1 || (h.orig % width)) {
            h.status = ST_CORRUPT;
        } else {
            const uint32_t wdt = (h.flags & 1) ? width : 1;
            const uint64_t table = (uint64_t)kSegEntry * S;
            uint64_t off = kHeader, remaining = h.orig, opos = 0;
            // iter_windows (stream.py:358-389)
            while (remaining > 0 && !bad) {
                if (table > len - off) { bad = true; break; }
                uint64_t wsum = 0;
                bool over = false, seg_aligned = true;
                for (uint64_t i = 0; i < S; i++) {
                    const uint64_t o = rd64(p + off + i * kSegEntry);
                    if (o > remaining - wsum) over = true;
                    else wsum += o;
                    if (o % B) seg_aligned = false;
                }
                const uint64_t toff = off;
                off += table;
                if (over || wsum == 0) { bad = true; break; }
                const uint64_t W = wsum;
                if ((h.flags & 1) && (W % width)) { bad = true; break; }  // reassemble_window
                const uint64_t wtiles = (W + kOutTile - 1) / kOutTile;
                if (nwin < cp.nwin && ntile + wtiles <= cp.ntile && scr + W <= cp.scratch) {
                    DecWin d;
                    d.W = W; d.n = W / wdt; d.w = wdt; d.stream = (uint32_t)s; d.pad = 0;
                    d.goff = cp.scratch0 + scr; d.ooff = cp.out0 + opos; d.soff = opos;
                    d.tile0 = cp.tile0 + ntile; d.ntile = (uint32_t)wtiles;
                    // xor_apply only with a prev of the payload's length (else k_finalize reports the mismatch)
                    d.prev = (in[s].prev && in[s].prev_len == h.orig) ? in[s].prev + opos : nullptr;
                    d.rec0 = cp.rec0 + nrec; d.seg0 = cp.seg0 + nseg; d.nseg = S;
                    d.fuse = fuse_ok && wdt == 2 && B >= 16384 && B <= 65536 && d.n >= B && d.n % B == 0 && seg_aligned &&
                             ((reinterpret_cast<uint64_t>(out) + d.ooff) & 15) == 0 &&
                             (reinterpret_cast<uint64_t>(d.prev) & 15) == 0;
                    wins[cp.win0 + nwin] = d;
                }
                uint64_t gpos = 0;
                for (uint64_t i = 0; i < S; i++) {
                    const uint64_t so = rd64(p + toff + i * kSegEntry), sc = rd64(p + toff + i * kSegEntry + 8);
                    if (sc > len - off) { bad = true; break; }
                    if ((so == 0) != (sc == 0)) { bad = true; break; }
                    // records are >= 6 bytes and decode to <= B bytes: anything more cannot
                    // walk (stream.py:240-250), so it is corrupt without looking further
                    if (so > (sc / 6) * (uint64_t)B) { bad = true; break; }
                    const uint64_t r = (so + B - 1) / B;
                    const uint64_t ch = (sc + kChunk - 1) / kChunk;
                    if (nseg < cp.nseg && nrec + r <= cp.nrec && nchunk + ch <= cp.nchunk && scr + W <= cp.scratch) {
                        DecSeg d;
                        d.base = p + off; d.comp = sc; d.orig = so;
                        d.goff = cp.scratch0 + scr + gpos;
                        d.rec0 = cp.rec0 + nrec; d.chunk0 = cp.chunk0 + nchunk;
                        d.nrec = (uint32_t)r; d.nchunk = (uint32_t)ch; d.block = B; d.stream = (uint32_t)s;
                        d.win = (uint32_t)(cp.win0 + nwin); d.pad = 0;
                        segs[cp.seg0 + nseg] = d;
                    }
                    nrec += r;
                    nchunk += ch;
                    nseg++;
                    off += sc;
                    gpos += so;
                }
                ntile += wtiles;
                scr += (W + 15) & ~15ull;
                nwin++;
                opos += W;
                remaining -= W;
            }
            if (!bad && off != len) bad = true;  // trailing bytes (stream.py:388-389)
            if (bad) h.status = ST_CORRUPT;
            else if (nwin > cp.nwin || nseg > cp.nseg || nrec > cp.nrec || nchunk > cp.nchunk || ntile > cp.ntile ||
                     scr > cp.scratch)
                h.status = ST_RETRY;
            else if (h.orig > cp.out)
                h.status = ST_CAPACITY;
        }
    }
    h.nwin = (uint32_t)nwin; h.nseg = (uint32_t)nseg; h.nrec = nrec; h.nchunk = nchunk; h.ntile = ntile; h.scratch = scr;
    sout[s] = h;
    // padding descriptors: unused (or rejected) capacity slots stay well-formed
    const bool ok = h.status == 0;
    const uint64_t used_w = ok ? nwin : 0, used_s = ok ? nseg : 0;
    const uint64_t end_rec = cp.rec0 + (ok ? nrec : 0), end_chunk = cp.chunk0 + (ok ? nchunk : 0);
    const uint64_t end_tile = cp.tile0 + (ok ? ntile : 0);
    for (uint64_t i = used_w; i < cp.nwin; i++) {
        DecWin d = {};
        d.tile0 = end_tile; d.stream = (uint32_t)s;
        wins[cp.win0 + i] = d;
    }
    for (uint64_t i = used_s; i < cp.nseg; i++) {
        DecSeg d = {};
        d.rec0 = end_rec; d.chunk0 = end_chunk; d.stream = (uint32_t)s; d.block = 4096;
        segs[cp.seg0 + i] = d;
    }
}

// ------------------------------------------------------- Huffman decoding
// Each record is decoded by one CTA: the bitstream is cut into one chunk of
// S bits per thread.  Pass 0 decodes every chunk from its nominal start
// (counting symbols, and marking the codeword boundaries of its first 64
// bits in a bitmap); a fix-up pass re-decodes a chunk from the end of its
// predecessor until it lands on one of those boundaries (Huffman codes
// self-synchronise within a few codewords); pass 2 re-decodes every chunk
// from its exact start and writes the symbols.  The decoder consumes up to
// three symbols per table lookup.
// Bitstream bytes staged in shared memory (longer payloads are read from
// global memory).  k_decrec runs twice: records whose payload fits
// kStageSmall at 4 CTAs per SM, then the larger ones with kStageLarge at 3
// (the staging area is the tail of the dynamic shared memory).
constexpr int kStageSmall = 30720, kStageLarge = 40960;
constexpr int kCheckpoints = 3;  // at 128, 256 and 512 bits into a chunk

struct DecSmem {
    uint32_t lut3[1 << kLut];           // tl(4)|pad(2)|n(2)|s3(8)|s2(8)|s1(8); 0: slow path (long or invalid prefix)
    uint16_t lut1[1 << kLut];           // (len << 8) | sym for codes <= kLut bits, else 0; entry i at lut1_at(i)
    uint8_t lutc[1 << kCntLut];         // count passes: n(4) | tl(4) of the whole codewords in a 12-bit window
    uint32_t bm[2][kThreads];           // pass-0 boundary bitmaps (first 64 bits of each chunk)
    uint32_t cp[kCheckpoints][kThreads];  // pass-0 checkpoints: (offset from p0) << 16 | symbol count
    uint32_t end[kThreads];
    uint8_t lens[256];
    uint8_t csym[256];
    uint32_t first_left[17], first_idx[17], bl_count[17];
    uint32_t cnt_w[kWarps][16];
    uint32_t wsum[kWarps];
    uint32_t kraft;
    int minlen, maxlen, lgcd;
    alignas(16) uint32_t bits[4];       // staged bitstream (TMA of the 16-byte aligned cover), big-endian
                                        // words; extends to the end of the dynamic shared memory
};
// dynamic shared memory of k_decrec / k_fallback for a staging capacity
__host__ __device__ constexpr size_t dec_smem_bytes(uint32_t stage) { return sizeof(DecSmem) + stage + 16; }

// Every kernel that decodes records keeps DecSmem at the start of its dynamic
// shared memory; the decoder addresses it through this symbol, so table and
// staging lookups are [register + constant] shared-memory loads (a DecSmem&
// handed through a call would cost a base-register add per lookup).
// lut1 is stored swizzled: entry i at i ^ (((i >> 6) & 31) << 1), i.e. the
// bank of an entry is bits 1..5 XOR bits 6..10 of its index.  The table
// builds look it up at (e << tl) & mask for the consecutive e of a warp (a
// power-of-two stride: up to 32 lanes in one bank of the plain layout, 8-11
// wavefronts per lookup measured); any five consecutive index bits now select
// five different bank bits, so those lookups are conflict-free.
__device__ __forceinline__ uint32_t lut1_at(uint32_t i) { return i ^ ((i >> 5) & 0x3Eu); }
extern __shared__ __align__(16) uint8_t g_dsmem[];
__device__ __forceinline__ DecSmem& dec_smem() { return *reinterpret_cast<DecSmem*>(g_dsmem); }
// The mbarrier of the payload bulk copy lives in the last 16 bytes of the
// dynamic shared memory (after the staging area: nothing else ever uses
// them) and is invalidated after every wait.  It used to sit inside DecSmem,
// which k_decpair overlays with its CRC tables after the decode: about one
// decompress in 300 then found the 8 bytes of barrier state written back over
// the table words in many CTAs at once (CRC-only IntegrityErrors on correct
// payloads) -- PTX requires mbarrier.inval before the memory of a barrier
// object is used for anything else.
__device__ __forceinline__ uint64_t* tma_bar(uint32_t stage_cap) {
    return reinterpret_cast<uint64_t*>(g_dsmem + sizeof(DecSmem) + stage_cap);
}

// Payload bit source: big-endian words, bit i of the payload is bit
// 31 - ((i + sh) & 31) of word (i + sh) >> 5; staged in shared memory when
// it fits (sw != null), else read from global memory.
struct Src {
    const uint32_t* sw;
    const uint8_t* gbase;      // 4-aligned global base
    uint64_t glimit;           // payload end in bytes from gbase
    uint64_t nwords_full;
    uint32_t sh;
    __device__ __forceinline__ uint32_t gword(uint64_t j) const {
        if (j < nwords_full) return bswap32(__ldg(reinterpret_cast<const uint32_t*>(gbase) + j));
        uint32_t v = 0;
        for (int q = 0; q < 4; q++) {
            const uint64_t o = j * 4 + q;
            v = (v << 8) | (o < glimit ? gbase[o] : 0u);
        }
        return v;
    }
    // the 32 payload bits starting at bit pos (zeros past the end)
    template <bool STAGED = false>
    __device__ __forceinline__ uint32_t peek(uint32_t pos) const {
        const uint32_t a = pos + sh;
        const uint32_t j = a >> 5;
        uint32_t w0, w1;
        if (STAGED) {
            w0 = sw[j];
            w1 = sw[j + 1];
        } else {
            w0 = gword(j);
            w1 = gword(j + 1);
        }
        return __funnelshift_l(w1, w0, a & 31);
    }
};

// One codeword at the window: returns its length (0 = invalid prefix).
__device__ __forceinline__ uint32_t step1(const DecSmem& s, uint32_t win, uint32_t& sym) {
    const uint32_t e = s.lut1[lut1_at(win >> (32 - kLut))];
    if (e) {
        sym = e & 0xFF;
        return e >> 8;
    }
    const uint32_t win15 = win >> 17;
    for (int q = kLut + 1; q <= s.maxlen; q++) {
        const uint32_t fl = s.first_left[q], endq = fl + (s.bl_count[q] << (kMaxLen - q));
        if (s.bl_count[q] && win15 >= fl && win15 < endq) {
            sym = s.csym[s.first_idx[q] + ((win15 - fl) >> (kMaxLen - q))];
            return q;
        }
    }
    return 0;
}

// Decode the codewords that start in [pos, lim).  Returns the first boundary
// >= lim (~0u on an invalid prefix) and the symbol count.
//   bm == 1: mark the boundaries within [p0, p0 + 64) in this thread's bitmap
//   bm == 2: stop as soon as a boundary hits that bitmap (*hit = the old
//            path's symbol count at that boundary, else ~0u)
//   EMIT:    write the symbols to dst
// The bulk loop is branch-free apart from codes longer than kLut bits:
// one 32-bit window (two word reads + funnel shift), one table lookup, up to
// three symbols.
template <bool EMIT, bool STAGED, bool RUN>
__device__ __forceinline__ uint32_t decode_span(DecSmem& s, const Src& src, uint32_t pos, uint32_t lim, uint32_t p0, int bm,
                                uint32_t& count, uint8_t* dst, uint32_t* hit, bool sparse = false) {
    // Lanes decode different chunks with different trip counts: every loop is
    // driven by a warp vote so the warp re-converges each iteration (instead of
    // drifting into independently scheduled, divergent lanes).
    const unsigned mask = __activemask();
    const int tid = threadIdx.x;
    uint32_t c = 0;
    bool bad = false, done = false;
    // staged payload: read through a two-word register bit buffer (hi:lo,
    // window = funnel shift by boff < 32), refilled branch-free (the next
    // word is always inside the staging area)
    uint32_t bhi = 0, blo = 0, boff = 0, bnj = 0;
    if (STAGED) {
        const uint32_t a0 = pos + src.sh, j0 = a0 >> 5;
        boff = a0 & 31;
        bhi = src.sw[j0];
        blo = src.sw[j0 + 1];
        bnj = j0 + 2;
    }
    auto win = [&]() -> uint32_t { return STAGED ? __funnelshift_l(blo, bhi, boff) : src.template peek<STAGED>(pos); };
    // a 1-bit codeword is '0' (canonical codes start at zero): every leading
    // zero bit of the window is one more of that symbol, so runs of it (XOR
    // deltas are mostly zero bytes) go many symbols per lookup
    constexpr bool run1 = RUN;   // (the record has a 1-bit codeword)
    const uint64_t rep8 = RUN ? s.csym[s.first_idx[1]] * 0x0101010101010101ull : 0ull;
    auto adv = [&](uint32_t l) {   // l <= 32
        pos += l;
        if (STAGED) {
            boff += l;
            const bool rf = boff >= 32;
            const uint32_t nw = src.sw[bnj];
            bhi = rf ? blo : bhi;
            blo = rf ? nw : blo;
            bnj += rf ? 1u : 0u;
            boff -= rf ? 32u : 0u;
        }
    };
    if (!EMIT) {
        // (every lane of the mask runs this loop's votes, also those with bm == 0)
        uint32_t m0 = 0, m1 = 0;
        if (bm == 2) { m0 = s.bm[0][tid]; m1 = s.bm[1][tid]; }
        bool act = bm != 0 && pos < lim && pos < p0 + 64;
        while (__any_sync(mask, act)) {
            if (act) {
                uint32_t sym;
                const uint32_t wv = win();
                // a run of the 1-bit symbol: its z boundaries pos+1 .. pos+z at once
                const uint32_t z = RUN ? min((uint32_t)__clz(wv), min(lim - pos, p0 + 64 - pos)) : 0u;
                if (RUN && z) {
                    const int r0 = (int)(pos - p0);          // may be negative (fix-up before p0)
                    const int lo = max(r0 + 1, 0), hi = min(r0 + (int)z, 63);
                    const uint64_t mk = lo <= hi ? ((~0ull >> (63 - hi + lo)) << lo) : 0ull;
                    uint32_t take = z;
                    if (bm == 1) {
                        m0 |= (uint32_t)mk;
                        m1 |= (uint32_t)(mk >> 32);
                    } else {
                        const uint64_t m = ((uint64_t)m1 << 32) | m0;
                        const uint64_t h = m & mk;
                        if (h) {   // synchronised at the first old boundary on the run
                            const int b = __ffsll((long long)h) - 1;
                            take = (uint32_t)(b - r0);
                            *hit = __popcll(m & (~0ull >> (63 - b)));
                            done = true;
                        }
                    }
                    adv(take);
                    c += take;
                } else {
                const uint32_t l = step1(s, wv, sym);
                if (!l) {
                    bad = true;
                } else {
                    adv(l);
                    c++;
                    const uint32_t rel = pos - p0;
                    if (rel < 64) {
                        const uint32_t bit = 1u << (rel & 31);
                        if (bm == 1) {
                            if (rel < 32) m0 |= bit; else m1 |= bit;
                        } else if ((rel < 32 ? m0 : m1) & bit) {
                            // synchronised: old count at this boundary = boundaries at or below rel
                            *hit = rel < 32 ? __popc(m0 & (bit | (bit - 1))) : __popc(m0) + __popc(m1 & (bit | (bit - 1)));
                            done = true;
                        }
                    }
                }
                }
                act = !bad && !done && pos < lim && pos < p0 + 64;
            }
        }
        if (bm == 1) { s.bm[0][tid] = m0; s.bm[1][tid] = m1; }
        // checkpoints: the first codeword boundary at or after p0 + (128 << k)
        // (pass 0 records it with its symbol count; a fix-up path that lands
        // on it is synchronised), for paths that do not resynchronise within
        // the 64-bit bitmap
#pragma unroll 1
        for (int k = 0; k < kCheckpoints; k++) {
            // pass 0 (bm == 1) records the first boundary at or after p0 + (128 << k);
            // a fix-up path (bm == 2) walks to the recorded boundary (whichever pass 0
            // recorded it) and is synchronised iff it lands on it
            const uint32_t cpk = bm == 2 ? s.cp[k][tid] : 0u;
            const uint32_t T = bm == 2 ? (cpk == ~0u ? lim : p0 + (cpk >> 16)) : p0 + (128u << k);
            const bool on = bm != 0 && !bad && !done && T < lim;
            constexpr int kCW = RUN ? kLut : kCntLut;
            bool a2 = on && pos + kCW <= T;
            while (__any_sync(mask, a2)) {
                if (a2) {
                    const uint32_t wv = win();
                    uint32_t n, tl;
                    if (RUN) {
                        const uint32_t e = s.lut3[wv >> (32 - kLut)];
                        n = (e >> 24) & 3; tl = e >> 28;
                    } else {
                        const uint32_t e = s.lutc[wv >> (32 - kCntLut)];
                        n = e >> 4; tl = e & 15;
                    }
                    if (run1) {
                        const uint32_t z = min((uint32_t)__clz(wv), T - pos);
                        if (z > n) { n = z; tl = z; }
                    }
                    if (n == 0) {
                        uint32_t sym;
                        tl = step1(s, wv, sym);
                        n = 1;
                        bad = tl == 0;
                    }
                    adv(tl);
                    c += n;
                    a2 = !bad && pos + kCW <= T;
                }
            }
            a2 = on && !bad && pos < T;
            while (__any_sync(mask, a2)) {
                if (a2) {
                    uint32_t sym;
                    const uint32_t l = step1(s, win(), sym);
                    if (!l) bad = true;
                    else { adv(l); c++; }
                    a2 = !bad && pos < T;
                }
            }
            if (on && !bad) {
                if (bm == 1) {
                    s.cp[k][tid] = ((pos - p0) << 16) | c;
                } else if (pos - p0 == (s.cp[k][tid] >> 16)) {
                    *hit = s.cp[k][tid] & 0xFFFF;
                    done = true;
                }
            }
        }
    }
    uint8_t* d = dst;
    if (EMIT && RUN && sparse) {
        // The plane is already filled with the run symbol (huff_passes): walk
        // the chunk, every leading zero bit of the window one run symbol (up to
        // 32 per step, nothing to store), and store only the other symbols.
        bool act = pos < lim;
        while (__any_sync(mask, act)) {
            if (act) {
                const uint32_t wv = win();
                const uint32_t z = min((uint32_t)__clz(wv), lim - pos);
                if (z) {
                    adv(z);
                    d += z;
                    c += z;
                } else {
                    uint32_t sym;
                    const uint32_t l = step1(s, wv, sym);
                    if (!l) {
                        bad = true;
                    } else {
                        adv(l);
                        *d++ = (uint8_t)sym;
                        c++;
                    }
                }
                act = !bad && pos < lim;
            }
        }
        count = c;
        return bad ? ~0u : pos;
    }
    if (EMIT) {
        // head: single symbols until the destination is 8-byte aligned
        bool act = pos < lim && (reinterpret_cast<uint64_t>(d) & 7);
        while (__any_sync(mask, act)) {
            if (act) {
                uint32_t sym;
                const uint32_t l = step1(s, win(), sym);
                if (!l) {
                    bad = true;
                } else {
                    adv(l);
                    c++;
                    *d++ = (uint8_t)sym;
                }
                act = !bad && pos < lim && (reinterpret_cast<uint64_t>(d) & 7);
            }
        }
    }
    uint64_t* w = reinterpret_cast<uint64_t*>(d);
    uint64_t acc = 0;
    uint32_t nacc = 0;
    constexpr int kW = (EMIT || RUN) ? kLut : kCntLut;   // window bits of the bulk lookups
    bool act = !bad && !done && pos + kW <= lim;
    // bulk: up to three symbols (count passes: twelve) per table lookup, two lookups per vote
    auto lookup = [&]() {
        const uint32_t wv = win();
        uint32_t n, tl;
        using PackT = typename std::conditional<RUN, uint64_t, uint32_t>::type;
        PackT packed = 0;
        if (EMIT) {
            const uint32_t e = s.lut3[wv >> (32 - kLut)];
            n = (e >> 24) & 3; tl = e >> 28; packed = e & 0xFFFFFF;
            if (run1) {   // up to 8 run symbols: one 8-byte store at most
                const uint32_t z = min((uint32_t)__clz(wv), 8u);
                if (z > n) { n = z; tl = z; packed = rep8 >> (64 - 8 * z); }
            }
        } else {
            if (RUN) {   // counting with the 3-symbol table (run records build no count LUT)
                const uint32_t e = s.lut3[wv >> (32 - kLut)];
                n = (e >> 24) & 3; tl = e >> 28;
            } else {
                const uint32_t e = s.lutc[wv >> (32 - kCntLut)];
                n = e >> 4; tl = e & 15;
            }
            if (run1) {
                const uint32_t z = min((uint32_t)__clz(wv), lim - pos);
                if (z > n) { n = z; tl = z; }
            }
        }
        if (n == 0) {
            uint32_t sym;
            tl = step1(s, wv, sym);
            n = 1;
            packed = sym;
            bad = tl == 0;
        }
        adv(tl);
        c += n;
        DBG_ADD(EMIT ? 25 : 26, 1);
        if (EMIT) {   // branch-free packing: predicated 8-byte store
            acc |= (uint64_t)packed << (8 * nacc);
            const uint32_t nn = nacc + n;
            const bool full = nn >= 8;   // (without runs: implies nacc >= 5)
            asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p st.global.u64 [%0], %1; }"
                         :: "l"(w), "l"(acc), "r"((uint32_t)full) : "memory");
            w += full ? 1 : 0;
            if (RUN) acc = full ? (nacc ? (uint64_t)packed >> (8 * (8 - nacc)) : 0ull) : acc;
            else acc = full ? ((uint64_t)packed >> (8 * (8 - nacc))) : acc;
            nacc = full ? nn - 8 : nn;
        }
    };
    while (__any_sync(mask, act)) {
        if (act) {
            lookup();
            if (!bad && pos + kW <= lim) lookup();
            act = !bad && pos + kW <= lim;
        }
    }
    act = !bad && !done && pos < lim;
    while (__any_sync(mask, act)) {
        if (act) {
            uint32_t sym;
            const uint32_t l = step1(s, win(), sym);
            if (!l) {
                bad = true;
            } else {
                adv(l);
                c++;
                if (EMIT) {
                    acc |= (uint64_t)sym << (8 * nacc);
                    if (++nacc == 8) {
                        *w++ = acc;
                        acc = 0;
                        nacc = 0;
                    }
                }
            }
            act = !bad && pos < lim;
        }
    }
    if (EMIT && !bad) {
        uint8_t* b = reinterpret_cast<uint8_t*>(w);
        for (uint32_t q = 0; q < nacc; q++) b[q] = (uint8_t)(acc >> (8 * q));
    }
    if (bm == 2 && !done) *hit = ~0u;
    DBG_ADD(EMIT ? 4 : bm * 2, 1);
    DBG_ADD((EMIT ? 4 : bm * 2) + 1, c);
    count = c;
    return bad ? ~0u : pos;
}

// ------------------------------------------------ lean passes (staged, no 1-bit code)
// Records whose payload is staged in shared memory and whose code has no
// 1-bit codeword (the weight exponent planes) take these loops: a two-word
// register bit buffer refilled branch-free after every lookup, K table
// lookups per warp vote, no branch per lookup (a window whose first codeword
// is longer than the table, or invalid, reads entry 0: the lookups of that
// lane consume nothing and one codeword is decoded by step1 after the vote),
// inactive lanes mask their lookups to no-ops.
struct BitBuf {
    uint32_t hi, lo, boff, j;   // window = funnelshift_l(lo, hi, boff); sw[j] is the next word
};
__device__ __forceinline__ void bb_init(BitBuf& b, const uint32_t* sw, uint32_t a) {
    b.j = a >> 5;
    b.boff = a & 31;
    b.hi = sw[b.j];
    b.lo = sw[b.j + 1];
    b.j += 2;
}
__device__ __forceinline__ uint32_t bb_win(const BitBuf& b) { return __funnelshift_l(b.lo, b.hi, b.boff); }
__device__ __forceinline__ void bb_adv(BitBuf& b, const uint32_t* sw, uint32_t l) {   // l <= 32
    b.boff += l;
    const bool rf = b.boff >= 32;
    const uint32_t nw = sw[b.j];
    b.hi = rf ? b.lo : b.hi;
    b.lo = rf ? nw : b.lo;
    b.j += rf ? 1u : 0u;
    b.boff -= rf ? 32u : 0u;
}

// Pass 0 of one chunk [p0, lim): the codeword boundaries of its first 32
// bits into the bitmap, checkpoints (the first lookup end at or after
// p0 + 128 / 256 / 512 bits, with the symbol count there) for the fix-up
// rounds, and the count.  Returns the first boundary >= lim (~0u: invalid).
// After its chunk the thread keeps decoding single codewords and marks the
// boundaries of its path inside the first 32 bits of the next chunk (np0 =
// that chunk's speculative start, ~0u: none) in `ov`, stopping at the first
// one that is also a boundary of the next chunk's own pass-0 path (its bitmap
// comes from lane + 1 by shuffle; lane 31 walks the 32 bits): the fix-up of the
// next chunk is then bit arithmetic on the two bitmaps (huff_passes).
template <int K>
__device__ __forceinline__ uint32_t pass0_lean(DecSmem& s, const uint32_t* sw, uint32_t sh, uint32_t p0, uint32_t lim,
                                               uint32_t& count, uint32_t np0, uint32_t bits, uint32_t& ov) {
    constexpr unsigned mask = 0xFFFFFFFFu;   // called by every thread (an empty chunk: p0 == lim)
    const int tid = threadIdx.x;
    BitBuf b;
    bb_init(b, sw, p0 + sh);
    uint32_t pos = p0, c = 0, m0 = 0, m1 = 0;
    bool bad = false;
    // (32 bits: the weight planes resynchronise within 20 bits; longer paths
    // meet a checkpoint)
    const uint32_t la = min(lim, p0 + 32);
    bool act = pos < la;
    while (__any_sync(mask, act)) {
        if (act) {
            uint32_t sym;
            const uint32_t l = step1(s, bb_win(b), sym);
            bad = l == 0;
            bb_adv(b, sw, l);
            pos += l;
            c += l ? 1u : 0u;
            const uint32_t rel = pos - p0;
            if (l && rel < 32) m0 |= 1u << rel;
            act = !bad && pos < la;
        }
    }
    s.bm[0][tid] = m0;
    s.bm[1][tid] = m1;
    uint32_t k = 0, T = p0 + 128;
    auto bulk = [&](auto kk) {
        constexpr int KK = decltype(kk)::value;
        bool a = !bad && pos + KK * kCntLut <= lim;
        while (__any_sync(mask, a)) {
            uint32_t tl = 0;
#pragma unroll
            for (int q = 0; q < KK; q++) {
                const uint32_t e = a ? (uint32_t)s.lutc[bb_win(b) >> (32 - kCntLut)] : 0u;
                tl = e & 15;
                c += e >> 4;
                pos += tl;
                bb_adv(b, sw, tl);
            }
            const bool st = a && tl == 0;   // a long (or invalid) codeword at the window
            if (__any_sync(mask, st)) {
                if (st) {
                    uint32_t sym;
                    const uint32_t l = step1(s, bb_win(b), sym);
                    bad = l == 0;
                    bb_adv(b, sw, l);
                    pos += l;
                    c += l ? 1u : 0u;
                }
            }
            if (a && k < kCheckpoints && pos >= T) {
                s.cp[k][tid] = ((pos - p0) << 16) | c;
                k++;
                T = p0 + (128u << k);
            }
            a = !bad && pos + KK * kCntLut <= lim;
        }
    };
    bulk(std::integral_constant<int, K>());
    bulk(std::integral_constant<int, 1>());
    act = !bad && pos < lim;
    while (__any_sync(mask, act)) {
        if (act) {
            uint32_t sym;
            const uint32_t l = step1(s, bb_win(b), sym);
            bad = l == 0;
            bb_adv(b, sw, l);
            pos += l;
            c += l ? 1u : 0u;
            act = !bad && pos < lim;
        }
    }
    count = c;
    {
        const int lane = tid & 31;
        // the next chunk's speculative boundaries (bit 0: its start), relative to np0
        uint32_t mnext = __shfl_down_sync(mask, m0 | 1u, 1);
        if (lane == 31) mnext = 0;
        const uint32_t pend = pos;
        uint32_t o = 0;
        const uint32_t stop = np0 == ~0u ? 0u : min(np0 + 32, bits);
        act = !bad && np0 != ~0u && pos < stop;
        while (__any_sync(mask, act)) {
            if (act) {
                bool hit = false;
                if (pos >= np0) {
                    o |= 1u << (pos - np0);
                    hit = (mnext >> (pos - np0)) & 1u;
                }
                uint32_t sym;
                const uint32_t l = hit ? 0u : step1(s, bb_win(b), sym);
                bb_adv(b, sw, l);
                pos += l;
                act = l != 0 && pos < stop;
            }
        }
        ov = o;
        pos = pend;
    }
    return bad ? ~0u : pos;
}

// Emit pass of one chunk: the codewords starting in [pos, lim) (validated by
// pass 0 and the fix-up rounds) as symbols at dst.  Up to three symbols per
// lookup are packed into a 32-bit accumulator; its full words queue in four
// registers and leave as 16-byte stores.
template <int K>
__device__ __forceinline__ void emit_lean(DecSmem& s, const uint32_t* sw, uint32_t sh, uint32_t pos, uint32_t lim,
                                          uint8_t* dst) {
    constexpr unsigned mask = 0xFFFFFFFFu;   // called by every thread (nothing to emit: pos == lim)
    BitBuf b;
    bb_init(b, sw, pos + sh);
    uint8_t* d = dst;
    // head: single symbols until the destination is 16-byte aligned
    bool act = pos < lim && (reinterpret_cast<uint64_t>(d) & 15);
    while (__any_sync(mask, act)) {
        if (act) {
            uint32_t sym;
            const uint32_t l = step1(s, bb_win(b), sym);
            bb_adv(b, sw, l);
            pos += l;
            *d++ = (uint8_t)sym;
            act = l && pos < lim && (reinterpret_cast<uint64_t>(d) & 15);
        }
    }
    // Full words collect in a four-register queue (oldest in q0 when it is
    // full) and leave as one 16-byte store: a warp's stores go to 32
    // different lines whatever their width, so 4-byte stores cost four times
    // the LSU wavefronts and L2 write sectors per byte (the kernel's LSU data
    // pipe ran at 68%, half of it these stores).
    uint4* w = reinterpret_cast<uint4*>(d);
    uint32_t acc = 0, nb = 0;   // accumulated bits (0, 8, 16 or 24)
    uint32_t q0 = 0, q1 = 0, q2 = 0, q3 = 0, wc = 0;
    auto put = [&](uint32_t packed, uint32_t nbits) {   // packed: up to 3 symbols, nbits = 8 * count
        acc |= packed << nb;
        const uint32_t ovf = __funnelshift_lc(packed, 0u, nb);   // the bytes beyond the word (packed >> (32 - nb))
        nb += nbits;
        if (nb >= 32) {
            q0 = q1; q1 = q2; q2 = q3; q3 = acc;
            acc = ovf;
            nb -= 32;
            if (++wc == 4) {
                *w++ = make_uint4(q0, q1, q2, q3);
                wc = 0;
            }
        }
    };
    auto bulk = [&](auto kk) {
        constexpr int KK = decltype(kk)::value;
        bool a = pos + KK * kLut <= lim;
        while (__any_sync(mask, a)) {
            uint32_t tl = 0;
#pragma unroll
            for (int q = 0; q < KK; q++) {
                const uint32_t e = a ? s.lut3[bb_win(b) >> (32 - kLut)] : 0u;
                tl = e >> 28;
                pos += tl;
                bb_adv(b, sw, tl);
                put(e & 0xFFFFFF, (e >> 21) & 0x18);
            }
            const bool st = a && tl == 0;   // a codeword longer than the table
            if (__any_sync(mask, st)) {
                if (st) {
                    uint32_t sym;
                    const uint32_t l = step1(s, bb_win(b), sym);
                    bb_adv(b, sw, l);
                    pos += l;
                    put(sym, 8);
                }
            }
            a = pos + KK * kLut <= lim;
        }
    };
    bulk(std::integral_constant<int, K>());   // (every lane of the mask runs the votes)
    bulk(std::integral_constant<int, 1>());
    act = pos < lim;
    while (__any_sync(mask, act)) {
        if (act) {
            uint32_t sym;
            const uint32_t l = step1(s, bb_win(b), sym);
            bb_adv(b, sw, l);
            pos += l;
            put(sym, 8);
            act = l && pos < lim;
        }
    }
    // the queue's wc words (the newest in q3), then the bytes of the open word
    uint32_t* tw = reinterpret_cast<uint32_t*>(w);
    if (wc == 3) { tw[0] = q1; tw[1] = q2; tw[2] = q3; }
    else if (wc == 2) { tw[0] = q2; tw[1] = q3; }
    else if (wc == 1) tw[0] = q3;
    uint8_t* tb = reinterpret_cast<uint8_t*>(tw + wc);
    for (uint32_t q = 0; q < nb / 8; q++) tb[q] = (uint8_t)(acc >> (8 * q));
}

// All passes over the chunks of one record (see huff_decode).
template <bool STAGED, bool RUN>
__device__ __forceinline__ bool huff_passes(DecSmem& s, const Src& src, uint32_t bits, uint32_t len, uint8_t* dst) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t S = (bits + kThreads - 1) / kThreads;
    S = max(128u, (S + 31) & ~31u);
    const uint32_t nch = (bits + S - 1) / S;
    // every codeword boundary is a multiple of the gcd of the code lengths:
    // chunk starts off that grid could never resynchronise
    const uint32_t gq = s.lgcd;
    const uint32_t c = tid;
    const uint32_t lim = min((c + 1) * S, bits);
    uint32_t p0 = 0, my_start = 0, my_end = 0, my_cnt = 0;
    DBG_T0(t_p0);
#pragma unroll
    for (int k = 0; k < kCheckpoints; k++) s.cp[k][tid] = ~0u;
    if (STAGED && !RUN) {
        // the lean loops vote over full warps: every thread runs them, empty chunks as [0, 0)
        if (c < nch) {
            p0 = c * S;
            if (gq > 1) p0 = ((p0 + gq - 1) / gq) * gq;
            my_start = p0;
        }
        const bool work = c < nch && my_start < lim;
        uint32_t cnt = 0, ov = 0, np0 = ~0u;
        if (work && c + 1 < nch) {
            np0 = (c + 1) * S;
            if (gq > 1) np0 = ((np0 + gq - 1) / gq) * gq;
        }
        const uint32_t e = pass0_lean<3>(s, src.sw, src.sh, work ? my_start : 0u, work ? lim : 0u, cnt, np0, bits, ov);
        if (c < nch) {
            my_end = work ? e : my_start;
            my_cnt = cnt;
            s.end[c] = my_end;
        }
        s.bm[1][tid] = ov;   // (for the bitmap fix-up below; zero again before the general rounds)
    } else if (c < nch) {
        p0 = c * S;
        if (gq > 1) p0 = ((p0 + gq - 1) / gq) * gq;
        my_start = p0;
        if (my_start >= lim) { my_end = my_start; s.bm[0][tid] = 0; s.bm[1][tid] = 0; }
        else my_end = decode_span<false, STAGED, RUN>(s, src, my_start, lim, p0, 1, my_cnt, nullptr, nullptr);
        s.end[c] = my_end;
    }
    __syncthreads();
    DBG_TADD(18, t_p0);
    DBG_T0(t_fix);
    const uint32_t p0_end = my_end, p0_cnt = my_cnt;   // the pass-0 path's end and count
    if (STAGED && !RUN) {
        // Bitmap fix-up: chunk c's true path starts at its predecessor's end
        // pe.  A = the boundaries of c's pass-0 path in its first 32 bits (bit
        // 0: its start), Bm = the predecessor's path there (pass0_lean's
        // overshoot).  The paths merge at the first common boundary x: the
        // codewords of the true path that start in [pe, x) replace those of
        // the pass-0 path that start before x; the end stays.  Chunks that do
        // not merge inside their 32 bits (or inside the chunk) are left to
        // the general rounds below, which also re-check every start.
        uint32_t pe = ~0u, Bm = 0;
        if (c < nch && c > 0) { pe = s.end[c - 1]; Bm = s.bm[1][tid - 1]; }
        __syncthreads();
        s.bm[1][tid] = 0;
        if (c < nch && c > 0 && pe != ~0u && pe != my_start && my_end != ~0u && pe >= p0 && my_start < lim) {
            const uint32_t A = s.bm[0][tid] | 1u;
            const uint32_t X = A & Bm;
            if (X) {
                const uint32_t x = __ffs(X) - 1;
                if (p0 + x < lim) {
                    const uint32_t below = (1u << x) - 1;
                    my_cnt = my_cnt - __popc(A & below) + __popc(Bm & below);
                    my_start = pe;
                }
            }
        }
    }
    // fix-up rounds until every chunk starts where its predecessor ended; a
    // re-decoded path that meets the pass-0 path (bitmap or checkpoint) takes
    // the rest of its count and its end from pass 0
    for (;;) {
        uint32_t pe = 0;
        if (c < nch && c > 0) pe = s.end[c - 1];
        __syncthreads();
        int changed = 0;
        if (c < nch && c > 0 && pe != ~0u && pe != my_start) {
            my_start = pe;
            if (my_start >= lim) {
                my_end = my_start;
                my_cnt = 0;
            } else {
                uint32_t h = ~0u, cnt2 = 0;
                const uint32_t e2 = decode_span<false, STAGED, RUN>(s, src, my_start, lim, p0, 2, cnt2, nullptr, &h);
                DBG_ADD(6, h == ~0u);
#if defined(LMCG_DEBUG) && !defined(LMCG_CHECK_TABLES)
                if (h == ~0u) {
                    const unsigned long long k = atomicAdd(&lmcg_dbg[10], 1ull);
                    if (k < 512) {
                        unsigned long long* e = lmcg_dbg_ev + 8 * k;
                        e[0] = blockIdx.x; e[1] = c; e[2] = p0; e[3] = pe; e[4] = lim; e[5] = bits;
                        e[6] = (unsigned long long)s.minlen << 32 | s.maxlen; e[7] = (unsigned long long)p0_cnt << 32 | cnt2;
                    }
                }
#endif
                DBG_ADD(9, h == ~0u && c == nch - 1);
                DBG_ADD(27, h == ~0u && e2 == ~0u);
                DBG_ADD(7, cnt2);
                if (e2 != ~0u && h != ~0u) {
                    my_cnt = cnt2 + (p0_cnt - h);  // the rest of the path is the pass-0 path
                    my_end = p0_end;
                } else {
                    my_end = e2;
                    my_cnt = cnt2;
                }
            }
            s.end[c] = my_end;
            changed = 1;
        }
        DBG_ADD(8, (tid == 0));
        if (!__syncthreads_or(changed)) break;
    }
    uint32_t v = (c < nch) ? my_cnt : 0;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s.wsum[warp] = incl;
    __syncthreads();
    uint32_t pre = 0, tot = 0;
    for (int w = 0; w < kWarps; w++) { if (w < warp) pre += s.wsum[w]; tot += s.wsum[w]; }
    const bool inv = (c < nch) && (my_end == ~0u);
    const bool bad = __syncthreads_or(inv) || tot != len || s.end[nch - 1] != bits;
    __syncthreads();
    DBG_TADD(19, t_fix);
    if (bad) return false;
    DBG_T0(t_emit);
    if (STAGED && !RUN) {
        const bool has = c < nch && my_cnt;
        emit_lean<3>(s, src.sw, src.sh, has ? my_start : 0u, has ? lim : 0u, dst + (has ? pre + incl - v : 0u));
    } else {
        // Records that are nearly all run symbol (<= 1.125 bits per symbol: the
        // high planes of XOR deltas): the CTA fills the plane with the run
        // symbol (coalesced 16-byte stores) and the emit pass stores only the
        // other symbols, taking up to 32 run symbols per step instead of the 8
        // that fill one store.
        const bool sparse = RUN && bits <= len + (len >> 3);
        if (sparse) {
            const uint32_t rs = s.csym[s.first_idx[1]] * 0x01010101u;
            const uint32_t head = min(len, (uint32_t)((16 - (reinterpret_cast<uint64_t>(dst) & 15)) & 15));
            const uint32_t n16 = (len - head) >> 4;
            if ((uint32_t)tid < head) dst[tid] = (uint8_t)rs;
            uint4* d16 = reinterpret_cast<uint4*>(dst + head);
            for (uint32_t i = tid; i < n16; i += kThreads) d16[i] = make_uint4(rs, rs, rs, rs);
            for (uint32_t i = head + (n16 << 4) + tid; i < len; i += kThreads) dst[i] = (uint8_t)rs;
            __syncthreads();
        }
        if (c < nch && my_cnt) {
            uint32_t cc;
            decode_span<true, STAGED, RUN>(s, src, my_start, lim, 0, 0, cc, dst + (pre + incl - v), nullptr, sparse);
        }
    }
    __syncthreads();
    DBG_TADD(20, t_emit);
    return true;
}

// TMA 1-D bulk copy global -> shared with an mbarrier (SASS UBLKCP).
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_inval(uint64_t* bar) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait0(uint64_t* bar) {
    asm volatile("{\n .reg .pred P;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n @!P bra WAIT_%=;\n}\n"
                 ::"r"(smem_u32(bar)) : "memory");
}

// CTA-wide decode of one Huffman record payload `pl` (codebook | bits u32 |
// bits) into dst[0, len).  Returns false on any corruption the reference
// would report (malformed codebook, zero bit count, invalid prefix, wrong end
// position or symbol count).
__device__ __forceinline__ uint64_t stage_cover(const uint8_t* pl) {   // staged bytes of a Huffman payload
    const uint32_t bits0 = rd32(pl + 128);
    const uint8_t* data0 = pl + kHuffOverhead;
    const uint64_t a16 = reinterpret_cast<uint64_t>(data0) & ~15ull;
    const uint64_t e16 = (reinterpret_cast<uint64_t>(data0) + ((uint64_t)bits0 + 7) / 8 + 15) & ~15ull;
    return e16 - a16;
}

__device__ bool huff_decode(DecSmem& /* the caller's view of dec_smem() */, const uint8_t* pl, uint32_t len, uint8_t* dst,
                            uint32_t stage_cap) {
    DecSmem& s = dec_smem();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    DBG_T0(t_setup);
    // the staging area below is rewritten by the bulk copy (async proxy);
    // every thread's earlier generic writes to this shared memory (byte swaps
    // of the last payload, k_decpair's CRC tables) must be ordered before it:
    // a proxy fence by each writer, then the barrier
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    // stage the payload in shared memory with one TMA bulk copy of its
    // 16-byte aligned cover, issued first so it lands while the tables are built
    const uint32_t bits0 = rd32(pl + 128);
    const uint8_t* data0 = pl + kHuffOverhead;
    const uint64_t a16 = reinterpret_cast<uint64_t>(data0) & ~15ull;
    const uint64_t e16 = (reinterpret_cast<uint64_t>(data0) + ((uint64_t)bits0 + 7) / 8 + 15) & ~15ull;
    const bool staged = bits0 != 0 && e16 - a16 <= (uint64_t)stage_cap;
    if (staged && tid == 0) {
        mbar_init1(tma_bar(stage_cap));
        tma_load_1d(s.bits, reinterpret_cast<const void*>(a16), (uint32_t)(e16 - a16), tma_bar(stage_cap));
    }
    const uint8_t wb = pl[tid >> 1];
    const uint32_t l = (tid & 1) ? (wb >> 4) : (wb & 15);
    s.lens[tid] = (uint8_t)l;
    if (tid < kWarps * 16) (&s.cnt_w[0][0])[tid] = 0;
    if (tid == 0) s.kraft = 0;
    __syncthreads();
    const uint32_t mm = __match_any_sync(0xFFFFFFFFu, l);
    const uint32_t rank_w = __popc(mm & ((1u << lane) - 1));
    if (lane == __ffs(mm) - 1) s.cnt_w[warp][l] = __popc(mm);
    uint32_t ku = l ? (1u << (kMaxLen - l)) : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) ku += __shfl_xor_sync(0xFFFFFFFFu, ku, o);
    if (lane == 0) atomicAdd(&s.kraft, ku);
    __syncthreads();
    if (warp == 0) {
        // lane q = code length q (1..15): its count, then exclusive scans of
        // the Kraft units (first_left) and of the counts (first_idx)
        const bool isq = lane >= 1 && lane <= kMaxLen;
        uint32_t c = 0;
        if (isq)
#pragma unroll
            for (int w = 0; w < kWarps; w++) c += s.cnt_w[w][lane];
        const uint32_t lf = isq ? c << (kMaxLen - lane) : 0u;
        uint32_t il = lf, ii = c;
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
            const uint32_t yl = __shfl_up_sync(0xFFFFFFFFu, il, o), yi = __shfl_up_sync(0xFFFFFFFFu, ii, o);
            if (lane >= o) { il += yl; ii += yi; }
        }
        if (isq) {
            s.bl_count[lane] = c;
            s.first_left[lane] = il - lf;
            s.first_idx[lane] = ii - c;
        }
        const uint32_t used = __ballot_sync(0xFFFFFFFFu, c != 0);   // bit q: length q in use
        if (lane == 0) {
            int gl = 0;   // gcd of the code lengths in use
            for (uint32_t u = used; u; u &= u - 1) {
                int a = gl, b = __ffs(u) - 1;
                while (b) { const int t = a % b; a = b; b = t; }
                gl = a;
            }
            s.minlen = used ? __ffs(used) - 1 : 16;
            s.maxlen = used ? 31 - __clz(used) : 0;
            s.lgcd = gl ? gl : 1;
        }
    }
    __syncthreads();
    const uint32_t bits = rd32(pl + 128);
    // _validate_codebook (huffman.py:191-210) and decode_block's bit-length check (:275)
    if (s.maxlen == 0 || s.kraft > (1u << kMaxLen) || bits == 0) {
        if (staged) {   // no bulk copy left in flight, no live barrier object
            mbar_wait0(tma_bar(stage_cap));
            __syncthreads();
            if (tid == 0) mbar_inval(tma_bar(stage_cap));
        }
        return false;
    }
    if (l) {
        uint32_t rk = rank_w;
        for (int w = 0; w < warp; w++) rk += s.cnt_w[w][l];
        s.csym[s.first_idx[l] + rk] = (uint8_t)tid;
    }
    const uint8_t* data = pl + kHuffOverhead;
    const uint64_t nbytes = ((uint64_t)bits + 7) / 8;
    Src G;
    G.sw = nullptr;
    G.gbase = reinterpret_cast<const uint8_t*>(reinterpret_cast<uint64_t>(data) & ~3ull);
    G.sh = (uint32_t)(reinterpret_cast<uint64_t>(data) & 3) * 8;
    G.glimit = (uint64_t)(data - G.gbase) + nbytes;
    G.nwords_full = G.glimit / 4;
    __syncthreads();
    // single-symbol LUT over kLut-bit prefixes
    // (canonical codes of one length occupy one interval of the code space,
    // the intervals in length order: a thread's increasing entries walk the
    // lengths forward once)
    {
        const int qmax = min(s.maxlen, kLut);
        int q = s.minlen;
        uint32_t fl = 0, endq = 0, base = 0;
        if (q <= qmax) { fl = s.first_left[q]; endq = fl + (s.bl_count[q] << (kMaxLen - q)); base = s.first_idx[q]; }
        for (int e = tid; e < (1 << kLut); e += kThreads) {
            const uint32_t v = (uint32_t)e << (kMaxLen - kLut);
            while (q <= qmax && v >= endq) {
                q++;
                if (q <= qmax) { fl = s.first_left[q]; endq = fl + (s.bl_count[q] << (kMaxLen - q)); base = s.first_idx[q]; }
            }
            s.lut1[lut1_at((uint32_t)e)] = q <= qmax ? (uint16_t)((q << 8) | s.csym[base + ((v - fl) >> (kMaxLen - q))]) : (uint16_t)0;
        }
    }
    __syncthreads();
    // three-symbol LUT: greedy codewords fully inside the kLut-bit prefix
    for (int e = tid; e < (1 << kLut); e += kThreads) {
        uint32_t ent = 0, n = 0, tl = 0, syms = 0;
        uint32_t rest = (uint32_t)e;
        while (n < 3) {
            const uint32_t a = s.lut1[lut1_at(rest & ((1u << kLut) - 1))];
            const uint32_t la = a >> 8;
            if (!a || tl + la > kLut) break;
            syms |= (a & 0xFF) << (8 * n);
            n++;
            tl += la;
            rest = (uint32_t)e << tl;
        }
        if (n) ent = (tl << 28) | (n << 24) | syms;
        s.lut3[e] = ent;
    }
    // count LUT: every whole codeword of a 12-bit window (greedy, continued
    // from the 3-symbol LUT's codewords of its first 11 bits); records with a
    // 1-bit code count with the 3-symbol LUT plus runs instead
    __syncthreads();
    if (!s.bl_count[1])
    for (int e = tid; e < (1 << kCntLut); e += kThreads) {
        const uint32_t e3 = s.lut3[e >> (kCntLut - kLut)];
        uint32_t n = (e3 >> 24) & 3, tl = e3 >> 28;
        for (;;) {
            const uint32_t rest = ((uint32_t)e << tl) & ((1u << kCntLut) - 1);
            const uint32_t a = s.lut1[lut1_at(rest >> (kCntLut - kLut))];
            const uint32_t la = a >> 8;
            if (!a || tl + la > kCntLut) break;
            n++;
            tl += la;
        }
        s.lutc[e] = (uint8_t)((n << 4) | tl);
    }
    __syncthreads();
    DBG_TADD(16, t_setup);
    DBG_ADD(17, staged ? 1 : 0);
    if (staged) {
        // the staged words in memory order -> big-endian words (bit i of the
        // payload is bit 31 - ((i + sh) & 31) of word (i + sh) >> 5)
        mbar_wait0(tma_bar(stage_cap));
        const uint32_t nw = (uint32_t)((e16 - a16) / 4);
        for (uint32_t j = tid; j < nw; j += kThreads) s.bits[j] = bswap32(s.bits[j]);
        __syncthreads();
        if (tid == 0) mbar_inval(tma_bar(stage_cap));   // (every thread is past its wait)
        Src St;
        St.sw = s.bits;
        St.gbase = reinterpret_cast<const uint8_t*>(a16);
        St.sh = (uint32_t)(reinterpret_cast<uint64_t>(data) - a16) * 8;
        St.glimit = (uint64_t)(data - St.gbase) + nbytes;
        St.nwords_full = St.glimit / 4;
        return s.bl_count[1] ? huff_passes<true, true>(s, St, bits, len, dst) : huff_passes<true, false>(s, St, bits, len, dst);
    }
    return s.bl_count[1] ? huff_passes<false, true>(s, G, bits, len, dst) : huff_passes<false, false>(s, G, bits, len, dst);
}

__device__ void copy_bytes(uint8_t* dst, const uint8_t* src, uint32_t n) {
    // dst 16-byte aligned; src arbitrary
    const int tid = threadIdx.x;
    const uint32_t nv = n / 16;
    const uint32_t sh = (uint32_t)(reinterpret_cast<uint64_t>(src) & 3) * 8;
    const uint32_t* w = reinterpret_cast<const uint32_t*>(reinterpret_cast<uint64_t>(src) & ~3ull);
    // four 16-byte pieces per thread in flight (loads first)
    for (uint32_t i0 = tid; i0 < nv; i0 += 4 * kThreads) {
        uint32_t a[4][5];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const uint32_t i = i0 + u * kThreads;
            if (i < nv) {
                const uint32_t* wi = w + 4 * i;
#pragma unroll
                for (int q = 0; q < 4; q++) a[u][q] = __ldg(wi + q);
                a[u][4] = (sh && 16 * i + 20 <= n) ? __ldg(wi + 4) : 0u;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const uint32_t i = i0 + u * kThreads;
            if (i >= nv) break;
            uint4 v;
            if (sh == 0) {
                v = make_uint4(a[u][0], a[u][1], a[u][2], a[u][3]);
            } else {
                uint32_t a4 = a[u][4];
                if (16 * i + 20 > n) {
                    const uint8_t* b4 = reinterpret_cast<const uint8_t*>(w + 4 * i + 4);
                    const int64_t lim = (int64_t)((uint64_t)(src + n) - reinterpret_cast<uint64_t>(b4));
                    for (int q = 0; q < 4 && q < lim; q++) a4 |= (uint32_t)b4[q] << (8 * q);
                }
                v = make_uint4(__funnelshift_r(a[u][0], a[u][1], sh), __funnelshift_r(a[u][1], a[u][2], sh),
                               __funnelshift_r(a[u][2], a[u][3], sh), __funnelshift_r(a[u][3], a4, sh));
            }
            reinterpret_cast<uint4*>(dst)[i] = v;
        }
    }
    for (uint32_t i = nv * 16 + tid; i < n; i += kThreads) dst[i] = src[i];
}

// Decode one record (mode u8 | len u32 | payload) at rec into dst.  The caller
// has validated the header and the payload bounds.  CTA-wide.
__device__ bool decode_record(DecSmem& s, const uint8_t* rec, uint32_t mode, uint32_t len, uint8_t* dst,
                              uint32_t stage_cap) {
    const uint8_t* pl = rec + 5;
    if (mode == MODE_RLE) {
        const uint32_t v = pl[0] * 0x01010101u;
        const uint32_t nv = len / 16;
        for (uint32_t i = threadIdx.x; i < nv; i += kThreads) reinterpret_cast<uint4*>(dst)[i] = make_uint4(v, v, v, v);
        for (uint32_t i = nv * 16 + threadIdx.x; i < len; i += kThreads) dst[i] = (uint8_t)v;
        return true;
    }
    if (mode == MODE_STORED) {
        copy_bytes(dst, pl, len);
        return true;
    }
    return huff_decode(s, pl, len, dst, stage_cap);
}

// payload size of the record at pos (stream.py:258-268); false when the
// header or payload does not fit in the segment.
__device__ __forceinline__ bool rec_size(const uint8_t* seg, uint64_t comp, uint64_t pos, uint32_t& mode, uint32_t& l,
                                         uint64_t& psize) {
    if (pos + 5 > comp) return false;
    mode = seg[pos];
    l = rd32(seg + pos + 1);
    if (mode == MODE_RLE) psize = 1;
    else if (mode == MODE_STORED) psize = l;
    else if (mode == MODE_HUFFMAN) {
        if (pos + 5 + kHuffOverhead > comp) return false;
        psize = kHuffOverhead + ((uint64_t)rd32(seg + pos + 5 + 128) + 7) / 8;
    } else return false;
    return pos + 5 + psize <= comp;
}

// -------------------------------------------------------------- k_scandec
constexpr uint64_t kFlagA = 1ull << 62, kFlagI = 2ull << 62, kMask = (1ull << 62) - 1;
__device__ __forceinline__ uint64_t ld_acq(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(uint64_t* p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ bool rec_size_dev(const uint8_t* seg, uint64_t comp, uint64_t pos, uint32_t& mode,
                                             uint32_t& l, uint64_t& psize) {
    if (pos + 5 > comp) return false;
    mode = seg[pos];
    l = rd32(seg + pos + 1);
    if (mode == MODE_RLE) psize = 1;
    else if (mode == MODE_STORED) psize = l;
    else if (mode == MODE_HUFFMAN) {
        if (pos + 5 + kHuffOverhead > comp) return false;
        psize = kHuffOverhead + ((uint64_t)rd32(seg + pos + 5 + 128) + 7) / 8;
    } else return false;
    return pos + 5 + psize <= comp;
}

// A record header "mode <= 2 | len == B" whose payload fits and whose
// successor is the segment end or another plausible header (len B, or the
// segment's tail length).  False positives inside payload bytes would have to
// pass both tests; any that does is caught by k_verify.
__device__ __forceinline__ bool is_cand(const uint8_t* seg, uint64_t comp, uint64_t pos, uint32_t B, uint32_t Ltail) {
    if (pos + 5 > comp || seg[pos] > 2 || rd32(seg + pos + 1) != B) return false;
    uint32_t mode, l;
    uint64_t ps;
    if (!rec_size_dev(seg, comp, pos, mode, l, ps)) return false;
    // what an encoder writes: a Huffman record has a non-empty bit stream
    // smaller than the stored record (stream.py:173) ...
    if (mode == MODE_HUFFMAN) {
        const uint32_t bits = rd32(seg + pos + 5 + 128);
        if (bits == 0 || kHuffOverhead + ((uint64_t)bits + 7) / 8 > B) return false;
    }
    // ... and is followed by the segment end or another record header (the
    // cheap test that rejects most byte patterns inside payloads) ...
    const uint64_t q = pos + 5 + ps;
    if (q != comp) {
        if (q + 5 > comp || seg[q] > 2) return false;
        const uint32_t l2 = rd32(seg + q + 1);
        if (l2 != B && l2 != Ltail) return false;
    }
    // ... and a codebook within the Kraft bound (huffman.py:191-210)
    if (mode == MODE_HUFFMAN) {
        uint32_t kraft = 0;
        const uint8_t* cb = seg + pos + 5;
        for (int i = 0; i < 128; i++) {
            const uint32_t v = cb[i], a = v & 15, b2 = v >> 4;
            kraft += (a ? 1u << (kMaxLen - a) : 0u) + (b2 ? 1u << (kMaxLen - b2) : 0u);
        }
        if (kraft == 0 || kraft > (1u << kMaxLen)) return false;
    }
    return true;
}

// Candidates of positions [pa, pe) of a segment, found by one warp with
// coalesced 16-byte loads: the little-endian block size has exactly one
// non-zero byte (at offset 1 + kb of a record header), so anchors are the
// bytes equal to it, compared 4 at a time with __vcmpeq4.  Appends the
// candidates in increasing order: emit(position, rank) with ranks counted
// from cnt (warp-uniform, updated); false if a lane overflowed its buffer.
constexpr int kLaneCand = 8;   // candidates per lane per 16 bytes (6-byte RLE records: true + offset-3 echoes)

template <class Emit>
__device__ bool warp_scan(const DecSeg& sg, uint64_t pa, uint64_t pe, uint32_t& cnt, int lane, Emit emit) {
    const uint32_t B = sg.block;
    const uint32_t Ltail = (uint32_t)(sg.orig - (uint64_t)(sg.nrec - 1) * B);
    const int kb = (__ffs(B) - 1) >> 3;
    const uint8_t* b = sg.base;
    const uint64_t qa = max(pa, (uint64_t)1) + 1 + kb;
    const uint64_t qe = min(pe + 1 + kb, sg.comp);
    if (qa >= qe) return true;
    const uint64_t A = (reinterpret_cast<uint64_t>(b) + qa - 1 - kb) & ~15ull;   // aligned row start (mode bytes)
    const uint64_t Aend = reinterpret_cast<uint64_t>(b) + qe;
    const uint64_t segend = reinterpret_cast<uint64_t>(b) + sg.comp;
    bool ok = true;
    constexpr int kRows = 4;  // 512-byte rows in flight per warp
    for (uint64_t gb = A; gb < Aend; gb += 512 * kRows) {
      uint4 rows[kRows];
#pragma unroll
      for (int rr = 0; rr < kRows; rr++) {
        const uint64_t g = gb + 512ull * rr + 16ull * lane;
        rows[rr] = make_uint4(0, 0, 0, 0);
        if (g < Aend && g + 16 <= segend) rows[rr] = __ldg(reinterpret_cast<const uint4*>(g));
      }
#pragma unroll 1
      for (int rr = 0; rr < kRows; rr++) {
        const uint64_t g0 = gb + 512ull * rr;
        if (g0 >= Aend) break;
        const uint64_t g = g0 + 16ull * lane;
        uint32_t w4[4] = {rows[rr].x, rows[rr].y, rows[rr].z, rows[rr].w};
        if (g < Aend && g + 16 > segend) {
            w4[0] = w4[1] = w4[2] = w4[3] = 0;
            for (int q = 0; q < 16; q++)
                if (g + q < segend) w4[q >> 2] |= (uint32_t)(*reinterpret_cast<const uint8_t*>(g + q)) << (8 * (q & 3));
        }
        // branch-free header test at all 16 byte positions of the lane:
        // mode byte <= 2 followed by the 4 little-endian bytes of B
        uint32_t w5 = __shfl_down_sync(0xFFFFFFFFu, w4[0], 1);
        if (lane == 31) {
            w5 = 0;
            const uint64_t gn = g + 16;
            if (gn + 4 <= segend) w5 = __ldg(reinterpret_cast<const uint32_t*>(gn));
            else for (int q = 0; q < 4; q++) if (gn + q < segend) w5 |= (uint32_t)(*reinterpret_cast<const uint8_t*>(gn + q)) << (8 * q);
        }
        // the u32 at byte p + 1 for p = 4i + j: funnel shifts of word pairs
        const uint32_t wv[5] = {w4[0], w4[1], w4[2], w4[3], w5};
        bool any = false;
#pragma unroll
        for (int i = 0; i < 4; i++) {
            any |= __funnelshift_r(wv[i], wv[i + 1], 8) == B;
            any |= __funnelshift_r(wv[i], wv[i + 1], 16) == B;
            any |= __funnelshift_r(wv[i], wv[i + 1], 24) == B;
            any |= wv[i + 1] == B;
        }
        uint32_t cm = 0;
        if (any) {
#pragma unroll
            for (int i = 0; i < 4; i++) {
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const uint32_t x = j == 3 ? wv[i + 1] : __funnelshift_r(wv[i], wv[i + 1], 8 * (j + 1));
                    const uint32_t mode = (wv[i] >> (8 * j)) & 0xFF;
                    if (x == B && mode <= 2) cm |= 1u << (4 * i + j);
                }
            }
        }
        uint32_t found[kLaneCand];
        uint32_t k = 0;
        while (cm) {
            const int j = __ffs(cm) - 1;
            cm &= cm - 1;
            const uint64_t p = g + j - reinterpret_cast<uint64_t>(b);
            if (p + 1 + kb >= qa && p + 1 + kb < qe && is_cand(b, sg.comp, p, B, Ltail)) {
                if (k < kLaneCand) found[k] = (uint32_t)p;
                k++;
            }
        }
        if (!__any_sync(0xFFFFFFFFu, k != 0)) continue;
        if (k > kLaneCand) ok = false;
        const uint32_t kk = min(k, (uint32_t)kLaneCand);
        uint32_t incl = kk;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t base = cnt + incl - kk;
        for (uint32_t i = 0; i < kk; i++) emit(found[i], base + i);
        cnt += __shfl_sync(0xFFFFFFFFu, incl, 31);
      }
    }
    return __all_sync(0xFFFFFFFFu, ok);
}

// Stored-grid shortcut for a span [pa, pe): a plane that does not compress
// (the low byte plane of bf16 weights) is a run of full stored records, each
// 5 + B bytes, so its records sit on the (B + 5)-byte grid from the segment
// start.  If every grid position whose record would cover a byte of the span
// holds a full stored header (mode 0, len B, payload inside the segment),
// the span's candidates are the grid positions inside it and its payload
// bytes are not read.  If those headers are not the segment's real records
// (payload bytes that look like them), record starts inside the span are
// missed, the chain does not verify (k_verify / k_resolve) and k_fallback
// walks the segment: the result is the same, only slower.  Returns false
// when the span is not of this shape (the caller scans it).
template <class Emit>
__device__ __forceinline__ bool stored_grid_span(const DecSeg& sg, uint64_t pa, uint64_t pe, uint32_t& cnt, int lane,
                                                 Emit emit) {
    const uint32_t B = sg.block;
    const uint64_t G = (uint64_t)B + 5;
    const uint64_t k_lo = pa / G, k_hi = (pe - 1) / G;
    if (k_hi - k_lo >= 32) return false;
    const uint64_t p = (k_lo + lane) * G;
    const bool mine = k_lo + lane <= k_hi;
    const uint32_t Ltail = (uint32_t)(sg.orig - (uint64_t)(sg.nrec - 1) * B);
    // each of them a full candidate (is_cand: the successor header too), so
    // that bit streams of delta payloads -- long zero runs with a stray 02 and
    // 01 byte look like "stored | B" about once in 1e5 positions -- do not
    // send segments to the serial walk
    bool good = true;
    if (mine) good = p + G <= sg.comp && sg.base[p] == MODE_STORED && is_cand(sg.base, sg.comp, p, B, Ltail);
    if (!__all_sync(0xFFFFFFFFu, good)) return false;
    // (position 0 is listed by the caller, as in warp_scan)
    const bool in = mine && p >= max(pa, (uint64_t)1) && p < pe;
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, in);
    if (in) emit(p, cnt + __popc(m & ((1u << lane) - 1)));
    cnt += __popc(m);
    return true;
}

// Owner maps (chunk -> segment, record slot -> segment, output tile ->
// window): one load per CTA in the kernels below instead of a binary search
// of dependent loads.  Unowned capacity slots keep the ~0u of the memset.
__global__ void k_maps(const DecSeg* __restrict__ segs, uint64_t nseg_total, const DecWin* __restrict__ wins,
                       uint64_t nwin_total, uint32_t* __restrict__ chunk2seg, uint32_t* __restrict__ rec2seg,
                       uint32_t* __restrict__ tile2win) {
    const uint64_t b = blockIdx.x;
    if (b < nseg_total) {
        const DecSeg sg = segs[b];
        for (uint32_t i = threadIdx.x; i < sg.nchunk; i += blockDim.x) chunk2seg[sg.chunk0 + i] = (uint32_t)b;
        for (uint32_t i = threadIdx.x; i < sg.nrec; i += blockDim.x) rec2seg[sg.rec0 + i] = (uint32_t)b;
    } else if (b - nseg_total < nwin_total) {
        const uint64_t w = b - nseg_total;
        const DecWin wd = wins[w];
        for (uint32_t i = threadIdx.x; i < wd.ntile; i += blockDim.x) tile2win[wd.tile0 + i] = (uint32_t)w;
    }
}

constexpr uint32_t kSpanCap = 64;                  // candidates listed per 8 KiB span (more: k_assign rescans)
constexpr uint32_t kDense = 0xFFFFFFFFu;            // a lane overflowed: the serial path takes the segment

// CTA per 64 KiB chunk slot of segment payload, warp per 8 KiB span: the
// candidate record headers of the span, in increasing order, into
// cand[span][0..kSpanCap) and their count (kDense on overflow) into ccnt.
__global__ void __launch_bounds__(kThreads) k_cand(const DecSeg* __restrict__ segs, const uint32_t* __restrict__ chunk2seg,
                                                 uint64_t nchunk_total, uint32_t* __restrict__ cand,
                                                 uint32_t* __restrict__ ccnt, uint32_t* __restrict__ ctot) {
    __shared__ uint32_t wcnt[kWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t t = blockIdx.x;
    if (t >= nchunk_total) return;
    const uint64_t span = t * kWarps + warp;
    const uint32_t owner = chunk2seg[t];
    if (owner == ~0u) {  // unused capacity slot
        if (lane == 0) ccnt[span] = 0;
        if (tid == 0) ctot[t] = 0;
        return;
    }
    const DecSeg sg = segs[owner];
    constexpr uint64_t kWarpSpan = kChunk / kWarps;
    const uint64_t c0 = (t - sg.chunk0) * kChunk, c1 = min(c0 + kChunk, sg.comp);
    const uint64_t pa = c0 + warp * kWarpSpan, pe = min(pa + kWarpSpan, c1);
    uint32_t* list = cand + span * kSpanCap;
    uint32_t n = 0;
    if (pa == 0 && pa < pe) {  // the segment start is always a record start
        if (lane == 0) list[0] = 0;
        n = 1;
    }
    bool ok = true;
    if (pa < pe) {
        auto put = [&](uint64_t p, uint32_t r) { if (r < kSpanCap) list[r] = (uint32_t)p; };
        if (!stored_grid_span(sg, pa, pe, n, lane, put)) ok = warp_scan(sg, pa, pe, n, lane, put);
    }
    if (lane == 0) {
        ccnt[span] = ok ? n : kDense;
        wcnt[warp] = ok ? n : kDense;
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t tot = 0;
        for (int w = 0; w < kWarps; w++) tot = (tot == kDense || wcnt[w] == kDense) ? kDense : tot + wcnt[w];
        ctot[t] = tot;
    }
}

// CTA per segment: exclusive scan of the chunk candidate totals (record
// number of each chunk's first candidate), the segment's candidate count,
// and failure for a segment with an overflowing span.
__global__ void __launch_bounds__(kThreads) k_number(const DecSeg* __restrict__ segs, uint64_t nseg_total,
                                                   const uint32_t* __restrict__ ctot, uint32_t* __restrict__ cpre,
                                                   uint32_t* __restrict__ seg_cnt, uint32_t* __restrict__ seg_fail) {
    __shared__ uint32_t wsum[kWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (uint64_t si = blockIdx.x; si < nseg_total; si += gridDim.x) {
        const DecSeg sg = segs[si];
        uint32_t carry = 0;
        bool bad = false;
        for (uint64_t c0 = 0; c0 < sg.nchunk; c0 += kThreads) {
            const uint64_t i = c0 + tid;
            uint32_t c = i < sg.nchunk ? ctot[sg.chunk0 + i] : 0u;
            if (c == kDense) { bad = true; c = 0; }
            uint32_t incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) wsum[warp] = incl;
            __syncthreads();
            uint32_t pre = carry, tot = 0;
#pragma unroll
            for (int w = 0; w < kWarps; w++) { if (w < warp) pre += wsum[w]; tot += wsum[w]; }
            if (i < sg.nchunk) cpre[sg.chunk0 + i] = pre + incl - c;
            carry += tot;
            __syncthreads();
        }
        bad = __syncthreads_or(bad);
        if (tid == 0) {
            seg_cnt[si] = carry;
            if (bad) { seg_fail[si] = 1; DBG_ADD(12, 1); }
        }
    }
}

// CTA per chunk slot: record slot r = (chunk prefix + span prefix + i) gets
// candidate i's position and the position its header says the next record
// starts at; after record R-2 the tail record (not a candidate when its
// length differs from the block size) follows.
__global__ void __launch_bounds__(kThreads) k_assign(const DecSeg* __restrict__ segs, const uint32_t* __restrict__ chunk2seg,
                                                   uint64_t nchunk_total, const uint32_t* __restrict__ cand,
                                                   const uint32_t* __restrict__ ccnt, const uint32_t* __restrict__ cpre,
                                                   uint32_t* __restrict__ seg_fail, uint64_t* __restrict__ rec_pos,
                                                   uint64_t* __restrict__ rec_next) {
    // one warp per chunk (a CTA per chunk spent its time being launched: a
    // chunk holds one to three records): lane w < kWarps holds span w's count
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t t = (uint64_t)blockIdx.x * kWarps + warp;
    if (t >= nchunk_total) return;
    const uint32_t lo = chunk2seg[t];
    if (lo == ~0u) return;
    const DecSeg sg = segs[lo];
    const uint32_t cw = lane < kWarps ? ccnt[t * kWarps + lane] : 0u;
    if (__any_sync(0xFFFFFFFFu, cw == kDense)) return;  // k_number failed the segment
    uint32_t incl = cw;
#pragma unroll
    for (int o = 1; o < kWarps; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    const uint32_t base = cpre[t];
    const uint32_t R = sg.nrec, B = sg.block;
    const uint32_t Ltail = R ? (uint32_t)(sg.orig - (uint64_t)(R - 1) * B) : 0;
    uint32_t pre = 0;   // record index of the current span's first candidate
    auto assign = [&](uint64_t pos, uint32_t k) {
        uint32_t r = pre + k;
        if (r >= R) { atomicOr(&seg_fail[lo], 1u); DBG_ADD(13, 1); return; }
        for (int part = 0; part < 2; part++) {
            uint32_t mode = 0, l = 0;
            uint64_t ps = 0;
            const bool rok = rec_size(sg.base, sg.comp, pos, mode, l, ps) && l == ((r + 1 == R) ? Ltail : B);
            rec_pos[sg.rec0 + r] = pos;
            rec_next[sg.rec0 + r] = rok ? pos + 5 + ps : ~0ull;
            if (!rok) { atomicOr(&seg_fail[lo], 1u); DBG_ADD(14, 1); }
            if (!(rok && part == 0 && r + 2 == R && Ltail != B)) break;
            pos += 5 + ps;
            r = R - 1;
        }
    };
    for (int sp = 0; sp < kWarps; sp++) {
        const uint32_t c = __shfl_sync(0xFFFFFFFFu, cw, sp);
        pre = base + __shfl_sync(0xFFFFFFFFu, incl - cw, sp);
        const uint64_t span = t * kWarps + sp;
        if (c <= kSpanCap) {
            for (uint32_t k = lane; k < c; k += 32) assign(cand[span * kSpanCap + k], k);
        } else {
            // dense span (e.g. runs of 6-byte RLE records): enumerate it again
            constexpr uint64_t kWarpSpan = kChunk / kWarps;
            const uint64_t c0 = (t - sg.chunk0) * kChunk, c1 = min(c0 + kChunk, sg.comp);
            const uint64_t pa = c0 + sp * kWarpSpan, pe = min(pa + kWarpSpan, c1);
            uint32_t n = 0;
            if (pa == 0 && pa < pe) {
                if (lane == 0) assign(0, 0);
                n = 1;
            }
            if (pa < pe) warp_scan(sg, pa, pe, n, lane, assign);
        }
    }
}

// CTA per record slot of the segments k_verify accepted: RLE fill, stored
// copy or CTA-wide Huffman decode into the grouped scratch.  A failure marks
// the segment for k_fallback, which re-walks it serially and reports the
// reference's error.
__device__ __forceinline__ bool is_large(const uint8_t* rec) {
    return rec[0] == MODE_HUFFMAN && stage_cover(rec + 5) > (uint64_t)kStageSmall;
}

// Decode record slot g into grouped scratch (CTA-wide).
__device__ __forceinline__ void decrec_one(DecSmem& s, const DecSeg* __restrict__ segs, const uint32_t* __restrict__ rec2seg,
                                           const DecWin* __restrict__ wins, uint64_t g, uint32_t* __restrict__ seg_fail,
                                           const uint64_t* __restrict__ rec_pos, uint8_t* __restrict__ scratch,
                                           bool skip_large, uint32_t stage_cap) {
    const uint32_t lo = rec2seg[g];
    if (lo == ~0u) return;
    if (__syncthreads_or(threadIdx.x == 0 && seg_fail[lo])) return;   // (one read: another CTA may be setting it)
    const DecSeg sg = segs[lo];
    if (wins[sg.win].fuse) return;   // (k_decpair has it)
    const uint32_t r = (uint32_t)(g - sg.rec0);
    const uint8_t* rec = sg.base + rec_pos[g];
    if (skip_large && is_large(rec)) return;   // (k_decrec_large has it)
    const uint32_t mode = rec[0], len = rd32(rec + 1);
    const bool ok = decode_record(s, rec, mode, len, scratch + sg.goff + (uint64_t)r * sg.block, stage_cap);
    if (!ok && threadIdx.x == 0) { atomicOr(&seg_fail[lo], 1u); DBG_ADD(16, 1); }
}

// CTA per record slot.  split: records listed by k_classify (Huffman payloads
// that do not stage in kStageSmall) are left to k_decrec_large, and this
// launch runs at 4 CTAs per SM with kStageSmall; otherwise (few records) it
// decodes everything with kStageLarge.
__global__ void __launch_bounds__(kThreads, 4) k_decrec(const DecSeg* __restrict__ segs, const uint32_t* __restrict__ rec2seg,
                                                   const DecWin* __restrict__ wins, uint64_t nrec_total, uint32_t* __restrict__ seg_fail,
                                                   const uint64_t* __restrict__ rec_pos, uint8_t* __restrict__ scratch,
                                                   int split) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    DecSmem& s = *reinterpret_cast<DecSmem*>(smem_raw);
    const uint64_t g = blockIdx.x;
    if (g >= nrec_total) return;
    decrec_one(s, segs, rec2seg, wins, g, seg_fail, rec_pos, scratch, split != 0, split ? kStageSmall : kStageLarge);
}

// The large records (k_classify's list), persistent CTAs with kStageLarge;
// runs on the side stream next to k_decrec.
__global__ void __launch_bounds__(kThreads, 3) k_decrec_large(const DecSeg* __restrict__ segs, const uint32_t* __restrict__ rec2seg,
                                                         const DecWin* __restrict__ wins, const uint32_t* __restrict__ list, const uint32_t* __restrict__ count,
                                                         uint32_t* __restrict__ seg_fail, const uint64_t* __restrict__ rec_pos,
                                                         uint8_t* __restrict__ scratch) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    DecSmem& s = *reinterpret_cast<DecSmem*>(smem_raw);
    const uint32_t n = *count;
    for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
        decrec_one(s, segs, rec2seg, wins, list[i], seg_fail, rec_pos, scratch, false, kStageLarge);
        __syncthreads();
    }
}

// Thread per record slot (after discovery): list the records for
// k_decrec_large.
__global__ void k_classify(const DecSeg* __restrict__ segs, const uint32_t* __restrict__ rec2seg, const DecWin* __restrict__ wins,
                           uint64_t nrec_total, const uint32_t* __restrict__ seg_fail, const uint64_t* __restrict__ rec_pos,
                           uint32_t* __restrict__ list, uint32_t* __restrict__ count) {
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (g >= nrec_total) return;
    const uint32_t lo = rec2seg[g];
    if (lo == ~0u || seg_fail[lo]) return;
    const DecSeg sg = segs[lo];
    if (wins[sg.win].fuse) return;
    const uint64_t pos = rec_pos[g];
    if (pos + 5 + kHuffOverhead > sg.comp) return;
    if (is_large(sg.base + pos)) list[atomicAdd(count, 1u)] = (uint32_t)g;
}

// ------------------------------------------------------------- k_decpair
// Fused decode + inverse byte-grouping + CRC for the fused windows (k_parse):
// the element range [kB, (k+1)B) of a two-plane window is low-plane record
// k and high-plane record n/B + k, and its 2B output bytes are
// out[2e] = low[e], out[2e+1] = high[e] (bytegroup.py:53-62,
// stream.py:392-403).  One persistent CTA per pair at a time (ticket order):
// Huffman planes are decoded (huff_decode, as k_decrec) into the CTA's 128 KiB
// ring slot in global memory -- written and read back by the same CTA within
// one pair, so the slot stays in L2 -- stored planes are read in place from
// the record, RLE planes are one byte; then the CTA writes the interleaved
// output with 16-byte streaming stores (XOR of the previous step for
// lmcg_decompress_apply) and folds the raw CRC-32 of each 32 KiB tile from the
// registers (slice-by-4 in the conflict-free 32 KiB layout rep4x8, laid over
// the decoder's shared memory).  No grouped scratch, no k_ungroup pass:
// decompress moves the stream once and the output once.  Any failure (a
// segment of the window that failed discovery, or a record that does not
// decode) marks every segment of the window failed, so k_fallback re-walks it
// into scratch and k_ungroup assembles it: the authoritative path decides.
constexpr uint32_t kPairRing = 2 * 65536;   // ring bytes per k_decpair CTA: low | high plane
constexpr int kCrcRepWords = 256 * 32;      // CrcTables::rep4x8 in shared memory

// k_decpair's work lists: the low-plane record slots of fused windows
// (pairs) and the records of the other windows (singles, decoded into the
// grouped scratch for k_ungroup).  ctl[0] = pairs, ctl[1] = k_decpair's
// ticket, ctl[2] = singles.
__device__ __forceinline__ void warp_append(bool is, uint32_t v, uint32_t* list, uint32_t* counter) {
    const unsigned m = __ballot_sync(0xFFFFFFFFu, is);
    if (!m) return;
    const int lane = threadIdx.x & 31, lead = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == lead) base = atomicAdd(counter, (uint32_t)__popc(m));
    base = __shfl_sync(0xFFFFFFFFu, base, lead);
    if (is) list[base + __popc(m & ((1u << lane) - 1))] = v;
}
__global__ void k_pairs(const DecSeg* __restrict__ segs, const uint32_t* __restrict__ rec2seg, uint64_t nrec_total,
                        const DecWin* __restrict__ wins, const uint32_t* __restrict__ seg_fail,
                        uint32_t* __restrict__ pairs, uint32_t* __restrict__ singles, uint32_t* __restrict__ ctl) {
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    bool is_pair = false, is_single = false;
    if (g < nrec_total) {
        const uint32_t lo = rec2seg[g];
        if (lo != ~0u) {
            const uint32_t wi = segs[lo].win;
            const uint32_t B = segs[lo].block;
            if (wins[wi].fuse) is_pair = (g - wins[wi].rec0) < wins[wi].n / B;
            else is_single = !seg_fail[lo];
        }
    }
    warp_append(is_pair, (uint32_t)g, pairs, &ctl[0]);
    warp_append(is_single, (uint32_t)g, singles, &ctl[2]);
}



// 16 plane bytes at element offset e (a multiple of 16) of a pair's plane
__device__ __forceinline__ uint4 plane16(const uint8_t* p, uint32_t mode, uint32_t rle, uint32_t e, uint32_t B) {
    if (mode == MODE_RLE) return make_uint4(rle, rle, rle, rle);
    if (mode == MODE_HUFFMAN) return __ldcg(reinterpret_cast<const uint4*>(p + e));   // ring slot (L2; never through L1)
    // stored payload, any alignment: the two aligned 16-byte chunks the piece
    // spans (two requests of 32 sectors; five 4-byte loads took five requests
    // of 16 sectors each).  The last piece's second chunk may reach up to 15
    // bytes past the payload, inside the same aligned 16 bytes as payload
    // bytes (as the bulk copy's aligned cover does).
    const uint64_t a = reinterpret_cast<uint64_t>(p) + e;
    const uint32_t lb = (uint32_t)(a & 15);   // (the same for every piece of a pair)
    const uint4* A = reinterpret_cast<const uint4*>(a & ~15ull);
    const uint4 P = __ldcs(A);
    if (lb == 0) return P;
    const uint4 N = __ldcs(A + 1);
    const uint32_t r = 8 * (lb & 3);
    switch (lb >> 2) {
    case 0: return make_uint4(__funnelshift_r(P.x, P.y, r), __funnelshift_r(P.y, P.z, r), __funnelshift_r(P.z, P.w, r), __funnelshift_r(P.w, N.x, r));
    case 1: return make_uint4(__funnelshift_r(P.y, P.z, r), __funnelshift_r(P.z, P.w, r), __funnelshift_r(P.w, N.x, r), __funnelshift_r(N.x, N.y, r));
    case 2: return make_uint4(__funnelshift_r(P.z, P.w, r), __funnelshift_r(P.w, N.x, r), __funnelshift_r(N.x, N.y, r), __funnelshift_r(N.y, N.z, r));
    default: return make_uint4(__funnelshift_r(P.w, N.x, r), __funnelshift_r(N.x, N.y, r), __funnelshift_r(N.y, N.z, r), __funnelshift_r(N.z, N.w, r));
    }
}


__global__ void __launch_bounds__(kThreads, 4) k_decpair(const DecSeg* __restrict__ segs, const uint32_t* __restrict__ rec2seg,
                                                    const DecWin* __restrict__ wins, const uint32_t* __restrict__ list,
                                                    const uint32_t* __restrict__ singles, uint32_t* __restrict__ ctl,
                                                    uint32_t* __restrict__ seg_fail,
                                                    const uint64_t* __restrict__ rec_pos, uint8_t* __restrict__ ring,
                                                    uint8_t* out /* may alias a window's prev */,
                                                    const CrcTables* __restrict__ ct, const uint32_t* __restrict__ sh992,
                                                    uint32_t* __restrict__ tile_crc, uint8_t* __restrict__ scratch) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    DecSmem& s = *reinterpret_cast<DecSmem*>(smem_raw);
    uint32_t* crctab = reinterpret_cast<uint32_t*>(smem_raw);   // after the decode: rep4x8 | 992-byte shift
    uint32_t* st992 = crctab + kCrcRepWords;
    __shared__ uint32_t sh_p;
    __shared__ uint32_t wcrc[kWarps];
    // the pair's descriptor, set up by thread 0 (nothing of it stays in
    // registers across the decoder calls)
    struct PairInfo {
        const uint8_t* rec[2];   // low, high record
        const uint8_t* prev;
        uint64_t ooff, tile0, k, seg0;
        uint32_t mode[2], B, nseg, ok;
    };
    __shared__ PairInfo pi;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (;;) {
        __syncthreads();   // the previous pair is done with sh_p and the shared memory
        if (tid == 0) sh_p = atomicAdd(&ctl[1], 1u);
        __syncthreads();
        const uint32_t p = sh_p;
        const uint32_t npairs = ctl[0];
        if (p >= npairs + ctl[2]) break;
        if (p >= npairs) {   // a record of a window that is not fused: into the grouped scratch (as k_decrec)
            const uint64_t g = singles[p - npairs];
            const uint32_t lo = rec2seg[g];
            if (__syncthreads_or(tid == 0 && seg_fail[lo])) continue;   // (one read: another CTA may be setting it)
            const DecSeg& sg = segs[lo];
            const uint8_t* rec = sg.base + rec_pos[g];
            const bool ok = decode_record(s, rec, rec[0], rd32(rec + 1), scratch + sg.goff + (g - sg.rec0) * sg.block,
                                          kStageSmall);
            if (!ok && tid == 0) atomicOr(&seg_fail[lo], 1u);
            continue;
        }
        if (tid == 0) {
            const uint64_t gL = list[p];
            const DecSeg& sgL = segs[rec2seg[gL]];
            const DecWin& wd = wins[sgL.win];
            const uint32_t B = sgL.block;
            const uint64_t gH = gL + wd.n / B;
            const DecSeg& sgH = segs[rec2seg[gH]];
            pi.rec[0] = sgL.base + rec_pos[gL];
            pi.rec[1] = sgH.base + rec_pos[gH];
            pi.prev = wd.prev;
            pi.ooff = wd.ooff;
            pi.tile0 = wd.tile0;
            pi.k = gL - wd.rec0;
            pi.seg0 = wd.seg0;
            pi.nseg = wd.nseg;
            pi.B = B;
        }
        __syncthreads();
        bool f = false;
        for (uint32_t i = tid; i < pi.nseg; i += kThreads) f |= seg_fail[pi.seg0 + i] != 0;
        bool ok = !__syncthreads_or(f);
        if (ok && tid == 0) {   // (record positions are valid once discovery passed)
            const uint32_t B = pi.B;
            pi.mode[0] = pi.rec[0][0];
            pi.mode[1] = pi.rec[1][0];
            // stored planes are read at the end of the pair: have them in L2 by then
            if (pi.mode[0] == MODE_STORED) prefetch_l2(pi.rec[0] + 5, B);
            if (pi.mode[1] == MODE_STORED) prefetch_l2(pi.rec[1] + 5, B);
        }
        __syncthreads();
        uint8_t* slot = ring + (uint64_t)blockIdx.x * kPairRing;   // low plane | high plane
        if (ok && pi.mode[1] == MODE_HUFFMAN) ok = huff_decode(s, pi.rec[1] + 5, pi.B, slot + 65536, kStageSmall);
        if (ok && pi.mode[0] == MODE_HUFFMAN) ok = huff_decode(s, pi.rec[0] + 5, pi.B, slot, kStageSmall);
        if (!ok) {
            for (uint32_t i = tid; i < pi.nseg; i += kThreads) seg_fail[pi.seg0 + i] = 1u;
            DBG_ADD(21, tid == 0);
            continue;
        }
        __syncthreads();   // decoded planes visible to the CTA; the decoder's shared memory is free
        DBG_T0(t_tab);
        for (int i = tid; i < kCrcRepWords / 4; i += kThreads)
            reinterpret_cast<uint4*>(crctab)[i] = __ldg(reinterpret_cast<const uint4*>(ct->rep4x8) + i);
        for (int i = tid; i < 1024; i += kThreads) st992[i] = __ldg(sh992 + i);
        __syncthreads();
        DBG_TADD(23, t_tab);
        DBG_T0(t_il);
        Crc4x8Lane cl;
        cl.init(crctab, lane);
        const uint32_t B = pi.B, mL = pi.mode[0], mH = pi.mode[1];
        const uint8_t* recL = pi.rec[0];
        const uint8_t* recH = pi.rec[1];
        const uint64_t k = pi.k;
        const uint8_t* dL = slot;
        const uint8_t* dH = slot + 65536;
        const uint8_t* pL = mL == MODE_HUFFMAN ? dL : recL + 5;
        const uint8_t* pH = mH == MODE_HUFFMAN ? dH : recH + 5;
        const uint32_t rL = recL[5] * 0x01010101u, rH = recH[5] * 0x01010101u;
        const uint64_t e0 = k * B;
        uint8_t* o = out + pi.ooff + 2 * e0;
        const uint8_t* pv = pi.prev ? pi.prev + 2 * e0 : nullptr;
        // warp w writes output rows [w R, (w + 1) R) of 1 KiB (lane l: bytes
        // 32 l .. 32 l + 31 of each row) as four chains of R / 4 rows
        const uint32_t R = B >> 12, Rc = R >> 2;
        uint32_t ch[4] = {0u, 0u, 0u, 0u};
        for (uint32_t r = 0; r < Rc; r++) {
            uint4 lo[4], hi[4];
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const uint32_t e = (warp * R + c * Rc + r) * 512u + 16u * lane;
                lo[c] = plane16(pL, mL, rL, e, B);
                hi[c] = plane16(pH, mH, rH, e, B);
            }
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const uint32_t e = (warp * R + c * Rc + r) * 512u + 16u * lane;
                const uint32_t l4[4] = {lo[c].x, lo[c].y, lo[c].z, lo[c].w}, h4[4] = {hi[c].x, hi[c].y, hi[c].z, hi[c].w};
                uint32_t v[8];
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    v[2 * q] = __byte_perm(l4[q], h4[q], 0x5140);
                    v[2 * q + 1] = __byte_perm(l4[q], h4[q], 0x7362);
                }
                uint4 s0 = make_uint4(v[0], v[1], v[2], v[3]), s1 = make_uint4(v[4], v[5], v[6], v[7]);
                if (pv) {
                    const uint4 a0 = __ldcs(reinterpret_cast<const uint4*>(pv + 2 * e));
                    const uint4 a1 = __ldcs(reinterpret_cast<const uint4*>(pv + 2 * e + 16));
                    s0.x ^= a0.x; s0.y ^= a0.y; s0.z ^= a0.z; s0.w ^= a0.w;
                    s1.x ^= a1.x; s1.y ^= a1.y; s1.z ^= a1.z; s1.w ^= a1.w;
                }
                __stcs(reinterpret_cast<uint4*>(o + 2 * e), s0);
                __stcs(reinterpret_cast<uint4*>(o + 2 * e + 16), s1);
                uint32_t x = ch[c];
                if (r) x = st992[x & 0xFF] ^ st992[256 + ((x >> 8) & 0xFF)] ^ st992[512 + ((x >> 16) & 0xFF)] ^ st992[768 + (x >> 24)];
#pragma unroll
                for (int q = 0; q < 8; q++) x = cl.word(x, v[q]);
                ch[c] = x;
            }
        }
        // chain c's last piece ends (3 - c) Rc KiB + 32 (31 - lane) bytes before the warp's rows end
        const int lc = 31 - __clz(Rc * 1024u);
        const uint32_t* tc = &ct->pow2[lc][0][0];
        uint32_t x = ch[0];
        x = crc_shift_tab(tc, x) ^ ch[1];
        x = crc_shift_tab(tc, x) ^ ch[2];
        x = crc_shift_tab(tc, x) ^ ch[3];
        x = crc_shift_bytes(ct, x, 32u * (31 - lane));
#pragma unroll
        for (int q = 16; q; q >>= 1) x ^= __shfl_xor_sync(0xFFFFFFFFu, x, q);
        if (lane == 0) wcrc[warp] = x;
        __syncthreads();
        // tiles of 32 KiB: 32 / R warps each
        const uint32_t T = (2 * B) / kOutTile, wpt = kWarps / T;
        if ((uint32_t)tid < T) {
            const uint32_t* tw = &ct->pow2[31 - __clz(R * 1024u)][0][0];
            uint32_t acc = 0;
            for (uint32_t j = 0; j < wpt; j++) acc = crc_shift_tab(tw, acc) ^ wcrc[tid * wpt + j];
            tile_crc[pi.tile0 + k * T + tid] = acc;
        }
        DBG_TADD(22, t_il);
#ifdef LMCG_CHECK_TABLES
        {   // experiment: are the CRC tables in shared memory still intact after the interleave?
            uint32_t badw = 0, first = ~0u, got = 0, want = 0;
            for (int i = tid; i < kCrcRepWords + 1024; i += kThreads) {
                const uint32_t wv = i < kCrcRepWords ? __ldg(ct->rep4x8 + i) : __ldg(sh992 + (i - kCrcRepWords));
                if (crctab[i] != wv) {
                    if (!badw) { first = i; got = crctab[i]; want = wv; }
                    badw++;
                }
            }
            if (badw) {
                atomicAdd(&lmcg_fallback_segs, (unsigned long long)badw);
#ifdef LMCG_DEBUG
                const unsigned long long kq = atomicAdd(&lmcg_dbg[31], 1ull);
                if (kq < 512) {
                    unsigned long long* e = lmcg_dbg_ev + 8 * kq;
                    e[0] = blockIdx.x; e[1] = tid; e[2] = first; e[3] = badw; e[4] = got; e[5] = want; e[6] = p; e[7] = clock64();
                }
#endif
            }
        }
#endif
    }
}

// --------------------------------------------------------------- k_verify
// One thread per record slot: the candidates must chain exactly.
__global__ void k_verify(const DecSeg* __restrict__ segs, const uint32_t* __restrict__ rec2seg, uint64_t nrec_total,
                         const uint32_t* __restrict__ seg_cnt, uint32_t* __restrict__ seg_fail,
                         const uint64_t* __restrict__ rec_pos, const uint64_t* __restrict__ rec_next) {
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (g >= nrec_total) return;
    const uint32_t lo = rec2seg[g];
    if (lo == ~0u) return;
    const DecSeg sg = segs[lo];
    const uint32_t r = (uint32_t)(g - sg.rec0);
    const uint32_t R = sg.nrec, B = sg.block;
    const uint32_t Ltail = (uint32_t)(sg.orig - (uint64_t)(R - 1) * B);
    bool ok = true;
    if (r == 0) {
        const uint32_t m_exp = (Ltail == B) ? R : (R > 1 ? R - 1 : 1);
        ok = seg_cnt[lo] == m_exp && rec_pos[g] == 0;
    }
    if (ok) {
        const uint64_t nx = rec_next[g];
        if (nx == ~0ull) ok = false;
        else if (r + 1 < R) ok = nx == rec_pos[g + 1];
        else ok = nx == sg.comp;
    }
    if (!ok) { atomicOr(&seg_fail[lo], 1u); DBG_ADD(15, 1); }
}

// ------------------------------------------------------------- k_resolve
// CTA per segment that failed verification (false candidates: header-like
// bytes inside payloads whose successor test also passed).  The true records
// are exactly the path that starts at candidate 0 (the segment start) and
// follows each record's size: gather the segment's candidates in position
// order, link each to the candidate (or tail record, or segment end) its
// header points to, mark the path from 0 by pointer doubling (log2 m rounds),
// and rank the marked ones.  A consistent path (R records ending at the
// segment end) clears the failure; anything else stays with k_fallback.
constexpr int kResMax = 8192;   // candidates per segment resolvable in shared memory
constexpr size_t kResSmem = (size_t)kResMax * (4 + 2 + 2 + 1) + 16;

__global__ void __launch_bounds__(kThreads) k_resolve(const DecSeg* __restrict__ segs, uint64_t nseg_total,
                                                    const uint32_t* __restrict__ cand, const uint32_t* __restrict__ ccnt,
                                                    const uint32_t* __restrict__ cpre, const uint32_t* __restrict__ seg_cnt,
                                                    uint32_t* __restrict__ seg_fail, uint64_t* __restrict__ rec_pos,
                                                    uint64_t* __restrict__ rec_next) {
    extern __shared__ __align__(16) uint8_t res_smem[];
    uint32_t* ps = reinterpret_cast<uint32_t*>(res_smem);                         // candidate positions
    int16_t (*nx)[kResMax] = reinterpret_cast<int16_t (*)[kResMax]>(ps + kResMax);  // successor index (kEnd / kTail / -1)
    uint8_t* mark = reinterpret_cast<uint8_t*>(nx[2]);
    __shared__ uint32_t wsum[kWarps];
    __shared__ int sh_ok;
    constexpr int16_t kEnd = 0x7FFF, kTail = 0x7FFE, kBad = -1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (uint64_t si = blockIdx.x; si < nseg_total; si += gridDim.x) {
        if (!seg_fail[si]) continue;
        const DecSeg sg = segs[si];
        const uint32_t m = seg_cnt[si];
        const uint32_t R = sg.nrec, B = sg.block;
        if (m == 0 || m > kResMax || R == 0) continue;
        const uint32_t Ltail = (uint32_t)(sg.orig - (uint64_t)(R - 1) * B);
        if (tid == 0) sh_ok = 1;
        __syncthreads();
        // gather (warp per chunk, spans in order)
        for (uint32_t cj = warp; cj < sg.nchunk; cj += kWarps) {
            const uint64_t t = sg.chunk0 + cj;
            uint32_t base = cpre[t];
            for (int w = 0; w < kWarps; w++) {
                const uint64_t span = t * kWarps + w;
                const uint32_t c = ccnt[span];
                if (c == kDense) { if (lane == 0) sh_ok = 0; break; }
                if (c <= kSpanCap) {
                    for (uint32_t k = lane; k < c; k += 32) ps[base + k] = cand[span * kSpanCap + k];
                } else {
                    constexpr uint64_t kWarpSpan = kChunk / kWarps;
                    const uint64_t c0 = cj * (uint64_t)kChunk, c1 = min(c0 + kChunk, sg.comp);
                    const uint64_t pa = c0 + w * kWarpSpan, pe = min(pa + kWarpSpan, c1);
                    uint32_t n = 0;
                    if (pa == 0 && pa < pe) { if (lane == 0) ps[base] = 0; n = 1; }
                    if (pa < pe) warp_scan(sg, pa, pe, n, lane, [&](uint64_t p, uint32_t r) { ps[base + r] = (uint32_t)p; });
                }
                base += c;
            }
        }
        __syncthreads();
        if (!sh_ok || ps[0] != 0) { __syncthreads(); continue; }
        // links
        for (uint32_t i = tid; i < m; i += kThreads) {
            int16_t v = kBad;
            uint32_t mode, l;
            uint64_t psz;
            if (rec_size(sg.base, sg.comp, ps[i], mode, l, psz) && (l == B || l == Ltail)) {
                const uint64_t q = ps[i] + 5 + psz;
                if (q == sg.comp) v = kEnd;
                else {
                    uint32_t lo = 0, hi = m;
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (ps[mid] < q) lo = mid + 1; else hi = mid;
                    }
                    if (lo < m && ps[lo] == q) v = (int16_t)lo;
                    else if (Ltail != B) {   // the tail record is not a candidate
                        uint32_t m2, l2;
                        uint64_t p2;
                        if (rec_size(sg.base, sg.comp, q, m2, l2, p2) && l2 == Ltail && q + 5 + p2 == sg.comp) v = kTail;
                    }
                }
            }
            nx[0][i] = v;
            mark[i] = i == 0;
        }
        if (tid == 0) mark[kResMax] = 0;
        __syncthreads();
        int cur = 0;
        for (uint32_t span = 1; span <= m + 1; span <<= 1) {
            for (uint32_t i = tid; i < m; i += kThreads) {
                const int16_t j = nx[cur][i];
                if (mark[i] && j >= 0 && j < (int16_t)m) mark[j] = 1;
            }
            __syncthreads();
            for (uint32_t i = tid; i < m; i += kThreads) {
                const int16_t j = nx[cur][i];
                nx[cur ^ 1][i] = (j >= 0 && j < (int16_t)m) ? nx[cur][j] : j;
            }
            cur ^= 1;
            __syncthreads();
        }
        // rank the marked candidates; rebuild their links from the headers
        uint32_t cnt = 0;
        const uint32_t per = (m + kThreads - 1) / kThreads;
        const uint32_t i0 = tid * per, i1 = min(m, i0 + per);
        for (uint32_t i = i0; i < i1; i++) cnt += mark[i];
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        uint32_t pre = 0, tot = 0;
        for (int w = 0; w < kWarps; w++) { if (w < warp) pre += wsum[w]; tot += wsum[w]; }
        pre += incl - cnt;
        const bool has_tail = Ltail != B;
        if (tot + (has_tail ? 1u : 0u) != R) { __syncthreads(); continue; }
        bool bad = false;
        const uint32_t nlast = tot - 1;   // rank of the last candidate record on the path
        for (uint32_t i = i0; i < i1; i++) {
            if (!mark[i]) continue;
            uint32_t mode, l;
            uint64_t psz;
            const uint64_t p = ps[i];
            rec_size(sg.base, sg.comp, p, mode, l, psz);
            const uint32_t r = pre++;
            const uint64_t q = p + 5 + psz;
            rec_pos[sg.rec0 + r] = p;
            rec_next[sg.rec0 + r] = q;
            if (l != ((r + 1 == R) ? Ltail : B)) bad = true;
            if (r == nlast) {
                if (!has_tail) {
                    if (q != sg.comp) bad = true;
                } else {
                    uint32_t m2, l2;
                    uint64_t p2;
                    if (rec_size(sg.base, sg.comp, q, m2, l2, p2) && l2 == Ltail && q + 5 + p2 == sg.comp) {
                        rec_pos[sg.rec0 + R - 1] = q;
                        rec_next[sg.rec0 + R - 1] = q + 5 + p2;
                    } else {
                        bad = true;
                    }
                }
            }
        }
        bad = __syncthreads_or(bad);
        if (tid == 0 && !bad) seg_fail[si] = 0;
        if (tid == 0) DBG_ADD(bad ? 10 : 9, 1);
        __syncthreads();
    }
}

// ------------------------------------------------------------- k_fallback
// Serial record walk with the reference's validation (stream.py:234-268) for
// every segment that failed verification; decodes each record in turn.
__global__ void __launch_bounds__(kThreads) k_fallback(const DecSeg* __restrict__ segs, uint64_t nseg_total,
                                                     const uint32_t* __restrict__ seg_fail, uint32_t* __restrict__ status,
                                                     uint8_t* __restrict__ scratch) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    DecSmem& s = *reinterpret_cast<DecSmem*>(smem_raw);
    __shared__ uint64_t sh_pos, sh_got, sh_ps;
    __shared__ uint32_t sh_mode, sh_len, sh_ok;
    for (uint64_t si = blockIdx.x; si < nseg_total; si += gridDim.x) {
        if (!seg_fail[si]) continue;
        DBG_ADD(11, threadIdx.x == 0);
        if (threadIdx.x == 0) atomicAdd(&lmcg_fallback_segs, 1ull);
        const DecSeg sg = segs[si];
        if (threadIdx.x == 0) { sh_pos = 0; sh_got = 0; }
        __syncthreads();
        bool corrupt = false;
        for (;;) {
            if (threadIdx.x == 0) {
                sh_ok = 1;
                const uint64_t pos = sh_pos, got = sh_got;
                if (got >= sg.orig) {
                    sh_ok = (pos == sg.comp) ? 2 : 0;
                } else {
                    uint32_t mode = 0, l = 0;
                    uint64_t ps = 0;
                    if (pos + 5 > sg.comp) sh_ok = 0;
                    else {
                        l = rd32(sg.base + pos + 1);
                        if (l == 0 || l > sg.block || l > sg.orig - got) sh_ok = 0;
                        else if (!rec_size(sg.base, sg.comp, pos, mode, l, ps)) sh_ok = 0;
                        else { sh_mode = mode; sh_len = l; sh_ps = ps; }
                    }
                }
            }
            __syncthreads();
            const uint32_t okv = sh_ok;
            if (okv == 2) break;
            if (okv == 0) { corrupt = true; break; }
            if (!decode_record(s, sg.base + sh_pos, sh_mode, sh_len, scratch + sg.goff + sh_got, kStageLarge)) { corrupt = true; break; }
            __syncthreads();
            if (threadIdx.x == 0) { sh_pos += 5 + sh_ps; sh_got += sh_len; }
            __syncthreads();
        }
        if (corrupt && threadIdx.x == 0) atomicOr(&status[sg.stream], ST_CORRUPT);
        __syncthreads();
    }
}

// -------------------------------------------------------------- k_ungroup
// Persistent warps over 32 KiB output tiles of the windows (the k_crc
// layout): out[e*w + g] = grouped[g*n + e].  The warp writes the tile as 32
// rows of 1 KiB, lane l producing the 32 output bytes at 1024 r + 32 l of
// each row (coalesced plane loads and 16-byte stores), and folds them into a
// raw CRC: two Horner chains per lane (rows 0-15, 16-31), a 992-byte shift
// (4 lookups) per row and the piece by slicing-by-4 through 32-fold
// replicated tables (crc4_rep: lane l reads copy l, no bank conflicts); lane values are then shifted to
// the tile end and XOR-reduced.  A short last tile is treated as left-padded
// with zero bytes, which leave a raw CRC unchanged.  lmcg_decompress_apply
// XORs the previous step into the stores (the CRC stays the payload's).
constexpr int kUngThreads = 1024;   // one CTA per SM shares the 32 KiB of conflict-free slicing tables (rep4x8)
constexpr int kUngWarps = kUngThreads / 32;
constexpr size_t kUngSmem = (kCrcRepWords + 1024) * sizeof(uint32_t);   // rep4x8 | 992-byte shift

__global__ void __launch_bounds__(kUngThreads, 1) k_ungroup(const DecWin* __restrict__ wins, const uint32_t* __restrict__ tile2win,
                                                    uint64_t ntile_total, const uint8_t* __restrict__ scratch,
                                                    uint8_t* out /* may alias a window's prev */, const CrcTables* __restrict__ ct,
                                                    const uint32_t* __restrict__ sh992, uint32_t* __restrict__ tile_crc,
                                                    const uint32_t* __restrict__ status, const uint32_t* __restrict__ seg_fail) {
    extern __shared__ uint32_t ung_tab[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < kCrcRepWords / 4; i += kUngThreads)
        reinterpret_cast<uint4*>(ung_tab)[i] = __ldg(reinterpret_cast<const uint4*>(ct->rep4x8) + i);
    uint32_t* st = ung_tab + kCrcRepWords;
    for (int i = tid; i < 1024; i += kUngThreads) st[i] = sh992[i];
    __syncthreads();
    Crc4x8Lane cl;
    cl.init(ung_tab, lane);
    auto shift992 = [&](uint32_t x) {
        return st[x & 0xFF] ^ st[256 + ((x >> 8) & 0xFF)] ^ st[512 + ((x >> 16) & 0xFF)] ^ st[768 + (x >> 24)];
    };
    static_assert(kOutTile == 32768, "k_ungroup rows");
    // tiles are dealt CTA-major (tile = blockIdx.x + gridDim.x * j, warp w
    // takes j = w, w + 32, ...), so a small window still spreads over every SM
    for (uint64_t j = warp, tile = blockIdx.x + (uint64_t)warp * gridDim.x; tile < ntile_total;
         j += kUngWarps, tile = blockIdx.x + j * gridDim.x) {
        const uint32_t wi = tile2win[tile];
        if (wi == ~0u) {   // unused capacity slot
            if (lane == 0) tile_crc[tile] = 0;
            continue;
        }
        const DecWin wd = wins[wi];
        if (status[wd.stream]) {
            if (lane == 0) tile_crc[tile] = 0;
            continue;
        }
        if (wd.fuse) {   // k_decpair wrote it, unless a segment of the window failed (then k_fallback decoded it to scratch)
            bool f = false;
            for (uint32_t i = lane; i < wd.nseg; i += 32) f |= seg_fail[wd.seg0 + i] != 0;
            if (!__any_sync(0xFFFFFFFFu, f)) continue;
        }
        const uint64_t t0 = (tile - wd.tile0) * kOutTile;
        const uint32_t L = (uint32_t)min((uint64_t)kOutTile, wd.W - t0);
        const uint32_t Z = kOutTile - L;   // leading zero padding of a short tile
        const uint32_t w = wd.w, lw = lg2w(w);
        const uint8_t* g = scratch + wd.goff;
        uint8_t* o = out + wd.ooff;
        const uint8_t* pv = wd.prev;
        // vector path for a whole piece: 16-byte aligned output (and prev),
        // plane loads of 32 >> lw bytes at an aligned element offset
        const bool avec = ((reinterpret_cast<uint64_t>(o) + t0) % 16 == 0) && (Z % 32 == 0) &&
                          (!pv || (reinterpret_cast<uint64_t>(pv) + t0) % 16 == 0) &&
                          (w == 1 ? ((reinterpret_cast<uint64_t>(g) + t0) % 16 == 0) : ((wd.n & 15) == 0));
        // the 32 output bytes at padded offset pb: written, and returned as 8 words
        auto piece = [&](uint32_t pb, uint32_t v[8]) {
            if (pb + 32 <= Z) {
#pragma unroll
                for (int q = 0; q < 8; q++) v[q] = 0;
                return;
            }
            const uint64_t ob = t0 + pb - Z;
            if (avec && pb >= Z) {
                if (w == 1) {
                    const uint4 a0 = *reinterpret_cast<const uint4*>(g + ob), a1 = *reinterpret_cast<const uint4*>(g + ob + 16);
                    v[0] = a0.x; v[1] = a0.y; v[2] = a0.z; v[3] = a0.w; v[4] = a1.x; v[5] = a1.y; v[6] = a1.z; v[7] = a1.w;
                } else if (w == 2) {
                    const uint64_t e = ob >> 1;
                    const uint4 a = *reinterpret_cast<const uint4*>(g + e), b = *reinterpret_cast<const uint4*>(g + wd.n + e);
                    const uint32_t lo4[4] = {a.x, a.y, a.z, a.w}, hi4[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        v[2 * q] = __byte_perm(lo4[q], hi4[q], 0x5140);
                        v[2 * q + 1] = __byte_perm(lo4[q], hi4[q], 0x7362);
                    }
                } else {
                    const uint64_t e = ob >> 2;
                    uint2 pl[4];
#pragma unroll
                    for (int q = 0; q < 4; q++) pl[q] = *reinterpret_cast<const uint2*>(g + q * wd.n + e);
#pragma unroll
                    for (int q = 0; q < 2; q++) {
                        const uint32_t p0 = q ? pl[0].y : pl[0].x, p1 = q ? pl[1].y : pl[1].x;
                        const uint32_t p2 = q ? pl[2].y : pl[2].x, p3 = q ? pl[3].y : pl[3].x;
                        const uint32_t x01lo = __byte_perm(p0, p1, 0x5140), x01hi = __byte_perm(p0, p1, 0x7362);
                        const uint32_t x23lo = __byte_perm(p2, p3, 0x5140), x23hi = __byte_perm(p2, p3, 0x7362);
                        v[4 * q + 0] = __byte_perm(x01lo, x23lo, 0x5410);
                        v[4 * q + 1] = __byte_perm(x01lo, x23lo, 0x7632);
                        v[4 * q + 2] = __byte_perm(x01hi, x23hi, 0x5410);
                        v[4 * q + 3] = __byte_perm(x01hi, x23hi, 0x7632);
                    }
                }
                uint4 s0 = make_uint4(v[0], v[1], v[2], v[3]), s1 = make_uint4(v[4], v[5], v[6], v[7]);
                if (pv) {
                    const uint4 p0 = *reinterpret_cast<const uint4*>(pv + ob), p1 = *reinterpret_cast<const uint4*>(pv + ob + 16);
                    s0.x ^= p0.x; s0.y ^= p0.y; s0.z ^= p0.z; s0.w ^= p0.w;
                    s1.x ^= p1.x; s1.y ^= p1.y; s1.z ^= p1.z; s1.w ^= p1.w;
                }
                *reinterpret_cast<uint4*>(o + ob) = s0;
                *reinterpret_cast<uint4*>(o + ob + 16) = s1;
                return;
            }
#pragma unroll
            for (int q = 0; q < 8; q++) v[q] = 0;
            for (uint32_t i = 0; i < 32; i++) {
                if (pb + i < Z) continue;
                const uint64_t ob1 = t0 + pb + i - Z;
                const uint64_t e = ob1 >> lw, gg = ob1 - (e << lw);
                const uint32_t x = g[gg * wd.n + e];
                o[ob1] = pv ? (uint8_t)(x ^ pv[ob1]) : (uint8_t)x;
                v[i >> 2] |= x << (8 * (i & 3));
            }
        };
        uint32_t ca = 0, cb = 0;
        for (uint32_t r = 0; r < 16; r++) {
            uint32_t va[8], vb[8];
            piece(1024 * r + 32 * lane, va);
            piece(1024 * (r + 16) + 32 * lane, vb);
            ca = shift992(ca);
            cb = shift992(cb);
#pragma unroll
            for (int q = 0; q < 8; q++) {
                ca = cl.word(ca, va[q]);
                cb = cl.word(cb, vb[q]);
            }
        }
        // chain a ends 16 rows (16 KiB) before chain b; lane l's value ends
        // 32 (31 - l) bytes before the tile end
        uint32_t crc = crc_shift_tab(&ct->pow2[14][0][0], ca) ^ cb;
        crc = crc_shift_bytes(ct, crc, 32u * (31 - lane));
#pragma unroll
        for (int q = 16; q; q >>= 1) crc ^= __shfl_xor_sync(0xFFFFFFFFu, crc, q);
        if (lane == 0) tile_crc[tile] = crc;
    }
}

// ------------------------------------------------------------- k_finalize
__global__ void __launch_bounds__(kThreads) k_finalize(const DecStreamOut* __restrict__ sout, const DecCaps* __restrict__ caps,
                                                     const DecWin* __restrict__ wins, int ns,
                                                     const uint32_t* __restrict__ tile_crc, const CrcTables* __restrict__ ct,
                                                     uint32_t* __restrict__ status, const DecStreamIn* __restrict__ in) {
    __shared__ uint32_t red[kThreads];
    const int s = blockIdx.x;
    if (s >= ns) return;
    const DecStreamOut h = sout[s];
    if (h.status || status[s]) return;
    const DecCaps cp = caps[s];
    uint32_t acc = 0;  // stream raw CRC so far (thread 0)
    for (uint32_t wl = 0; wl < h.nwin; wl++) {
        const DecWin wd = wins[cp.win0 + wl];
        const uint64_t full = wd.W / kOutTile, rem = wd.W % kOutTile;
        const uint32_t* tc = tile_crc + wd.tile0;
        uint32_t wc = crc_combine_uniform(ct, full, kOutTile, [&](uint64_t i) { return tc[i]; }, red);
        if (threadIdx.x == 0) {
            if (rem) wc = crc_shift_bytes(ct, wc, rem) ^ tc[full];
            acc = crc_shift_bytes(ct, acc, wd.W) ^ wc;
        }
    }
    if (threadIdx.x == 0) {
        const uint32_t crc = acc ^ crc_shift_bytes(ct, 0xFFFFFFFFu, h.orig) ^ 0xFFFFFFFFu;
        if (crc != h.crc) atomicOr(&status[s], ST_INTEGRITY);
        // lmcg_decompress_apply: xor_bytes' length check comes after the decode
        // and its CRC check (chain.py:296-300 -> delta.py:20-21)
        else if (in[s].prev && in[s].prev_len != h.orig) atomicOr(&status[s], ST_SHAPE);
    }
}

// ----------------------------------------------------- plan helper kernels
// Stream inputs of a decompress plan: n streams at base + offsets[i].
__global__ void k_mkin(const uint8_t* __restrict__ base, const uint64_t* __restrict__ offsets,
                       const uint64_t* __restrict__ lengths, int n, DecStreamIn* __restrict__ in) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) in[i] = DecStreamIn{base + offsets[i], lengths[i], nullptr, 0};
}

// Final per-stream status as C-ABI codes (LMCG_*), written to device memory.
__global__ void k_status(const DecStreamOut* __restrict__ sout, const uint32_t* __restrict__ status, int n,
                         int32_t* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t s = sout[i].status | status[i];
    int32_t code = 0;
    if (s & ST_UNSUPPORTED) code = 1;
    else if (s & ST_CORRUPT) code = 2;
    else if (s & ST_RETRY) code = 10;
    else if (s & ST_CAPACITY) code = 8;
    else if (s & ST_INTEGRITY) code = 3;
    else if (s & ST_SHAPE) code = 11;
    out[i] = code;
}

}  // namespace lmcg
