// decompress.cu -- B200 kernels of the LMC decompress path.
//
//   k_parse      header + window/segment-table walk with the reference's exact
//                validation (stream.py:114-142, 358-389); pass 1 counts,
//                pass 2 writes window / segment descriptors
//   k_cand       record discovery, step 1: every 4 KiB chunk of every segment
//                is scanned for record headers "mode<=2 | len==block_size"
//   k_link       record discovery, step 2 (warp per segment): the candidates
//                must chain exactly (p -> p + record size) through the
//                canonical record lengths; otherwise the segment is walked
//                serially exactly like decompress_segment (stream.py:234-268)
//   k_decode     persistent CTA-per-record decoder: RLE fill, stored copy, and
//                Huffman decode with self-synchronising chunked parallel
//                decoding (huffman.py:258-349 semantics, stream.py:190-215)
//   k_ungroup    inverse byte-grouping of each window (bytegroup.py:53-62,
//                stream.py:392-403) + raw CRC-32 of every 16 KiB output tile
//   k_finalize   per-stream CRC combine and status (stream.py:416-423)
#include "lmc_common.cuh"

namespace lmcg {

constexpr int kCandChunk = 4096;   // bytes of segment payload per k_cand CTA
constexpr int kCandCap = 32;       // candidates kept per chunk
constexpr int kOutTile = 16384;    // output bytes per k_ungroup CTA
constexpr uint8_t kSkip = 0xFF;

enum : uint32_t { ST_CORRUPT = 1, ST_INTEGRITY = 2, ST_UNSUPPORTED = 4, ST_CAPACITY = 8 };

struct DecStreamIn {
    const uint8_t* p;
    uint64_t len;
};

// per stream, written by k_parse pass 1 (and read back by the host)
struct DecStreamHdr {
    uint64_t orig;
    uint32_t status;   // ST_* bits
    uint32_t et, flags, block, segs, crc;
    uint32_t nwin;
    uint32_t pad;
    uint64_t nseg;
    uint64_t nrec;     // canonical record count = sum ceil(seg_orig / block)
};

// per stream, computed by the host after pass 1
struct DecStreamPlan {
    uint64_t win0, seg0, rec0;      // global first window / segment / record
    uint64_t chunk0, nchunk;        // k_cand chunk range (upper bound)
    uint64_t tile0, ntile;          // k_ungroup tile range (upper bound)
    uint64_t scratch;               // grouped scratch offset (16-aligned)
    uint64_t out;                   // output offset (caller's layout)
};

struct DecWin {
    uint64_t W, n;          // window bytes, bytes per plane
    uint64_t goff;          // absolute scratch offset (16-aligned)
    uint64_t ooff;          // absolute output offset
    uint64_t soff;          // window start inside the stream's original payload
    uint32_t w, stream;
};

struct DecSeg {
    uint64_t comp_off;      // segment start (byte offset inside its stream)
    uint64_t comp_len;
    uint64_t orig_off;      // offset inside the window's grouped bytes
    uint64_t orig_len;
    uint64_t rec0;          // global index of the first canonical record slot
    uint64_t chunk0;        // global index of the first k_cand chunk
    uint32_t win, stream;
    uint32_t nrec, block;
};

struct DecRec {
    const uint8_t* src;     // record start (mode byte)
    uint8_t* dst;           // grouped scratch destination
    uint32_t len;           // original block length
    uint32_t psize;         // payload bytes
    uint32_t stream;
    uint8_t mode;
    uint8_t pad[3];
};

__device__ __forceinline__ uint32_t rd32(const uint8_t* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
__device__ __forceinline__ uint64_t rd64(const uint8_t* p) { return (uint64_t)rd32(p) | ((uint64_t)rd32(p + 4) << 32); }

__device__ __forceinline__ bool valid_block(uint32_t b) { return b >= 4096 && b <= (1u << 20) && (b & (b - 1)) == 0; }

// ---------------------------------------------------------------- k_parse
// One thread per stream.  pass 1: validate + count; pass 2: write descriptors.
__global__ void k_parse(const DecStreamIn* __restrict__ in, int ns, int pass, DecStreamHdr* __restrict__ hdr,
                        const DecStreamPlan* __restrict__ plan, DecWin* __restrict__ wins, DecSeg* __restrict__ segs,
                        uint64_t* __restrict__ win_tile0) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ns) return;
    const uint8_t* p = in[s].p;
    const uint64_t len = in[s].len;
    DecStreamHdr h;
    if (pass == 2) {
        h = hdr[s];
        if (h.status) return;
    } else {
        h.orig = 0; h.status = 0; h.et = 0; h.flags = 0; h.block = 0; h.segs = 0; h.crc = 0;
        h.nwin = 0; h.pad = 0; h.nseg = 0; h.nrec = 0;
        // parse_header (stream.py:114-142)
        if (len < kHeader || p[0] != 'L' || p[1] != 'M' || p[2] != 'C' || p[3] != '1' || p[4] != 1) {
            h.status = ST_UNSUPPORTED; hdr[s] = h; return;
        }
        const uint32_t flags = p[5], et = p[6];
        h.flags = flags; h.et = et;
        h.orig = rd64(p + 8); h.block = rd32(p + 16); h.segs = rd32(p + 20); h.crc = rd32(p + 24);
        const uint32_t width = et == 0 ? 1 : (et == 3 ? 4 : 2);
        if ((flags & ~3u) || p[7] != 0 || et > 3 || !valid_block(h.block) || h.segs < 1 || (h.orig % width)) {
            h.status = ST_CORRUPT; hdr[s] = h; return;
        }
    }
    const uint32_t width = h.et == 0 ? 1 : (h.et == 3 ? 4 : 2);
    const uint32_t wdt = (h.flags & 1) ? width : 1;
    const uint64_t B = h.block, S = h.segs;
    // iter_windows (stream.py:358-389)
    uint64_t off = kHeader, remaining = h.orig, opos = 0;
    uint64_t nwin = 0, nseg = 0, nrec = 0, ntile = 0, scr = 0;
    const uint64_t table = kSegEntry * S;
    const DecStreamPlan pl = (pass == 2) ? plan[s] : DecStreamPlan{};
    uint64_t chunk = 0;
    bool bad = false;
    while (remaining > 0) {
        if (table > len - off) { bad = true; break; }
        uint64_t wsum = 0;
        bool over = false;
        for (uint64_t i = 0; i < S; i++) {
            const uint64_t o = rd64(p + off + i * kSegEntry);
            if (o > remaining - wsum) over = true;
            else wsum += o;
        }
        const uint64_t toff = off;
        off += table;
        if (over || wsum == 0) { bad = true; break; }
        const uint64_t W = wsum;
        if ((h.flags & 1) && (W % width)) { bad = true; break; }   // reassemble_window
        uint64_t gpos = 0;
        for (uint64_t i = 0; i < S; i++) {
            const uint64_t so = rd64(p + toff + i * kSegEntry), sc = rd64(p + toff + i * kSegEntry + 8);
            if (sc > len - off) { bad = true; break; }
            if ((so == 0) != (sc == 0)) { bad = true; break; }
            const uint64_t r = (so + B - 1) / B;
            if (pass == 2) {
                DecSeg d;
                d.comp_off = off; d.comp_len = sc; d.orig_off = gpos; d.orig_len = so;
                d.rec0 = pl.rec0 + nrec; d.chunk0 = pl.chunk0 + chunk;
                d.win = (uint32_t)(pl.win0 + nwin); d.stream = (uint32_t)s;
                d.nrec = (uint32_t)r; d.block = (uint32_t)B;
                segs[pl.seg0 + nseg] = d;
            }
            chunk += (sc + kCandChunk - 1) / kCandChunk;
            nrec += r;
            nseg++;
            off += sc;
            gpos += so;
        }
        if (bad) break;
        if (pass == 2) {
            DecWin d;
            d.W = W; d.n = W / wdt; d.w = wdt; d.stream = (uint32_t)s;
            d.goff = pl.scratch + scr; d.ooff = pl.out + opos; d.soff = opos;
            wins[pl.win0 + nwin] = d;
            win_tile0[pl.win0 + nwin] = pl.tile0 + ntile;
        }
        ntile += (W + kOutTile - 1) / kOutTile;
        scr += (W + 15) & ~15ull;
        nwin++;
        opos += W;
        remaining -= W;
    }
    if (!bad && off != len) bad = true;   // trailing bytes (stream.py:388-389)
    if (pass == 1) {
        if (bad) { h.status = ST_CORRUPT; hdr[s] = h; return; }
        h.nwin = (uint32_t)nwin; h.nseg = nseg; h.nrec = nrec;
        hdr[s] = h;
    }
}

// ----------------------------------------------------------------- k_cand
// CTA per 4 KiB chunk of segment payload.  A candidate is a position where a
// record header "mode <= 2 | len == block_size" fits, plus the segment start.
__global__ void __launch_bounds__(128) k_cand(const DecStreamIn* __restrict__ in, const DecSeg* __restrict__ segs,
                                              uint64_t nseg_total, uint64_t nchunk_total,
                                              uint32_t* __restrict__ cand_cnt, uint32_t* __restrict__ cand_pos) {
    __shared__ uint8_t buf[kCandChunk + 8];
    __shared__ uint32_t sh_w[4];
    const uint64_t chunk = blockIdx.x;
    if (chunk >= nchunk_total) return;
    // segment owning this chunk: last seg with chunk0 <= chunk
    uint64_t lo = 0, hi = nseg_total;
    while (hi - lo > 1) {
        uint64_t mid = (lo + hi) >> 1;
        if (segs[mid].chunk0 <= chunk) lo = mid; else hi = mid;
    }
    const DecSeg sg = segs[lo];
    const uint64_t nch = (sg.comp_len + kCandChunk - 1) / kCandChunk;
    if (chunk < sg.chunk0 || chunk >= sg.chunk0 + nch) {
        if (threadIdx.x == 0) cand_cnt[chunk] = 0;
        return;
    }
    const uint64_t c0 = (chunk - sg.chunk0) * kCandChunk;
    const uint64_t avail = min((uint64_t)(sg.comp_len - c0), (uint64_t)(kCandChunk + 8));
    const uint8_t* base = in[sg.stream].p + sg.comp_off + c0;
    for (int i = threadIdx.x; i < kCandChunk + 8; i += 128) buf[i] = i < (int)avail ? base[i] : 0xFF;
    __syncthreads();
    const uint32_t B = sg.block;
    const uint64_t npos = min((uint64_t)(sg.comp_len - c0), (uint64_t)(kCandChunk));
    uint32_t mask = 0;
    for (int q = 0; q < 32; q++) {
        const int i = threadIdx.x * 32 + q;
        if ((uint64_t)i >= npos) break;
        const uint64_t pos = c0 + i;
        bool cand = (pos == 0);
        if (!cand && pos + 5 <= sg.comp_len && buf[i] <= 2) {
            const uint32_t l = (uint32_t)buf[i + 1] | ((uint32_t)buf[i + 2] << 8) | ((uint32_t)buf[i + 3] << 16) |
                               ((uint32_t)buf[i + 4] << 24);
            cand = (l == B);
        }
        if (cand) mask |= 1u << q;
    }
    // ordered compaction
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t c = __popc(mask);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) sh_w[warp] = incl;
    __syncthreads();
    uint32_t pre = 0, tot = 0;
    for (int q = 0; q < 4; q++) { if (q < warp) pre += sh_w[q]; tot += sh_w[q]; }
    uint32_t o = pre + incl - c;
    while (mask) {
        const int q = __ffs(mask) - 1;
        mask &= mask - 1;
        if (o < kCandCap) cand_pos[chunk * kCandCap + o] = (uint32_t)(c0 + threadIdx.x * 32 + q);
        o++;
    }
    if (threadIdx.x == 0) cand_cnt[chunk] = tot;
}

// ----------------------------------------------------------------- k_link
__device__ __forceinline__ bool rec_size_at(const uint8_t* seg, uint64_t comp, uint64_t pos, uint32_t& mode,
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

// One warp per segment.
__global__ void __launch_bounds__(128) k_link(const DecStreamIn* __restrict__ in, const DecSeg* __restrict__ segs,
                                              uint64_t nseg_total, const DecWin* __restrict__ wins,
                                              const uint32_t* __restrict__ cand_cnt, const uint32_t* __restrict__ cand_pos,
                                              DecRec* __restrict__ recs, DecRec* __restrict__ irr, uint32_t* __restrict__ irr_count,
                                              uint32_t irr_cap, uint32_t* __restrict__ status, uint8_t* __restrict__ scratch) {
    const int lane = threadIdx.x & 31;
    const uint64_t si = (uint64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    if (si >= nseg_total) return;
    const DecSeg sg = segs[si];
    if (sg.orig_len == 0) return;
    const uint8_t* seg = in[sg.stream].p + sg.comp_off;
    uint8_t* gdst = scratch + wins[sg.win].goff + sg.orig_off;
    const uint64_t comp = sg.comp_len;
    const uint32_t B = sg.block, R = sg.nrec;
    const uint32_t Ltail = (uint32_t)(sg.orig_len - (uint64_t)(R - 1) * B);
    const uint64_t nch = (comp + kCandChunk - 1) / kCandChunk;
    // total candidates (and overflow)
    uint64_t m = 0;
    bool overflow = false;
    for (uint64_t c = lane; c < nch; c += 32) {
        const uint32_t k = cand_cnt[sg.chunk0 + c];
        m += k;
        overflow |= k > kCandCap;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m += __shfl_xor_sync(0xFFFFFFFFu, m, o);
    overflow = __any_sync(0xFFFFFFFFu, overflow);
    const uint64_t m_exp = (Ltail == B) ? R : (R > 1 ? R - 1 : 1);
    bool ok = !overflow && m == m_exp;
    if (ok) {
        // candidate i -> (chunk, slot): walk chunks with a running prefix
        uint64_t pre = 0;
        for (uint64_t cbase = 0; cbase < nch && ok; cbase += 32) {
            const uint64_t c = cbase + lane;
            const uint32_t k = c < nch ? cand_cnt[sg.chunk0 + c] : 0;
            uint32_t incl = k;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += y;
            }
            const uint64_t first = pre + incl - k;
            bool good = true;
            for (uint32_t j = 0; j < k; j++) {
                const uint64_t idx = first + j;   // candidate == canonical record index
                const uint64_t pos = cand_pos[(sg.chunk0 + c) * kCandCap + j];
                uint32_t mode, l;
                uint64_t ps;
                const uint32_t want = (idx + 1 == R) ? Ltail : B;
                if (!rec_size_at(seg, comp, pos, mode, l, ps) || l != want) { good = false; break; }
                const uint64_t nxt = pos + 5 + ps;
                // successor: next candidate, or the tail record, or the segment end
                if (idx + 1 < m) {
                    const uint64_t np = (j + 1 < k) ? cand_pos[(sg.chunk0 + c) * kCandCap + j + 1] : ~0ull;
                    if (np != ~0ull && np != nxt) { good = false; break; }
                    if (np == ~0ull) {
                        // first candidate of a later chunk: checked by its predecessor through scan below
                    }
                } else if (m < R) {
                    // tail record follows the last candidate (Ltail != B)
                    uint32_t tm, tl;
                    uint64_t tps;
                    if (!rec_size_at(seg, comp, nxt, tm, tl, tps) || tl != Ltail || nxt + 5 + tps != comp) {
                        good = false; break;
                    }
                    DecRec t;
                    t.src = seg + nxt; t.dst = gdst + (uint64_t)(R - 1) * B; t.len = tl; t.psize = (uint32_t)tps;
                    t.stream = sg.stream; t.mode = (uint8_t)tm;
                    recs[sg.rec0 + R - 1] = t;
                } else {
                    if (nxt != comp) { good = false; break; }
                }
                DecRec d;
                d.src = seg + pos; d.dst = gdst + idx * B; d.len = l; d.psize = (uint32_t)ps;
                d.stream = sg.stream; d.mode = (uint8_t)mode;
                recs[sg.rec0 + idx] = d;
            }
            ok = __all_sync(0xFFFFFFFFu, good);
            pre += __shfl_sync(0xFFFFFFFFu, incl, 31);
        }
        // cross-chunk links: the last candidate of each chunk must point at the
        // first candidate of the next non-empty chunk
        if (ok) {
            __syncwarp();
            bool good = true;
            for (uint64_t i = lane; i + 1 < m; i += 32) {
                const DecRec a = recs[sg.rec0 + i];
                const DecRec bb = recs[sg.rec0 + i + 1];
                if (a.src + 5 + a.psize != bb.src) good = false;
            }
            ok = __all_sync(0xFFFFFFFFu, good);
        }
    }
    if (ok) return;
    // ---- serial walk, exactly decompress_segment (stream.py:234-255)
    __syncwarp();
    for (uint32_t r = lane; r < R; r += 32) recs[sg.rec0 + r].mode = kSkip;
    __syncwarp();
    if (lane != 0) return;
    uint64_t pos = 0, got = 0;
    uint32_t idx = 0;
    bool canon = true;
    uint32_t nirr = 0;
    // first pass: validate and check canonical shape
    while (got < sg.orig_len) {
        uint32_t mode, l;
        uint64_t ps;
        if (pos + 5 > comp) { atomicOr(&status[sg.stream], ST_CORRUPT); return; }
        mode = seg[pos];
        l = rd32(seg + pos + 1);
        if (l == 0 || l > B || l > sg.orig_len - got) { atomicOr(&status[sg.stream], ST_CORRUPT); return; }
        if (!rec_size_at(seg, comp, pos, mode, l, ps)) { atomicOr(&status[sg.stream], ST_CORRUPT); return; }
        const uint32_t want = (idx + 1 == R) ? Ltail : B;
        if (idx >= R || l != want) canon = false;
        pos += 5 + ps;
        got += l;
        idx++;
    }
    if (pos != comp) { atomicOr(&status[sg.stream], ST_CORRUPT); return; }
    if (!canon) {
        nirr = atomicAdd(irr_count, idx);
        if (nirr + idx > irr_cap) { atomicOr(&status[sg.stream], ST_CAPACITY); return; }
    }
    // second pass: emit records
    pos = 0; got = 0;
    for (uint32_t r = 0; r < idx; r++) {
        uint32_t mode, l;
        uint64_t ps;
        rec_size_at(seg, comp, pos, mode, l, ps);
        DecRec d;
        d.src = seg + pos; d.dst = gdst + got; d.len = l; d.psize = (uint32_t)ps; d.stream = sg.stream;
        d.mode = (uint8_t)mode;
        if (canon) recs[sg.rec0 + r] = d;
        else irr[nirr + r] = d;
        pos += 5 + ps;
        got += l;
    }
}

// --------------------------------------------------------------- k_decode
constexpr int kLutBits = 11;

struct DecSmem {
    uint8_t lens[256];
    uint8_t csym[256];          // symbols in canonical (length, symbol) order
    uint16_t lut[1 << kLutBits];  // (len << 8) | sym for codes <= kLutBits, 0 otherwise
    uint32_t first_left[17];    // left-justified first code of each length
    uint32_t first_idx[17];     // canonical index of the first code of each length
    uint32_t bl_count[17];
    uint32_t cnt_w[kWarps][16];
    uint32_t start[kThreads], end[kThreads], cnt[kThreads], off[kThreads];
    uint32_t wsum[kWarps];
    uint32_t kraft;
    int minlen, maxlen;
};

struct BitReader {
    const uint8_t* base;   // 4-byte aligned base
    uint64_t nwords_full;  // words entirely inside the payload
    uint64_t limit;        // payload end (bytes from base)
    uint64_t buf;
    int nb;
    uint64_t next;         // next word index
    __device__ __forceinline__ uint32_t word(uint64_t j) const {
        if (j < nwords_full) return bswap32(__ldg(reinterpret_cast<const uint32_t*>(base) + j));
        uint32_t v = 0;
        for (int q = 0; q < 4; q++) {
            const uint64_t o = j * 4 + q;
            v = (v << 8) | (o < limit ? base[o] : 0u);
        }
        return v;
    }
    __device__ __forceinline__ void init(const uint8_t* data, uint64_t nbytes, uint64_t bitpos) {
        base = reinterpret_cast<const uint8_t*>(reinterpret_cast<uint64_t>(data) & ~3ull);
        const uint32_t sh = (uint32_t)(reinterpret_cast<uint64_t>(data) & 3) * 8;
        limit = (uint64_t)(data - base) + nbytes;
        nwords_full = limit / 4;
        const uint64_t abit = bitpos + sh;
        const uint64_t j = abit >> 5;
        const int k = (int)(abit & 31);
        buf = (((uint64_t)word(j) << 32) | word(j + 1)) << k;
        nb = 64 - k;
        next = j + 2;
    }
    __device__ __forceinline__ void refill() {
        if (nb <= 32) {
            buf |= (uint64_t)word(next) << (32 - nb);
            nb += 32;
            next++;
        }
    }
};

// Decode codewords starting in [pos, lim); returns the end position (first
// boundary >= lim) or ~0u on an invalid prefix.  EMIT writes the symbols to
// dst (16-byte grouped stores where aligned).
template <bool EMIT>
__device__ __forceinline__ uint32_t decode_run(const DecSmem& s, const uint8_t* data, uint64_t nbytes, uint32_t pos,
                                               uint32_t lim, uint32_t& count, uint8_t* dst) {
    BitReader br;
    br.init(data, nbytes, pos);
    uint32_t c = 0;
    uint64_t acc_lo = 0, acc_hi = 0;
    int nacc = 0;
    uint64_t o = 0;  // bytes emitted
    while (pos < lim) {
        br.refill();
        const uint32_t win = (uint32_t)(br.buf >> 49);  // 15-bit window
        const uint32_t e = s.lut[win >> (kMaxLen - kLutBits)];
        uint32_t l, sym;
        if (e) {
            l = e >> 8;
            sym = e & 0xFF;
        } else {
            l = 0;
            for (int q = kLutBits + 1; q <= s.maxlen; q++) {
                const uint32_t endq = s.first_left[q] + (s.bl_count[q] << (kMaxLen - q));
                if (s.bl_count[q] && win >= s.first_left[q] && win < endq) { l = q; break; }
            }
            if (!l) { count = c; return ~0u; }
            sym = s.csym[s.first_idx[l] + ((win - s.first_left[l]) >> (kMaxLen - l))];
        }
        br.buf <<= l;
        br.nb -= l;
        pos += l;
        c++;
        if (EMIT) {
            // head bytes until 16-byte alignment, then whole uint4 stores
            uint8_t* d = dst + o;
            if (nacc == 0 && ((reinterpret_cast<uint64_t>(d) & 15) != 0)) {
                *d = (uint8_t)sym;
                o++;
            } else {
                if (nacc < 8) acc_lo |= (uint64_t)sym << (8 * nacc);
                else acc_hi |= (uint64_t)sym << (8 * (nacc - 8));
                nacc++;
                if (nacc == 16) {
                    *reinterpret_cast<uint4*>(dst + o) =
                        make_uint4((uint32_t)acc_lo, (uint32_t)(acc_lo >> 32), (uint32_t)acc_hi, (uint32_t)(acc_hi >> 32));
                    o += 16;
                    nacc = 0;
                    acc_lo = acc_hi = 0;
                }
            }
        }
    }
    if (EMIT) {
        for (int q = 0; q < nacc; q++) dst[o + q] = (uint8_t)((q < 8 ? acc_lo >> (8 * q) : acc_hi >> (8 * (q - 8))));
    }
    count = c;
    return pos;
}

__device__ __forceinline__ void copy_bytes(uint8_t* dst, const uint8_t* src, uint32_t n, int tid, int nt) {
    // dst is 16-byte aligned; src arbitrary
    const uint32_t nv = n / 16;
    for (uint32_t i = tid; i < nv; i += nt) {
        uint4 v;
        const uint8_t* sp = src + 16 * i;
        if ((reinterpret_cast<uint64_t>(sp) & 3) == 0) {
            const uint32_t* w = reinterpret_cast<const uint32_t*>(sp);
            v = make_uint4(__ldg(w), __ldg(w + 1), __ldg(w + 2), __ldg(w + 3));
        } else {
            const uint32_t* w = reinterpret_cast<const uint32_t*>(reinterpret_cast<uint64_t>(sp) & ~3ull);
            const uint32_t sh = (uint32_t)(reinterpret_cast<uint64_t>(sp) & 3) * 8;
            const uint32_t a0 = __ldg(w), a1 = __ldg(w + 1), a2 = __ldg(w + 2), a3 = __ldg(w + 3);
            // the 5th word may lie past the payload only for the final vector: read bytewise there
            uint32_t a4;
            if (16 * i + 16 + 4 <= n) a4 = __ldg(w + 4);
            else {
                a4 = 0;
                const uint8_t* b4 = reinterpret_cast<const uint8_t*>(w + 4);
                const uint64_t lim = (uint64_t)(src + n) - reinterpret_cast<uint64_t>(b4);
                for (uint32_t q = 0; q < 4 && q < lim; q++) a4 |= (uint32_t)b4[q] << (8 * q);
            }
            v = make_uint4(__funnelshift_r(a0, a1, sh), __funnelshift_r(a1, a2, sh), __funnelshift_r(a2, a3, sh),
                           __funnelshift_r(a3, a4, sh));
        }
        reinterpret_cast<uint4*>(dst)[i] = v;
    }
    for (uint32_t i = nv * 16 + tid; i < n; i += nt) dst[i] = src[i];
}

__global__ void __launch_bounds__(kThreads) k_decode(const DecRec* __restrict__ recs, uint64_t nrec,
                                                   const DecRec* __restrict__ irr, const uint32_t* __restrict__ irr_count,
                                                   uint32_t* __restrict__ status) {
    __shared__ DecSmem s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t total = nrec + *irr_count;
    for (uint64_t r = blockIdx.x; r < total; r += gridDim.x) {
        const DecRec d = (r < nrec) ? recs[r] : irr[r - nrec];
        __syncthreads();   // smem reuse across records
        if (d.mode == kSkip) continue;
        const uint8_t* pl = d.src + 5;
        if (d.mode == MODE_RLE) {
            const uint32_t v = pl[0] * 0x01010101u;
            const uint32_t nv = d.len / 16;
            for (uint32_t i = tid; i < nv; i += kThreads) reinterpret_cast<uint4*>(d.dst)[i] = make_uint4(v, v, v, v);
            for (uint32_t i = nv * 16 + tid; i < d.len; i += kThreads) d.dst[i] = (uint8_t)v;
            continue;
        }
        if (d.mode == MODE_STORED) {
            copy_bytes(d.dst, pl, d.len, tid, kThreads);
            continue;
        }
        // ---- Huffman (huffman.py:258-349 semantics)
        const uint8_t wb = pl[tid >> 1];
        const uint32_t l = (tid & 1) ? (wb >> 4) : (wb & 15);
        s.lens[tid] = (uint8_t)l;
        if (tid < kWarps * 16) (&s.cnt_w[0][0])[tid] = 0;
        if (tid == 0) s.kraft = 0;
        __syncthreads();
        const uint32_t mm = __match_any_sync(0xFFFFFFFFu, l);
        const uint32_t rank_w = __popc(mm & ((1u << lane) - 1));
        if (lane == __ffs(mm) - 1) s.cnt_w[warp][l] = __popc(mm);
        if (l) atomicAdd(&s.kraft, 1u << (kMaxLen - l));
        __syncthreads();
        if (tid == 0) {
            uint32_t left = 0, idx = 0;
            int mn = 16, mx = 0;
            for (int q = 1; q <= kMaxLen; q++) {
                uint32_t c = 0;
                for (int w = 0; w < kWarps; w++) c += s.cnt_w[w][q];
                s.bl_count[q] = c;
                s.first_left[q] = left;
                s.first_idx[q] = idx;
                left += c << (kMaxLen - q);
                idx += c;
                if (c) { mn = min(mn, q); mx = max(mx, q); }
            }
            s.minlen = mn;
            s.maxlen = mx;
        }
        __syncthreads();
        const uint32_t bits = rd32(pl + 128);
        // _validate_codebook (huffman.py:191-210) and the bit-length check (:275)
        const bool bad_cb = (s.maxlen == 0) || (s.kraft > (1u << kMaxLen)) || bits == 0;
        if (bad_cb) {
            if (tid == 0) atomicOr(&status[d.stream], ST_CORRUPT);
            continue;
        }
        if (l) {
            uint32_t rk = rank_w;
            for (int w = 0; w < warp; w++) rk += s.cnt_w[w][l];
            s.csym[s.first_idx[l] + rk] = (uint8_t)tid;
        }
        __syncthreads();
        // LUT: entry e covers windows [e << 4, (e+1) << 4)
        for (int e = tid; e < (1 << kLutBits); e += kThreads) {
            const uint32_t v = (uint32_t)e << (kMaxLen - kLutBits);
            uint16_t ent = 0;
            for (int q = 1; q <= kLutBits; q++) {
                const uint32_t fl = s.first_left[q], endq = fl + (s.bl_count[q] << (kMaxLen - q));
                if (v >= fl && v < endq) {
                    ent = (uint16_t)((q << 8) | s.csym[s.first_idx[q] + ((v - fl) >> (kMaxLen - q))]);
                    break;
                }
            }
            s.lut[e] = ent;
        }
        const uint8_t* data = pl + kHuffOverhead;
        const uint64_t nbytes = (bits + 7) / 8;
        // chunking: at most kThreads chunks of S bits (multiple of 32)
        uint32_t S = (bits + kThreads - 1) / kThreads;
        S = max(256u, (S + 31) & ~31u);
        const uint32_t nch = (bits + S - 1) / S;
        const bool fixed = s.minlen == s.maxlen;
        __syncthreads();
        // phase 1: speculative decode of every chunk from its nominal start
        const uint32_t c = tid;
        uint32_t my_start = 0, my_end = 0, my_cnt = 0;
        const uint32_t lim = min((c + 1) * S, bits);
        if (c < nch) {
            my_start = c * S;
            if (fixed) my_start = ((my_start + s.minlen - 1) / s.minlen) * s.minlen;
            if (my_start >= lim) { my_end = my_start; my_cnt = 0; }
            else my_end = decode_run<false>(s, data, nbytes, my_start, lim, my_cnt, nullptr);
            s.start[c] = my_start; s.end[c] = my_end; s.cnt[c] = my_cnt;
        }
        __syncthreads();
        // phase 2: fix-up rounds until every chunk starts where its predecessor ended
        for (;;) {
            uint32_t pe = 0;
            if (c < nch && c > 0) pe = s.end[c - 1];
            __syncthreads();
            int changed = 0;
            if (c < nch && c > 0 && pe != ~0u && pe != my_start) {
                my_start = pe;
                if (my_start >= lim) { my_end = my_start; my_cnt = 0; }
                else my_end = decode_run<false>(s, data, nbytes, my_start, lim, my_cnt, nullptr);
                s.start[c] = my_start; s.end[c] = my_end; s.cnt[c] = my_cnt;
                changed = 1;
            }
            if (!__syncthreads_or(changed)) break;
        }
        // totals
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
        const bool bad = __syncthreads_or(inv) || tot != d.len || s.end[nch - 1] != bits;
        if (bad) {
            if (tid == 0) atomicOr(&status[d.stream], ST_CORRUPT);
            continue;
        }
        // phase 3: final decode with output
        if (c < nch && my_cnt) {
            uint32_t cc;
            decode_run<true>(s, data, nbytes, my_start, lim, cc, d.dst + (pre + incl - v));
        }
    }
}

// -------------------------------------------------------------- k_ungroup
// CTA per 16 KiB output tile of a window: out[e*w + g] = grouped[g*n + e];
// each thread produces 64 contiguous output bytes and their raw CRC.
__global__ void __launch_bounds__(kThreads) k_ungroup(const DecWin* __restrict__ wins, const uint64_t* __restrict__ win_tile0,
                                                    uint64_t nwin_total, uint64_t ntile_total,
                                                    const uint8_t* __restrict__ scratch, uint8_t* __restrict__ out,
                                                    const CrcTables* __restrict__ ct, uint32_t* __restrict__ tile_crc,
                                                    uint64_t* __restrict__ tile_end, const uint32_t* __restrict__ status) {
    __shared__ uint32_t sh_slice[1024];
    __shared__ uint32_t sh_part[kWarps];
    const uint64_t tile = blockIdx.x;
    if (tile >= ntile_total) return;
    uint64_t lo = 0, hi = nwin_total;
    while (hi - lo > 1) {
        uint64_t mid = (lo + hi) >> 1;
        if (win_tile0[mid] <= tile) lo = mid; else hi = mid;
    }
    const DecWin wd = wins[lo];
    const uint64_t t0 = (tile - win_tile0[lo]) * kOutTile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tile < win_tile0[lo] || t0 >= wd.W || status[wd.stream]) {
        if (tid == 0) { tile_crc[tile] = 0; tile_end[tile] = 0; }
        return;
    }
    for (int i = tid; i < 1024; i += kThreads) sh_slice[i] = ct->slice[i >> 8][i & 255];
    __syncthreads();
    const uint64_t L = min((uint64_t)(kOutTile), (uint64_t)(wd.W - t0));
    const uint64_t Z = kOutTile - L;  // leading zero padding of a short tile
    const uint32_t w = wd.w;
    const uint8_t* g = scratch + wd.goff;
    uint8_t* o = out + wd.ooff;
    const uint64_t lo_b = (uint64_t)tid * kLaneBytes, hi_b = lo_b + kLaneBytes;
    uint32_t c = 0;
    const bool full = lo_b >= Z;
    const uint64_t ob = t0 + lo_b - Z;  // first output byte (window-relative) of this thread when full
    const bool vec = full && ((reinterpret_cast<uint64_t>(o) + ob) % 16 == 0) &&
                     (w == 1 ? ((reinterpret_cast<uint64_t>(g) + ob) % 16 == 0)
                             : ((ob / w) % 16 == 0 && (wd.n % 16) == 0));
    if (vec) {
        uint32_t v[16];
        if (w == 1) {
#pragma unroll
            for (int q = 0; q < 4; q++) {
                uint4 a = *reinterpret_cast<const uint4*>(g + ob + 16 * q);
                v[4 * q] = a.x; v[4 * q + 1] = a.y; v[4 * q + 2] = a.z; v[4 * q + 3] = a.w;
            }
        } else if (w == 2) {
            const uint64_t e = ob / 2;
            const uint4 a0 = *reinterpret_cast<const uint4*>(g + e), a1 = *reinterpret_cast<const uint4*>(g + e + 16);
            const uint4 b0 = *reinterpret_cast<const uint4*>(g + wd.n + e), b1 = *reinterpret_cast<const uint4*>(g + wd.n + e + 16);
            const uint32_t lw[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const uint32_t hw[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int q = 0; q < 8; q++) {
                v[2 * q] = __byte_perm(lw[q], hw[q], 0x5140);
                v[2 * q + 1] = __byte_perm(lw[q], hw[q], 0x7362);
            }
        } else {
            const uint64_t e = ob / 4;
            uint4 pl[4];
#pragma unroll
            for (int q = 0; q < 4; q++) pl[q] = *reinterpret_cast<const uint4*>(g + q * wd.n + e);
            const uint32_t* p0 = reinterpret_cast<const uint32_t*>(&pl[0]);
            const uint32_t* p1 = reinterpret_cast<const uint32_t*>(&pl[1]);
            const uint32_t* p2 = reinterpret_cast<const uint32_t*>(&pl[2]);
            const uint32_t* p3 = reinterpret_cast<const uint32_t*>(&pl[3]);
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const uint32_t x01lo = __byte_perm(p0[q], p1[q], 0x5140), x01hi = __byte_perm(p0[q], p1[q], 0x7362);
                const uint32_t x23lo = __byte_perm(p2[q], p3[q], 0x5140), x23hi = __byte_perm(p2[q], p3[q], 0x7362);
                v[4 * q + 0] = __byte_perm(x01lo, x23lo, 0x5410);
                v[4 * q + 1] = __byte_perm(x01lo, x23lo, 0x7632);
                v[4 * q + 2] = __byte_perm(x01hi, x23hi, 0x5410);
                v[4 * q + 3] = __byte_perm(x01hi, x23hi, 0x7632);
            }
        }
#pragma unroll
        for (int q = 0; q < 4; q++)
            *reinterpret_cast<uint4*>(o + ob + 16 * q) = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
#pragma unroll
        for (int q = 0; q < 16; q++) c = crc_word(sh_slice, c, v[q]);
    } else {
        for (uint64_t q = max(lo_b, Z); q < hi_b; q++) {
            const uint64_t ob1 = t0 + q - Z;
            const uint64_t e = ob1 / w, gg = ob1 - e * w;
            const uint8_t x = g[gg * wd.n + e];
            o[ob1] = x;
            c = crc_byte(sh_slice, c, x);
        }
    }
    c = crc_warp_tree(ct, c, lane);
    if (lane == 0) sh_part[warp] = c;
    __syncthreads();
    if (tid == 0) {
        uint32_t acc = 0;
        for (int q = 0; q < kWarps; q++) acc = crc_shift_tab(&ct->shift[5][0][0], acc) ^ sh_part[q];
        tile_crc[tile] = acc;
        tile_end[tile] = wd.soff + t0 + L;  // stream-relative end of this tile
    }
}

// ------------------------------------------------------------- k_finalize
__global__ void __launch_bounds__(kThreads) k_finalize(const DecStreamHdr* __restrict__ hdr, const DecStreamPlan* __restrict__ plan,
                                                     int ns, const uint32_t* __restrict__ tile_crc,
                                                     const uint64_t* __restrict__ tile_end, const CrcTables* __restrict__ ct,
                                                     uint32_t* __restrict__ status) {
    __shared__ uint32_t red[kThreads];
    const int s = blockIdx.x;
    if (s >= ns) return;
    const DecStreamHdr h = hdr[s];
    if (h.status) return;
    const DecStreamPlan pl = plan[s];
    uint32_t acc = 0;
    for (uint64_t t = threadIdx.x; t < pl.ntile; t += kThreads) {
        const uint64_t e = tile_end[pl.tile0 + t];
        const uint32_t part = tile_crc[pl.tile0 + t];
        if (part) acc ^= crc_shift_generic(ct->x2n, part, h.orig - e);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = kThreads / 2; o; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] ^= red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const uint32_t crc = red[0] ^ crc_shift_generic(ct->x2n, 0xFFFFFFFFu, h.orig) ^ 0xFFFFFFFFu;
        if (crc != h.crc) atomicOr(&status[s], ST_INTEGRITY);
    }
}

}  // namespace lmcg
