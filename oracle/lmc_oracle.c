/*
 * lmc_oracle.c -- CPU restatement of the reference LMC codec (TEST INFRASTRUCTURE).
 *
 * This file is the parity oracle for the B200 hot path.  It restates, function
 * by function, the reference Python package `lmc` 0.1.0 (the reference lives
 * under /root/reference/pkg/src/lmc in the build container only):
 *
 *   histogram            <- entropy.py:53-59
 *   build_codebook       <- huffman.py:79-103
 *   huffman_depths       <- huffman.py:106-137   (two-queue, ties prefer leaves)
 *   package_merge        <- huffman.py:140-180   (14 rounds, leaves first on ties)
 *   assign_canonical     <- huffman.py:183-225
 *   encode_block         <- huffman.py:228-255   (MSB-first, zero-padded)
 *   decode_block         <- huffman.py:258-349   (end-position check semantics)
 *   pack/unpack_codebook <- huffman.py:374-395
 *   encode_record        <- stream.py:161-177
 *   segment_bounds       <- stream.py:271-284
 *   lmc_compress         <- stream.py:311-355
 *   parse_header         <- stream.py:114-142
 *   iter_windows / decompress_segment / lmc_decompress <- stream.py:234-268,358-423
 *   group/ungroup        <- bytegroup.py:39-62
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and the
 * --impl reference arm) may load this library, and only as the checker or the
 * timed CPU baseline.  The product path (paper_2505_09810_b200) never links it.
 *
 * Parity pin: tests/golden/ holds streams produced by the live reference
 * (tests/golden/make_golden.py); tests/test_oracle.py checks this restatement
 * against them byte for byte.
 *
 * Block encoding and decoding are parallelised over pthreads (blocks are
 * independent, exactly like the reference's segment-level ProcessPool in
 * parallel.py:92-102); output bytes never depend on the thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define MAXLEN 15
#define KRAFT_ONE (1u << MAXLEN)
#define HDR 28
#define SEG_ENTRY 16
#define HUFF_OVERHEAD 132 /* 128-byte codebook + u32 bit count, stream.py:80 */

enum { LMCO_OK = 0, LMCO_UNSUPPORTED = 1, LMCO_CORRUPT = 2, LMCO_INTEGRITY = 3,
       LMCO_CONFIG = 4, LMCO_ALIGNMENT = 5, LMCO_EMPTY = 6, LMCO_NOMEM = 7,
       LMCO_CAPACITY = 8 };

/* ------------------------------------------------------------------ CRC-32 */
/* IEEE reflected polynomial 0xEDB88320, init/xorout 0xFFFFFFFF == zlib.crc32. */
static uint32_t crc_tab[8][256];
static pthread_once_t crc_once = PTHREAD_ONCE_INIT;
static void crc_init(void) {
    for (uint32_t i = 0; i < 256; i++) {
        uint32_t c = i;
        for (int k = 0; k < 8; k++) c = (c & 1) ? (c >> 1) ^ 0xEDB88320u : c >> 1;
        crc_tab[0][i] = c;
    }
    for (int t = 1; t < 8; t++)
        for (int i = 0; i < 256; i++)
            crc_tab[t][i] = (crc_tab[t - 1][i] >> 8) ^ crc_tab[0][crc_tab[t - 1][i] & 0xFF];
}
uint32_t lmco_crc32(const uint8_t* p, uint64_t n, uint32_t crc) {
    pthread_once(&crc_once, crc_init);
    crc = ~crc;
    while (n >= 8) {
        uint32_t a = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
        a ^= crc;
        crc = crc_tab[7][a & 0xFF] ^ crc_tab[6][(a >> 8) & 0xFF] ^ crc_tab[5][(a >> 16) & 0xFF] ^
              crc_tab[4][a >> 24] ^ crc_tab[3][p[4]] ^ crc_tab[2][p[5]] ^ crc_tab[1][p[6]] ^ crc_tab[0][p[7]];
        p += 8; n -= 8;
    }
    while (n--) crc = (crc >> 8) ^ crc_tab[0][(crc ^ *p++) & 0xFF];
    return ~crc;
}

/* -------------------------------------------------------------- histogram */
/* entropy.py:53-59 -- np.bincount(block, minlength=256) */
void lmco_histogram(const uint8_t* b, uint64_t n, uint64_t counts[256]) {
    memset(counts, 0, 256 * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; i++) counts[b[i]]++;
}

/* ------------------------------------------------------- codebook builder */
/* huffman.py:106-137: two-queue Huffman over ascending-sorted weights; ties
 * prefer the leaf queue (`w[leaf_head] <= w[node_head]`). */
static int huffman_depths(const uint64_t* w_in, int n, uint8_t* depth_out) {
    int total = 2 * n - 1;
    uint64_t w[511];
    int parent[511];
    int depth[511];
    for (int i = 0; i < n; i++) w[i] = w_in[i];
    int leaf_head = 0, node_head = n;
    for (int nxt = n; nxt < total; nxt++) {
        uint64_t acc = 0;
        for (int k = 0; k < 2; k++) {
            int child;
            if (leaf_head < n && (node_head >= nxt || w[leaf_head] <= w[node_head])) child = leaf_head++;
            else child = node_head++;
            parent[child] = nxt;
            acc += w[child];
        }
        w[nxt] = acc;
    }
    depth[total - 1] = 0;
    for (int node = total - 2; node >= 0; node--) depth[node] = depth[parent[node]] + 1;
    int mx = 0;
    for (int i = 0; i < n; i++) { depth_out[i] = (uint8_t)(depth[i] > 255 ? 255 : depth[i]); if (depth[i] > mx) mx = depth[i]; }
    return mx;
}

/* huffman.py:140-180: package-merge, literal restatement.  Each item carries
 * the multiset of leaves it contains (as per-leaf occurrence counts); packages
 * pair consecutive items (k, k+1) for even k; merge(leaves, packages) keeps
 * leaves first on equal weight; the length of a leaf is its number of
 * occurrences among the first 2n-2 items after limit-1 rounds. */
typedef struct { uint64_t w; uint16_t cnt[256]; } pm_item;
static void package_merge(const uint64_t* weights, int n, int limit, uint8_t* lengths) {
    pm_item* leaves = calloc((size_t)n, sizeof(pm_item));
    pm_item* items = calloc((size_t)2 * n, sizeof(pm_item));
    pm_item* pk = calloc((size_t)n, sizeof(pm_item));
    pm_item* nxt = calloc((size_t)2 * n, sizeof(pm_item));
    for (int i = 0; i < n; i++) { leaves[i].w = weights[i]; leaves[i].cnt[i] = 1; items[i] = leaves[i]; }
    int nitems = n;
    for (int round = 0; round < limit - 1; round++) {
        int np = 0;
        for (int k = 0; k + 1 < nitems; k += 2) {
            pk[np].w = items[k].w + items[k + 1].w;
            for (int j = 0; j < n; j++) pk[np].cnt[j] = (uint16_t)(items[k].cnt[j] + items[k + 1].cnt[j]);
            np++;
        }
        /* _merge_by_weight(leaves, packages): ties keep items from `a` (leaves) first */
        int i = 0, j = 0, o = 0;
        while (i < n && j < np) {
            if (leaves[i].w <= pk[j].w) nxt[o++] = leaves[i++];
            else nxt[o++] = pk[j++];
        }
        while (i < n) nxt[o++] = leaves[i++];
        while (j < np) nxt[o++] = pk[j++];
        pm_item* t = items; items = nxt; nxt = t;
        nitems = o;
    }
    for (int i = 0; i < n; i++) lengths[i] = 0;
    for (int k = 0; k < 2 * n - 2 && k < nitems; k++)
        for (int j = 0; j < n; j++) lengths[j] = (uint8_t)(lengths[j] + items[k].cnt[j]);
    free(leaves); free(items); free(pk); free(nxt);
}

/* huffman.py:79-103.  Returns 0, or LMCO_EMPTY for an all-zero histogram.
 * *used_pm reports whether the package-merge fallback ran. */
int lmco_build_codebook(const uint64_t counts[256], uint8_t lengths[256], int* used_pm) {
    int syms[256], n = 0;
    uint64_t total = 0;
    for (int s = 0; s < 256; s++) { total += counts[s]; if (counts[s]) syms[n++] = s; }
    memset(lengths, 0, 256);
    if (used_pm) *used_pm = 0;
    if (total == 0) return LMCO_EMPTY;
    if (n == 1) { lengths[syms[0]] = 1; return LMCO_OK; }
    /* np.lexsort((syms, counts)): ascending count, then ascending symbol.
     * Insertion sort is stable, and syms[] is already ascending. */
    for (int i = 1; i < n; i++) {
        int s = syms[i], j = i - 1;
        while (j >= 0 && counts[syms[j]] > counts[s]) { syms[j + 1] = syms[j]; j--; }
        syms[j + 1] = s;
    }
    uint64_t w[256];
    uint8_t depth[256];
    for (int i = 0; i < n; i++) w[i] = counts[syms[i]];
    int mx = huffman_depths(w, n, depth);
    if (mx > MAXLEN) {
        package_merge(w, n, MAXLEN, depth);
        if (used_pm) *used_pm = 1;
    }
    for (int i = 0; i < n; i++) lengths[syms[i]] = depth[i];
    return LMCO_OK;
}

/* huffman.py:191-210 (_validate_codebook): lengths <= 15, not empty, Kraft <= 1. */
static int validate_codebook(const uint8_t lengths[256]) {
    uint64_t units = 0;
    int any = 0;
    for (int s = 0; s < 256; s++) {
        if (lengths[s] > MAXLEN) return LMCO_CORRUPT;
        if (lengths[s]) { any = 1; units += 1u << (MAXLEN - lengths[s]); }
    }
    if (!any) return LMCO_CORRUPT;
    if (units > KRAFT_ONE) return LMCO_CORRUPT;
    return LMCO_OK;
}

/* huffman.py:183-188,213-225: canonical order is (length, symbol); each code
 * value is its cumulative Kraft offset (in 2^-15 units) shifted back down. */
int lmco_assign_canonical(const uint8_t lengths[256], uint16_t codes[256]) {
    int r = validate_codebook(lengths);
    if (r) return r;
    memset(codes, 0, 256 * sizeof(uint16_t));
    uint32_t start = 0;
    for (int len = 1; len <= MAXLEN; len++)
        for (int s = 0; s < 256; s++)
            if (lengths[s] == len) {
                codes[s] = (uint16_t)(start >> (MAXLEN - len));
                start += 1u << (MAXLEN - len);
            }
    return LMCO_OK;
}

/* huffman.py:369-371 */
uint64_t lmco_cost_bits(const uint8_t lengths[256], const uint64_t counts[256]) {
    uint64_t c = 0;
    for (int s = 0; s < 256; s++) c += (uint64_t)lengths[s] * counts[s];
    return c;
}

/* huffman.py:374-377: low nibble = even symbol. */
void lmco_pack_codebook(const uint8_t lengths[256], uint8_t wire[128]) {
    for (int i = 0; i < 128; i++) wire[i] = (uint8_t)(lengths[2 * i] | (lengths[2 * i + 1] << 4));
}
/* huffman.py:383-395 (validation included). */
int lmco_unpack_codebook(const uint8_t wire[128], uint8_t lengths[256]) {
    for (int i = 0; i < 128; i++) { lengths[2 * i] = wire[i] & 0x0F; lengths[2 * i + 1] = wire[i] >> 4; }
    return validate_codebook(lengths);
}

/* huffman.py:228-255: MSB-first packing; final byte zero-padded.  `out` must
 * hold ceil(bits/8) bytes.  Returns the bit count. */
uint64_t lmco_encode_block(const uint8_t* blk, uint64_t n, const uint8_t lengths[256],
                           const uint16_t codes[256], uint8_t* out) {
    uint64_t bitpos = 0;
    uint64_t acc = 0; int nacc = 0; /* MSB-first accumulator */
    uint64_t o = 0;
    for (uint64_t i = 0; i < n; i++) {
        int l = lengths[blk[i]];
        acc = (acc << l) | codes[blk[i]];
        nacc += l;
        bitpos += (uint64_t)l;
        while (nacc >= 8) { out[o++] = (uint8_t)(acc >> (nacc - 8)); nacc -= 8; }
    }
    if (nacc) out[o++] = (uint8_t)(acc << (8 - nacc));
    return bitpos;
}

/* huffman.py:258-349.  Sequential restatement of the pointer-doubling decoder:
 * the symbol at chain position p is read from the 15-bit window starting at p
 * (bits past the payload are zero); an unassigned window (incomplete code) or
 * any chain position at/after bit_length makes the final position differ from
 * bit_length, which is the single corruption check the reference performs. */
int lmco_decode_block(const uint8_t* data, uint64_t nbytes, uint64_t bit_length,
                      const uint8_t lengths[256], uint64_t out_len, uint8_t* out) {
    if (out_len == 0) return LMCO_OK;
    if (bit_length > nbytes * 8 || bit_length == 0) return LMCO_CORRUPT;
    if (validate_codebook(lengths)) return LMCO_CORRUPT;
    /* canonical (length, symbol) order and left-justified range ends */
    uint8_t csym[256]; uint32_t cend[256]; uint8_t clen[256]; int nc = 0;
    uint32_t start = 0;
    for (int len = 1; len <= MAXLEN; len++)
        for (int s = 0; s < 256; s++)
            if (lengths[s] == len) {
                start += 1u << (MAXLEN - len);
                csym[nc] = (uint8_t)s; clen[nc] = (uint8_t)len; cend[nc] = start; nc++;
            }
    uint64_t pos = 0;
    uint64_t nb = (bit_length + 7) / 8;
    for (uint64_t i = 0; i < out_len; i++) {
        if (pos >= bit_length) return LMCO_CORRUPT;     /* drift zone */
        uint64_t byte = pos >> 3; int r = (int)(pos & 7);
        uint32_t b0 = data[byte];
        uint32_t b1 = byte + 1 < nb ? data[byte + 1] : 0;
        uint32_t b2 = byte + 2 < nb ? data[byte + 2] : 0;
        uint32_t win = ((((b0 << 16) | (b1 << 8) | b2) << r) >> 9) & 0x7FFF;
        /* binary search for the first canonical range end > win */
        int lo = 0, hi = nc;
        while (lo < hi) { int mid = (lo + hi) >> 1; if (cend[mid] > win) hi = mid; else lo = mid + 1; }
        if (lo == nc) return LMCO_CORRUPT;               /* unassigned window */
        out[i] = csym[lo];
        pos += clen[lo];
    }
    if (pos != bit_length) return LMCO_CORRUPT;
    return LMCO_OK;
}

/* -------------------------------------------------------- byte grouping */
/* bytegroup.py:39-50 / 53-62 */
void lmco_group_bytes(const uint8_t* in, uint64_t n, int width, uint8_t* out) {
    if (width == 1) { memcpy(out, in, n); return; }
    uint64_t ne = n / (uint64_t)width;
    for (uint64_t e = 0; e < ne; e++)
        for (int g = 0; g < width; g++) out[(uint64_t)g * ne + e] = in[e * width + g];
}
void lmco_ungroup_bytes(const uint8_t* in, uint64_t n, int width, uint8_t* out) {
    if (width == 1) { memcpy(out, in, n); return; }
    uint64_t ne = n / (uint64_t)width;
    for (uint64_t e = 0; e < ne; e++)
        for (int g = 0; g < width; g++) out[e * width + g] = in[(uint64_t)g * ne + e];
}

/* ------------------------------------------------------------- records */
static void put32(uint8_t* p, uint32_t v) { p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); p[2] = (uint8_t)(v >> 16); p[3] = (uint8_t)(v >> 24); }
static void put64(uint8_t* p, uint64_t v) { put32(p, (uint32_t)v); put32(p + 4, (uint32_t)(v >> 32)); }
static uint32_t get32(const uint8_t* p) { return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24); }
static uint64_t get64(const uint8_t* p) { return (uint64_t)get32(p) | ((uint64_t)get32(p + 4) << 32); }

/* stream.py:161-177.  Writes the serialized record (mode u8 | len u32 |
 * payload) to `out` (capacity n + 5 suffices) and returns its size.  Optional
 * per-block diagnostics: mode, bit count, lengths, package-merge flag. */
uint64_t lmco_encode_record(const uint8_t* blk, uint64_t n, uint8_t* out,
                            int* mode_out, uint64_t* bits_out, uint8_t* lengths_out, int* pm_out) {
    uint64_t counts[256];
    lmco_histogram(blk, n, counts);
    uint64_t mx = 0;
    for (int s = 0; s < 256; s++) if (counts[s] > mx) mx = counts[s];
    uint8_t lengths[256];
    int pm = 0;
    if (pm_out) *pm_out = 0;
    if (mx == n) {
        out[0] = 1; put32(out + 1, (uint32_t)n); out[5] = blk[0];
        if (mode_out) *mode_out = 1;
        if (bits_out) *bits_out = 0;
        if (lengths_out) memset(lengths_out, 0, 256);
        return 6;
    }
    lmco_build_codebook(counts, lengths, &pm);
    if (pm_out) *pm_out = pm;
    if (lengths_out) memcpy(lengths_out, lengths, 256);
    uint64_t bits = lmco_cost_bits(lengths, counts);
    uint64_t hsize = HUFF_OVERHEAD + (bits + 7) / 8;
    if (bits_out) *bits_out = bits;
    if (hsize <= n) {
        uint16_t codes[256];
        lmco_assign_canonical(lengths, codes);
        out[0] = 0; put32(out + 1, (uint32_t)n);
        lmco_pack_codebook(lengths, out + 5);
        put32(out + 5 + 128, (uint32_t)bits);
        lmco_encode_block(blk, n, lengths, codes, out + 5 + HUFF_OVERHEAD);
        if (mode_out) *mode_out = 0;
        return 5 + hsize;
    }
    out[0] = 2; put32(out + 1, (uint32_t)n); memcpy(out + 5, blk, n);
    if (mode_out) *mode_out = 2;
    return 5 + n;
}

/* stream.py:271-284 */
void lmco_segment_bounds(uint64_t wlen, uint64_t block, uint32_t segs, uint64_t* edges /* segs+1 */) {
    uint64_t nblocks = (wlen + block - 1) / block;
    for (uint32_t i = 0; i < segs; i++) {
        uint64_t e = ((uint64_t)i * nblocks / segs) * block;
        edges[i] = e < wlen ? e : wlen;
    }
    edges[segs] = wlen;
}

/* entropy.py:27-37 */
static int valid_block_size(uint64_t b) { return b >= 4096 && b <= (1u << 20) && (b & (b - 1)) == 0; }

/* stream.py:287-301 */
int lmco_validate_options(int width, uint64_t block, uint32_t segs, uint64_t bufsize) {
    if (!valid_block_size(block)) return LMCO_CONFIG;
    if (segs < 1) return LMCO_CONFIG;
    if (bufsize < block) return LMCO_CONFIG;
    if (bufsize % (uint64_t)width) return LMCO_CONFIG;
    return LMCO_OK;
}

/* Upper bound of a stream (test_stream.py:106-111 generalised to windows). */
uint64_t lmco_compress_bound(uint64_t n, uint64_t block, uint32_t segs, uint64_t bufsize) {
    uint64_t nwin = (n + bufsize - 1) / bufsize;
    uint64_t blocks = 0;
    for (uint64_t w = 0; w < nwin; w++) {
        uint64_t wl = (w + 1) * bufsize <= n ? bufsize : n - w * bufsize;
        blocks += (wl + block - 1) / block;
    }
    return HDR + nwin * SEG_ENTRY * (uint64_t)segs + n + 5 * blocks;
}

/* ------------------------------------------------- parallel block workers */
typedef struct {
    const uint8_t* win; uint64_t wlen; uint64_t block;
    uint8_t* recbuf;            /* nblocks * (block+5) scratch */
    uint64_t* recsize;
    uint64_t nblocks;
    uint64_t next;              /* atomic work counter */
} enc_job;

static void* enc_worker(void* arg) {
    enc_job* j = (enc_job*)arg;
    for (;;) {
        uint64_t k = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
        if (k >= j->nblocks) break;
        uint64_t off = k * j->block;
        uint64_t n = j->wlen - off < j->block ? j->wlen - off : j->block;
        j->recsize[k] = lmco_encode_record(j->win + off, n, j->recbuf + k * (j->block + 5), 0, 0, 0, 0);
    }
    return 0;
}

static void run_workers(void* (*fn)(void*), void* job, int nthreads) {
    if (nthreads <= 1) { fn(job); return; }
    pthread_t th[256];
    if (nthreads > 256) nthreads = 256;
    for (int t = 0; t < nthreads; t++) pthread_create(&th[t], 0, fn, job);
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], 0);
}

/* stream.py:311-355 (lmc_compress).  Returns the stream length, or a negative
 * LMCO_* code.  `delta` selects FLAG_DELTA (the input is a DeltaBuffer). */
int64_t lmco_compress(const uint8_t* data, uint64_t n, int et_code, int width, int delta,
                      int byte_group, uint64_t block, uint32_t segs, uint64_t bufsize,
                      uint8_t* out, uint64_t cap, int nthreads) {
    int r = lmco_validate_options(width, block, segs, bufsize);
    if (r) return -r;
    if (n % (uint64_t)width) return -LMCO_ALIGNMENT;
    if (cap < lmco_compress_bound(n, block, segs, bufsize)) return -LMCO_CAPACITY;
    uint8_t flags = (uint8_t)((byte_group ? 1 : 0) | (delta ? 2 : 0));
    memcpy(out, "LMC1", 4); out[4] = 1; out[5] = flags; out[6] = (uint8_t)et_code; out[7] = 0;
    put64(out + 8, n); put32(out + 16, (uint32_t)block); put32(out + 20, segs);
    put32(out + 24, lmco_crc32(data, n, 0));
    uint64_t o = HDR;
    uint64_t wmax = bufsize < n ? bufsize : n;
    uint8_t* grouped = wmax ? malloc(wmax) : 0;
    uint64_t maxblocks = (wmax + block - 1) / block;
    uint8_t* recbuf = maxblocks ? malloc(maxblocks * (block + 5)) : 0;
    uint64_t* recsize = maxblocks ? malloc(maxblocks * sizeof(uint64_t)) : 0;
    uint64_t* edges = malloc(((uint64_t)segs + 1) * sizeof(uint64_t));
    if ((wmax && (!grouped || !recbuf || !recsize)) || !edges) { free(grouped); free(recbuf); free(recsize); free(edges); return -LMCO_NOMEM; }
    for (uint64_t woff = 0; woff < n; woff += bufsize) {
        uint64_t wlen = n - woff < bufsize ? n - woff : bufsize;
        const uint8_t* win = data + woff;
        if (byte_group && width > 1) { lmco_group_bytes(win, wlen, width, grouped); win = grouped; }
        enc_job job = { win, wlen, block, recbuf, recsize, (wlen + block - 1) / block, 0 };
        run_workers(enc_worker, &job, nthreads);
        lmco_segment_bounds(wlen, block, segs, edges);
        uint64_t tab = o;
        o += (uint64_t)SEG_ENTRY * segs;
        for (uint32_t s = 0; s < segs; s++) {
            uint64_t b0 = edges[s] / block, b1 = (edges[s + 1] + block - 1) / block;
            if (edges[s + 1] == edges[s]) b1 = b0;
            uint64_t comp = 0;
            for (uint64_t k = b0; k < b1; k++) {
                memcpy(out + o, recbuf + k * (block + 5), recsize[k]);
                o += recsize[k]; comp += recsize[k];
            }
            put64(out + tab + (uint64_t)s * SEG_ENTRY, edges[s + 1] - edges[s]);
            put64(out + tab + (uint64_t)s * SEG_ENTRY + 8, comp);
        }
    }
    free(grouped); free(recbuf); free(recsize); free(edges);
    return (int64_t)o;
}

/* ----------------------------------------------------------- decompress */
typedef struct { uint64_t soff; uint64_t ooff; uint32_t mode; uint32_t len; uint64_t plen; } rec_ref;

/* stream.py:114-142 */
int lmco_parse_header(const uint8_t* s, uint64_t len, int* et_code, int* width, int* flags,
                      uint64_t* orig, uint32_t* block, uint32_t* segs, uint32_t* crc) {
    if (len < HDR) return LMCO_UNSUPPORTED;
    if (memcmp(s, "LMC1", 4)) return LMCO_UNSUPPORTED;
    if (s[4] != 1) return LMCO_UNSUPPORTED;
    if (s[5] & ~3) return LMCO_CORRUPT;
    if (s[7] != 0) return LMCO_CORRUPT;
    static const int widths[4] = { 1, 2, 2, 4 };
    if (s[6] > 3) return LMCO_CORRUPT;
    *et_code = s[6]; *width = widths[s[6]]; *flags = s[5];
    *orig = get64(s + 8); *block = get32(s + 16); *segs = get32(s + 20); *crc = get32(s + 24);
    if (!valid_block_size(*block)) return LMCO_CORRUPT;
    if (*segs < 1) return LMCO_CORRUPT;
    if (*orig % (uint64_t)*width) return LMCO_CORRUPT;
    return LMCO_OK;
}

typedef struct {
    const uint8_t* s; uint8_t* out; const rec_ref* recs; uint64_t nrec; uint64_t next; int err;
} dec_job;

/* stream.py:190-215 (_decode_record) */
static int decode_record(const uint8_t* s, const rec_ref* r, uint8_t* out) {
    const uint8_t* p = s + r->soff;
    if (r->mode == 1) { memset(out, p[0], r->len); return LMCO_OK; }
    if (r->mode == 2) { memcpy(out, p, r->len); return LMCO_OK; }
    uint8_t lengths[256];
    if (lmco_unpack_codebook(p, lengths)) return LMCO_CORRUPT;
    uint64_t bits = get32(p + 128);
    return lmco_decode_block(p + HUFF_OVERHEAD, r->plen - HUFF_OVERHEAD, bits, lengths, r->len, out);
}

static void* dec_worker(void* arg) {
    dec_job* j = (dec_job*)arg;
    for (;;) {
        uint64_t k = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
        if (k >= j->nrec) break;
        if (decode_record(j->s, &j->recs[k], j->out + j->recs[k].ooff)) __atomic_store_n(&j->err, 1, __ATOMIC_RELAXED);
    }
    return 0;
}

/* stream.py:406-423 with iter_windows (358-389), decompress_segment (234-255),
 * _payload_size (258-268) and reassemble_window (392-403).  All structural
 * failures map to LMCO_CORRUPT, CRC failure to LMCO_INTEGRITY. */
int lmco_decompress(const uint8_t* s, uint64_t len, uint8_t* out, uint64_t cap,
                    uint64_t* out_len, int* et_code_out, int* flags_out, int nthreads) {
    int et, width, flags; uint64_t orig; uint32_t block, segs, crc;
    int r = lmco_parse_header(s, len, &et, &width, &flags, &orig, &block, &segs, &crc);
    if (r) return r;
    *et_code_out = et; *out_len = orig;
    if (flags_out) *flags_out = flags;
    if (cap < orig) return LMCO_CAPACITY;
    uint64_t off = HDR, remaining = orig, opos = 0;
    uint64_t table = (uint64_t)SEG_ENTRY * segs;
    uint8_t* wbuf = 0; uint64_t wcap = 0;
    rec_ref* recs = 0; uint64_t rcap = 0;
    int err = LMCO_OK;
    while (remaining > 0) {
        if (table > len - off) { err = LMCO_CORRUPT; break; }
        uint64_t wsum = 0; int bad = 0;
        for (uint32_t i = 0; i < segs; i++) {
            uint64_t o = get64(s + off + (uint64_t)i * SEG_ENTRY);
            if (o > remaining || wsum + o > remaining) bad = 1;
            else wsum += o;
        }
        uint64_t toff = off;
        off += table;
        if (bad || wsum == 0) { err = LMCO_CORRUPT; break; }
        uint64_t wlen = wsum;
        int grouped = (flags & 1) && width > 1;
        if ((flags & 1) && wlen % (uint64_t)width) { /* checked after segment decode in the reference */ }
        if (wlen > wcap) { free(wbuf); wbuf = malloc(wlen); wcap = wlen; if (!wbuf) { err = LMCO_NOMEM; break; } }
        uint8_t* dst = grouped ? wbuf : out + opos;
        uint64_t nrec = 0, wpos = 0;
        for (uint32_t i = 0; i < segs && !err; i++) {
            uint64_t so = get64(s + toff + (uint64_t)i * SEG_ENTRY);
            uint64_t sc = get64(s + toff + (uint64_t)i * SEG_ENTRY + 8);
            if (sc > len - off) { err = LMCO_CORRUPT; break; }
            if ((so == 0) != (sc == 0)) { err = LMCO_CORRUPT; break; }
            /* decompress_segment: serial record walk (header parsing only) */
            uint64_t p = 0, got = 0;
            const uint8_t* seg = s + off;
            while (got < so) {
                if (p + 5 > sc) { err = LMCO_CORRUPT; break; }
                uint32_t mode = seg[p]; uint32_t l = get32(seg + p + 1);
                p += 5;
                if (l == 0 || l > block) { err = LMCO_CORRUPT; break; }
                if (l > so - got) { err = LMCO_CORRUPT; break; }
                uint64_t plen;
                if (mode == 1) plen = 1;
                else if (mode == 2) plen = l;
                else if (mode == 0) {
                    if (p + HUFF_OVERHEAD > sc) { err = LMCO_CORRUPT; break; }
                    plen = HUFF_OVERHEAD + ((uint64_t)get32(seg + p + 128) + 7) / 8;
                } else { err = LMCO_CORRUPT; break; }
                if (plen > sc - p) { err = LMCO_CORRUPT; break; }
                if (nrec == rcap) { rcap = rcap ? rcap * 2 : 1024; rec_ref* t = realloc(recs, rcap * sizeof(rec_ref)); if (!t) { err = LMCO_NOMEM; break; } recs = t; }
                recs[nrec].soff = off + p; recs[nrec].ooff = wpos + got; recs[nrec].mode = mode;
                recs[nrec].len = l; recs[nrec].plen = plen; nrec++;
                p += plen; got += l;
            }
            if (err) break;
            if (p != sc) { err = LMCO_CORRUPT; break; }
            off += sc; wpos += so;
        }
        if (err) break;
        dec_job job = { s, dst, recs, nrec, 0, 0 };
        run_workers(dec_worker, &job, nthreads);
        if (job.err) { err = LMCO_CORRUPT; break; }
        if (flags & 1) {
            if (wlen % (uint64_t)width) { err = LMCO_CORRUPT; break; }
            if (grouped) lmco_ungroup_bytes(wbuf, wlen, width, out + opos);
        }
        opos += wlen; remaining -= wlen;
    }
    free(wbuf); free(recs);
    if (err) return err;
    if (off != len) return LMCO_CORRUPT;
    if (lmco_crc32(out, orig, 0) != crc) return LMCO_INTEGRITY;
    return LMCO_OK;
}

/* Per-block diagnostics over one grouped window: modes, bit counts, record
 * sizes, code lengths and package-merge flags (parity of kernels K2/K3). */
void lmco_analyze_blocks(const uint8_t* grouped, uint64_t wlen, uint64_t block,
                         int32_t* modes, uint64_t* bits, uint64_t* sizes, uint8_t* lengths, int32_t* pm) {
    uint8_t* tmp = malloc(block + 5);
    uint64_t nb = (wlen + block - 1) / block;
    for (uint64_t k = 0; k < nb; k++) {
        uint64_t off = k * block, n = wlen - off < block ? wlen - off : block;
        int m, p; uint64_t b;
        sizes[k] = lmco_encode_record(grouped + off, n, tmp, &m, &b, lengths + 256 * k, &p);
        modes[k] = m; bits[k] = b; pm[k] = p;
    }
    free(tmp);
}
