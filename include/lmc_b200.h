/*
 * lmc_b200.h -- C-ABI of the B200-native LMC hot path (liblmc_b200.so).
 *
 * Drop-in boundary for the reference package `lmc` 0.1.0 (pure Python).  Each
 * entry point below replaces one reference interface; the ctypes binding a
 * maintainer would add to the reference is shown in INTEGRATION.md.
 *
 *   lmcg_compress / lmcg_compress_host
 *       <- lmc.stream.lmc_compress          (pkg/src/lmc/stream.py:311-341)
 *       <- lmc.parallel.plmc_compress       (pkg/src/lmc/parallel.py:53-103)
 *   lmcg_decompress (+ lmcg_read_hints, lmcg_decompress_result) / lmcg_decompress_host
 *       <- lmc.stream.lmc_decompress        (pkg/src/lmc/stream.py:406-423)
 *       <- lmc.parallel.plmc_decompress     (pkg/src/lmc/parallel.py:106-128)
 *   lmcg_decompress_apply
 *       <- lmc.delta.xor_apply(prev, lmc_decompress(delta stream))
 *          (pkg/src/lmc/delta.py:50-52, as lmc.chain.restore_step uses it,
 *          pkg/src/lmc/chain.py:293-300), fused into the decode
 *   lmcg_validate_options
 *       <- lmc.stream._validate_options     (pkg/src/lmc/stream.py:287-301)
 *   lmcg_build_codebooks
 *       <- lmc.huffman.build_codebook       (pkg/src/lmc/huffman.py:79-180), batched
 *   lmcg_block_info
 *       per-block (mode, bit count, record size, lengths) of the last compress:
 *       the values lmc.stream._encode_record (stream.py:161-177) derives.
 *
 * Status codes map 1:1 onto the reference exception classes
 * (pkg/src/lmc/errors.py:8-53); see LMCG_* below.  All device pointers are
 * plain CUDA device addresses (PyTorch-owned in the Python front-end); the
 * `cuda_stream` arguments are cudaStream_t values (0 = legacy default).
 * Functions are reentrant per context; one context must not be used by two
 * host threads at once.  There is no CPU fallback: without a CUDA device every
 * compute entry point returns LMCG_ERR_CUDA.
 */
#ifndef LMC_B200_H
#define LMC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -> reference exception classes (errors.py) */
#define LMCG_OK 0
#define LMCG_ERR_UNSUPPORTED 1        /* UnsupportedFormatError (magic/version/short) */
#define LMCG_ERR_CORRUPT 2            /* CorruptStreamError (any structural failure)  */
#define LMCG_ERR_INTEGRITY 3          /* IntegrityError (payload CRC mismatch)        */
#define LMCG_ERR_CONFIG 4             /* ConfigError (block/segment/buffer options)   */
#define LMCG_ERR_ALIGNMENT 5          /* AlignmentError (length % element width)      */
#define LMCG_ERR_EMPTY 6              /* EmptyInputError (empty histogram)            */
#define LMCG_ERR_CUDA 7               /* no device / CUDA runtime failure             */
#define LMCG_ERR_CAPACITY 8           /* caller buffer too small                      */
#define LMCG_ERR_ARGUMENT 9           /* bad argument (NULL pointer, n < 0, ...)      */
#define LMCG_ERR_RETRY 10             /* decompress hints too small: call again        */
#define LMCG_ERR_SHAPE 11             /* ShapeMismatchError (xor_apply length mismatch) */

/* ElementType wire codes (types.py:24-27) */
#define LMCG_RAW8 0
#define LMCG_BF16 1
#define LMCG_FP16 2
#define LMCG_FP32 3

typedef struct lmcg_ctx lmcg_ctx;

/* One tensor to compress.  `data` (and `prev`) are device pointers. */
typedef struct {
    const void* data;      /* payload bytes, or the NEXT step when prev != NULL         */
    const void* prev;      /* previous step: fused XOR delta (delta.py:18-47), or NULL  */
    uint64_t nbytes;       /* payload length in bytes                                   */
    int32_t element_type;  /* LMCG_RAW8 .. LMCG_FP32                                    */
    int32_t delta;         /* nonzero: header FLAG_DELTA (a DeltaBuffer input)          */
} lmcg_tensor;

/* lmc_compress keyword options (stream.py:311-318). */
typedef struct {
    int32_t byte_group;      /* FLAG_BYTE_GROUPED                          */
    uint32_t block_size;     /* power of two in [4096, 1048576]            */
    uint32_t segment_count;  /* >= 1                                       */
    uint32_t reserved;       /* must be 0                                  */
    uint64_t buffer_size;    /* window bytes, >= block_size, % width == 0  */
} lmcg_options;

lmcg_ctx* lmcg_create(int device);
void lmcg_destroy(lmcg_ctx* ctx);
const char* lmcg_last_error(lmcg_ctx* ctx);
int lmcg_version(void); /* stream format version written (1) */

/* stream.py:287-301 plus the TensorBuffer alignment check (types.py:85-90). */
int lmcg_validate_options(const lmcg_options* opts, int element_type, uint64_t nbytes);

/* Exact upper bound of the packed output of lmcg_compress for these tensors. */
uint64_t lmcg_compress_bound(const lmcg_tensor* tensors, int n, const lmcg_options* opts);
/* Device scratch needed by lmcg_compress (pass 0/NULL workspace to let the
 * context allocate and cache it). */
uint64_t lmcg_compress_workspace(const lmcg_tensor* tensors, int n, const lmcg_options* opts);

/* Compress n tensors into n independent LMC1 streams packed back to back in
 * d_out.  d_offsets / d_lengths (device, n x u64) receive each stream's start
 * and length inside d_out.  Asynchronous on cuda_stream; no host sync. */
int lmcg_compress(lmcg_ctx* ctx, const lmcg_tensor* tensors, int n, const lmcg_options* opts,
                  void* d_out, uint64_t out_capacity, uint64_t* d_offsets, uint64_t* d_lengths,
                  void* d_workspace, uint64_t workspace_bytes, void* cuda_stream);

/* What the caller knows about a stream before decoding it: the header's
 * original_length / segment_count / block_size and, if known, the number of
 * windows (0 = assume the default 128 MiB buffer).  Used only to size the
 * device work areas; a wrong hint costs a retry, never a wrong result. */
typedef struct {
    uint64_t orig;
    uint32_t segments;
    uint32_t block;
    uint64_t windows;
} lmcg_stream_hint;

/* One part of a stream compressed on several GPUs (a tensor
 * larger than a rank's fair share is split by block range).  The records of
 * blocks [blk_begin, blk_end) of the tensor's stream (global record order:
 * windows in turn, each window's blocks in grouped order) are written back to
 * back into d_out and their sizes into d_rec_sizes (u32 each); the raw CRC-32
 * (no pre/post inversion) of the element bytes [crc_begin, crc_end) of the
 * payload (XOR delta applied) goes to *d_crc.  With every rank's sizes and
 * CRCs all-gathered, paper_2505_09810_b200.shard assembles the 28-byte header
 * (CRC combined), the segment tables (stream.py:271-284, 344-355) and the
 * records into the stream lmcg_compress writes, byte for byte.  Same
 * compression path as lmcg_compress (stream.py:161-187, huffman.py:79-255). */
int lmcg_compress_part(lmcg_ctx* ctx, const lmcg_tensor* tensor, const lmcg_options* opts, uint64_t blk_begin,
                       uint64_t blk_end, void* d_out, uint64_t out_capacity, uint32_t* d_rec_sizes, uint64_t crc_begin,
                       uint64_t crc_end, uint32_t* d_crc, void* cuda_stream);

/* Exact hints for n device streams: validates headers and segment tables on
 * the device (nothing is decoded) and reports their structure (synchronises).
 * Streams the walk rejects get all-zero hints; lmcg_decompress then reports
 * their error. */
int lmcg_read_hints(lmcg_ctx* ctx, const void* const* d_streams, const uint64_t* stream_lengths, int n,
                    lmcg_stream_hint* hints, void* cuda_stream);

/* Decompress n device-resident streams (stream.py:406-423 semantics, all
 * validation of stream.py:114-142, 234-268, 358-389 on the device).  Stream
 * i's payload goes to d_out + h_out_offsets[i] (or, when h_out_offsets is
 * NULL, packed at 16-byte aligned offsets in stream order).  Asynchronous:
 * no host synchronisation; read the outcome with lmcg_decompress_result. */
int lmcg_decompress(lmcg_ctx* ctx, const void* const* d_streams, const uint64_t* stream_lengths, int n,
                    const lmcg_stream_hint* hints, void* d_out, uint64_t out_capacity,
                    const uint64_t* h_out_offsets, void* cuda_stream);

/* lmcg_decompress followed by xor_apply (delta.py:50-52): stream i's payload
 * is XORed with the prev_lengths[i] bytes at d_prev[i] on its way out, so
 * d_out + offset receives prev ^ payload (the next checkpoint step when the
 * stream holds the XOR delta against prev).  d_prev[i] may be the output
 * location itself (in-place restore of a resident step) and may be NULL (plain
 * decode of that stream).  The CRC check is on the payload, as in the
 * reference; a payload whose length differs from prev_lengths[i] is reported
 * as LMCG_ERR_SHAPE (xor_bytes, delta.py:20-21) after the decode's own
 * errors, and nothing is XORed.  On any error the output bytes of that stream
 * are unspecified (with d_prev[i] == output, the prev bytes are lost). */
int lmcg_decompress_apply(lmcg_ctx* ctx, const void* const* d_streams, const uint64_t* stream_lengths, int n,
                          const lmcg_stream_hint* hints, const void* const* d_prev, const uint64_t* prev_lengths,
                          void* d_out, uint64_t out_capacity, const uint64_t* h_out_offsets, void* cuda_stream);

/* Synchronise and report the last lmcg_decompress per stream: status
 * (LMCG_OK / UNSUPPORTED / CORRUPT / INTEGRITY / SHAPE, or LMCG_ERR_RETRY /
 * LMCG_ERR_CAPACITY when the hints were too small), original length, element
 * type, flags and window count.  Any pointer may be NULL. */
int lmcg_decompress_result(lmcg_ctx* ctx, int n, int32_t* h_status, uint64_t* h_orig_lengths,
                           int32_t* h_element_types, int32_t* h_flags, uint64_t* h_windows);

/* Plans: everything that depends only on shapes/options is validated, laid
 * out and uploaded once; a run only launches kernels (no host synchronisation,
 * no allocation), so runs can be captured in a CUDA graph and replayed for
 * every checkpoint of the same model.
 *
 * Compress plan: the tensors' device addresses and sizes are fixed; each run
 * compresses their current contents (identical bytes to lmcg_compress). */
typedef struct lmcg_plan lmcg_plan;
lmcg_plan* lmcg_compress_plan_create(lmcg_ctx* ctx, const lmcg_tensor* tensors, int n, const lmcg_options* opts);
int lmcg_compress_plan_run(lmcg_ctx* ctx, lmcg_plan* plan, void* d_out, uint64_t out_capacity, uint64_t* d_offsets,
                           uint64_t* d_lengths, void* cuda_stream);
/* Decompress plan for n streams whose structure the hints describe exactly
 * (e.g. those of a compress plan) and whose lengths never exceed len_bounds.
 * Each run decodes the streams found at d_base + d_offsets[i] (device arrays,
 * e.g. the output of lmcg_compress_plan_run) into d_out at 16-byte aligned
 * packed offsets, and writes per-stream LMCG_* codes to d_status (device). */
lmcg_plan* lmcg_decompress_plan_create(lmcg_ctx* ctx, int n, const lmcg_stream_hint* hints, const uint64_t* len_bounds);
int lmcg_decompress_plan_run(lmcg_ctx* ctx, lmcg_plan* plan, const void* d_base, const uint64_t* d_offsets,
                             const uint64_t* d_lengths, void* d_out, int32_t* d_status, void* cuda_stream);
/* SM-driven copy of a few bytes (e.g. a plan's stream offsets / lengths) into
 * page-locked host memory, ordered on cuda_stream: unlike cudaMemcpyAsync it
 * is not queued behind bulk transfers on the copy engines, so the host can
 * learn the stream sizes while large copies are in flight.  h_dst must be
 * pinned (cudaHostAlloc / torch pin_memory). */
int lmcg_copy_to_host(void* h_dst, const void* d_src, uint64_t bytes, void* cuda_stream);

/* Diagnostics: segments decoded by the serial fallback walk (stream.py:234-268
 * restated on the device) since the last reset, across all contexts of the
 * process (synchronises the device).  Well-formed streams stay on the
 * parallel path; corrupt ones end there to report the reference's error. */
uint64_t lmcg_fallback_segments(int reset);

/* Output bytes a run needs: compress bound / decompressed payload bytes. */
uint64_t lmcg_plan_output_bytes(const lmcg_plan* plan);
void lmcg_plan_destroy(lmcg_plan* plan);

/* Host-buffer conveniences (the call a ctypes binding in lmc.stream makes):
 * host -> device copy, the GPU path above, device -> host copy. */
int lmcg_compress_host(lmcg_ctx* ctx, const void* data, uint64_t nbytes, int element_type, int delta,
                       const lmcg_options* opts, void* out, uint64_t out_capacity, uint64_t* out_len);
int lmcg_decompress_host(lmcg_ctx* ctx, const void* stream, uint64_t len, void* out, uint64_t out_capacity,
                         uint64_t* out_len, int32_t* element_type, int32_t* flags);

/* Stage level: code lengths for nhist 256-bin histograms (device u32 [nhist][256]
 * -> device u8 [nhist][256]); identical to build_codebook including the
 * package-merge fallback and its tie rules.  Empty histograms yield all zeros
 * and LMCG_ERR_EMPTY. */
int lmcg_build_codebooks(lmcg_ctx* ctx, const uint32_t* d_hists, int nhist, uint8_t* d_lengths,
                         void* cuda_stream);

/* Per-block diagnostics of the most recent lmcg_compress on this context, in
 * global block order (streams, then windows, then blocks).  Host arrays of
 * capacity `cap` blocks; any pointer may be NULL.  Returns the block count. */
int64_t lmcg_block_info(lmcg_ctx* ctx, int32_t* modes, uint32_t* bits, uint32_t* record_sizes,
                        uint8_t* codebook_wire /* cap x 128 */, uint32_t* pm_flags, int64_t cap);

/* Decode fusion switch (default on from 16384 record slots; environment
 * LMCG_NOFUSE=1 / LMCG_FUSE_FROM=n set the defaults of a new context).  On:
 * in decodes of at least min_records record slots, two-plane windows with 16-64 KiB blocks are
 * decoded, byte-interleaved and CRC-checked in one pass (k_decpair) instead
 * of decode -> grouped scratch -> k_ungroup.  Output and errors are identical
 * either way; the switch exists so the tests exercise both paths. */
int lmcg_set_decode_fusion(lmcg_ctx* ctx, int enable, uint64_t min_records);

/* Measurement hooks (bench.py): bracket every kernel launch with CUDA events
 * while enabled; lmcg_profile_report synchronises, writes lines
 * "<kernel> <launches> <total_ms>" into buf, clears the counters and returns
 * the report length. */
int lmcg_profile(lmcg_ctx* ctx, int enable);
int64_t lmcg_profile_report(lmcg_ctx* ctx, char* buf, uint64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* LMC_B200_H */
