/*
 * bitsnap_b200.h — C-ABI of the B200-native BitSnap codec (sm_100a).
 *
 * Drop-in boundary for the reference's codec entry points
 * (/root/reference/pkg/src/bitsnap, exported from __init__.py:4-39).  The
 * reference is pure Python with no FFI; each function below replaces one
 * reference function and is what a ctypes binding in the reference package
 * would call.  Conventions:
 *
 *   - every data pointer is a DEVICE pointer; `stream` is a cudaStream_t
 *     (NULL = legacy default stream); calls are asynchronous on that stream;
 *   - the library never allocates and never synchronises: the caller passes
 *     a workspace `ws` of at least bsnp_*_ws_bytes(...) bytes;
 *   - return value: BSNP_OK or a BSNP_E_* host-side error (argument checks,
 *     launch failures).  Data-dependent errors the reference raises
 *     (DeltaError / QuantizerError) are reported through device-side status
 *     words (BSNP_ERR_* bit flags) that the host wrapper reads back and turns
 *     into the reference's exception types and messages;
 *   - element data is little-endian; F16 tensors are raw 16-bit patterns
 *     (fp16 or bf16 — the bitmask codec never interprets values).
 */
#ifndef BITSNAP_B200_H
#define BITSNAP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BSNP_ABI_VERSION 1

/* host-side return codes */
#define BSNP_OK 0
#define BSNP_E_INVALID 1   /* null pointer with n > 0, m outside [2,16], ... */
#define BSNP_E_ALIGN 2     /* element pointer not aligned to its element size */
#define BSNP_E_WORKSPACE 3 /* ws_bytes smaller than the required workspace */
#define BSNP_E_CUDA 4      /* CUDA runtime error, text in bsnp_last_error() */

/* device-side status flags (bsnp_status.err_flags) */
#define BSNP_ERR_PADDING 0x1u     /* nonzero mask padding bits (bitmask.py:128-129) */
#define BSNP_ERR_POPCOUNT 0x2u    /* popcount != changed_count  (bitmask.py:130-135) */
#define BSNP_ERR_PAYLOAD_CAP 0x4u /* encode: n_c > payload_cap (payload truncated)   */
#define BSNP_ERR_LABEL 0x8u       /* label >= m                 (quantizer.py:196-197) */
#define BSNP_ERR_NONFINITE 0x10u  /* NaN/Inf in a cluster-fit unit    */

/* 16-byte device status block written by every codec call. */
typedef struct bsnp_status {
  uint64_t count;     /* encode: n_c; decode: popcount of mask[:n]; dequant: max label */
  uint32_t err_flags; /* BSNP_ERR_* */
  uint32_t aux;       /* reserved (0) */
} bsnp_status;

int bsnp_abi_version(void);
/* Text of the last BSNP_E_CUDA error on the calling thread. */
const char* bsnp_last_error(void);
/* Number of SMs of the current device (0 if none). */
int bsnp_device_sm_count(void);
/* Page-lock / release an existing host range for DMA (cudaHostRegister):
 * the staging slot region's mapping (replaces the host memcpy of
 * reference engine.py:225-227 SlotRegion.stage).  A range that cannot be
 * registered (disk-backed mapping) returns BSNP_E_CUDA and leaves no pending
 * CUDA error. */
int bsnp_host_register(void* ptr, size_t bytes);
int bsnp_host_unregister(void* ptr);

/* ------------------------------------------------------------------------
 * Bitmask delta codec
 * ---------------------------------------------------------------------- */

/* Workspace of one encode call over n elements (tile status words plus an
 * L2-resident payload staging area of 2*n bytes rounded up to whole tiles). */
size_t bsnp_delta_encode_ws_bytes(uint64_t n);
/* Workspace of one decode call over n elements (about n/1024 bytes). */
size_t bsnp_delta_decode_ws_bytes(uint64_t n);

/*
 * Replaces bitmask.encode_delta (bitmask.py:94-111).
 *   changed[i] = base[i] != target[i] (raw 16-bit patterns)
 *   mask[ceil(n/8)]: bit (i & 7) of byte (i >> 3) = changed[i], padding 0
 *   payload[0..n_c): target[i] for changed i, ascending i
 * payload_cap bounds the payload writes; status->count = n_c always, and
 * BSNP_ERR_PAYLOAD_CAP is raised if n_c > payload_cap.
 */
int bsnp_delta_encode(const uint16_t* base, const uint16_t* target, uint64_t n,
                      uint8_t* mask, uint16_t* payload, uint64_t payload_cap,
                      bsnp_status* status, void* ws, size_t ws_bytes, void* stream);

/*
 * Replaces bitmask.decode_delta (bitmask.py:114-140).
 *   out[i] = changed[i] ? payload[rank(i)] : base[i]
 * out may equal base (in-place chain replay, store.py:441-454): the mask is
 * validated by a separate pre-pass first so that base is left untouched when
 * BSNP_ERR_PADDING / BSNP_ERR_POPCOUNT is raised.  Out of place, the decode
 * does not wait for the validation: `out` is undefined when a flag is raised.
 */
int bsnp_delta_decode(const uint16_t* base, const uint8_t* mask, const uint16_t* payload,
                      uint64_t n, uint64_t n_c, uint16_t* out, bsnp_status* status,
                      void* ws, size_t ws_bytes, void* stream);

/*
 * bsnp_delta_decode out of place with n_c read ON THE DEVICE from n_c_dev
 * (e.g. &encode_status->count): an encode and the decode of its record run
 * back to back with no host round trip.  payload holds the record's n_c
 * elements; base, out and mask 16-byte aligned; out != base.  Same flags
 * and status->count as bsnp_delta_decode.
 */
int bsnp_delta_decode_dn(const uint16_t* base, const uint8_t* mask, const uint16_t* payload,
                         uint64_t n, const uint64_t* n_c_dev, uint16_t* out,
                         bsnp_status* status, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Cluster quantizer (reference quantizer.py:100-204)
 *
 * A "unit" is the slice that gets its own ClusterTable: the whole tensor when
 * block == 0 (the reference's per-tensor behaviour, store.py:261-263) or
 * consecutive `block`-element slices (block % 8 == 0; the last slice may be
 * shorter), the per-block mode of BASELINE configs[2] whose oracle is the
 * reference applied to each slice.  Units are laid out back to back:
 *   tables[u]                  one bsnp_cluster_table per unit
 *   labels  + u * block / 2    packed 4-bit labels of unit u (ceil(len/2) B,
 *                              low nibble = even index, quantizer.py:146-150)
 *   codes   + u * block        one u8 code per element
 * ---------------------------------------------------------------------- */

/* ClusterTable (quantizer.py:45-65) in device memory, 256 bytes. */
typedef struct bsnp_cluster_table {
  float mean;            /* f32(mean), quantizer.py:350, 368 */
  float std;             /* f32(std),  quantizer.py:351, 369 */
  float boundaries[15];  /* m-1 used: f32(mu + std * ndtri(k/m)) */
  float scales[16];      /* m used: f32(max - min) per cluster, 0 if empty */
  float offsets[16];     /* m used: f32(min) per cluster, 0 if empty */
  uint32_t m;            /* clusters, 2..16 */
  uint32_t flags;        /* BSNP_ERR_NONFINITE if the unit had NaN/Inf statistics */
  uint32_t reserved[13];
} bsnp_cluster_table;

/* Workspace of a fit / quantize / dequantize call over n elements. */
size_t bsnp_cluster_ws_bytes(uint64_t n, uint64_t block);

/*
 * Replaces build_clusters (quantizer.py:100-135) for every unit: mean/std in
 * float64 with numpy's pairwise summation tree reproduced exactly, normal-
 * quantile boundaries, per-cluster min/max with fit-time labels taken against
 * the unrounded float64 boundaries.  Bit-identical tables.
 */
int bsnp_cluster_fit(const float* x, uint64_t n, uint64_t block, int m,
                     bsnp_cluster_table* tables, void* ws, size_t ws_bytes, void* stream);

/*
 * Replaces quantize (quantizer.py:161-189) for every unit with the given
 * tables: label = #(boundaries < v), code = ceil(clip((v-b)/S,0,1)*255 - 0.5)
 * evaluated exactly as the reference's float64 expression.
 */
int bsnp_cluster_quantize(const float* x, uint64_t n, uint64_t block,
                          const bsnp_cluster_table* tables, uint8_t* labels, uint8_t* codes,
                          void* ws, size_t ws_bytes, void* stream);

/* fit + quantize in one call (the store's optimizer-state path). */
int bsnp_cluster_encode(const float* x, uint64_t n, uint64_t block, int m,
                        bsnp_cluster_table* tables, uint8_t* labels, uint8_t* codes,
                        void* ws, size_t ws_bytes, void* stream);

/*
 * Replaces dequantize (quantizer.py:192-204): out = f32(f64(code)/255 * S + b).
 * status->count = largest label seen; BSNP_ERR_LABEL if it is >= m.
 */
int bsnp_cluster_dequantize(const uint8_t* labels, const uint8_t* codes, uint64_t n,
                            uint64_t block, const bsnp_cluster_table* tables, float* out,
                            bsnp_status* status, void* ws, size_t ws_bytes, void* stream);

/* One per-tensor (block 0) quantized state of a restore batch. */
typedef struct bsnp_dequant_item {
  const uint8_t* labels;            /* (n + 1) / 2 bytes */
  const uint8_t* codes;             /* n bytes */
  const bsnp_cluster_table* table;  /* 16-byte aligned */
  float* out;                       /* n floats, 4-byte aligned */
  uint64_t n;
} bsnp_dequant_item;

/* Elements per CTA of bsnp_cluster_dequantize_batch. */
#define BSNP_DEQUANT_CHUNK 65536u

/*
 * The restore loop's per-record dequantize (store.py:458-468 calls
 * quantizer.dequantize once per optimizer record) for many records in one
 * launch.  items / first / status live in device memory: first[i] is the
 * index of item i's first BSNP_DEQUANT_CHUNK chunk, nchunks = first[nitems];
 * status[i] is item i's bsnp_cluster_dequantize status (zeroed here).
 */
int bsnp_cluster_dequantize_batch(const bsnp_dequant_item* items, const uint32_t* first,
                                  uint32_t nitems, uint32_t nchunks, bsnp_status* status,
                                  void* stream);

/*
 * n bytes from device memory to page-locked host memory (dst: a pinned or
 * registered host address, device-accessible under unified addressing) by
 * SM stores, not a copy engine: the encoder's status words and cluster
 * tables come back without queueing behind the bulk device-to-host copies
 * of earlier record groups (store.py:240-270 reads them synchronously).
 */
int bsnp_copy_sm(const void* src, void* dst, uint64_t n, void* stream);

/* ------------------------------------------------------------------------
 * Checkpoint blob assembly
 * ---------------------------------------------------------------------- */

/* len bytes from device address src to blob + dst_off */
typedef struct bsnp_segment {
  const void* src;
  uint64_t dst_off;
  uint64_t len;
} bsnp_segment;

/* Chunk size of bsnp_gather_segments (bytes per CTA). */
#define BSNP_GATHER_CHUNK 65536u

/*
 * Assembles tensors.bin in device memory: every record's header and bodies
 * at its store offset (store.py:240-270 writes them one by one into a host
 * buffer).  segs / first live in device memory; first[s] is the index of
 * segment s's first BSNP_GATHER_CHUNK chunk and nchunks = first[nsegs] (the
 * chunk total, passed by value so the launch needs no read-back).  The blob
 * then leaves HBM in a single device-to-host copy.
 */
int bsnp_gather_segments(const bsnp_segment* segs, const uint32_t* first, uint32_t nsegs,
                         uint32_t nchunks, uint8_t* blob, void* stream);

/*
 * Reduction behind precision_report (quantizer.py:280-296): acc3 receives
 * (sum (o-r)^2, sum |o-r|/|o| over |o| > 1e-12, count of those o) in float64.
 * Deterministic: a fixed partition of [0, n) into kPrecParts contiguous
 * ranges (independent of the GPU), each reduced in a fixed order into the
 * workspace, then one fixed tree over the partials - the same bits on every
 * run.  ws: bsnp_precision_ws_bytes() bytes of device memory.
 */
size_t bsnp_precision_ws_bytes(void);
int bsnp_precision_report(const float* original, const float* restored, uint64_t n,
                          double* acc3, void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BITSNAP_B200_H */
