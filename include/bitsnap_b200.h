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
 * BSNP_ERR_PADDING / BSNP_ERR_POPCOUNT is raised.  Out-of-place decode is a
 * single pass; its `out` is undefined when a flag is raised.
 */
int bsnp_delta_decode(const uint16_t* base, const uint8_t* mask, const uint16_t* payload,
                      uint64_t n, uint64_t n_c, uint16_t* out, bsnp_status* status,
                      void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BITSNAP_B200_H */
