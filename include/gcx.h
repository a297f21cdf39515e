/*
 * gcx.h — C-ABI of the B200-native compressed-allreduce hot path
 * (libgcx.so, sm_100a).  Plain pointers and sizes only: no torch or C++
 * types cross this boundary.  Every launcher is asynchronous on the given
 * CUDA stream (passed as void*; NULL = legacy default stream), never
 * allocates, and returns 0 on success or a negative GCX_E* code with a
 * message in gcx_last_error() (thread-local).
 *
 * Reference interfaces replaced (paths under /root/reference/proj):
 *   gcx_quantize        codec::quantize        src/codec.cpp:24-69,  include/gcomm/codec.hpp:50
 *   gcx_dequantize      codec::dequantize      src/codec.cpp:71-95,  include/gcomm/codec.hpp:51
 *   gcx_compressed_size codec::compressed_size_bytes src/codec.cpp:151-156
 *   gcx_encode_pieces   encode_pieces (quantize+serialize per piece)  src/collectives.cpp:143-163
 *   gcx_decode_pieces   decode_pieces (+ finalize's average)          src/collectives.cpp:165-194, :213-228
 *   gcx_fold_pieces     run_sra owner fold (ascending id, own raw)   src/collectives.cpp:258-279
 *   gcx_sra_reduce      run_sra owner step: fold, hop-1 re-encode,
 *                       owner decodes its own bytes                  src/collectives.cpp:258-292
 *   gcx_hop_seed        collectives::hop_seed  src/collectives.cpp:29-31
 *   gcx_uniform01       uniform01              include/gcomm/util.hpp:26-29
 *
 * Device payload layout ("message"): a list of pieces, each at a 16-byte
 * aligned byte offset chosen by the caller.  A quantized piece stores
 * ceil(len/bucket) f32 norms at `norms` and the (bits+1)-bit LSB-first
 * packed stream (byte-identical to codec::pack_levels) at `packed`; a raw
 * piece stores len f32 at `norms` (`packed` unused).  The reference's
 * 17-byte wire header is not materialised on device: every rank derives the
 * layout from the segment table, so headers would carry no information.
 */
#ifndef GCX_H_
#define GCX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GCX_OK 0
#define GCX_E_INVALID (-1)   /* bad parameter (reference: std::invalid_argument) */
#define GCX_E_CUDA (-2)      /* CUDA launch/runtime failure */
#define GCX_E_RANGE (-3)     /* payload too short (reference: std::runtime_error) */

/* launch flags (from gcx_plan_tiles) */
#define GCX_F_BIG_BUCKETS 1u   /* some piece has bucket > GCX_TILE: norm pre-pass */
#define GCX_F_NEEDS_ZERO 2u    /* some piece's tiles share packed words: zero first */
#define GCX_F_PIECE_SEEDS 4u   /* use gcx_piece.seed instead of the launch seed */
#define GCX_F_ODD_BUCKETS 8u   /* some quantized piece has bucket % 32 != 0: generic K1b */
#define GCX_F_NORM_PASS 16u    /* some piece's norms come from the K1a pre-pass (bucket not 32/64/128) */
#define GCX_F_LANE_GROUP 32u   /* some piece has bucket % 32 == 0 other than 32/64/128 (k_quant32) */
#define GCX_F_KEY_PREFIX 64u   /* the key table holds seed-independent prefixes (gcx_make_prefix) */
#define GCX_F_SPAN_DEC 128u    /* every piece is raw or quantized with a power-of-two bucket in
                                  [128, 4096]: the span decode serves the table */
#define GCX_F_SPAN_ENC 256u    /* every quantized piece has the same bits and bucket, bucket in
                                  {32, 64, 128}: the span K1 serves the table; its key runs use
                                  the span key layout (gcx_plan_keys) */
#define GCX_F_SPAN_DEC_WIDE 512u /* with GCX_F_SPAN_DEC: some piece has bits 5..8 (per-element
                                   values instead of shuffle tables) */
#define GCX_F_SEED_DEVICE 1024u /* the launch `seed` argument carries the device address of
                                   a uint64 seed written earlier on the stream
                                   (gcx_sra_step_seeds): a step captured in a CUDA graph
                                   replays with fresh seeds.  Span tables only
                                   (GCX_F_SPAN_ENC); other tables are rejected. */
#define GCX_F_SPAN_BITS_SHIFT 16 /* with GCX_F_SPAN_ENC: bits at flags[16..19], */
#define GCX_F_SPAN_LGB_SHIFT 20  /* log2(bucket) at flags[20..23] */

#define GCX_TILE 4096          /* max elements per CTA tile */

/* One maximal run of a chunk with one codec (collectives.cpp:69-75 Piece). */
typedef struct gcx_piece {
  uint64_t src;    /* element offset of the piece in the float buffer it reads/writes */
  uint64_t len;    /* elements */
  uint64_t norms;  /* byte offset (from the message base) of the norms / raw f32 payload */
  uint64_t packed; /* byte offset (from the message base) of the packed stream */
  uint64_t seed;   /* per-piece seed (only with GCX_F_PIECE_SEEDS) */
  uint32_t bucket; /* bucket size (quantized pieces) */
  int32_t bits;    /* 1..8 magnitude bits; 0 = raw f32 (CodecMode::uncompressed) */
  uint64_t keys;   /* element offset of this piece's run in a key table
                      (gcx_plan_keys), or UINT64_MAX: draw keys inline */
} gcx_piece;

/* One run of a key table: slot off + i holds the uniform01 key of piece-local
 * index i (< len) for bucket size `bucket` (util.hpp:26-29 before the >> 11).
 * Runs start on multiples of 1024 slots; a table of `total` slots occupies
 * total * 8 bytes, laid out for coalesced reads by the quantizer (the high
 * and low key words of each 1024-slot block are stored apart, gcx_kernels.cu
 * key_pos). */
typedef struct gcx_keygroup {
  uint64_t off;
  uint64_t len;
  uint32_t bucket;
  uint32_t pad;
} gcx_keygroup;

int gcx_version(void);
const char* gcx_last_error(void);

/* ---- host-side sizing / planning (no GPU needed) ---- */
uint64_t gcx_compressed_size(uint64_t n, int bits, uint64_t bucket);
uint64_t gcx_packed_bytes(uint64_t n, int bits);    /* ceil(n*(bits+1)/8) */
uint64_t gcx_packed_capacity(uint64_t n, int bits); /* rounded up to whole 32-bit words */
uint64_t gcx_hop_seed(uint64_t step_seed, uint64_t hop, uint64_t node);
double gcx_uniform01(uint64_t seed, uint64_t a, uint64_t b);
/* Tile decomposition of a piece table: tile_prefix[npieces+1] (first tile of
 * each piece, total last) and launch flags.  Returns total tiles or <0. */
int64_t gcx_plan_tiles(const gcx_piece* pieces, uint32_t npieces, uint32_t* tile_prefix,
                       uint32_t* flags);

/* ---- single vector codec ----
 * norms: ceil(n/bucket) f32; packed: gcx_packed_capacity(n,bits) bytes.
 * bad_key (device u64, may be NULL): atomic-min of the first non-finite input
 * index; caller presets it to UINT64_MAX and checks it after the stream syncs
 * (reference message: "non-finite gradient value at index i"). */
int gcx_quantize(const float* x, uint64_t n, int bits, uint64_t bucket, uint64_t seed,
                 float* norms, uint8_t* packed, unsigned long long* bad_key, void* stream);
int gcx_dequantize(const float* norms, const uint8_t* packed, uint64_t n, int bits,
                   uint64_t bucket, float* out, void* stream);
/* Key prefixes: the reference keys every draw as uniform01(seed, b, i) =
 * mix64(seed ^ T(i)) >> 11 with T(i) = mix64(b ^ mix64(i)), b = i / bucket
 * (util.hpp:26-29).  T depends only on (i, bucket), so a caller that
 * quantizes same-shaped buffers every step (a gradient buffer) builds the
 * table once and each step hashes one finalizer per element instead of
 * three.  table: gcx_prefix_slots(n) entries of 8 bytes (laid out like a key
 * table).  gcx_quantize_prefixed == gcx_quantize bit for bit. */
uint64_t gcx_prefix_slots(uint64_t n);
int gcx_make_prefix(uint64_t n, uint64_t bucket, unsigned long long* table, void* stream);
int gcx_quantize_prefixed(const float* x, uint64_t n, int bits, uint64_t bucket, uint64_t seed,
                          const unsigned long long* prefix, float* norms, uint8_t* packed,
                          unsigned long long* bad_key, void* stream);

/* ---- piece-table codec (device tables; tile_prefix from gcx_plan_tiles) ----
 * encode: src + pieces[k].src ... -> msg + pieces[k].norms/packed.  Raw pieces
 *         are copied.  bad_key = (piece << 40) | piece-local index.  keys: a
 *         key table made by gcx_make_keys for this seed (or NULL: inline).
 * decode: msg -> dst + pieces[k].src, each value divided by `divisor` when
 *         divisor != 1 (IEEE f32 division, finalize() average).  flags from
 *         gcx_plan_tiles (GCX_F_ODD_BUCKETS selects the generic kernel too). */
int gcx_encode_pieces(const gcx_piece* pieces, const uint32_t* tile_prefix, uint32_t npieces,
                      uint32_t ntiles, uint32_t flags, uint64_t seed, const float* src,
                      uint8_t* msg, const unsigned long long* keys,
                      unsigned long long* bad_key, void* stream);
/* Key tables for a piece table quantized under ONE seed (SRA stage 1 uses
 * one seed for every piece of a sender's hop, collectives.cpp:252-253; the
 * owner's re-encode one seed for its whole chunk): pieces of one bucket size
 * draw the same key at the same piece-local index (codec.cpp:60), so one run
 * per bucket size, as long as its longest piece, serves them all.
 * plan_keys sets pieces[k].keys, fills groups[], returns the table length. */
int64_t gcx_plan_keys(gcx_piece* pieces, uint32_t npieces, gcx_keygroup* groups,
                      uint32_t group_cap, uint32_t* ngroups);
/* Same, choosing the key-table layout: GCX_KEYS_AUTO = the span layout when
 * the table qualifies for the span K1 (GCX_F_SPAN_ENC), GCX_KEYS_LANE_GROUP =
 * always the lane-group layout (the caller then clears GCX_F_SPAN_ENC from the
 * table's flags, so the lane-group K1 kernels read it). */
#define GCX_KEYS_AUTO 0
#define GCX_KEYS_LANE_GROUP 1
int64_t gcx_plan_keys_layout(gcx_piece* pieces, uint32_t npieces, gcx_keygroup* groups,
                             uint32_t group_cap, uint32_t* ngroups, int layout);
int gcx_make_keys(const gcx_keygroup* groups, uint32_t ngroups, uint64_t total, uint64_t seed,
                  unsigned long long* keys, void* stream);
/* The same table in two steps for layouts that are reused every step (an
 * SRA reducer): make_key_prefix stores the seed-independent T(slot) once;
 * make_keys_prefixed then derives the step's keys with one finalizer per
 * slot (key = mix64(seed ^ T), util.hpp:26-29).  Identical keys. */
int gcx_make_key_prefix(const gcx_keygroup* groups, uint32_t ngroups, uint64_t total,
                        unsigned long long* prefix, void* stream);
int gcx_make_keys_prefixed(uint64_t total, uint64_t seed, const unsigned long long* prefix,
                           unsigned long long* keys, void* stream);
/* make_keys_prefixed with the seed read from device memory (*seed_dev) */
int gcx_make_keys_prefixed_dev(uint64_t total, const unsigned long long* seed_dev,
                               const unsigned long long* prefix, unsigned long long* keys,
                               void* stream);
/* Per-step SRA seeds on the device (a graph-replayable step): state[0] =
 * base seed, state[1] = step, state[2] = buffer index, state[3] = node id.
 * Writes state[4] = hop_seed(S, 0, node), state[5] = hop_seed(S, 1, node)
 * with S = hash_combine(hash_combine(base, step), buffer) (engine.cpp:208-209,
 * collectives.cpp:252-253, :283), then state[1] = step + 1. */
int gcx_sra_step_seeds(unsigned long long* state, void* stream);
int gcx_decode_pieces(const gcx_piece* pieces, const uint32_t* tile_prefix, uint32_t npieces,
                      uint32_t ntiles, uint32_t flags, const uint8_t* msg, float* dst,
                      float divisor, void* stream);

/* ---- SRA owner step ----
 * fold: the contribution of node id is `own` when id == me, else the message
 * in recv slot (id < me ? id : id-1) at recv + slot*slot_stride; folds
 * ascending id in f32 (collectives.cpp:268-279) and writes the aggregate to
 * out + pieces[k].src (pieces are the owner's chunk, src = buffer offsets).
 * sra_reduce: fold, re-encode the aggregate with `seed` into bcast, and write
 * the owner's decoded result (divided by divisor) to out
 * (collectives.cpp:283-292). */
int gcx_fold_pieces(const gcx_piece* pieces, const uint32_t* tile_prefix, uint32_t npieces,
                    uint32_t ntiles, uint32_t flags, const uint8_t* recv, uint64_t slot_stride,
                    const float* own, uint32_t nodes, uint32_t me, float* out, void* stream);
/* fold_encode: the owner's fold and hop-1 re-encode in one pass
 * (collectives.cpp:266-284): the aggregate goes straight into bcast, never
 * to HBM.  One launch when the table qualifies (GCX_F_SPAN_ENC, bits <= 4,
 * bucket 128, nodes <= 8; keys = the table's span-layout prefixes with
 * GCX_F_KEY_PREFIX, or NULL to hash inline), else fold into out and encode
 * out (keys as gcx_encode_pieces). */
int gcx_sra_fold_encode(const gcx_piece* pieces, const uint32_t* tile_prefix, uint32_t npieces,
                        uint32_t ntiles, uint32_t flags, const uint8_t* recv, uint64_t slot_stride,
                        const float* own, uint32_t nodes, uint32_t me, uint64_t seed,
                        uint8_t* bcast, float* out, const unsigned long long* keys,
                        unsigned long long* bad_key, void* stream);
int gcx_sra_reduce(const gcx_piece* pieces, const uint32_t* tile_prefix, uint32_t npieces,
                   uint32_t ntiles, uint32_t flags, const uint8_t* recv, uint64_t slot_stride,
                   const float* own, uint32_t nodes, uint32_t me, uint64_t seed,
                   uint8_t* bcast, float* out, float divisor, const unsigned long long* keys,
                   unsigned long long* bad_key, void* stream);

/* ---- exact wire framing (codec.cpp:216-259, collectives.cpp:143-194) ----
 * The reference's message bytes for a piece table: per quantized piece the
 * 17-byte LE header {u32 count, u8 bits, u32 bucket, u64 seed}, the f32
 * norms and the ceil(len*(bits+1)/8) packed bytes; per raw piece its f32s.
 * wire_layout (host): wire_off[k] per piece, returns the message length.
 * frame: device message -> wire bytes (seed = the encode's seed, or the
 *        pieces' own with GCX_F_PIECE_SEEDS).
 * unframe: wire bytes -> device message; *err |= 1 when a header disagrees
 *        with the layout (the reference's "chunk payload does not match piece
 *        layout"); the caller checks the total length (trailing / short). */
int64_t gcx_wire_layout(const gcx_piece* pieces, uint32_t npieces, uint64_t* wire_off);
int gcx_frame_pieces(const gcx_piece* pieces, const uint64_t* wire_off, uint32_t npieces,
                     const uint8_t* msg, uint64_t seed, uint32_t flags, uint8_t* wire,
                     void* stream);
int gcx_unframe_pieces(const gcx_piece* pieces, const uint64_t* wire_off, uint32_t npieces,
                       const uint8_t* wire, uint8_t* msg, unsigned int* err, void* stream);

/* acc[i] = acc[i] + x[i] in f32 (the ring and tree topologies' folds,
 * collectives.cpp:359-361 and :412-413). */
int gcx_add_f32(float* acc, const float* x, uint64_t n, void* stream);
/* x[i] = x[i] / divisor (IEEE f32; finalize's average). */
int gcx_div_f32(float* x, uint64_t n, float divisor, void* stream);

/* ---- microbenchmarks ----
 * Integer ceiling of the reference RNG: n draws of uniform01(seed, i/bucket, i),
 * xor-reduced into *sink (device u64).  variant 0 = reference 64-bit form,
 * 1 = pipe-balanced split form used by K1/K2, 2 = split form, 2-way ILP. */
int gcx_hash_bench(uint64_t n, uint64_t seed, uint32_t bucket, int variant,
                   unsigned long long* sink, void* stream);

/* ---- K4: adaptive-selector statistics (adaptive.cpp:21-97, :390-415) ----
 * accumulate: sum[i] += (double)v[i]; *nonfinite |= 1 on a non-finite v.
 * snapshot:   out[i] = (float)sum[i].
 * reduce:     out[0] = sum_i sum[i]^2, out[1] = sum of the `keep` largest
 *             squares; scratch >= gcx_stats_scratch_bytes(n).
 * sq_error:   *out = sum_i (double(a_i) - double(b_i))^2; scratch >= 4736 B. */
int gcx_stats_accumulate(double* sum, const float* v, uint64_t n, unsigned int* nonfinite,
                         void* stream);
int gcx_stats_snapshot(const double* sum, float* out, uint64_t n, void* stream);
uint64_t gcx_stats_scratch_bytes(uint64_t n);
int gcx_stats_reduce(const double* sum, uint64_t n, uint64_t keep, void* scratch,
                     uint64_t scratch_bytes, double* out, void* stream);
int gcx_sq_error(const float* a, const float* b, uint64_t n, double* scratch, double* out,
                 void* stream);
/* mean over nodes, folded in node order then divided by nodes (the adaptive
 * observation feed, engine.cpp:268-283); stack = nodes rows of n floats */
int gcx_mean_nodes(const float* stack, uint32_t nodes, uint64_t n, float* out, void* stream);
const char* gcx_stats_last_error(void);

/* ---- TopK + error feedback, the reference's sparse codec (codec.cpp:158-214) ----
 * compress: residual <- v + residual; idx_out[0..k) = the k largest |acc|
 *           (ties to the lower index) in increasing order, val_out = their
 *           acc values, residual[idx] = 0.  *bad = min non-finite index of v
 *           (preset to UINT64_MAX).  scratch >= gcx_topk_scratch_bytes(n).
 * densify:  dense = 0, dense[idx[j]] = val[j]  (topk_decompress). */
uint64_t gcx_topk_scratch_bytes(uint64_t n);
int gcx_topk_compress(const float* v, uint64_t n, uint64_t k, float* residual, uint32_t* idx_out,
                      float* val_out, void* scratch, uint64_t scratch_bytes,
                      unsigned long long* bad, void* stream);
int gcx_topk_densify(const uint32_t* idx, const float* val, uint64_t k, uint64_t n, float* dense,
                     void* stream);

/* Number of SMs and the kernels' resident CTAs per SM (device 0..). */
int gcx_device_info(int device, int* sms, int* encode_ctas_per_sm);

#ifdef __cplusplus
}
#endif
#endif /* GCX_H_ */
