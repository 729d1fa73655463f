/*
 * smol_preproc.h -- C ABI of the B200-native Smol preprocessing hot path.
 *
 * The operation (§2 "Breakdown of end-to-end DNN inference",
 * P:366-382, steps 1-4; §6.4 "Partial and Low-Fidelity Decoding",
 * P:1037-1148): for each image of a batch of entropy-decoded baseline JPEGs
 * (Huffman decoding stays on the host), compute
 *
 *   dequantize -> 8x8 IDCT at scale 1, 1/2, 1/4 or 1/8 (reduced-fidelity
 *   decode, reading R1) -> level shift / round / clamp to u8 (R3) -> 4:2:0
 *   centred triangle chroma upsample (R2) -> exact JFIF YCbCr->RGB (R6) ->
 *   bilinear resize (half-pixel, no antialias, R8) to the short-side or exact
 *   size (R7/R11) -> centre crop or per-image ROI
 *    -> float, /255, -mean, /std -> NCHW
 *    fp32 or fp16.
 *
 * Only the coefficient blocks under the bilinear tap footprint of the crop are
 * read and transformed (ROI decoding).  Decoded pixels never go
 * to HBM: one fused sm_100a kernel per (scale, output dtype).
 *
 * Conventions
 *  - Every function returns an int32_t smol_status and never throws.  On
 *    failure smol_last_error() returns a thread-local message naming the
 *    failing image index and field where applicable.
 *  - Pointer kinds are stated per field: DEVICE = cudaMalloc'd memory of the
 *    plan's device; HOST = ordinary host memory.  Coefficient pointers given
 *    to smol_preproc_run_host may be host memory that was pinned with
 *    cudaHostRegister / cudaMallocHost (read by the kernel over PCIe).
 *  - The caller owns every buffer it passes and must keep it alive until the
 *    work on `stream` has finished.  The plan owns its own device scratch.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *    Work is asynchronous; kernel faults surface at the caller's next sync.
 *  - One run per plan may be in flight per stream; plans are not thread-safe.
 */
#ifndef SMOL_PREPROC_H
#define SMOL_PREPROC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMOL_ABI_VERSION 3

typedef enum {
  SMOL_OK = 0,
  SMOL_ERR_INVALID = 1,      /* bad argument / descriptor field             */
  SMOL_ERR_UNSUPPORTED = 2,  /* valid but not implemented (e.g. 4:4:4)      */
  SMOL_ERR_CUDA = 3,         /* CUDA runtime error (message has the name)   */
  SMOL_ERR_NOMEM = 4,        /* device/host allocation failed               */
  SMOL_ERR_CAPACITY = 5      /* n_images > plan capacity, or tile too large */
} smol_status;

typedef enum { SMOL_OUT_F32_NCHW = 0, SMOL_OUT_F16_NCHW = 1 } smol_out_dtype;
typedef enum { SMOL_RESIZE_SHORT_SIDE = 0, SMOL_RESIZE_EXACT = 1 } smol_resize_mode;
/* Coefficient block layout (per component plane, block-raster rows):
 *  DENSE64: 64 int16 per block, natural order (libjpeg JBLOCK).
 *  PACKED : only the coefficients the plan's scale uses (reading R1: the
 *           box-averaged basis of the others is exactly zero), row-major over
 *           the index set, padded to 8 bytes per block:
 *             1/1: = DENSE64;  1/2: u,v in {0,1,2,3,5,6,7} -> 52 int16 (104 B);
 *             1/4: u,v in {0,1,3,5,7} -> 28 int16 (56 B);  1/8: DC -> 1 int16 (2 B). */
typedef enum { SMOL_LAYOUT_DENSE64 = 0, SMOL_LAYOUT_PACKED = 1 } smol_coef_layout;

/* Plan parameters (fixed for the plan's lifetime). */
typedef struct {
  int32_t scale_denom;      /* k in {1,2,4,8}: decode at scale 1/k (R1)            */
  int32_t resize_mode;      /* smol_resize_mode                                    */
  int32_t resize_short;     /* SHORT_SIDE: short edge -> resize_short, long edge
                               -> floor(resize_short*long/short) (torchvision)   */
  int32_t resize_w, resize_h;  /* EXACT: resized size                            */
  int32_t crop_w, crop_h;   /* centre crop in resized coordinates; 0,0 = none
                               (required for SHORT_SIDE: fixed output size)      */
  float mean[3], std[3];    /* RGB; y = (x/255 - mean)/std, std > 0              */
  int32_t out_dtype;        /* smol_out_dtype                                      */
  int32_t layout;           /* smol_coef_layout                                    */
  int32_t tile_rows;        /* output rows per CTA tile; 0 = automatic           */
  int32_t idct_def;         /* reduced-scale IDCT (reading R1 / R16):
                               SMOL_IDCT_BOX_MEAN (0, Definition A: k x k box
                               mean of the 8x8 IDCT) or SMOL_IDCT_TRUNCATED (1,
                               Definition B: orthonormal (8/k)-point IDCT of
                               the top-left (8/k)^2 coefficients x (8/k)/8);
                               both equal the 8x8 IDCT at k = 1 and DC/8 at
                               k = 8                                              */
  int32_t max_width, max_height; /* optional staging capacity: when both > 0,
                               plan allocates the staging of the staged paths
                               (run_host, run_compact) for max_images images of
                               at most this SOF size, and those runs never
                               allocate (a larger image -> SMOL_ERR_CAPACITY);
                               0 = allocate on first use, grow on demand         */
  int32_t chroma_2s;        /* 1: libjpeg-turbo-style scaled decoding of 4:2:0
                               (reading R18): chroma blocks IDCT'd at twice the
                               luma scale (1/(k/2)), giving chroma at the luma
                               resolution, and no upsampling; k >= 2, DENSE64,
                               Definition A, 4:2:0 (and gray) images only;
                               0 = all components at 1/k + triangle upsample (R2) */
} smol_preproc_params;

typedef enum { SMOL_IDCT_BOX_MEAN = 0, SMOL_IDCT_TRUNCATED = 1 } smol_idct_def;

/* One entropy-decoded 4:2:0 image. */
typedef struct {
  int32_t width, height;           /* SOF size in pixels, > 0                        */
  int32_t subsampling;             /* chroma sampling (T.81 A.1.1): 420 (chroma
                                      W/2 x H/2), 422 (W/2 x H), 444 (W x H), or
                                      400 = grayscale (one component, Nf = 1:
                                      coef[1..2], their blocks/strides and
                                      qtable[1..2] are ignored; R = G = B = Y);
                                      anything else: SMOL_ERR_UNSUPPORTED            */
  int32_t qtable[3];               /* Y, Cb, Cr index into batch qtables             */
  const int16_t* coef[3];          /* DEVICE (or pinned HOST for run_host):
                                      [blocks_h][blocks_w][E] int16 blocks of the
                                      plan's layout (E = 64 for DENSE64: natural
                                      row-major v*8+u order), absolute DC;
                                      16-byte aligned                               */
  int32_t blocks_w[3], blocks_h[3];/* >= ceil(W/8), ceil(H/8) luma; chroma
                                      >= ceil(Wc/8), ceil(Hc/8) with Wc, Hc the
                                      chroma size (420: ceil(W/2), ceil(H/2))       */
  int32_t row_stride_bytes[3];     /* >= blocks_w*2*E, multiple of 16                 */
  int32_t roi_left, roi_top;       /* optional ROI: crop window origin in resized
                                      coordinates (window = crop_w x crop_h);
                                      -1,-1 = centre crop                            */
  int32_t roi_x, roi_y, roi_w, roi_h;  /* optional ROI rectangle (PAPER.md P:1080-1083,
                                      P:1107-1109: "the ROIs are the face crops"), in
                                      SOF pixel coordinates; roi_w, roi_h > 0 enable
                                      it (roi_left/top must then be -1): the
                                      rectangle's decoded window at scale 1/k,
                                      [floor(x/k), ceil((x+w)/k)) x [floor(y/k),
                                      ceil((y+h)/k)) (reading R15), is resized
                                      (bilinear, R8, taps clamped to the window) to
                                      the plan's output size -- torchvision
                                      resized_crop; 0,0,0,0 = no rectangle          */
} smol_image_desc;

typedef struct {
  int32_t n_images;                /* 0 is allowed (no-op)                           */
  const smol_image_desc* images;   /* HOST array of n_images                          */
  const uint16_t* qtables;         /* DEVICE [n_qtables][64] natural order, 1..65535 */
  int32_t n_qtables;               /* 1..4                                            */
} smol_batch_desc;

typedef struct smol_preproc_plan smol_preproc_plan_t;   /* opaque */

/* Geometry of one image under a plan (test/introspection; host only). */
typedef struct {
  int32_t Wd, Hd;               /* decoded luma size at scale 1/k (R4)          */
  int32_t Wc, Hc;               /* decoded chroma size                          */
  int32_t Wr, Hr;               /* resized size                                  */
  int32_t left, top;            /* crop origin in resized coordinates            */
  int32_t OW, OH;               /* output size                                   */
  int32_t lx0, lx1, ly0, ly1;   /* luma tap footprint (inclusive, decoded px)    */
  int32_t cx0, cx1, cy0, cy1;   /* chroma footprint incl. upsample neighbours    */
  int32_t bx0[3], bx1[3], by0[3], by1[3];  /* ROI block ranges per component   */
  int64_t roi_blocks;           /* blocks under the footprint (sum over comps)  */
  int64_t roi_coef_bytes;       /* algorithmic coefficient bytes of the image
                                   (SURVEY 8(d)): roi_blocks x 2 B x the K_s
                                   coefficients scale 1/k uses (64/49/25/1 at
                                   k = 1/2/4/8, reading R1), in any layout     */
  int32_t sx0, sy0, sw, sh;     /* source window of the resize (decoded px): the
                                   whole image, or the ROI rectangle's window   */
  int64_t storage_coef_bytes;   /* bytes the plan's layout stores for those
                                   blocks: 128 (DENSE64; 32 at k = 8, the DC's
                                   sector) or 128/104/56/2 (PACKED)            */
} smol_geometry;

/* Create a plan on the current CUDA device for batches of <= max_images.
 * Validates params, allocates all device scratch once (no allocation in
 * run).  *out = NULL on failure. */
int32_t smol_preproc_plan(const smol_preproc_params* params, int32_t max_images,
                          smol_preproc_plan_t** out);

/* Run the fused path on `stream`.  out: DEVICE [n][3][OH][OW] fp32/fp16,
 * aligned to its element size (vector stores are used when it is 16-B
 * (fp32) / 8-B (fp16) aligned).  Validates every descriptor before any
 * launch (status + smol_last_error); consecutive descriptors that differ only
 * in their coef pointers share one validated "kind" (only the pointers are
 * checked for them).  The per-run descriptors are uploaded on the plan's
 * internal copy stream and `stream` waits on that upload, so the next run's
 * upload overlaps this run's kernel (while `stream` is being captured into a
 * CUDA graph every operation stays on `stream`).  The plan's device must be
 * the current device (SMOL_ERR_INVALID otherwise). */
int32_t smol_preproc_run(smol_preproc_plan_t* plan, const smol_batch_desc* batch,
                         void* out, void* stream);

/* Same as smol_preproc_run, but coefficient pointers may be pinned HOST
 * memory (qtables stay DEVICE).  Only the ROI block rows cross PCIe: a gather
 * kernel on the plan's internal copy stream stages them into plan-owned device
 * memory (3 staging slots: the next call's transfer overlaps this call's fused
 * kernel while the host prepares the call after it), then the fused kernel runs on `stream`.  The staging buffers are
 * sized in plan when params.max_width / max_height are set (no allocation in
 * any run call; a batch that does not fit returns SMOL_ERR_CAPACITY), else
 * allocated on first use and grown when a larger batch arrives.  Every
 * plane's first and last byte must be pinned host (or device) memory:
 * checked per image (SMOL_ERR_INVALID), verified allocation ranges cached.
 * out: DEVICE. */
int32_t smol_preproc_run_host(smol_preproc_plan_t* plan, const smol_batch_desc* batch,
                              void* out, void* stream);

/* ---- Compact coefficient transport (§6.4
 * Huffman decoding stays on the host, so what crosses PCIe is
 * the entropy decoder's output; P:959-968 / P:1790-1796: pinned buffers
 * allocated once and reused).  A Huffman decoder produces each block as a
 * short list of nonzero coefficients; shipping 64 int16 per block instead
 * makes PCIe the end-to-end bound.  A compact record holds, for one image and
 * one plan, only the ROI blocks (the tap footprint of the whole output, the
 * same ranges smol_debug_geometry reports) and, per block, only the nonzero
 * coefficients among those the plan's scale uses (reading R1):
 *
 *   offset 0   header, 64 B: uint32 magic 0x32434D53 ("SMC2"), uint32 E
 *              (elements per block of the plan's layout), uint32 n_units
 *              (u16 units of the entry stream), uint32 0, int32 bx0[3], by0[3],
 *              nbx[3], nby[3] (ROI block ranges per component Y, Cb, Cr)
 *   64         uint8 len[nblocks]: per ROI block (component-major, then
 *              block-raster), the units of its entries (<= 128)
 *   align 4    uint32 row_start[nrows]: per ROI block row (component-major),
 *              index of the row's first unit in the entry stream
 *   align 16   uint16 entry stream: per block, one entry per nonzero element
 *              in ascending element index e: the unit e | v << 6 when
 *              -511 <= v <= 511 (v as 10-bit two's complement), else the
 *              escape e | (-512 << 6) followed by v as int16
 *   +2, align 16  (end: >= 2 zero bytes after the stream; record size is a
 *              multiple of 16)
 *
 * Everything outside the ROI and every element the scale does not use
 * (reading R1: u or v = 4 at 1/2, u or v in {2,4,6} at 1/4, AC at 1/8;
 * PACKED padding) is dropped, which leaves the output bit-identical to
 * smol_preproc_run on the dense planes. */
typedef struct {
  int32_t width, height;           /* SOF size in pixels, > 0                        */
  int32_t subsampling;             /* 420, 422, 444 or 400 (grayscale: the record
                                      has no chroma rows)                            */
  int32_t qtable[3];               /* Y, Cb, Cr index into batch qtables             */
  int32_t roi_left, roi_top;       /* as smol_image_desc (-1,-1 = centre crop)       */
  int32_t roi_x, roi_y, roi_w, roi_h;  /* as smol_image_desc (0,0,0,0 = none)        */
  int64_t offset;                  /* byte offset of the image's record in `arena`,
                                      multiple of 16                                 */
} smol_compact_image;

typedef struct {
  int32_t n_images;                /* 0 is allowed (no-op)                           */
  const smol_compact_image* images;/* HOST array of n_images                          */
  const void* arena;               /* records: pinned HOST (cudaMallocHost /
                                      cudaHostRegister) or DEVICE memory, 16-B aligned */
  int64_t arena_bytes;             /* every record lies inside [0, arena_bytes)      */
  const uint16_t* qtables;         /* DEVICE [n_qtables][64] natural order           */
  int32_t n_qtables;               /* 1..4                                            */
} smol_compact_batch;

/* Host only (no CUDA call): encode one image into a compact record for plans
 * with `params`.  image->coef[] are HOST planes in the params' layout (the
 * smol_image_desc rules apply; 16-B alignment is not required here).  With
 * dst == NULL only *written = record size is returned; otherwise the record is
 * written to dst (capacity bytes; SMOL_ERR_CAPACITY if too small) and
 * *written = its size. */
int32_t smol_compact_encode(const smol_preproc_params* params, const smol_image_desc* image,
                            void* dst, int64_t capacity, int64_t* written);

/* End-to-end run from compact records.  The byte range of the arena the batch
 * uses is copied host->device in one DMA on the plan's copy stream (skipped
 * when the arena is DEVICE memory); then, on `stream`, an expand kernel
 * rebuilds the ROI blocks of the plan's layout in plan-owned staging and the
 * fused kernel runs (3 staging slots: the next call's DMA overlaps this
 * call's expand + fused kernel while the host prepares the call after it).  Each record's header must match the ROI ranges
 * the plan computes for its image and lie inside the arena: checked on the
 * host (SMOL_ERR_INVALID) when the arena is host memory; a DEVICE arena is
 * not read by the host, so only its record offsets are checked.  Block
 * lengths and row starts are not re-scanned on the host: the expand kernel
 * clamps them (units per block <= 2E, every unit inside the record's
 * n_units), so a corrupt record gives wrong samples for its image but never
 * an out-of-bounds access.  Staging is sized in plan when params.max_width /
 * max_height are set (a batch that does not fit: SMOL_ERR_CAPACITY), else
 * allocated on first use and grown for a larger batch.  out: DEVICE. */
int32_t smol_preproc_run_compact(smol_preproc_plan_t* plan, const smol_compact_batch* batch,
                                 void* out, void* stream);

void smol_preproc_destroy(smol_preproc_plan_t* plan);

/* Output tensor shape (C=3, OH, OW) of the plan. */
int32_t smol_preproc_output_shape(const smol_preproc_plan_t* plan, int32_t* c, int32_t* h,
                                  int32_t* w);

/* ---------------------------------------------------------------------
 * JPEG input (entropy decoding on the GPU).
 *
 * The paper leaves Huffman decoding on the host because it "requires
 * substantial branching" (§6.4).  This entry point takes the
 * JPEG files themselves: the host parses only the headers (ITU-T T.81 Annex
 * B markers: SOF0/SOF1, DQT, DHT, DRI, SOS; a header byte-identical to the
 * previous image's is parsed once), then on the GPU one kernel finds the
 * restart markers (RSTm, T.81 B.2.1) and one thread per restart interval
 * Huffman-decodes its MCUs (T.81 F.2.2: DC prediction reset at every
 * interval, F.2.1.3.1; run-length AC, Figure F.13; zig-zag, Figure A.6),
 * writing only the blocks inside each image's ROI (the plan's tap footprint)
 * in the plan's layout; the fused kernel follows as for run_compact.  The
 * output equals smol_preproc_run on the entropy-decoded planes bit for bit.
 * Parallelism comes from restart intervals: a file without DRI decodes on one
 * thread (correct, slow).
 *
 * Supported: baseline sequential Huffman (SOF0, or SOF1 with 8-bit tables),
 * 8-bit samples, one interleaved scan of 1 (grayscale) or 3 components with
 * luma sampling 2x2 (4:2:0), 2x1 (4:2:2) or 1x1 (4:4:4) and chroma 1x1;
 * else SMOL_ERR_UNSUPPORTED.  Quantization tables come from each file's DQT
 * (at most 64 distinct tables and 16 distinct sets of Huffman tables per
 * batch: SMOL_ERR_CAPACITY).
 * Malformed entropy-coded data cannot make a kernel read or write out of
 * bounds (the bit reader stops at the file end; runs past 63 end the block);
 * it yields wrong samples.  A header error is SMOL_ERR_INVALID with the image
 * index in smol_last_error(). */
typedef struct {
  int64_t offset;                  /* byte offset of the file (SOI..EOI) in arena,
                                      multiple of 16                                 */
  int64_t size;                    /* bytes                                         */
  int32_t roi_left, roi_top;       /* as smol_image_desc (-1,-1 = centre crop)      */
  int32_t roi_x, roi_y, roi_w, roi_h;  /* as smol_image_desc (0,0,0,0 = none)       */
} smol_jpeg_image;

typedef struct {
  int32_t n_images;                /* 0 is allowed (no-op)                          */
  const smol_jpeg_image* images;   /* HOST array of n_images                        */
  const void* arena;               /* the files: pinned HOST memory (cudaMallocHost /
                                      cudaHostRegister); read by the host (headers)
                                      and copied to the device in one DMA            */
  int64_t arena_bytes;             /* every file lies inside [0, arena_bytes)       */
} smol_jpeg_batch;

/* Header of one JPEG file as this library reads it (host only, no CUDA). */
typedef struct {
  int32_t width, height;           /* SOF size                                      */
  int32_t subsampling;             /* 420, 422, 444 or 400                           */
  int32_t ncomp;
  int32_t blocks_w[3], blocks_h[3];/* coefficient blocks per component incl. MCU padding */
  int32_t mcus_x, mcus_y;
  int32_t restart_interval;        /* MCUs per interval (0 = none)                   */
  int32_t n_segments;              /* restart intervals in the scan                 */
  int32_t scan_offset;             /* first byte of the entropy-coded data          */
} smol_jpeg_header;

int32_t smol_jpeg_parse_header(const void* data, int64_t size, smol_jpeg_header* out);

/* Files -> output tensor (see above).  Stream ordering, staging and
 * ownership as smol_preproc_run_compact: one DMA of the batch's byte range on
 * the plan's copy stream, the index + decode kernels, then the fused kernel
 * on `stream`.  Errors: SMOL_ERR_CAPACITY (n_images > the plan's max_images,
 * or too many distinct tables), SMOL_ERR_INVALID (arena not pinned host
 * memory, a file outside it or at an offset not a multiple of 16, a bad
 * header), SMOL_ERR_UNSUPPORTED (a non-baseline file, a chroma_2s plan); no
 * work is queued when a check fails.  The arena must stay untouched until the call after next has
 * returned (3 staging slots). */
int32_t smol_preproc_run_jpeg(smol_preproc_plan_t* plan, const smol_jpeg_batch* batch, void* out,
                              void* stream);

/* Test-only: Huffman-decode every block of every image (no ROI, no plan)
 * into caller-owned DEVICE planes: planes[3 i + c] = [blocks_h][blocks_w][64]
 * int16, natural order, absolute DC (sizes from smol_jpeg_parse_header;
 * NULL for the chroma of a grayscale file).  Synchronous; allocates and frees
 * its own scratch. */
int32_t smol_jpeg_decode_planes(const smol_jpeg_batch* batch, int16_t* const* planes, void* stream);

/* Number of kernel launches one smol_preproc_run issues (for accounting): 1.
 * smol_preproc_run_host and smol_preproc_run_compact issue one more (the
 * gather or expand kernel before the fused kernel), smol_preproc_run_jpeg two
 * more (marker index + Huffman decode). */
int32_t smol_preproc_launches_per_run(const smol_preproc_plan_t* plan);

/* Host-only: geometry of one image under `params` (no CUDA needed). */
int32_t smol_debug_geometry(const smol_preproc_params* params, const smol_image_desc* image,
                            smol_geometry* out);

/* Test-only: run the SAME fused kernel with its debug store enabled: besides
 * `out`, writes the u8 samples it decoded into DEVICE int16 planes
 * (initialised by the caller to -1): y_dbg[n][Hd][Wd], cb_dbg/cr_dbg
 * [n][Hc][Wc], rgb_dbg[n][Hd][Wd][3] (per-image slices of size
 * dbg_stride_* elements).  Only samples inside each image's footprint are
 * written. */
int32_t smol_debug_run(smol_preproc_plan_t* plan, const smol_batch_desc* batch, void* out,
                       int16_t* y_dbg, int16_t* cb_dbg, int16_t* cr_dbg, int16_t* rgb_dbg,
                       int64_t dbg_stride_y, int64_t dbg_stride_c, int64_t dbg_stride_rgb,
                       void* stream);

/* Thread-local message of the last failing call ("" if none). */
const char* smol_last_error(void);

/* SMOL_ABI_VERSION of the loaded library. */
int32_t smol_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SMOL_PREPROC_H */
