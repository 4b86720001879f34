/*
 * slcs.h -- C ABI of the B200-native SLCS/ImgQL primitive layer.
 *
 * This is the drop-in boundary below the reference executor's opcode dispatch
 * `evalTask` (proj/src/executor.cpp:74-115, declared proj/include/pixlog/executor.hpp:54-55).
 * Every entry point is plain C: opaque handles, plain pointers and sizes, int
 * status codes, no C++ or torch types.  INTEGRATION.md shows the C++ shim a
 * reference maintainer adds (a device variant of `Value`, a rethrowing
 * wrapper) and the ctypes binding used by this repository's Python host.
 *
 * Semantics are bit-exact with the reference CPU path.
 *
 * Threading: all entry points are safe to call concurrently from several host
 * threads (the reference evaluates independent DAG nodes on WorkerPool
 * threads, executor.cpp:220,259).  Work is enqueued in call order on the
 * context's stream; only volume/download/program outputs synchronise.
 *
 * Errors: a non-zero status plus a thread-local message (slcs_last_error)
 * that reuses the reference's RunError texts, e.g. "dimension mismatch"
 * (kernels.cpp:16-21), "expects a boolean image, got u16" (kernels.cpp:10-14),
 * "reach expects boolean images" (reach.cpp:13-14), "image too large for
 * packed coordinate labels" (image.cpp:26-28).
 */
#ifndef SLCS_H
#define SLCS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SLCS_ABI_VERSION 1

typedef struct slcs_ctx slcs_ctx;         /* one device + one stream + memory pool */
typedef struct slcs_image slcs_image;     /* refcounted immutable device image      */
typedef struct slcs_program slcs_program; /* a whole task DAG compiled for replay   */

/* PixelKind, proj/include/pixlog/image.hpp:16 */
typedef enum { SLCS_BOOL = 0, SLCS_U16 = 1, SLCS_LABEL = 2 } slcs_kind;

/* kernels::CmpOp, proj/include/pixlog/kernels.hpp:10 (">." ">=." "<." "<=." "=.") */
typedef enum { SLCS_GT = 0, SLCS_GE = 1, SLCS_LT = 2, SLCS_LE = 3, SLCS_EQ = 4 } slcs_cmp;

typedef enum {
  SLCS_OK = 0,
  SLCS_ERR_KIND = 1,      /* wrong pixel kind (RunError "expects a ... image")        */
  SLCS_ERR_SHAPE = 2,     /* dimension mismatch / bad dimensions                      */
  SLCS_ERR_TOO_LARGE = 3, /* labels need W*H < 0xFFFFFFFE (image.cpp:26-28)           */
  SLCS_ERR_OOM = 4,       /* device allocation failed                                 */
  SLCS_ERR_CUDA = 5,      /* CUDA runtime error                                       */
  SLCS_ERR_NCCL = 6,      /* collective failure (multi-GPU)                           */
  SLCS_ERR_ARG = 7,       /* invalid argument (null handle, bad enum, ...)            */
  SLCS_ERR_RUN = 8,       /* evaluation error (division by zero, unknown opcode, ...) */
  SLCS_ERR_NOGPU = 9      /* no CUDA device: the product path has no CPU fallback     */
} slcs_status;

/* ---- library / context --------------------------------------------------- */

int slcs_abi_version(void);
/* Message of the last failing call on this thread ("" if none). */
const char* slcs_last_error(void);

/* Creates a context on `device`.  `cuda_stream` is a cudaStream_t to enqueue
 * on (e.g. torch.cuda.current_stream().cuda_stream) or NULL for a private
 * non-blocking stream. */
int slcs_ctx_create(int device, void* cuda_stream, slcs_ctx** out);
int slcs_ctx_destroy(slcs_ctx* ctx);
int slcs_ctx_synchronize(slcs_ctx* ctx);
void* slcs_ctx_stream(slcs_ctx* ctx);
/* Number of kernels this context has launched (for bench gpu_launches). */
int64_t slcs_ctx_launch_count(slcs_ctx* ctx);

/* ---- device images (refcounted, mirror shared_ptr<const ImageBuffer>) ----
 * Host layout is the reference ImageBuffer layout (image.hpp:36-75): row-major,
 * Bool = 1 byte/pixel (0 or nonzero), U16 = 2 bytes, LABEL = uint32 idx+1.
 * `batch` stacks same-shape slices (slice s at offset s*W*H in host memory);
 * the single-image reference API uses batch = 1.
 * Device layout: Bool is bit-packed, 32 px per uint32 word,
 * LSB = lowest column, row pitch padded to 16 B, padding bits zero; U16 rows
 * are padded to 32 pixels; labels are dense uint32. */
int slcs_image_upload(slcs_ctx* ctx, slcs_kind kind, int w, int h, int batch,
                      const void* host, slcs_image** out);
/* Same, from DEVICE memory already in the reference dense layout. */
int slcs_image_from_device(slcs_ctx* ctx, slcs_kind kind, int w, int h, int batch,
                           const void* dev, slcs_image** out);
/* Copies into host memory in the reference layout (Bool -> bytes 0/1).
 * `bytes` must be >= W*H*batch*sizeof(pixel).  Synchronises. */
int slcs_image_download(slcs_ctx* ctx, const slcs_image* img, void* host, size_t bytes);
/* Device-to-device copy into the reference dense layout (no sync). */
int slcs_image_to_device(slcs_ctx* ctx, const slcs_image* img, void* dev, size_t bytes);
/* Rows [row0, row0 + h) of the reference's randomMask(w, H, density, Rng(seed))
 * fixture (proj/tests/oracles.cpp:44-49, splitmix64 proj/include/pixlog/rng.hpp:14-19)
 * generated on the device, bit-identical to the CPU stream: pixel i consumes
 * draw i.  Lets each rank of a banded run generate its own band. */
int slcs_random_mask(slcs_ctx* ctx, int w, int h, long long row0, uint64_t seed, double density,
                     slcs_image** out);
/* Rows [row0, row0 + h) of a uniform U16 fixture, pixel i of the w-wide image
 * = (draw i of splitmix64(seed)) % 65536 -- the reference's Rng::below(65536)
 * per pixel (proj/include/pixlog/rng.hpp:21-23), as make_golden uses it.
 * Fixture for the 65536^2 threshold parity/bench (no reference function). */
int slcs_random_u16(slcs_ctx* ctx, int w, int h, long long row0, uint64_t seed,
                    slcs_image** out);
int slcs_image_retain(slcs_image* img);
int slcs_image_release(slcs_image* img);
int slcs_image_info(const slcs_image* img, int* kind, int* w, int* h, int* batch);
/* Raw device storage (bit-packed for Bool) for zero-copy interop. */
int slcs_image_storage(const slcs_image* img, void** dev, size_t* row_pitch_bytes,
                       size_t* slice_bytes);

/* ---- image ingest / egress (png_io, proj/src/png_io.cpp:30-144) ----------
 * loadPng: 8/16-bit grey, grey+alpha, RGB or RGBA (Adam7 allowed) -> U16, the
 * first channel, 8-bit samples widened by v*257; palette images and other bit
 * depths fail with the reference's messages.  savePng: Bool -> 16-bit grey
 * (true = 65535), U16 verbatim, labels -> 8-bit RGB (slcs_label_color).
 * Decoding of the byte stream (zlib) is host work; the per-pixel conversion
 * runs on the device. */
int slcs_png_load(slcs_ctx* ctx, const char* path, slcs_image** out);
int slcs_png_decode(slcs_ctx* ctx, const void* bytes, size_t n, slcs_image** out);
int slcs_png_save(slcs_ctx* ctx, const slcs_image* img, const char* path);
/* labelColor (png_io.cpp:75-90): lowbias32 hash of a packed label, null -> black */
void slcs_label_color(uint32_t packed, uint8_t rgb[3]);

/* ---- primitives: each returns a NEW image (*out, refcount 1) --------------
 * Boolean operands that are U16 are coerced by `p > 0` (boolArg,
 * executor.cpp:43-50).  Label images are rejected. */

/* kernels::threshold (kernels.cpp:75-97): U16 -> Bool, double(p) op n. */
int slcs_threshold(slcs_ctx* ctx, slcs_cmp op, const slcs_image* img, double n,
                   slcs_image** out);
/* kernels::logicalNot / logicalAnd / logicalOr (kernels.cpp:36-73). */
int slcs_not(slcs_ctx* ctx, const slcs_image* a, slcs_image** out);
int slcs_and(slcs_ctx* ctx, const slcs_image* a, const slcs_image* b, slcs_image** out);
int slcs_or(slcs_ctx* ctx, const slcs_image* a, const slcs_image* b, slcs_image** out);
/* kernels::dilate = near (kernels.cpp:99-124); near_k = near applied k times
 * (one launch, (2k+1)^2 clipped box). */
int slcs_near(slcs_ctx* ctx, const slcs_image* a, slcs_image** out);
int slcs_near_k(slcs_ctx* ctx, const slcs_image* a, int k, slcs_image** out);
/* stdlib interior = !near(!a) (stdlib.imgql:5) as one erosion launch. */
int slcs_interior(slcs_ctx* ctx, const slcs_image* a, slcs_image** out);
int slcs_interior_k(slcs_ctx* ctx, const slcs_image* a, int k, slcs_image** out);
/* kernels::countTrue = volume (kernels.cpp:126-136).  `out` holds `batch`
 * counts (one per slice).  Synchronises. */
int slcs_volume(slcs_ctx* ctx, const slcs_image* a, int64_t* out);
/* volume without a host round trip: `batch` int64 counts are written to DEVICE
 * memory `dev_counts` in stream order (no synchronisation) -- the device-side
 * volume -> print path of SURVEY §8(f) rank 3. */
int slcs_volume_async(slcs_ctx* ctx, const slcs_image* a, int64_t* dev_counts);
/* ccl::label (ccl.cpp:127-165): 8-connected labels, each component labelled
 * with its max row-major index + 1 (ccl.hpp:52-60), background 0. */
int slcs_ccl(slcs_ctx* ctx, const slcs_image* a, slcs_image** out);
/* reach(target, through) (reach.cpp:10-50). */
int slcs_reach(slcs_ctx* ctx, const slcs_image* target, const slcs_image* through,
               slcs_image** out);
/* NEW opcode maxvol: union of the 8-connected components of maximal pixel
 * count (ties keep all maxima; per slice for batches).  No reference pin. */
int slcs_maxvol(slcs_ctx* ctx, const slcs_image* a, slcs_image** out);

/* ---- row bands (multi-GPU) ------------------------------------
 * A 65536^2 image is split into row bands, one per GPU (one process per GPU).
 * Each band runs the single-image kernels on its rows; what crosses a band
 * border is exchanged on the device:
 *   near/interior: k halo rows from each neighbour (e.g. NCCL send/recv of the
 *     neighbours' first/last k packed rows, slcs_image_storage) feed one
 *     slcs_near_k_halo launch -- no band copies;
 *   reach: slcs_reach_prepare labels the band; slcs_reach_border_record writes
 *     the band's BORDER RECORD (roots/classes of its first and last row and its
 *     first and last target row, slcs_band_record_bytes(0, w) bytes of device
 *     memory); the caller all-gathers the records of all nb bands (in band
 *     order, e.g. ncclAllGather); slcs_band_reach_merge resolves the
 *     components that cross borders with a small device union-find and flags
 *     this band's newly seeded roots; slcs_reach_finish(k_out = 0) gives
 *     target | selected, closed by slcs_near_k_halo;
 *   ccl: band-local labels (slcs_ccl), slcs_ccl_border_record, all-gather,
 *     slcs_band_ccl_relabel -> global 64-bit labels equal to the whole-image
 *     ccl::label (component max index + 1), which 65536^2 needs; or, with no
 *     u32 label image, slcs_ccl_band_begin / all-gather / slcs_ccl_band_finish.
 * Halo buffers are packed rows with the band image's row pitch. */
int slcs_near_k_halo(slcs_ctx* ctx, const slcs_image* a, int k, int erode, const void* top_dev,
                     int top_rows, const void* bot_dev, int bot_rows, slcs_image** out);
/* kind 0 = reach record, 1 = label record, for a band of width w */
size_t slcs_band_record_bytes(int kind, int w);
int slcs_ccl_border_record(slcs_ctx* ctx, const slcs_image* labels, void* record_dev);
/* records_dev: nb records in band order; band_heights: host array of nb heights;
 * out_dev: W*H uint64 device memory for this band (band `me`). */
int slcs_band_ccl_relabel(slcs_ctx* ctx, const slcs_image* labels, int nb, int me,
                          const void* records_dev, const long long* band_heights,
                          uint64_t* out_dev);
/* The same band CCL without a u32 label image in between: begin runs the
 * band's union-find and writes its label record (as slcs_ccl_border_record
 * would from slcs_ccl's labels); after the all-gather, finish writes the
 * global 64-bit labels straight from the union-find (8 B/px written once,
 * instead of 4 B/px labels written, read back and relabelled).  A job is
 * destroyed with slcs_ccl_job_destroy, finished or not. */
typedef struct slcs_ccl_job slcs_ccl_job;
typedef struct slcs_reach_state slcs_reach_state;
int slcs_ccl_band_begin(slcs_ctx* ctx, const slcs_image* band, void* record_dev,
                        slcs_ccl_job** job);
/* The band's ccl::label from the labelling of a band reach on the same image
 * (slcs_reach_prepare_labels: reach's `through` is the ccl input): no second
 * union-find.  The job keeps the reach state's labelling alive: the two may
 * be destroyed in either order. */
int slcs_ccl_band_begin_reach(slcs_reach_state* st, void* record_dev, slcs_ccl_job** job);
int slcs_ccl_band_finish(slcs_ccl_job* job, int nb, int me, const void* records_dev,
                         const long long* band_heights, uint64_t* out_dev);
int slcs_ccl_job_destroy(slcs_ccl_job* job);
/* reach in phases: prepare labels `through` and flags the components holding a
 * seed (through & near(target)); reach_row copies, per pixel of one row, the
 * component's root node and a class byte (0 background, 1 unseeded, 2 seeded)
 * to the host; reach_set_flags seeds host-listed roots; finish writes
 * near^k_out(target | selected components) (k_out = 0: no closing near). */
int slcs_reach_prepare(slcs_ctx* ctx, const slcs_image* target, const slcs_image* through,
                       slcs_reach_state** out);
/* slcs_reach_prepare whose labelling also keeps each component's max key, for
 * slcs_ccl_band_begin_reach (ccl::label of `through` at no second labelling). */
int slcs_reach_prepare_labels(slcs_ctx* ctx, const slcs_image* target, const slcs_image* through,
                              slcs_reach_state** out);
int slcs_reach_row(slcs_reach_state* st, int row, uint32_t* roots, uint8_t* cls);
int slcs_reach_set_flags(slcs_reach_state* st, int n, const uint32_t* roots);
int slcs_reach_border_record(slcs_reach_state* st, void* record_dev);
int slcs_band_reach_merge(slcs_reach_state* st, int nb, int me, const void* records_dev);
int slcs_reach_finish(slcs_reach_state* st, int k_out, slcs_image** out);
int slcs_reach_state_destroy(slcs_reach_state* st);
/* Rows [row0, row0 + nrows) of an image / vertical concatenation (same kind
 * and width) -- halo assembly for banded stencils. */
int slcs_image_rows(slcs_ctx* ctx, const slcs_image* img, int row0, int nrows, slcs_image** out);
int slcs_image_vstack(slcs_ctx* ctx, int n, const slcs_image* const* imgs, slcs_image** out);

/* ---- host-in / host-out wrappers with the reference signatures -----------
 * kernels::threshold / logicalNot / logicalAnd / logicalOr / dilate /
 * countTrue, ccl::label, reach -- for callers holding host ImageBuffers. */
int slcs_h_threshold(slcs_ctx* ctx, slcs_cmp op, const uint16_t* img, int w, int h, double n,
                     uint8_t* out);
int slcs_h_not(slcs_ctx* ctx, const uint8_t* a, int w, int h, uint8_t* out);
int slcs_h_and(slcs_ctx* ctx, const uint8_t* a, const uint8_t* b, int w, int h, uint8_t* out);
int slcs_h_or(slcs_ctx* ctx, const uint8_t* a, const uint8_t* b, int w, int h, uint8_t* out);
int slcs_h_dilate(slcs_ctx* ctx, const uint8_t* a, int w, int h, uint8_t* out);
int slcs_h_count_true(slcs_ctx* ctx, const uint8_t* a, int w, int h, int64_t* out);
int slcs_h_ccl_label(slcs_ctx* ctx, const uint8_t* a, int w, int h, uint32_t* out);
int slcs_h_reach(slcs_ctx* ctx, const uint8_t* target, const uint8_t* through, int w, int h,
                 uint8_t* out);

/* ---- programs: a whole TaskGraph evaluated device-resident ----------------
 * Replaces executor::run's per-node scheduling (executor.cpp:117-282) below
 * the same Task contract (task_graph.hpp:20-24): tasks in id order (deps have
 * smaller ids, task_graph.cpp:64-70), opcode strings from the builtin table
 * (task_graph.cpp:131-139) plus "const", "load", "save", "print", and the new
 * "maxvol".  payload_num is used by "const"; payload_str by load/save/print.
 * deps of task i are deps[dep_off[i] .. dep_off[i+1]).
 * The program binds "load" names to images, plans device memory by liveness,
 * fuses elementwise/threshold chains and near runs, and records the whole
 * evaluation into a CUDA graph that is replayed by slcs_program_run. */
int slcs_program_create(slcs_ctx* ctx, int n_tasks, const char* const* opcodes,
                        const double* payload_num, const char* const* payload_str,
                        const int* dep_off, const int* deps, slcs_program** out);
int slcs_program_destroy(slcs_program* prog);
/* Binds the image loaded by `load` tasks with payload `name`. */
int slcs_program_bind(slcs_program* prog, const char* name, const slcs_image* img);
/* flags: bit 0 = capture/replay as a CUDA graph, bit 1 = disable fusion,
 * bit 2 = disable label CSE (reaches sharing one `through` node label it once),
 * bit 3 = disable reach chains (consecutive label-CSE reaches in one persistent
 * cooperative launch), bit 4 = timeline: launch eagerly with a CUDA event after
 * every device step (per-task device times, slcs_program_task_time; the
 * reference's TaskEvent start/end, executor.hpp:28-35). */
int slcs_program_run(slcs_program* prog, int flags);
/* Copies host pixels (reference layout) straight into the program's input
 * slot for `load` name `name` -- the end-to-end path: no intermediate image. */
int slcs_program_set_input_host(slcs_program* prog, const char* name, slcs_kind kind, int w,
                                int h, int batch, const void* host);
/* Downloads the result of task `task` into host memory in the reference
 * layout (Bool -> bytes 0/1; a number -> one double).  Synchronises. */
int slcs_program_download(slcs_program* prog, int task, void* host, size_t bytes);
/* Result of task `task` (an image; *out gets a new reference) or a number
 * (synchronises).  kind_out: 0 image, 1 number. */
int slcs_program_result(slcs_program* prog, int task, int* kind_out, slcs_image** img_out,
                        double* num_out);
/* Outcome of task `task` in the last run: *state 0 = evaluated, 1 = failed
 * (*message = the RunError text, e.g. "division by zero"), 2 = aborted because a
 * dependency failed (executor.cpp:204-218).  *message stays valid until the
 * next run. */
int slcs_program_task_state(slcs_program* prog, int task, int* state, const char** message);
/* After a run with the timeline flag: the device interval (ms from the start of
 * the run) of the step that evaluated task `task`; -1 when the task has no step
 * of its own (host-side const/load/save/print, or fused into a consumer's step). */
int slcs_program_task_time(slcs_program* prog, int task, float* start_ms, float* end_ms);
/* Kernel launches issued by one run (after fusion). */
int slcs_program_launches(slcs_program* prog, int* out);
/* Human-readable execution plan (fused groups, buffer slots). */
const char* slcs_program_plan(slcs_program* prog);

#ifdef __cplusplus
}
#endif
#endif /* SLCS_H */
