/* lpm6cu — C ABI of the B200-native batched IPv6 longest-prefix-match lookup.
 *
 * This is the drop-in boundary for PlanB's hot path. It replaces, on the GPU,
 * the reference interfaces below (all under /root/reference/proj/):
 *
 *   reference                                            here
 *   ---------------------------------------------------  ------------------------------
 *   FibTable -> build_intervals -> build_tree            lpm6cu_fib_build
 *     (fib.hpp:74-105, intervals.hpp:34, tree.hpp:74)
 *   build_intervals (intervals.hpp:34)                   lpm6_build_intervals
 *   plan_geometry / build_tree (tree.hpp:36, :74)        lpm6_plan_layout / lpm6_build_tree
 *   search_batch / lookup (bodies absent,     lpm6cu_lookup_batch
 *     CMakeLists.txt:27-28,35,42) behind the runtime
 *     backend table detail::vector_backend()
 *     (intervals.cpp:121, CMakeLists.txt:18-46)
 *   lpm6::Error{Errc} (types.hpp:27-49)                  int status = (int)Errc + 1, lpm6cu_last_error()
 *
 * Conventions
 *   - Every function returns 0 on success or a status code below; the message of
 *     the last failure on the calling thread is lpm6cu_last_error(). No C++
 *     exception crosses this boundary.
 *   - Addresses are 16-byte little-endian unsigned __int128 values (lo word first),
 *     the type lpm6::lookup_linear_oracle takes (intervals.hpp:37). The lookup key
 *     is the top 64 bits (fib.hpp:27), clamped to 0xFFFF_FFFF_FFFF_FFFE (types.hpp:25).
 *   - Next hops are written at the FIB's value width (1, 2 or 4 bytes, little-endian).
 *   - A FIB handle is immutable after creation: any number of lookups on any
 *     streams may run on it concurrently (the reference's contract).
 *     The tuning calls (lpm6cu_fib_set_kernel_config, lpm6cu_fib_set_checked)
 *     change how later lookups run and must not race with lookups on the handle.
 *   - There is no CPU fallback: a lookup without a usable CUDA device fails with
 *     LPM6CU_E_CUDA.
 *   - Device buffers must live on the FIB's own device (InvalidArgument otherwise:
 *     a kernel touching another GPU's memory would poison the CUDA context).
 */
#ifndef LPM6CU_H
#define LPM6CU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  LPM6CU_OK = 0,
  LPM6CU_E_MALFORMED_ADDRESS = 1,       /* Errc::MalformedAddress */
  LPM6CU_E_UNSUPPORTED_PREFIX_LENGTH = 2,
  LPM6CU_E_MISSING_NEXT_HOP = 3,
  LPM6CU_E_RESERVED_NEXT_HOP = 4,
  LPM6CU_E_DUPLICATE_PREFIX = 5,
  LPM6CU_E_UNKNOWN_PREFIX = 6,
  LPM6CU_E_SENTINEL_COLLISION = 7,
  LPM6CU_E_EXHAUSTED_PREFIX_SPACE = 8,
  LPM6CU_E_INVALID_ARGUMENT = 9,
  LPM6CU_E_BAD_TRACE_FILE = 10,
  LPM6CU_E_BAD_SNAPSHOT_FILE = 11,
  LPM6CU_E_IO = 12,
  LPM6CU_E_CUDA = 13,
  LPM6CU_E_NCCL = 14,
};

/* Same memory layout as lpm6::Prefix (fib.hpp:22-29): u128 value (text order,
 * canonical), int length 0..64, u32 next hop; 32 bytes. A reference
 * FibTable::entries().data() can be passed directly. */
typedef struct {
  uint64_t value_lo;
  uint64_t value_hi;
  int32_t length;
  uint32_t next_hop;
  uint64_t reserved;
} lpm6cu_prefix;

#define LPM6CU_MAX_LEVELS 9

/* Geometry of the B200 tree layout: one array of 128-byte lines. Internal
 * lines hold k = 15 separator keys (arity 16); leaf lines hold leaf_keys boundary keys
 * followed by their next hops. Counterpart of lpm6::TreeGeometry (tree.hpp:18-33). */
typedef struct {
  uint32_t k;           /* separator keys per internal node (15; word 15 is padding) */
  uint32_t b;           /* arity, k + 1 */
  uint32_t depth;       /* internal levels; a lookup visits depth + 1 lines */
  uint32_t value_bytes; /* next-hop width: 1, 2 or 4 */
  uint32_t leaf_keys;   /* keys per leaf line: 14, 12 or 8 for 1-, 2-, 4-byte next hops */
  uint32_t image_levels;/* internal levels [0, image_levels) have a shared-memory image */
  uint64_t num_keys;    /* m, real interval boundaries */
  uint64_t leaf_nodes;  /* ceil(m / leaf_keys) */
  uint64_t total_words; /* length of the array in u64 words: tree lines, then the image */
  uint64_t image_start; /* word offset of that image: the 15 keys of each node at a 120-byte
                           stride (bank skew), staged into shared memory by one TMA copy */
  uint64_t level_nodes[LPM6CU_MAX_LEVELS]; /* reachable nodes per level (level depth = leaves) */
  uint64_t level_start[LPM6CU_MAX_LEVELS]; /* u64-word offset of each level */
  uint32_t default_next_hop;
  uint32_t leaf_image;   /* 1: small tree — the leaf lines also have a shared-memory image (16 words
                            at a 17-word stride) right after the internal image; smem_levels =
                            depth + 1 then serves the whole lookup from shared memory */
  uint32_t leaf_words;   /* words per leaf: 16 (one 128-byte line) or 8 (half-line leaves: 6 keys in
                            words 0-5, their 1- or 2-byte next hops in words 6-7) */
  uint32_t reserved;
} lpm6cu_geometry;

typedef struct {
  uint32_t merge_adjacent; /* IntervalBuildOptions::merge_adjacent (intervals.hpp:28); default 1 */
  uint32_t value_bytes;    /* 0 = narrowest width holding every next hop */
  uint32_t leaf_format;    /* 0 = automatic (half-line leaves where they keep the depth and the
                              shared-memory levels of a tree with an L2 internal level), 1 = full
                              128-byte leaf lines, 2 = half-line leaves (1- or 2-byte next hops) */
  uint32_t reserved;
} lpm6cu_build_opts;

/* Kernel shape; 0 in a field = automatic. */
typedef struct {
  uint32_t lanes_per_query; /* lanes cooperating on one 128-byte line in the L2 levels (4) */
  uint32_t smem_levels;     /* top levels staged in shared memory by TMA and searched one
                               thread per query; 0xFF = auto */
  uint32_t ctas_per_sm;      /* cap on resident CTAs per SM used for the grid; 0 = occupancy */
  uint32_t threads_per_cta;  /* 1024 (default), 512 or 256 */
  uint32_t queries_per_lane; /* 32-query tiles each warp carries at once: 1; 2 at 256 threads; 2 or
                                4 at 1024 threads on the texture leaf paths 1 and 4 (the tiles'
                                shared-memory descents overlap, their L2 levels run one tile at a
                                time; other line paths then run one tile). The tuner picks it. */
  uint32_t min_ctas_per_sm;  /* register cap (__launch_bounds__ min blocks): 1 at 1024 threads,
                                2 at 512, 0 or 4 at 256 */
  uint32_t line_path;        /* which L1TEX pipe carries the 128-byte L2 lines (address / key
                                input, and packets over half-line leaves; default shape, unchecked): 0 = leaves through the LSU,
                                internal L2 levels through the texture pipe (default); 1 = leaves
                                through the texture pipe too, faster when leaf lines often hit L1
                                (skewed traffic); 2 = half of each warp's leaf lines through each
                                pipe; 3 = as 1 with half of the internal-level lines through the
                                LSU; 4 = as 1 with another extraction of 1-byte next hops (same as 1
                                for wider ones). Pick it on representative traffic with
                                lpm6cu_fib_tune_line_path. */
  uint32_t plane_levels;     /* split-plane descent of the staged levels (2 or 4 tiles per warp on
                                line paths 1 and 4; other plans ignore it): P >= 2 = levels 1 .. P - 1
                                are staged as a plane of the nodes' high 32-bit words followed by a
                                plane of their low words and probed with 4-byte loads (fewer
                                shared-memory bank conflicts), a low word read only when a lane of
                                the warp ties on a high word; deeper staged levels keep the packed
                                8-byte keys. 0 (default) or 1 = packed everywhere. Kernels exist for
                                P = 2, 3 and every staged level (P >= smem_levels, reported as
                                smem_levels; other values run as 3), on trees of depth >= 3 with all
                                or all but one internal level staged. Results are identical; the
                                tuner picks P with the line path (levels whose high words tie often
                                are better left packed). */
} lpm6cu_kernel_config;

typedef struct lpm6cu_fib lpm6cu_fib;
typedef struct lpm6cu_querygen lpm6cu_querygen;

const char* lpm6cu_last_error(void);
const char* lpm6cu_status_name(int status);
const char* lpm6cu_version(void);

/* ---- host-side FIB build (no GPU needed) ---------------------------------- */

/* build_intervals (intervals.cpp:33-93): boundaries/next_hops need capacity >= 2n+1. */
int lpm6_build_intervals(const lpm6cu_prefix* rules, uint64_t n, uint32_t default_next_hop,
                         int merge_adjacent, uint64_t* boundaries, uint32_t* next_hops,
                         uint64_t capacity, uint64_t* m_out);

/* Geometry for m boundaries at a next-hop width of value_bytes. */
int lpm6_plan_layout(uint64_t m, uint32_t value_bytes, lpm6cu_geometry* g);
/* The same with an explicit leaf format (lpm6cu_build_opts.leaf_format). */
int lpm6_plan_layout_ex(uint64_t m, uint32_t value_bytes, uint32_t leaf_format, lpm6cu_geometry* g);

/* Lay out the tree. With lines == NULL only *g is filled (to size the arrays:
 * g->total_words u64 words of lines, g->leaf_nodes * g->leaf_keys leaf values).
 * leaf_values (optional) receives the next hop of every leaf slot as u32. */
int lpm6_build_tree(const uint64_t* boundaries, const uint32_t* next_hops, uint64_t m,
                    uint32_t default_next_hop, uint32_t value_bytes, lpm6cu_geometry* g,
                    uint64_t* lines, uint32_t* leaf_values);
/* The same with an explicit leaf format (lpm6cu_build_opts.leaf_format). */
int lpm6_build_tree_ex(const uint64_t* boundaries, const uint32_t* next_hops, uint64_t m,
                       uint32_t default_next_hop, uint32_t value_bytes, uint32_t leaf_format,
                       lpm6cu_geometry* g, uint64_t* lines, uint32_t* leaf_values);

/* Parse "<ipv6>/<len> <next_hop>" (fib.cpp:72-105). */
int lpm6_parse_prefix(const char* text, lpm6cu_prefix* out, int* host_bits_masked);

/* ---- device FIB ----------------------------------------------------------- */

/* FibTable -> intervals -> B200 layout -> device memory of `device`. */
int lpm6cu_fib_build(int device, const lpm6cu_prefix* rules, uint64_t n, uint32_t default_next_hop,
                     const lpm6cu_build_opts* opts, lpm6cu_fib** out);

/* The same build done entirely on the GPU: rules (host or device
 * memory) -> intervals -> layout, bit-identical to lpm6cu_fib_build. Stream-ordered
 * on `stream`; returns when the FIB is ready. */
int lpm6cu_fib_build_device(int device, const lpm6cu_prefix* rules, uint64_t n, uint32_t default_next_hop,
                            const lpm6cu_build_opts* opts, void* stream, lpm6cu_fib** out);

/* Device-built intervals copied to host arrays (capacity >= 2n+1), for checking
 * against lpm6_build_intervals and the reference. */
int lpm6cu_build_intervals_device(int device, const lpm6cu_prefix* rules, uint64_t n, uint32_t default_next_hop,
                                  int merge_adjacent, uint64_t* boundaries, uint32_t* next_hops,
                                  uint64_t capacity, uint64_t* m_out);

/* From a host layout (lpm6_build_tree output); copies into device memory it owns. */
int lpm6cu_fib_create(int device, const lpm6cu_geometry* g, const uint64_t* lines, lpm6cu_fib** out);

/* Over a device line array the caller owns (e.g. filled by an NCCL broadcast); not
 * freed by lpm6cu_fib_destroy. */
int lpm6cu_fib_wrap_device(int device, const lpm6cu_geometry* g, const void* d_lines, lpm6cu_fib** out);

/* Like wrap_device, but the handle takes ownership: cudaFree on destroy. */
int lpm6cu_fib_adopt_device(int device, const lpm6cu_geometry* g, void* d_lines, lpm6cu_fib** out);

/* Single-process replication: broadcast src's line array to
 * devices[1..ndev-1] with one grouped ncclBroadcast over NVLink (devices[0] must
 * be src's device; out[0] is a fresh copy there). NCCL is loaded at run time
 * (libnccl.so.2); failures report LPM6CU_E_NCCL. The one-process-per-GPU path
 * broadcasts the same array with torch.distributed (dispatch.py). */
int lpm6cu_fib_replicate(const lpm6cu_fib* src, const int* devices, int ndev, lpm6cu_fib** out);

int lpm6cu_fib_geometry(const lpm6cu_fib* fib, lpm6cu_geometry* g);
int lpm6cu_fib_device_lines(const lpm6cu_fib* fib, const void** d_lines);
/* Copy the device line array (g.total_words u64 words) to host memory. */
int lpm6cu_fib_copy_lines(const lpm6cu_fib* fib, uint64_t* host_lines, uint64_t words);
int lpm6cu_fib_set_kernel_config(lpm6cu_fib* fib, const lpm6cu_kernel_config* cfg);
int lpm6cu_fib_kernel_config(const lpm6cu_fib* fib, lpm6cu_kernel_config* cfg);
/* Times the line paths on a representative batch (device buffers; two interleaved
 * rounds of `reps` timed launches per path after one untimed, the faster round
 * kept; on `stream`, which it synchronizes) — the texture leaf paths 1 and 4 also
 * with 2 and 4 tiles per warp (queries_per_lane, at 1024 threads) and, on those, the
 * split-plane descent (plane_levels 2, 3 and every staged level) — keeps the
 * fastest in the kernel config and returns its line path in *line_path (0..4, see
 * lpm6cu_kernel_config; 3 only when the tree has internal L2 levels, 4 only with
 * 1-byte next hops). Results are
 * identical on every path; like the other tuning calls it must not race with
 * lookups on the handle. */
int lpm6cu_fib_tune_line_path(lpm6cu_fib* fib, const void* d_addrs, uint64_t n, void* d_out, void* stream,
                              uint32_t reps, uint32_t* line_path);
/* Waits for the device (as cudaFree would), then releases the handle's memory; device-built
 * line arrays return to a library-private pool instead of being unmapped. */
void lpm6cu_fib_destroy(lpm6cu_fib* fib);

/* Checked mode: lookups run a bounds-checked kernel that never reads outside the
 * tree and records violations (only a corrupted tree can cause one: bit 0 node
 * index past a shared-memory level, bit 1 past an L2 level, bit 2 leaf rank 0). */
int lpm6cu_fib_set_checked(lpm6cu_fib* fib, int on);
/* OR of the violation bits since the last reset (synchronizes the device). */
int lpm6cu_fib_violations(lpm6cu_fib* fib, uint32_t* bits, int reset);
/* Checked mode also counts the tree lines each query visited (shared-memory
 * image levels included): always depth + 1 per query. */
int lpm6cu_fib_node_visits(lpm6cu_fib* fib, uint64_t* visits, int reset);

/* ---- lookup --------------------------------------------------------------- */

/* n next hops for n addresses. With device pointers: one kernel launch on
 * `stream` (a cudaStream_t; NULL = legacy default), asynchronous, no host sync,
 * no allocation — when `out` is 4*value_bytes-byte aligned; at any other byte
 * offset the results go through a stream-ordered scratch buffer and one
 * device-to-device copy. With host pointers: page-locked buffers of up to 2^20
 * queries are read and written by the kernel over PCIe (zero-copy: one launch,
 * one sync); larger or pageable buffers go through a chunked host->device copy /
 * lookup / device->host copy pipeline. Either way the work is ordered after
 * `stream` and the call returns when `out` holds the results. */
int lpm6cu_lookup_batch(const lpm6cu_fib* fib, const void* addrs, uint64_t n, void* out,
                        void* stream);

/* The serving-size fast path of lpm6cu_lookup_batch for buffers the caller knows
 * are device memory on the FIB's device (the reference's search_batch over keys
 * already in memory): no pointer-kind queries, no host pipeline — the
 * launch only (plus the device switch when the calling thread is on another
 * device). Host pointers here are undefined behaviour (the kernel faults). */
int lpm6cu_lookup_batch_device(const lpm6cu_fib* fib, const void* d_addrs, uint64_t n, void* d_out,
                               void* stream);

/* 8-byte keys instead of 16-byte addresses — the input of the reference's
 * search_batch(t, keys[B]) and of its PBTR traces. Keys are clamped
 * like address keys. Device buffers: one kernel launch on `stream`; host buffers:
 * the pipelined H2D / kernel / D2H path with half the PCIe bytes of addresses. */
int lpm6cu_lookup_keys(const lpm6cu_fib* fib, const uint64_t* keys, uint64_t n, void* out, void* stream);

/* search_batch: for n 8-byte keys, the interval ordinal of each —
 * SearchResult::interval_ordinal, the index i into the interval map with
 * boundaries[i] <= key < boundaries[i+1] — and, when next_hops is not NULL, its
 * next hop. Device buffers; one kernel launch on `stream`. */
int lpm6cu_search_batch(const lpm6cu_fib* fib, const uint64_t* keys, uint64_t n, uint32_t* ordinals, void* next_hops,
                        void* stream);

/* Packet-path ingest: n frames `stride` bytes apart in device memory
 * (e.g. a NIC RX ring written by GPUDirect), the IPv6 destination address at byte
 * `dst_offset` of each frame in network byte order (38 for Ethernet + IPv6). The
 * kernel reads the destination's first 8 bytes straight from the frame — no
 * separate extraction pass — and writes one next hop per frame. */
int lpm6cu_lookup_packets(const lpm6cu_fib* fib, const void* frames, uint64_t n, uint64_t stride, uint32_t dst_offset,
                          void* out, void* stream);

/* The layout step alone on the GPU, from host intervals (an IntervalMap:
 * boundaries[0] = 0, strictly increasing, no sentinel, no reserved next hop) —
 * the device counterpart of build_tree(map) (tree.hpp:74). merge_adjacent in
 * opts is ignored (the map is final). */
int lpm6cu_fib_build_from_intervals(int device, const uint64_t* boundaries, const uint32_t* next_hops, uint64_t m,
                                    uint32_t default_next_hop, const lpm6cu_build_opts* opts, void* stream,
                                    lpm6cu_fib** out);

/* ---- reference file formats ---------------------------------------
 * PBT1 snapshot (tree.hpp:90-96): "PBT1", u16 version 1, u16 k, u16 depth,
 * u64 m, u64 allocated_leaf_nodes (26 header bytes), the reference LinearizedTree's
 * keys (u64 LE) and values (u32 LE). PBTR trace: "PBTR", u16 version 1,
 * u16 reserved, u64 count, count u64 LE keys. Errors: BadSnapshotFile /
 * BadTraceFile / Io. */

/* Interval map -> PBT1 bytes in the reference layout at k keys per node (8 = the
 * reference default). buf NULL: *size only. */
int lpm6_snapshot_encode(const uint64_t* boundaries, const uint32_t* next_hops, uint64_t m, uint32_t k, void* buf,
                         uint64_t cap, uint64_t* size);
int lpm6_snapshot_save(const uint64_t* boundaries, const uint32_t* next_hops, uint64_t m, uint32_t k,
                       const char* path);
/* Validate a PBT1 image and extract its interval map (arrays NULL: *m, *k only). */
int lpm6_snapshot_decode(const void* buf, uint64_t size, uint64_t* boundaries, uint32_t* next_hops, uint64_t cap,
                         uint64_t* m, uint32_t* k);
/* memory_footprint (tree.hpp:76-88): exact bytes of each array. */
typedef struct {
  uint64_t leaf_bytes;     /* leaf keys (B200: whole leaf lines, next hops included) */
  uint64_t internal_bytes; /* internal levels */
  uint64_t value_bytes;    /* separate value array (reference: u32 per leaf slot; B200: 0) */
  uint64_t image_bytes;    /* B200: the shared-memory image copy (reference: 0) */
  uint64_t total_bytes;
  double bytes_per_interval;
  uint64_t total_bytes_value8;       /* with 8-byte value slots (the paper's 18 B/interval basis) */
  double bytes_per_interval_value8;
} lpm6cu_footprint;
int lpm6_memory_footprint(const lpm6cu_geometry* g, lpm6cu_footprint* out);
/* The reference layout's footprint for m intervals at k keys per node. */
int lpm6_ref_memory_footprint(uint64_t m, uint32_t k, lpm6cu_footprint* out);

/* PBT1 file -> device FIB without an interval sweep (load_snapshot_file, tree.hpp:96). */
int lpm6cu_fib_load_snapshot(int device, const char* path, uint32_t default_next_hop, const lpm6cu_build_opts* opts,
                             void* stream, lpm6cu_fib** out);
int lpm6_trace_save(const uint64_t* keys, uint64_t n, const char* path);
/* Validate a PBTR image in memory; *n = key count. */
int lpm6_trace_count(const void* buf, uint64_t size, uint64_t* n);
/* PBTR file -> d_keys (device, capacity cap keys) through pinned double-buffered
 * staging, ordered on `stream`; returns when the keys are resident. d_keys NULL:
 * validate and count only. */
int lpm6cu_trace_load(int device, const char* path, uint64_t* d_keys, uint64_t cap, uint64_t* count, void* stream);

/* ---- rebuild-and-swap FIB store (SPEC update-engine) ---
 *
 * Replaces the reference's FibStore: route changes are staged,
 * commit rebuilds the whole FIB on the GPU (lpm6cu_fib_build_device, off the
 * lookup streams) and publishes it with one pointer swap; readers pin a snapshot
 * with acquire/release and never wait for a commit. Release is stream-ordered:
 * it records an event on the reader's stream, and a retired snapshot's device
 * memory is freed only after its last release AND every lookup queued before
 * those releases has finished on the device. */

enum {
  LPM6_UPDATE_INSERT = 0,   /* must not exist (DuplicatePrefix) */
  LPM6_UPDATE_DELETE = 1,   /* must exist (UnknownPrefix); next_hop ignored */
  LPM6_UPDATE_MODIFY = 2,   /* must exist (UnknownPrefix) */
  LPM6_UPDATE_ANNOUNCE = 3, /* insert-or-modify: the trace's "A" line */
};

/* lpm6::UpdateOp; 48 bytes. */
typedef struct {
  uint32_t kind;
  uint32_t reserved0;
  uint64_t reserved1;
  lpm6cu_prefix prefix;
} lpm6_update_op;

typedef struct {
  uint64_t epoch;         /* active snapshot's epoch: 1 after create, +1 per effective commit */
  uint64_t pending_ops;   /* staged, not yet committed */
  uint64_t active_rules;  /* rules in the active snapshot */
  uint64_t retired;       /* snapshots replaced but not yet reclaimed */
  uint64_t reclaimed;     /* snapshots whose device memory was freed */
  uint64_t commits;       /* effective commits */
  double last_build_ms;   /* wall time of the last device rebuild */
  double last_publish_us; /* time the active-pointer swap was held */
  uint64_t fences;        /* outstanding release fences over all snapshots (<= reader streams each) */
} lpm6cu_store_stats;

typedef struct lpm6cu_store lpm6cu_store;
typedef struct lpm6cu_snapshot lpm6cu_snapshot;

/* Parse one update-trace line "A <ipv6>/<len> <next_hop>" | "W <ipv6>/<len> [next_hop]". */
int lpm6_parse_update(const char* line, lpm6_update_op* op);

/* The store's staging rule on host arrays (no GPU): apply ops in order to the rule
 * set `rules` (n entries); op_status[i] (optional) receives 0 or the status of op i,
 * invalid ops are skipped. The resulting rules go to out (capacity cap; order is
 * the store's, not sorted) and *out_n; *staged counts the applied ops. */
int lpm6_apply_updates(const lpm6cu_prefix* rules, uint64_t n, const lpm6_update_op* ops, uint64_t n_ops,
                       lpm6cu_prefix* out, uint64_t cap, uint64_t* out_n, uint64_t* staged, int32_t* op_status);

/* Epoch 1 = rules built on `device`. opts as lpm6cu_fib_build (value_bytes 0 =
 * re-derived at every commit). */
int lpm6cu_store_create(int device, const lpm6cu_prefix* rules, uint64_t n, uint32_t default_next_hop,
                        const lpm6cu_build_opts* opts, lpm6cu_store** out);
/* Waits for every outstanding release fence; fails (InvalidArgument) while a
 * snapshot is still acquired. */
int lpm6cu_store_destroy(lpm6cu_store* store);
/* Validate and append ops (any thread). Invalid ops are skipped and reported in
 * op_status (optional, n entries: 0 or a status); *staged = ops appended. */
int lpm6cu_store_stage(lpm6cu_store* store, const lpm6_update_op* ops, uint64_t n, uint64_t* staged,
                       int32_t* op_status);
/* Rebuild from the staged view and publish (one committer at a time). Empty
 * pending: no-op. On failure (e.g. SentinelCollision) the old snapshot stays
 * active and the pending ops stay staged. *epoch (optional) = active epoch. */
int lpm6cu_store_commit(lpm6cu_store* store, uint64_t* epoch);
/* Pin the current snapshot. */
int lpm6cu_store_acquire(lpm6cu_store* store, lpm6cu_snapshot** snap);
/* Unpin. Work already queued on `stream` (cudaStream_t, NULL = legacy default)
 * that uses the snapshot keeps it alive until it finishes on the device. */
int lpm6cu_store_release(lpm6cu_snapshot* snap, void* stream);
/* The snapshot's epoch, device FIB (for lpm6cu_lookup_batch) and rule count. */
int lpm6cu_snapshot_info(const lpm6cu_snapshot* snap, uint64_t* epoch, const lpm6cu_fib** fib, uint64_t* n_rules);
/* Copy the snapshot's rules (n_rules entries, store order). */
int lpm6cu_snapshot_rules(const lpm6cu_snapshot* snap, lpm6cu_prefix* out, uint64_t cap);
/* acquire -> lpm6cu_lookup_batch -> release(stream) in one call. */
int lpm6cu_store_lookup_batch(lpm6cu_store* store, const void* addrs, uint64_t n, void* out, void* stream,
                              uint64_t* epoch);
/* Free retired snapshots whose fences have completed (non-blocking). */
int lpm6cu_store_reclaim(lpm6cu_store* store);
int lpm6cu_store_stats_get(lpm6cu_store* store, lpm6cu_store_stats* stats);

/* ---- synthetic workloads C0..C4 (BASELINE.json configs) ---------------------- */

typedef struct {
  int32_t id;         /* 0 C0, 1 C1, 2 C2, 3 C3a, 4 C3b, 5 C4 */
  int32_t fib_kind;   /* 0: C0 FIB, 1: 200K backbone FIB, 2: 1M projected FIB */
  uint64_t n_queries;
  uint64_t chunk;     /* queries per chunk (C4), 0 = one */
  uint32_t value_bytes;
  uint32_t reserved;
  char name[8];
} lpm6_workload_info;

int lpm6_workload_info_get(int workload, lpm6_workload_info* info);

/* The FIB of fib_kind; with out == NULL only *n_out / *default_next_hop are set. */
int lpm6_workload_fib(int fib_kind, lpm6cu_prefix* out, uint64_t capacity, uint64_t* n_out,
                      uint32_t* default_next_hop);

/* Queries [first, first+n) of `workload` over `rules`, generated on the host. */
int lpm6_workload_queries_host(int workload, const lpm6cu_prefix* rules, uint64_t nrules,
                               uint64_t first, uint64_t n, void* out_addrs, int threads);

/* The same queries generated on the GPU (bit-identical to the host generator). */
int lpm6cu_querygen_create(int device, int workload, const lpm6cu_prefix* rules, uint64_t nrules,
                           lpm6cu_querygen** out);
int lpm6cu_querygen_run(const lpm6cu_querygen* gen, uint64_t first, uint64_t n, void* d_out_addrs,
                        void* stream);
void lpm6cu_querygen_destroy(lpm6cu_querygen* gen);

/* ---- measurement probes (roofline denominators) ----------------------------- */

/* Random gather of `line_bytes`-sized lines (32 or 128) from an L2-resident
 * buffer of `buffer_bytes`; returns achieved GB/s of requested bytes. */
int lpm6cu_probe_l2_gather(int device, uint64_t buffer_bytes, uint32_t line_bytes, double* gbps);
/* Shared-memory read bandwidth (all SMs, conflict-free 128-byte rows), GB/s. */
int lpm6cu_probe_smem(int device, double* gbps);

#ifdef __cplusplus
}
#endif
#endif /* LPM6CU_H */
