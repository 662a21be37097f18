/*
 * pyrit_b200.h -- C ABI of the B200-native PYRIT ring codec.
 *
 * Drop-in boundary for the reference's hot path (paths relative to
 * /root/reference/proj/include/pyrit/):
 *
 *   reference (C++, header only)                    here
 *   ----------------------------------------------  -------------------------------
 *   FieldSpec            field.hpp:30-51          pyrit_field
 *   CodeSpec             matrix.hpp:16-23         pyrit_code
 *   cauchy_parity_matrix matrix.hpp:54-80         pyrit_cauchy_parity_matrix
 *   decode_matrix        matrix.hpp:193-220         pyrit_decode_matrix
 *   sparse_transform     ring.hpp:77-90             pyrit_sparse_transform
 *   compile_schedule     schedule.hpp:94-163        pyrit_plan_create (+ _encode/_decode)
 *   schedule_stats       schedule.hpp:216-223       pyrit_plan_get_stats
 *   replay / parallel_replay codec.hpp:118-193      pyrit_cu_apply, pyrit_apply_host
 *   RingElem masks (to_shift_set) ring.hpp:94-102   pyrit_ringmat, pyrit_cu_apply_ringmat
 *   (any XorSchedule)    schedule.hpp:40-58         pyrit_plan_from_schedule
 *   encode               codec.hpp:212-220          pyrit_cu_encode   (device buffers)
 *   encode_crs           codec.hpp:223-231          pyrit_cu_encode_crs
 *                                                    pyrit_encode_host (host buffers)
 *   decode               codec.hpp:241-284          pyrit_cu_decode   (device buffers)
 *                                                    pyrit_decode_host (host buffers)
 *   (per-stripe calls)   container.hpp:207-218      pyrit_cu_encode_batch / _decode_batch
 *   serialize/parse_header container.hpp:114-161    pyrit_header_serialize / _parse
 *   encode_file          container.hpp:168-222      pyrit_encode_file
 *   decode_file          container.hpp:249-299      pyrit_decode_file
 *   Errc / Error         errors.hpp:12-39           return codes, pyrit_strerror
 *
 * Symbols are bit-sliced exactly as SymbolBuffer stores them
 * (codec.hpp:24-73): a symbol of symbol_size bytes is w contiguous strips
 * of symbol_size / w bytes, strip i holding coefficient i of every bit
 * column.  symbol_size must be a positive multiple of w and of 8
 * (codec.hpp:28-30).
 *
 * Return codes: 0 ok; 1 + Errc (1..11, errors.hpp:12-24) for argument,
 * shape and algebra errors; negative for device failures: -e for a
 * cudaError_t e, -1000 - r for an nvrtcResult r, -2000 - r for a driver
 * CUresult r.  Nothing throws across this boundary.
 *
 * Ownership: the caller owns every buffer; device entry points allocate
 * nothing per call and run asynchronously on the given stream (a
 * cudaStream_t passed as void*; NULL = legacy default stream).  Plans are
 * immutable once created and may be used from any thread concurrently.
 */
#ifndef PYRIT_B200_H
#define PYRIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* field.hpp:30-51 (ring elements widened: n <= 32, any p | x^n + 1) */
typedef struct pyrit_field {
    uint32_t w;       /* extension degree, elements are w-bit (<= 16) */
    uint32_t n;       /* ring length, w < n <= 32 */
    uint32_t kind;    /* 0 = Aop, 1 = Esp (FieldKind, field.hpp:14-17) */
    uint32_t s;       /* coefficient spacing */
    uint32_t r_esp;   /* degree of the ESP base polynomial (w for AOP) */
    uint32_t modulus; /* p(x), bit i = coefficient of x^i */
} pyrit_field;

/* matrix.hpp:16-23 */
typedef struct pyrit_code {
    uint32_t k;         /* data symbols */
    uint32_t r;         /* parity symbols */
    pyrit_field field;
    uint32_t transform; /* 0 = Embedding, 1 = Parity (transform.hpp:24) */
} pyrit_code;

/* schedule.hpp:61-67 ScheduleStats, extended with the fused-program counts */
typedef struct pyrit_plan_stats {
    uint32_t rows, cols;       /* outputs x inputs */
    uint64_t matrix_ones;      /* sum of representative weights x w (schedule.hpp:112) */
    uint64_t ref_region_ops;   /* ops compile_schedule emits (pre+core+post), generalized fold */
    uint64_t naive_xors;       /* 2-input XORs of the unshared ring program */
    uint64_t xors;             /* 2-input XORs of the compiled program */
    uint64_t loads, stores;    /* strip words read / written per column word */
    uint32_t group;            /* input symbols whose strips are live together */
    uint32_t parts;            /* output parts (row groups) of the staged / split kernels */
    uint64_t part_xors;        /* 2-input XORs per column word summed over the parts */
} pyrit_plan_stats;

typedef struct pyrit_plan pyrit_plan;

/* ---- host algebra ---------------------------------------------------- */
const char* pyrit_version(void);
const char* pyrit_strerror(int code);

/* FieldSpec::gf16_aop / gf64_esp (field.hpp:38-43) and the BASELINE fields */
int pyrit_field_named(const char* name, pyrit_field* out); /* "gf16", "gf64", "gf256_r17", "gf1024", "gf4096" */
int pyrit_field_validate(const pyrit_field* f);
int pyrit_gf_mul(const pyrit_field* f, uint32_t a, uint32_t b, uint32_t* out);   /* field.hpp:68 */
int pyrit_gf_inv(const pyrit_field* f, uint32_t a, uint32_t* out);               /* field.hpp:82 */
int pyrit_sparse_transform(const pyrit_field* f, uint32_t u, uint32_t* rep);     /* ring.hpp:77 */
int pyrit_fold_table(const pyrit_field* f, uint32_t* fold /* n - w entries */);  /* x^t mod p */
/* out: r x k row-major (matrix.hpp:54) */
int pyrit_cauchy_parity_matrix(const pyrit_code* code, uint16_t* out);
/* out: (#erased data) x k rows of A^-1, survivors in given order (matrix.hpp:193) */
int pyrit_decode_matrix(const pyrit_code* code, const uint32_t* survivors, uint16_t* out, uint32_t* rows);
/* fused repair matrix: survivors (k, lowest index first), outputs (erased,
 * data then parity, each ascending), matrix outputs x k */
int pyrit_repair_matrix(const pyrit_code* code, const uint32_t* erased, uint32_t n_erased,
                        uint32_t* survivors, uint32_t* outputs, uint16_t* matrix);

/* ---- compiled plans (schedule.hpp:94 compile_schedule) ---------------- */
/* rep: 0 = RingRep::Sparse (minimal weight), 1 = Dense (schedule.hpp:78),
 * 2 = the plain-field Cauchy-RS bitmatrix program instead of the ring
 * (compile_crs_schedule, schedule.hpp:168-203: the GPU CRS baseline);
 * group: input symbols per register group, 0 = automatic */
int pyrit_plan_create(const pyrit_field* f, uint32_t transform, const uint16_t* matrix, uint32_t rows,
                      uint32_t cols, uint32_t rep, uint32_t group, pyrit_plan** out);
int pyrit_plan_encode(const pyrit_code* code, pyrit_plan** out);
int pyrit_plan_decode(const pyrit_code* code, const uint32_t* erased, uint32_t n_erased, pyrit_plan** out,
                      uint32_t* survivors, uint32_t* outputs);
int pyrit_plan_get_stats(const pyrit_plan* plan, pyrit_plan_stats* out);
/* Negative control (the reference's hidden `pyrit verify --inject-theta-fault`,
 * tools/pyrit.cpp:281-282, selfcheck.hpp:28-34, flips one bit of the embedding
 * idempotent): flip bit `bit` of the ring representative of matrix entry
 * `entry` (row-major) and recompile the plan, so that tests can show the GPU
 * parity checks detect a wrong program.  Test hook; never used by the codec. */
int pyrit_plan_inject_fault(pyrit_plan* plan, uint32_t entry, uint32_t bit);
int pyrit_plan_reps(const pyrit_plan* plan, uint32_t* reps /* rows x cols */);
/* key of the plan in the staged-kernel tuning table (tuned.tsv next to the library) */
int pyrit_plan_key(const pyrit_plan* plan, char* buf, size_t cap);
/* generated CUDA source of the fused kernel; *len receives the full size.
 * lanes: 1/2/4 = direct LDG kernel with that many 32-bit words per thread per
 * strip, 0 = byte mode, PYRIT_SOURCE_STAGED = the staged kernel (its
 * producer as chosen for the plan; PYRIT_SOURCE_STAGED + 1 = the variant for
 * equally spaced inputs -- one 4D TMA map; + 8 / + 4 = cp.async with 8- / 4-byte
 * chunks for strips with only that alignment) */
#define PYRIT_SOURCE_STAGED 100u
int pyrit_plan_source(const pyrit_plan* plan, uint32_t lanes, char* buf, size_t cap, size_t* len,
                      char* name, size_t name_cap);
/* verification aid: interprets the compiled program on HOST buffers (no
 * device involved); used to test the compiler where no GPU exists */
int pyrit_plan_interpret(const pyrit_plan* plan, const uint8_t* const* in, uint8_t* const* out,
                         uint64_t strip_bytes, uint64_t off, uint64_t len);
/* verification aid: runs, on HOST buffers, the launch plan the runtime-matrix
 * ring kernel would get for this stripe batch (output groups and parts, op
 * lists read back from its kernel parameters) -- the CPU check of that planner.
 * Same arguments as pyrit_cu_apply_batch minus the stream; buffers 16-byte
 * aligned, strip/off/len multiples of 16, a ring geometry with an AOT kernel. */
int pyrit_rt_interpret(const pyrit_plan* plan, const uint8_t* const* in, uint8_t* const* out, uint64_t strip_bytes,
                       uint64_t off, uint64_t len, uint64_t stripes, uint64_t in_pitch, uint64_t out_pitch);
/* verification aid: how the runtime-matrix planner would run this plan, no device
 * involved: info[0] launches, info[1] ring terms of the matrix (set bits of the
 * representatives, schedule.hpp:132-161), info[2] ops the launches run for them (a
 * paired-shift op covers two terms with 3-input XORs), info[3] bytes of dispatch-case
 * code the largest launch names (kept within the instruction cache) */
int pyrit_rt_plan_info(const pyrit_plan* plan, uint32_t info[4]);
void pyrit_plan_destroy(pyrit_plan* plan);

/* ---- a raw ring-representative matrix (SURVEY 8(b) pyrit_cu_ringmat) --- */
/* rows x cols ring elements, row-major n-bit shift masks: the reference's
 * RingElem / to_shift_set form (ring.hpp:94-102, schedule.hpp:78), any
 * element of each coset under the Embedding transform -- it stands for the
 * field element u mod p (phi_E^{-1}); the Parity transform takes the
 * canonical (sparse_transform) representative only.  Applied by the runtime-matrix ring kernel with the masks in
 * its kernel parameters: no code generation and no compile (16-byte aligned
 * buffers, strip, window; the AOT ring geometries -- anything else runs the
 * generated kernel of the field matrix, the same symbols). */
typedef struct pyrit_ringmat {
    pyrit_field field;
    uint32_t transform; /* 0 Embedding, 1 Parity */
    uint32_t rows, cols;
    const uint32_t* reps;
} pyrit_ringmat;
/* a plan of it (all the pyrit_cu_apply* / interpret entry points take it) */
int pyrit_plan_from_ringmat(const pyrit_ringmat* m, pyrit_plan** out);
/* one call: out[i] = sum_j reps[i][j] * in[j] over the window, the program
 * cached by matrix (replay, codec.hpp:118-157, with the masks as the operand) */
int pyrit_cu_apply_ringmat(const pyrit_ringmat* m, const uint8_t* const* in, uint8_t* const* out,
                           uint64_t strip_bytes, uint64_t off, uint64_t len, void* stream);

/* ---- plans from a reference schedule (the replay operator) ------------ */
/* One region op of an XorSchedule, laid out like the reference's XorOp
 * (schedule.hpp:42-48; mode = OpMode: 0 Copy, 1 Xor, 2 Zero), so a
 * std::vector<XorOp> can be passed as is. */
typedef struct pyrit_xor_op {
    uint16_t src_sym, src_pkt, dst_sym, dst_pkt;
    uint8_t mode;
} pyrit_xor_op;
/* Compiles any XorSchedule -- compile_schedule / compile_crs_schedule output
 * or hand-written -- into one fused GPU kernel with replay()'s semantics
 * (codec.hpp:118-157): ops = pre, core, post concatenated in replay order;
 * sym < k is input slot sym (in_map), sym >= k output slot sym - k
 * (out_map); packets >= w are workspace scratch, zero at entry (the fresh
 * Workspace parallel_replay makes, codec.hpp:176-193).  labels (k + outputs
 * entries, or NULL = all distinct): slots with equal labels share storage
 * (decode() replays with one SymbolBuffer as in and out), so a write
 * through one slot is seen by later reads through another.  Output packets
 * no op writes are left untouched.  Errors as replay: BufferShape for a
 * slot/packet out of range or a write to an input data packet.
 * The plan is applied with pyrit_cu_apply / _batch / pyrit_apply_host with
 * in[k] and out[outputs] indexed by slot. */
int pyrit_plan_from_schedule(const pyrit_field* f, uint32_t k, uint32_t outputs, const pyrit_xor_op* ops,
                             size_t n_ops, const uint32_t* labels, pyrit_plan** out);

/* ---- device path ------------------------------------------------------ */
/* replay (codec.hpp:118): window [off, off+len) of every strip; in[j] /
 * out[i] are device base pointers of the input / output symbols */
int pyrit_cu_apply(const pyrit_plan* plan, const uint8_t* const* in, uint8_t* const* out, uint64_t strip_bytes,
                   uint64_t off, uint64_t len, void* stream);
/* compile + load the plan's kernel for the current device (no launch) */
int pyrit_cu_prepare(const pyrit_plan* plan);
/* encode (codec.hpp:212): data[k], parity[r] device symbol pointers */
int pyrit_cu_encode(const pyrit_code* code, const uint8_t* const* data, uint8_t* const* parity,
                    uint64_t symbol_size, void* stream);
/* encode_crs (codec.hpp:223-231): the same parity through the plain-field
 * Cauchy-RS bitmatrix program (compile_crs_schedule) -- the baseline codec */
int pyrit_cu_encode_crs(const pyrit_code* code, const uint8_t* const* data, uint8_t* const* parity,
                        uint64_t symbol_size, void* stream);
/* decode (codec.hpp:241): symbols[k + r] device pointers, repaired in place */
int pyrit_cu_decode(const pyrit_code* code, uint8_t* const* symbols, const uint32_t* erased, uint32_t n_erased,
                    uint64_t symbol_size, void* stream);

/* ---- stripe batches (encode_file / decode_file call encode()/decode()
 * once per stripe, container.hpp:207-218, :284-297; here one launch covers
 * `stripes` stripes).  Input symbol j of stripe b is at in[j] + b * in_pitch,
 * output i at out[i] + b * out_pitch; each symbol is w strips of
 * strip_bytes (apply) or symbol_size / w (encode/decode) bytes. */
int pyrit_cu_apply_batch(const pyrit_plan* plan, const uint8_t* const* in, uint8_t* const* out,
                         uint64_t strip_bytes, uint64_t off, uint64_t len, uint64_t stripes, uint64_t in_pitch,
                         uint64_t out_pitch, void* stream);
int pyrit_cu_encode_batch(const pyrit_code* code, const uint8_t* const* data, uint8_t* const* parity,
                          uint64_t symbol_size, uint64_t stripes, uint64_t data_pitch, uint64_t parity_pitch,
                          void* stream);
/* symbols[k + r]: symbol i of stripe b at symbols[i] + b * pitch, repaired in place */
int pyrit_cu_decode_batch(const pyrit_code* code, uint8_t* const* symbols, const uint32_t* erased,
                          uint32_t n_erased, uint64_t symbol_size, uint64_t stripes, uint64_t pitch, void* stream);

/* ---- host-buffer path (end to end: H2D, fused kernel, D2H, pipelined) -- */
/* parallel_replay / replay (codec.hpp:118-193) on HOST symbols: in[j] /
 * out[i] are host base pointers (w strips of strip_bytes each), window
 * [off, off+len) of every strip.  Synchronous. */
int pyrit_apply_host(const pyrit_plan* plan, const uint8_t* const* in, uint8_t* const* out, uint64_t strip_bytes,
                     uint64_t off, uint64_t len, int device);
/* data: k * symbol_size contiguous host bytes (SymbolBuffer layout);
 * parity: r * symbol_size host bytes.  Synchronous. Pinned buffers overlap. */
int pyrit_encode_host(const pyrit_code* code, const uint8_t* data, uint8_t* parity, uint64_t symbol_size,
                      int device);
/* the same over several GPUs of one process: every strip is split into
 * byte-offset shards (16-byte aligned), one per listed device, processed
 * concurrently with no exchange; a device may repeat */
int pyrit_encode_host_devices(const pyrit_code* code, const uint8_t* data, uint8_t* parity, uint64_t symbol_size,
                              const int* devices, uint32_t n_devices);
int pyrit_decode_host_devices(const pyrit_code* code, uint8_t* symbols, const uint32_t* erased, uint32_t n_erased,
                              uint64_t symbol_size, const int* devices, uint32_t n_devices);
/* encode_crs (codec.hpp:223-231) with host buffers */
int pyrit_encode_crs_host(const pyrit_code* code, const uint8_t* data, uint8_t* parity, uint64_t symbol_size,
                          int device);
/* symbols: (k + r) * symbol_size host bytes, repaired in place.  Synchronous. */
int pyrit_decode_host(const pyrit_code* code, uint8_t* symbols, const uint32_t* erased, uint32_t n_erased,
                      uint64_t symbol_size, int device);
/* bytes per strip per pipeline chunk (0 = automatic) */
int pyrit_set_host_chunk(uint64_t strip_chunk_bytes);
/* Multi-GPU hosts: restrict the CALLING thread to the CPUs of the NUMA node the device's
 * PCIe slot belongs to, so the host buffers it allocates and touches next (and the copies it
 * makes) are local to that GPU's link -- call it in each per-GPU worker before allocating its
 * pinned buffers (the reference's parallel_replay workers, codec.hpp:176-193, have no such
 * notion: they share one memory).  Best effort: returns the node, or -1 (and changes nothing)
 * when the platform does not say, PYRIT_B200_NUMA=0, or the node's CPUs are outside the
 * process's cpuset.  pyrit_*_host_devices does this for its per-device threads. */
int pyrit_numa_bind_thread(int device);
/* the same from a sysfs-style CPU list ("0-13,28-41") for callers that know their topology:
 * the calling thread keeps the listed CPUs it is allowed on; returns the CPUs listed, or -1
 * (nothing changed) for an empty or malformed list or one disjoint from the thread's cpuset */
int pyrit_bind_thread_cpulist(const char* cpulist);

/* ---- shard container and file codec (container.hpp) ------------------ */
#define PYRIT_HEADER_SIZE 29 /* container.hpp:38 */
/* container.hpp:57-84; serialized little-endian as container.hpp:16-36 */
typedef struct pyrit_shard_header {
    uint8_t version;   /* 1 */
    uint8_t field;     /* field id (pyrit_field_id) */
    uint8_t transform; /* 0 = Embedding, 1 = Parity */
    uint16_t k, r, shard_index;
    uint32_t symbol_size;
    uint64_t original_length;
} pyrit_shard_header;
uint32_t pyrit_crc32(const uint8_t* bytes, size_t len);                         /* container.hpp:41-55 */
int pyrit_header_serialize(const pyrit_shard_header* h, uint8_t* out /* 29 */); /* container.hpp:114-127 */
int pyrit_header_parse(const uint8_t* bytes, size_t len, pyrit_shard_header* out); /* container.hpp:132-161 */
/* header field ids: 0 = gf16_aop, 1 = gf64_esp (field.hpp:54-62), and for
 * the fields the reference cannot record: 2 = GF(2^8) in R_{2,17} (0x139),
 * 3 = GF(2^10) AOP, 4 = GF(2^12) AOP */
int pyrit_field_id(const pyrit_field* f, uint8_t* id);
int pyrit_field_from_id(uint8_t id, pyrit_field* out);
/* "<out_dir>/<basename(input)>.sNNN.pyrit" (container.hpp:186-189) */
int pyrit_shard_path(const char* input, const char* out_dir, uint32_t index, char* buf, size_t cap);
/* encode_file (container.hpp:168-222): writes k + r shard files; batches of
 * stripes go through `device` (pinned staging, three streams).  Synchronous. */
int pyrit_encode_file(const pyrit_code* code, const char* input, const char* out_dir, uint32_t symbol_size,
                      int device);
/* decode_file (container.hpp:249-299) from any k (or more) shard files */
int pyrit_decode_file(const char* const* shard_paths, uint32_t n_paths, const char* output, int device);
/* source bytes per pipeline chunk of the file codec (0 = automatic) */
int pyrit_set_file_chunk(uint64_t bytes);

/* ---- synthetic inputs and verification digests ----------------------- */
int pyrit_cu_fill(uint64_t seed, uint64_t frag, uint8_t* dst, uint64_t begin, uint64_t len, uint64_t valid,
                  void* stream);
/* *out (device uint64) += digest of src[0, len) whose first word has global
 * index word_offset; src 8-byte aligned */
int pyrit_cu_digest(const uint8_t* src, uint64_t len, uint64_t word_offset, uint64_t* out, void* stream);

/* ---- runtime knobs and counters -------------------------------------- */
int pyrit_set_lanes(uint32_t lanes); /* 32-bit words per thread per strip: 1, 2 or 4 */
/* 0 = auto (TMA-staged kernel whenever pointers/pitch/window are 16-byte
 * aligned and the tiles fit in shared memory), 1 = direct kernel only,
 * 2 = staged whenever possible, 3 = the generic bit-matrix kernel (no
 * per-code compilation; 4-byte aligned launches), 4 = the runtime-matrix ring
 * kernel (no per-code compilation; 16-byte aligned launches of the AOT ring
 * geometries).  In mode 0 the runtime-matrix kernel (else the generic one)
 * serves decode patterns and launches whose specialised kernel is still
 * compiling (PYRIT_B200_TIERED, default on) */
int pyrit_set_kernel_mode(int mode);
int pyrit_set_kernel_dir(const char* dir);
/* name and geometry of this thread's most recent generated-kernel launch */
int pyrit_cu_last_launch(char* kernel, size_t cap, uint32_t* blocks, uint32_t* threads);
uint64_t pyrit_jit_compiles(void);
/* wall time of the most recent kernel compile and of all compiles so far, in
 * milliseconds (NVRTC in process, or the background helper process) -- what a
 * new code or a hot erasure pattern costs before its specialised kernel runs */
int pyrit_jit_time(double* last_ms, double* total_ms);
/* which NVRTC compiles kernels that are not prebuilt: "nvrtc 12.9 (<file>)" */
int pyrit_jit_info(char* buf, size_t cap);
/* wait until every background compile started so far has finished (their
 * kernels serve the next launches): call it before capturing a CUDA graph */
int pyrit_jit_wait(void);
uint64_t pyrit_kernel_launches(void);
/* Load, on `device`, what a first call would otherwise load on its own path: the
 * runtime-matrix kernel's modules (~29 ms on the first decode of a new pattern in
 * a process otherwise).  Optional; for services that want flat first-call latency. */
int pyrit_warmup(int device);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif

#endif /* PYRIT_B200_H */
