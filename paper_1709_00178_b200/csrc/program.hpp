// Ring program compiler: the B200 replacement for compile_schedule
// (schedule.hpp:94-163).
//
// The reference compiles a generator matrix into a flat list of
// whole-strip region ops (Copy/Xor/Zero) that replay() streams through
// memory one op at a time (codec.hpp:118-157).  Here the same ring
// semantics -- output ring row t of output i accumulates input strip
// (t - sh) mod n for every shift sh of the entry's minimal-weight
// representative, strips >= w of an embedded input are identically zero,
// and the top rows are folded back by x^t mod p -- are compiled into a
// straight-line SSA program over per-thread registers, which the code
// generator turns into one fused CUDA kernel: every input byte is read
// from HBM once and every output byte written once.
//
// XOR is associative and commutative, so the compiler is free to share
// common pairs between ring rows (greedy pair elimination inside a group
// of fragments whose strips are live in registers at the same time); the
// bytes are identical to the reference's op-by-op replay.
#pragma once

#include <atomic>
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "algebra.hpp"

namespace pyrit_b200 {

struct Instr {
    enum Op : std::uint8_t { Load, Xor, Store } op;
    std::uint32_t dst = 0;            // Load/Xor: defined variable
    std::uint32_t sym = 0, strip = 0; // Load: input fragment/strip; Store: output fragment/strip
    std::vector<std::uint32_t> src;   // Xor/Store: XOR of these variables (Store: empty = zero)
};

struct ProgramStats {
    std::uint64_t matrix_ones = 0;   // sum of representative weights x w (schedule.hpp:112)
    std::uint64_t ref_region_ops = 0; // what compile_schedule would emit (pre + core + post)
    std::uint64_t naive_xors = 0;    // 2-input XORs of the ring program without sharing
    std::uint64_t xors = 0;          // 2-input XORs after pair elimination
    std::uint64_t loads = 0, stores = 0, vars = 0;
};

struct Program {
    Field field;
    TransformKind kind = TransformKind::Embedding;
    std::uint32_t rows = 0, cols = 0; // outputs x inputs
    std::uint32_t group = 1;          // input fragments whose strips are live together
    bool cse = true;                  // pair sharing applied
    bool crs = false;                 // plain-field bitmatrix program (compile_crs_schedule)
    bool sched = false;               // compiled from an explicit XorSchedule (bits/written below)
    std::vector<std::uint32_t> bits;  // sched: rows x cols x w masks, bit c of [(i*cols+j)*w+b] = strip c of input j
                                      //        feeds strip b of output i
    std::vector<std::uint8_t> written; // sched: rows x w, strip b of output i is stored (else left untouched)
    std::vector<std::uint32_t> reps;  // rows x cols ring representatives (n-bit masks)
    std::vector<std::uint16_t> matrix; // rows x cols GF(2^w) entries the program was compiled from
    std::vector<std::uint32_t> fold;  // fold[t - w] = x^t mod p
    std::vector<Instr> code;          // canonical order (next group's loads before this group's XORs)
    std::vector<std::vector<Instr>> group_loads, group_compute; // per fragment group
    std::vector<Instr> tail;          // inverse transform + stores
    std::uint32_t nvars = 0;
    // staged kernels split the outputs across consumer warp groups: part r
    // computes rows [part_row0[r], part_row0[r] + parts[r].rows)
    std::vector<Program> parts;
    std::vector<std::uint32_t> part_row0;
    std::uint32_t staged_threads = 0; // staged CTA size override (0 = 256)
    std::uint32_t staged_producer = 0; // 0 auto, 1 cp.async, 2 TMA tensor, 3 TMA tensor + producer warp
    ProgramStats stats;
    // plain-field bitmatrix of the program for the generic kernel: mask[(i*w + b)*cols + j] = strips of
    // input j feeding strip b of output i (empty for schedule programs that leave strips unwritten)
    std::vector<std::uint16_t> field_masks;
    // one of many programs of a code (a decode erasure pattern): served by the
    // runtime-matrix ring kernel, never compiled (runtime.cpp launch_batch)
    bool adhoc = false;
    // light: only field, kind, shape, matrix, reps and fold are set (what the
    // runtime-matrix kernel needs); full_program() compiles the rest on first
    // use.  key = plan_key, computed once.
    bool light = false;
    std::string key;
    std::shared_ptr<struct LazyCompile> lazy;
    std::uint64_t ir_hash = 0; // hash of every instruction list a kernel is generated from (code, parts):
                               // part of the kernel name, so a cached cubin never outlives its program
};

struct CompileOptions {
    std::uint32_t group = 0;   // 0: choose automatically
    bool cse = true;           // greedy pair elimination
    bool dense = false;        // RingRep::Dense (plain phi1) instead of Sparse (schedule.hpp:78)
    bool crs = false;          // Cauchy-RS bitmatrix baseline instead of the ring (schedule.hpp:168-203)
    std::uint32_t parts = 0;   // output parts for the staged kernel: 0 auto, 1 = do not split
    std::uint32_t part_group = 0; // fragment group of the parts: 0 auto
    std::uint32_t max_temps = 0;  // cap on shared pair temporaries per group (0 = no cap)
    std::uint32_t cse_window = 0; // pair sharing within windows of this many targets (0 = whole group)
    std::uint32_t staged_threads = 0; // staged CTA size (0 = tuned table / 256)
    // explicit linear map instead of a matrix (compile_schedule_program): the
    // matrix passed alongside only gives the shape
    const std::vector<std::uint32_t>* bits = nullptr;
    const std::vector<std::uint8_t>* written = nullptr;
    // representatives to use instead of sparse_transform of the matrix (the
    // negative-control fault injection, pyrit_plan_inject_fault)
    const std::vector<std::uint32_t>* reps = nullptr;
};

// Measured staged-kernel choices for specific programs (tuned.tsv):
//   <plan_key> <parts> <part_group> <part_cse>
struct TunedEntry {
    std::string key;
    std::uint32_t parts = 1, part_group = 1;
    int part_cse = 0;
    std::uint32_t threads = 0; // staged CTA size (0 = default)
    std::uint32_t producer = 0; // 0 auto, 1 cp.async, 2 TMA tensor, 3 TMA tensor + producer warp
};
std::string plan_key(const Program& p); // field + transform + ring representatives
void set_tuned_path(const std::string& path);
const TunedEntry* find_tuned(const std::string& key);

// compile_schedule analogue: matrix (rows x cols, GF(2^w) entries) -> program
Program compile_program(const Field& f, TransformKind kind, const Matrix& m, const CompileOptions& opt);

// Shared state of a light program and its copies: the full program, compiled
// once on demand, and how many launches the pattern has had (hot patterns get
// a specialised kernel compiled in the background, runtime.cpp)
struct LazyCompile {
    std::once_flag once;
    std::shared_ptr<const Program> prog;
    std::atomic<std::uint32_t> uses{0};
};

// A light ad-hoc program (decode patterns): representatives and fold only,
// microseconds to build; full_program() compiles it (once, shared by copies)
// when something needs the instruction lists -- a generated kernel, the
// interpreter or the statistics.
Program light_program(const Field& f, TransformKind kind, const Matrix& m);
const Program& full_program(const Program& p);
// a light program from ring representatives as given (n-bit shift masks, any
// element of each coset): the runtime-matrix kernel applies them as they are;
// a compiled kernel, if one is ever built for it, uses the field matrix
// u mod p, which computes the same symbols (SURVEY 8(b) pyrit_cu_ringmat)
Program ring_program(const Field& f, TransformKind kind, const std::uint32_t* reps, std::uint32_t rows,
                     std::uint32_t cols);

// One region op of a reference XorSchedule (schedule.hpp:40-48); mode is
// OpMode: 0 Copy, 1 Xor, 2 Zero.
struct ScheduleOp {
    std::uint16_t src_sym = 0, src_pkt = 0, dst_sym = 0, dst_pkt = 0;
    std::uint8_t mode = 0;
};

// A reference XorSchedule compiled for the GPU: the B200 replacement for
// replay()/parallel_replay() over an arbitrary schedule (codec.hpp:118-193).
// The schedule (pre, core, post concatenated in replay order) is evaluated
// symbolically over GF(2): every output packet it writes is a XOR of
// initial input packets, which one fused kernel computes column word by
// column word.  Slots follow replay(): sym < k is input slot sym (in_map),
// sym >= k output slot sym - k (out_map); packets >= w are workspace
// scratch, zero at entry (a fresh Workspace, as parallel_replay makes).
// Slots that share storage (decode() passes one SymbolBuffer as in and out)
// carry equal labels, so a write through one slot is seen by later reads
// through another, as in the reference's op-by-op replay.
//   kernel input q reads slot src_slot[q] (>= 0: input slot; < 0: output
//   slot -1-src_slot[q], its contents before the call); kernel output r is
//   output slot dst_slot[r], written only on the strips in prog.written.
struct ScheduleProgram {
    Program prog;
    std::vector<std::int32_t> src_slot;
    std::vector<std::uint32_t> dst_slot;
    std::uint32_t k = 0, outputs = 0;
};
// labels: k + outputs storage labels (empty = all slots distinct)
ScheduleProgram compile_schedule_program(const Field& f, std::uint32_t k, std::uint32_t outputs,
                                         const std::vector<ScheduleOp>& ops, const std::vector<std::uint32_t>& labels,
                                         const CompileOptions& opt);

// Host interpreter of a compiled program (verification of the compiler on
// machines without a GPU; never used by the device path).  Window
// [off, off+len) of every strip; strip i of symbol j is in[j] + i*strip.
void interpret_program(const Program& p, const std::uint8_t* const* in, std::uint8_t* const* out,
                       std::uint64_t strip, std::uint64_t off, std::uint64_t len);

// CUDA C source of the fused kernel for this program.
//
// Direct mode: every thread streams its column word of every strip with
//   vector LDG (lanes 32-bit words per thread per strip; 0 = byte mode),
//   grid-stride over the window.
// Staged mode (the sm_100a main path): a persistent CTA per SM; warp 0 is a
//   TMA producer that moves [k*w strips x tile] tiles of the window into a
//   ring of shared-memory stages with cp.async.bulk, completion tracked by
//   one mbarrier per (stage, fragment group); the consumer warps evaluate the
//   ring program reading their 4-byte column word of each strip from shared
//   memory and store the folded outputs straight to HBM.  Needs 16-byte
//   aligned pointers, strip pitch, window offset and length.
struct KernelShape {
    std::uint32_t lanes = 1;
    std::uint32_t threads = 256;
    std::uint32_t min_blocks = 2;
    bool staged = false;
    std::uint32_t tile = 512;       // staged: bytes per strip per tile (= 4 x consumer threads)
    std::uint32_t stages = 2;       // staged: shared-memory ring depth
    std::uint32_t bar_bytes = 128;  // staged: mbarrier area at the start of shared memory
    std::uint32_t smem_bytes = 0;   // staged: dynamic shared memory per CTA
    std::uint32_t copy = 2;         // staged producer: 2 = TMA tensor boxes (one elected thread), 1 = cp.async by
                                    // every thread (any 4/8/16-byte alignment), 0 = TMA 1D bulk copies by warp 0
    std::uint32_t chunk = 16;       // staged cp.async: bytes per copy (16; 8 or 4 for less aligned strips)
    std::uint32_t split = 0;        // direct: rows split over p.parts.size() thread groups (0/1 = no split)
    std::uint32_t half = 0;         // direct sub-word mode: 1 = 2-byte elements (u16), 0 = bytes
    std::uint32_t ws = 0;           // staged TMA: 1 = a dedicated producer warp (blockDim = threads + 32)
    std::uint32_t tmap4 = 0;        // staged TMA: 1 = inputs equally spaced, one 4D map / one box per unit
    std::uint32_t spb = 0;          // staged TMA: strips per box (0 = all w strips of a fragment in one box)
};
std::string kernel_name(const Program& p, const KernelShape& ks);
std::string generate_cuda(const Program& p, const KernelShape& ks);
// Staged-mode shape for this program, or staged=false if the tiles do not fit.
KernelShape staged_shape(const Program& p, std::uint32_t smem_limit);

std::uint64_t fnv1a(const std::string& s);

} // namespace pyrit_b200
