/* mrb200.h -- C ABI of the B200-native backend for Relay's fused-group
 * execution path (arXiv 1904.08368; reference: MicroRelay, /root/reference).
 *
 * The reference executes a fused module -- the output of run_pipeline with
 * "fuse" (fuse.cpp:318-328) and optionally "quantize" (quantize.cpp:212-245)
 * -- with its tree-walking interpreter:
 *
 *     ValueRef interp(const ModuleEnv&, const std::string& entry,
 *                     const std::vector<ValueRef>& args, InterpOptions);
 *                                                       (interp.hpp:50-51)
 *
 * evaluating every `let %fusedN = fn(...) [Primitive=true] {...}` group op by
 * op through OperatorDecl::eval / KernelFn (registry.hpp:58-68,
 * interp.cpp:86-111).  This library is the drop-in replacement for that
 * call on a B200: it takes the same fused module (as the reference's own
 * text format, printer.cpp / parser.cpp), lowers each Primitive group to one
 * hand-written sm_100a kernel launch (plus hoisted weight prologues), plans
 * every intermediate into one device arena, and replays the launch list as
 * a CUDA graph.
 *
 * Conventions
 *  - Plain C types only; no torch / STL types cross this boundary.
 *  - Every function returns an mr_status (0 = ok).  Non-zero codes mirror the
 *    reference's DiagCode (diagnostics.hpp:32-93) where one applies; CUDA
 *    failures and unsupported group patterns have their own codes.  Nothing
 *    throws across the ABI; mr_last_error_message() is thread-local.
 *  - Unsupported group patterns are rejected at mr_exec_create (compile
 *    time), never at launch.  There is no CPU fallback.
 *  - Tensors at the boundary use the reference's layout: row-major NCHW
 *    float32 (TensorLiteral, literal.hpp:17-24).  Internal storage (NHWC,
 *    int8 codes, bf16) is private to the executor.
 */
#ifndef MRB200_H_
#define MRB200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum mr_status {
  MR_OK = 0,
  /* mirrors of microrelay::DiagCode (diagnostics.hpp:32-93), offset by 1 */
  MR_ERR_UNBOUND_VARIABLE = 1,
  MR_ERR_UNKNOWN_OPERATOR = 2,
  MR_ERR_SYNTAX = 6,
  MR_ERR_META_INDEX = 7,
  MR_ERR_TYPE_MISMATCH = 9,
  MR_ERR_ARITY_MISMATCH = 13,
  MR_ERR_CALIBRATION_FAILED = 15,
  MR_ERR_UNCALIBRATED = 16,
  MR_ERR_INTERNAL = 24,
  /* backend-specific */
  MR_ERR_UNSUPPORTED_GROUP = 100, /* a Primitive body with no kernel pattern */
  MR_ERR_CUDA = 101,
  MR_ERR_INVALID_ARGUMENT = 102,
  MR_ERR_OUT_OF_MEMORY = 103,
  MR_ERR_INEXACT_INT8 = 104       /* an int8 contraction whose partial sums are not
                                     proven below 2^24 quanta: the int32 tensor-core
                                     sum could differ from interp()'s fp32 sum, so
                                     mr_exec_set_weights refuses the weights */
} mr_status;

/* Element type, matching microrelay::BaseType (dtype.hpp:18-43). */
typedef enum mr_type_code { MR_INT = 0, MR_UINT = 1, MR_FLOAT = 2, MR_BOOL = 3 } mr_type_code;

typedef struct mr_tensor {
  void* data;          /* host or device pointer, see each call */
  int32_t ndim;
  int64_t shape[8];    /* row-major (NCHW for 4-D activations) */
  int32_t type_code;   /* mr_type_code */
  int32_t bits;        /* 32 for float32 */
} mr_tensor;

/* How the float (non-quantized) parts of a module are computed.  A module
 * realized by the reference's quantize pass always runs its quantized
 * contractions as int8 x int8 -> int32 on tcgen05 (kind::i8) and is
 * bit-exact with interp(); the choice below only affects modules (or
 * groups) without quantize chains. */
typedef enum mr_float_mode {
  MR_FLOAT_BF16 = 0,        /* bf16 operands, fp32 accumulate (tcgen05 kind::f16) */
  MR_FLOAT_FP32_STRICT = 1, /* fp32, reference accumulation order, no FMA:
                               bit-exact with kernels.cpp, slow (for checking) */
  MR_FLOAT_TF32 = 2         /* float32 activations; convs and dense on tcgen05
                               kind::tf32 (fp32 accumulate); groups with no tf32
                               formulation (3-channel stems, pooling, depthwise)
                               run the strict fp32 kernels */
} mr_float_mode;

typedef struct mr_exec_options {
  int32_t device;          /* CUDA device ordinal */
  int64_t batch;           /* binds the symbolic batch dim (?n) of @main's inputs */
  int32_t n_data_inputs;   /* leading @main params that change per call (default 1);
                              the rest are weights, set once by mr_exec_set_weights */
  int32_t float_mode;      /* mr_float_mode */
  int32_t use_cuda_graph;  /* 1: capture the launch list once, replay per run */
  int32_t force_simt;      /* 1: use the CUDA-core kernels even where a tcgen05
                              kernel exists (baseline / debugging) */
} mr_exec_options;

typedef struct mr_exec_s* mr_exec_t;

/* Fills defaults: device 0, batch 1, 1 data input, bf16, graphs on. */
void mr_exec_default_options(mr_exec_options* opts);

/* Replaces constructing an Interpreter over the fused ModuleEnv
 * (interp.cpp:16-19): parses `fused_module_text` (print_module output of a
 * run_pipeline(...,fuse) module), lowers every Primitive group, plans device
 * memory.  Fails with MR_ERR_UNSUPPORTED_GROUP naming the group if a body
 * matches no kernel pattern. */
mr_status mr_exec_create(const char* fused_module_text, const mr_exec_options* opts,
                         mr_exec_t* out);

/* Uploads the non-data @main arguments (weights, biases, shape-only windows)
 * from HOST float32 NCHW/OIHW buffers, in @main parameter order, and runs
 * the hoisted weight prologues (folded-BN multiply, weight quantize chains)
 * once on the device.  Must precede mr_exec_run. */
mr_status mr_exec_set_weights(mr_exec_t ex, int32_t n, const mr_tensor* weights);

/* The interp(m, "main", args) replacement, device-resident: `inputs` are the
 * n_data_inputs leading @main args as DEVICE float32 NCHW buffers, `output`
 * a DEVICE buffer for @main's result, written by the final launch itself (no
 * extra copy; one captured graph per (input, output) address set).
 * Stream-ordered on `stream` (a cudaStream_t; NULL = legacy default stream);
 * does not synchronize.  Every mr_exec_* call makes the executor's device
 * current for its duration and restores the caller's device on return. */
mr_status mr_exec_run(mr_exec_t ex, const mr_tensor* inputs, mr_tensor* output, void* stream);

/* Same, end to end from HOST buffers: copies inputs H2D (pinned staging),
 * runs, copies the result D2H and synchronizes the stream. */
mr_status mr_exec_run_host(mr_exec_t ex, const mr_tensor* inputs, mr_tensor* output,
                           void* stream);

/* Shape of @main's result at the bound batch. */
/* Asynchronous end-to-end call for streaming inference: enqueues the H2D copy
 * of inputs[0] (HOST float32, pinned for true asynchrony) into one of two
 * device stages on an internal copy stream, the run on `stream` once that
 * copy lands, and the D2H of the result into output->data (HOST) on `stream`,
 * then returns without waiting.  Consecutive submissions pipeline: batch
 * i+1's upload overlaps batch i's kernels.  Host buffers must stay untouched
 * until mr_exec_sync returns.  Results are identical to mr_exec_run_host. */
mr_status mr_exec_submit_host(mr_exec_t ex, const mr_tensor* inputs, mr_tensor* output, void* stream);

/* Waits for every mr_exec_submit_host issued since the last sync. */
mr_status mr_exec_sync(mr_exec_t ex);

mr_status mr_exec_output_shape(mr_exec_t ex, mr_tensor* shape_only);

/* JSON description of the lowered program: groups, kernels, formats, arena
 * plan, per-launch algorithmic bytes/flops.  Pointer valid until destroy. */
const char* mr_exec_describe(mr_exec_t ex);

/* Kernel launches issued by one mr_exec_run (graph nodes). */
int32_t mr_exec_launch_count(mr_exec_t ex);

/* Per-launch device timing of one (non-graph) run on `stream`: writes up to
 * `cap` milliseconds into ms[] in launch order; returns the count. */
int32_t mr_exec_profile(mr_exec_t ex, const mr_tensor* inputs, mr_tensor* output, void* stream,
                        float* ms, int32_t cap);

void mr_exec_destroy(mr_exec_t ex);

const char* mr_last_error_message(void);

/* Host-only compile check (no device touched): parses the fused module and
 * lowers every Primitive group exactly as mr_exec_create does, then returns a
 * JSON description of the lowered groups (kind, anchor attrs, prologue and
 * epilogue op lists) in *json (valid until the next call on this thread).
 * The error contract matches mr_exec_create's (MR_ERR_SYNTAX,
 * MR_ERR_UNSUPPORTED_GROUP ...).  Mirrors what FuseOps' consumer learns from
 * the reference's per-group type check (passes.cpp:452-486). */
mr_status mr_module_lower(const char* fused_module_text, int64_t batch, int32_t n_data_inputs,
                          const char** json);

/* GPU calibration sweep: the global power-of-two
 * scale the reference's quant_calibrate (quantize.cpp:138-177) picks -- the
 * first k in [k_min, k_max] (the reference: [-16, 16]) such that no quantize
 * site of the module at rho = 2^k sees |nearbyint(x / rho * 2^(bits-sign))|
 * above 2^(bits-1), over the weights and every calibration batch.
 * `fused_module_text` is a realized + fused module at ANY global scale (the
 * sweep rewrites every site, as with_global_scale does, quantize.cpp:123-134);
 * inputs[i] is calibration batch i (HOST float32, opts->batch images each).
 * Fails with MR_ERR_CALIBRATION_FAILED when every k overflows. */
mr_status mr_calibrate(const char* fused_module_text, const mr_exec_options* opts, int32_t n_weights,
                       const mr_tensor* weights, int32_t n_sets, const mr_tensor* inputs, int32_t k_min,
                       int32_t k_max, int32_t* k_out, int32_t* trials_out);

/* ---- group level: one Primitive closure application ----------------------
 * Replaces Interpreter::apply on a Primitive Closure (interp.cpp:86-101): the
 * group `group` (its function name %fusedN or the value its call binds) of
 * `fused_module_text`, compiled on its own with the same kernels the executor
 * uses for it (opts->batch binds ?n of the module).  The group's operands are
 * its call arguments (= fn params in order, fuse.cpp:296-302). */
typedef struct mr_group_s* mr_group_t;

mr_status mr_group_compile(const char* fused_module_text, const char* group, const mr_exec_options* opts,
                           mr_group_t* out);

/* Number of operands and the result's shape. */
mr_status mr_group_signature(mr_group_t g, int32_t* n_operands, mr_tensor* out_shape);

/* Applies the group: in[i] = argument i (DEVICE float32, row-major, the types
 * the module binds), *out = DEVICE float32 result.  Stream-ordered, no sync.
 * Weight operands (the @main weight params the group reads) are staged and
 * their prologues (folded-BN multiply, weight realize chain) run when a weight
 * operand's address differs from the previous launch; contents at an
 * unchanged address are assumed unchanged (mr_group_reload forces a restage).
 * Fails with MR_ERR_ARITY_MISMATCH / MR_ERR_TYPE_MISMATCH like apply(). */
mr_status mr_group_launch(mr_group_t g, const mr_tensor* in, int32_t n_in, mr_tensor* out, void* stream);

/* Forces the next mr_group_launch to restage the weight operands. */
void mr_group_reload(mr_group_t g);

void mr_group_destroy(mr_group_t g);

/* Library build identification (arch, kernels compiled). */
const char* mr_build_info(void);

#ifdef __cplusplus
}
#endif

#endif /* MRB200_H_ */
