// Internal host-side structures of libgpulet (not part of the C-ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/gpulet.h"
#include "program.h"

namespace gl {

// ---- driver entry points (resolved through cudart; no link-time libcuda) ----
struct Driver {
  decltype(&::cuTensorMapEncodeTiled) tensorMapEncodeTiled = nullptr;
  decltype(&::cuTensorMapEncodeIm2col) tensorMapEncodeIm2col = nullptr;
  decltype(&::cuDeviceGetDevResource) deviceGetDevResource = nullptr;
  decltype(&::cuDevSmResourceSplitByCount) devSmResourceSplitByCount = nullptr;
  decltype(&::cuDevResourceGenerateDesc) devResourceGenerateDesc = nullptr;
  decltype(&::cuGreenCtxCreate) greenCtxCreate = nullptr;
  decltype(&::cuGreenCtxDestroy) greenCtxDestroy = nullptr;
  decltype(&::cuGreenCtxStreamCreate) greenCtxStreamCreate = nullptr;
  decltype(&::cuLaunchKernelEx) launchKernelEx = nullptr;
  decltype(&::cuKernelSetAttribute) kernelSetAttribute = nullptr;
  decltype(&::cuStreamDestroy) streamDestroy = nullptr;
  decltype(&::cuDeviceGet) deviceGet = nullptr;
  bool ok = false;
};
Driver& driver();
// cudaFree / cudaFreeHost, deferred while persistent executors are running.
void release_device(void* p, bool host);

// ---- weights -------------------------------------------------------------------
struct Param {
  std::vector<int> shape;
  std::vector<uint16_t> data;  // bf16 bits
  size_t numel() const {
    size_t n = 1;
    for (int d : shape) n *= (size_t)d;
    return n;
  }
};
using ParamMap = std::map<std::string, Param>;
bool load_glw(const std::string& path, ParamMap& out, std::string& err);

// Device-side copies of (repacked) weights of one model on one GPU.
struct DevWeights {
  std::vector<void*> allocs;
  std::map<std::string, void*> ptr;
  size_t bytes = 0;
  ~DevWeights();
};

// ---- programs -------------------------------------------------------------------
struct Program {
  std::vector<OpDesc> ops;
  size_t in_copy_bytes = 0; // tests: bytes of the input copied into the workspace before launch
  size_t in_copy_off = 0;   //   ... at this workspace offset
  OpDesc* dev = nullptr;   // device copy
  size_t ws_bytes = 0;     // activation workspace needed
  double flops = 0;        // algorithmic FLOPs of one batch (2 * MACs)
  double weight_bytes = 0; // weight bytes read once per batch
};

struct Model {
  int kind = 0;
  int gpu = 0;
  ParamMap host;                 // host copy of the file (kept: programs for other gpu-let sizes are built later)
  std::unique_ptr<DevWeights> w;
  Program prog[33];              // per batch 1..32, tiles for a whole B200 (148 SMs)
  size_t in_bytes[33] = {0}, out_bytes[33] = {0};
  std::map<int, std::vector<Program>> prog_sm;   // SM count -> [batch] programs tiled for that gpu-let size
};

// Program-builder tuning overrides (gl_set_tuning; 0 = automatic choice).
enum TuneKey {
  TUNE_BN = 0, TUNE_SPLIT = 1, TUNE_MISC = 2, TUNE_WARM = 3, TUNE_GATHER = 4, TUNE_SMS = 5,
  TUNE_DATAFLOW = 6,   // 1: barrier-free GEMM step joins in programs built afterwards; 2: also log the plan
  TUNE_SERVE_RT = 7,   // 1: gl_serve runs its polling loop SCHED_FIFO when permitted
  kTuneKeys = 8
};
extern int g_tune[kTuneKeys];
// thread-local gl_last_error text (runtime.cpp); returns s
gl_status set_error(gl_status s, const char* m);

// Build the layer program of model `kind` at batch b (models.cpp).
// sm_target: the SM count of the gpu-let the program is built for (tile
// decomposition: N tile, split-K); 148 = a whole B200.
bool build_program(int kind, int batch, const ParamMap& host, DevWeights& dw, int gpu, Program& out,
                   size_t& in_bytes, size_t& out_bytes, std::string& err, int sm_target = 148);

// Single-op programs for kernel unit tests (models.cpp).
// in_ws: the input is first copied into the workspace so the TMA operand paths run.
bool build_test_gemm(int M, int N, int K, int act, int swap_ab, int splitk, int out_fp32, const uint16_t* w_host,
                     const uint16_t* b_host, int in_ws, DevWeights& dw, Program& out, std::string& err);
bool build_test_conv(int N, int H, int W, int C, int Cout, int KH, int stride, int pad, int act,
                     const uint16_t* w_host, const uint16_t* b_host, int in_ws, DevWeights& dw, Program& out,
                     std::string& err);
// Bind a program to a workspace: encode the tensor maps of workspace-resident
// activation operands (their addresses are only known per workspace).
bool bind_program(const Program& p, char* ws, std::vector<OpDesc>& out, std::string& err);
// Barrier-free joins of GEMM steps with completion counters (models.cpp; GL_DATAFLOW=1 enables).
bool dataflow_enabled();
bool build_test_misc(int type, const int* iargs, int n_iargs, const uint16_t* w_host, size_t w_len, DevWeights& dw,
                     Program& out, std::string& err);

void op_cost(const OpDesc& op, double& flops, double& bytes);
int model_kind_count();
const char* model_name(int kind);

}  // namespace gl
