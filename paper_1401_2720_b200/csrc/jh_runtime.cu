// Host-side runtime shared by the launchers: launch accounting, per-kernel
// class event timing (bench.py), library options, and per-device launch
// attributes.
//
// Launch attributes (dynamic shared memory above 48 KB) are device state:
// they are set once per (kernel, device) -- not once per process -- so a
// process that solves on several GPUs, or from several host threads, sees
// every kernel configured on every device it launches on.
#include "jh_kernels.h"

#include <cudaTypedefs.h>

#include <mutex>
#include <unordered_map>

namespace jh {

unsigned long long g_launches = 0;

static bool g_overlap = true;   // engine 1: programmatic overlap of inner + update
static bool g_simple = false;   // SIMT reference-order kernels only (parity tests)

bool opt_overlap() { return g_overlap; }
bool opt_simple() { return g_simple; }

void ensure_smem(const void *fn, int bytes) {
  static std::mutex mu;
  static std::unordered_map<const void *, int> set_per_dev[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  std::lock_guard<std::mutex> lock(mu);
  int &have = set_per_dev[dev][fn];
  if (have >= bytes) return;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  have = bytes;
}

bool make_col_tmap(CUtensorMap *map, const double *A, int64_t rows, int64_t cols, int64_t ld,
                   int box_rows, int box_cols) {
  // the driver's encoder through the runtime (no link against libcuda)
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }();
  if (!encode || (ld * 8) % 16 || ((uintptr_t)A) % 16) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  const cuuint32_t box[2] = {(cuuint32_t)box_rows, (cuuint32_t)box_cols};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(A), dims, strides,
                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int sm_count() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

// ---------------------------------------------------------------------------
// per-kernel-class event timing

struct Profiler {
  bool on = false;
  int cap = 0, used = 0;
  cudaEvent_t *ev = nullptr;  // pairs (before, after)
  int *cls = nullptr;
};
static Profiler g_prof;

void prof_mark(cudaStream_t st, int cls, bool after) {
  if (!g_prof.on || g_prof.used >= g_prof.cap) return;
  if (!after) {
    cudaEventRecord(g_prof.ev[2 * g_prof.used], st);
    g_prof.cls[g_prof.used] = cls;
  } else {
    cudaEventRecord(g_prof.ev[2 * g_prof.used + 1], st);
    g_prof.used++;
  }
}

}  // namespace jh

using namespace jh;

extern "C" {

// Number of kernels this library has launched (all entry points).
unsigned long long jh_launch_count(void) { return g_launches; }

// Start timing every p-step kernel launch (up to max_launches launches).
int jh_profile_begin(int max_launches) {
  if (g_prof.cap < max_launches) {
    for (int i = 0; i < 2 * g_prof.cap; i++) cudaEventDestroy(g_prof.ev[i]);
    delete[] g_prof.ev;
    delete[] g_prof.cls;
    g_prof.ev = new cudaEvent_t[2 * (size_t)max_launches];
    g_prof.cls = new int[max_launches];
    for (int i = 0; i < 2 * max_launches; i++) cudaEventCreate(&g_prof.ev[i]);
    g_prof.cap = max_launches;
  }
  g_prof.used = 0;
  g_prof.on = true;
  return 0;
}

// Stop timing; synchronizes on the recorded events and returns per kernel
// class (0 Gram, 1 factor + inner, 2 update, 3 V-only update launches) the
// summed milliseconds and the number of timed launches (arrays of 4).
int jh_profile_end(double *ms, int64_t *count) {
  g_prof.on = false;
  for (int k = 0; k < 4; k++) {
    ms[k] = 0.0;
    count[k] = 0;
  }
  for (int i = 0; i < g_prof.used; i++) {
    float t = 0.f;
    cudaEventSynchronize(g_prof.ev[2 * i + 1]);
    cudaEventElapsedTime(&t, g_prof.ev[2 * i], g_prof.ev[2 * i + 1]);
    ms[g_prof.cls[i]] += t;
    count[g_prof.cls[i]]++;
  }
  return 0;
}

// Engine 1: overlap the update launch with the inner Jacobi's tail (1,
// default) or keep every kernel apart (0, for per-kernel timing).
int jh_set_overlap(int on) {
  g_overlap = on != 0;
  return 0;
}

// 1: run the sweep with the generic SIMT kernels only (reference-order fma
// loops, any even width); 0 (default): DMMA / TMA kernels where they apply.
// Results are bitwise identical; the parity tests check exactly that.
int jh_set_simple_kernels(int on) {
  g_simple = on != 0;
  return 0;
}

}  // extern "C"
