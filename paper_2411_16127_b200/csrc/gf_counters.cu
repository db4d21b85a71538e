// Measured hardware counters of a host-defined region (the "measured bytes"
// column of the bench harness next to the reference's modelled counters,
// bench.cpp:172-187, and bench.py's live roofline `traffic`): the CUPTI range
// profiler (user range, user replay) around a callback that launches the
// region's kernels, evaluated with the CUPTI profiler host API.
//
// libcupti is loaded lazily with dlopen, so the library has no link-time
// dependency on it; without CUPTI or without profiling permission the call
// returns GF_ERR_UNSUPPORTED and the caller reports the column as absent.
// Host code only (no kernels).
#include <cuda.h>
#include <cupti_profiler_host.h>
#include <cupti_profiler_target.h>
#include <cupti_range_profiler.h>
#include <cupti_target.h>
#include <dlfcn.h>

#include <mutex>
#include <string>
#include <vector>

#include "gf_internal.cuh"

namespace {

struct Cupti {
  void* h = nullptr;
#define GF_CUPTI_FN(name) decltype(&::name) name = nullptr;
  GF_CUPTI_FN(cuptiProfilerInitialize)
  GF_CUPTI_FN(cuptiDeviceGetChipName)
  GF_CUPTI_FN(cuptiProfilerGetCounterAvailability)
  GF_CUPTI_FN(cuptiProfilerHostInitialize)
  GF_CUPTI_FN(cuptiProfilerHostDeinitialize)
  GF_CUPTI_FN(cuptiProfilerHostConfigAddMetrics)
  GF_CUPTI_FN(cuptiProfilerHostGetConfigImageSize)
  GF_CUPTI_FN(cuptiProfilerHostGetConfigImage)
  GF_CUPTI_FN(cuptiProfilerHostEvaluateToGpuValues)
  GF_CUPTI_FN(cuptiRangeProfilerEnable)
  GF_CUPTI_FN(cuptiRangeProfilerDisable)
  GF_CUPTI_FN(cuptiRangeProfilerGetCounterDataSize)
  GF_CUPTI_FN(cuptiRangeProfilerCounterDataImageInitialize)
  GF_CUPTI_FN(cuptiRangeProfilerSetConfig)
  GF_CUPTI_FN(cuptiRangeProfilerStart)
  GF_CUPTI_FN(cuptiRangeProfilerStop)
  GF_CUPTI_FN(cuptiRangeProfilerPushRange)
  GF_CUPTI_FN(cuptiRangeProfilerPopRange)
  GF_CUPTI_FN(cuptiRangeProfilerDecodeData)
  GF_CUPTI_FN(cuptiGetResultString)
#undef GF_CUPTI_FN
  std::string why;
  bool ok = false;
};

Cupti& cupti() {
  static Cupti c;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* paths[] = {"libcupti.so.12", "libcupti.so", "/usr/local/cuda/lib64/libcupti.so.12",
                           "/usr/local/cuda/extras/CUPTI/lib64/libcupti.so.12"};
    for (const char* p : paths)
      if ((c.h = dlopen(p, RTLD_NOW | RTLD_LOCAL))) break;
    if (!c.h) {
      c.why = "libcupti.so.12 not found";
      return;
    }
    bool all = true;
#define GF_CUPTI_SYM(name)                                              \
  c.name = reinterpret_cast<decltype(c.name)>(dlsym(c.h, #name));        \
  all = all && c.name != nullptr;
    GF_CUPTI_SYM(cuptiProfilerInitialize)
    GF_CUPTI_SYM(cuptiDeviceGetChipName)
    GF_CUPTI_SYM(cuptiProfilerGetCounterAvailability)
    GF_CUPTI_SYM(cuptiProfilerHostInitialize)
    GF_CUPTI_SYM(cuptiProfilerHostDeinitialize)
    GF_CUPTI_SYM(cuptiProfilerHostConfigAddMetrics)
    GF_CUPTI_SYM(cuptiProfilerHostGetConfigImageSize)
    GF_CUPTI_SYM(cuptiProfilerHostGetConfigImage)
    GF_CUPTI_SYM(cuptiProfilerHostEvaluateToGpuValues)
    GF_CUPTI_SYM(cuptiRangeProfilerEnable)
    GF_CUPTI_SYM(cuptiRangeProfilerDisable)
    GF_CUPTI_SYM(cuptiRangeProfilerGetCounterDataSize)
    GF_CUPTI_SYM(cuptiRangeProfilerCounterDataImageInitialize)
    GF_CUPTI_SYM(cuptiRangeProfilerSetConfig)
    GF_CUPTI_SYM(cuptiRangeProfilerStart)
    GF_CUPTI_SYM(cuptiRangeProfilerStop)
    GF_CUPTI_SYM(cuptiRangeProfilerPushRange)
    GF_CUPTI_SYM(cuptiRangeProfilerPopRange)
    GF_CUPTI_SYM(cuptiRangeProfilerDecodeData)
    GF_CUPTI_SYM(cuptiGetResultString)
#undef GF_CUPTI_SYM
    if (!all) {
      c.why = "libcupti lacks the range-profiler API (CUDA >= 12.6 needed)";
      return;
    }
    CUpti_Profiler_Initialize_Params ip = {CUpti_Profiler_Initialize_Params_STRUCT_SIZE};
    if (c.cuptiProfilerInitialize(&ip) != CUPTI_SUCCESS) {
      c.why = "cuptiProfilerInitialize failed";
      return;
    }
    c.ok = true;
  });
  return c;
}

std::string cupti_msg(const Cupti& c, CUptiResult r) {
  const char* s = nullptr;
  if (c.cuptiGetResultString) c.cuptiGetResultString(r, &s);
  return s ? s : ("CUPTI error " + std::to_string(static_cast<int>(r)));
}

}  // namespace

#define GF_CUPTI(call)                                                                  \
  do {                                                                                  \
    CUptiResult _r = (call);                                                            \
    if (_r != CUPTI_SUCCESS) {                                                          \
      gfb::set_error(std::string("gf_measure_metrics: " #call ": ") + cupti_msg(c, _r)); \
      rc = _r == CUPTI_ERROR_INSUFFICIENT_PRIVILEGES ? GF_ERR_UNSUPPORTED : GF_ERR_CUDA;   \
      goto done;                                                                        \
    }                                                                                   \
  } while (0)

extern "C" int gf_measure_metrics(void (*prep)(void*), void (*fn)(void*), void* user,
                                  const char* const* metrics, int32_t n_metrics, double* values) {
  if (!fn || !metrics || n_metrics < 1 || n_metrics > 16 || !values) {
    gfb::set_error("gf_measure_metrics: invalid arguments");
    return GF_ERR_INVALID;
  }
  Cupti& c = cupti();
  if (!c.ok) {
    gfb::set_error("gf_measure_metrics: " + c.why);
    return GF_ERR_UNSUPPORTED;
  }
  static std::mutex mu;  // one profiling session at a time per process
  std::lock_guard<std::mutex> lock(mu);
  int rc = GF_OK;
  int dev = 0;
  CUcontext ctx = nullptr;
  CUpti_Profiler_Host_Object* host = nullptr;
  CUpti_RangeProfiler_Object* rp = nullptr;
  std::vector<uint8_t> avail, config, counter;
  std::vector<const char*> names(metrics, metrics + n_metrics);
  {
    GF_CHECK_CUDA(cudaFree(nullptr));
    GF_CHECK_CUDA(cudaGetDevice(&dev));
    void* get_ctx = nullptr;
    cudaDriverEntryPointQueryResult q;
    GF_CHECK_CUDA(cudaGetDriverEntryPoint("cuCtxGetCurrent", &get_ctx, cudaEnableDefault, &q));
    if (!get_ctx || reinterpret_cast<CUresult (*)(CUcontext*)>(get_ctx)(&ctx) != CUDA_SUCCESS) {
      gfb::set_error("gf_measure_metrics: no current CUDA context");
      return GF_ERR_CUDA;
    }
  }
  {
    CUpti_Device_GetChipName_Params cp = {CUpti_Device_GetChipName_Params_STRUCT_SIZE};
    cp.deviceIndex = static_cast<size_t>(dev);
    GF_CUPTI(c.cuptiDeviceGetChipName(&cp));
    CUpti_Profiler_GetCounterAvailability_Params ap = {
        CUpti_Profiler_GetCounterAvailability_Params_STRUCT_SIZE};
    ap.ctx = ctx;
    GF_CUPTI(c.cuptiProfilerGetCounterAvailability(&ap));
    avail.resize(ap.counterAvailabilityImageSize);
    ap.pCounterAvailabilityImage = avail.data();
    GF_CUPTI(c.cuptiProfilerGetCounterAvailability(&ap));

    CUpti_Profiler_Host_Initialize_Params hp = {CUpti_Profiler_Host_Initialize_Params_STRUCT_SIZE};
    hp.profilerType = CUPTI_PROFILER_TYPE_RANGE_PROFILER;
    hp.pChipName = cp.pChipName;
    hp.pCounterAvailabilityImage = avail.data();
    GF_CUPTI(c.cuptiProfilerHostInitialize(&hp));
    host = hp.pHostObject;
    CUpti_Profiler_Host_ConfigAddMetrics_Params am = {
        CUpti_Profiler_Host_ConfigAddMetrics_Params_STRUCT_SIZE};
    am.pHostObject = host;
    am.ppMetricNames = names.data();
    am.numMetrics = names.size();
    GF_CUPTI(c.cuptiProfilerHostConfigAddMetrics(&am));
    CUpti_Profiler_Host_GetConfigImageSize_Params cs = {
        CUpti_Profiler_Host_GetConfigImageSize_Params_STRUCT_SIZE};
    cs.pHostObject = host;
    GF_CUPTI(c.cuptiProfilerHostGetConfigImageSize(&cs));
    config.resize(cs.configImageSize);
    CUpti_Profiler_Host_GetConfigImage_Params ci = {
        CUpti_Profiler_Host_GetConfigImage_Params_STRUCT_SIZE};
    ci.pHostObject = host;
    ci.configImageSize = config.size();
    ci.pConfigImage = config.data();
    GF_CUPTI(c.cuptiProfilerHostGetConfigImage(&ci));

    CUpti_RangeProfiler_Enable_Params ep = {CUpti_RangeProfiler_Enable_Params_STRUCT_SIZE};
    ep.ctx = ctx;
    GF_CUPTI(c.cuptiRangeProfilerEnable(&ep));
    rp = ep.pRangeProfilerObject;
    CUpti_RangeProfiler_GetCounterDataSize_Params ds = {
        CUpti_RangeProfiler_GetCounterDataSize_Params_STRUCT_SIZE};
    ds.pRangeProfilerObject = rp;
    ds.pMetricNames = names.data();
    ds.numMetrics = names.size();
    ds.maxNumOfRanges = 1;
    ds.maxNumRangeTreeNodes = 1;
    GF_CUPTI(c.cuptiRangeProfilerGetCounterDataSize(&ds));
    counter.resize(ds.counterDataSize);
    CUpti_RangeProfiler_CounterDataImage_Initialize_Params di = {
        CUpti_RangeProfiler_CounterDataImage_Initialize_Params_STRUCT_SIZE};
    di.pRangeProfilerObject = rp;
    di.counterDataSize = counter.size();
    di.pCounterData = counter.data();
    GF_CUPTI(c.cuptiRangeProfilerCounterDataImageInitialize(&di));
    CUpti_RangeProfiler_SetConfig_Params sc = {CUpti_RangeProfiler_SetConfig_Params_STRUCT_SIZE};
    sc.pRangeProfilerObject = rp;
    sc.configSize = config.size();
    sc.pConfig = config.data();
    sc.counterDataImageSize = counter.size();
    sc.pCounterDataImage = counter.data();
    sc.range = CUPTI_UserRange;
    sc.replayMode = CUPTI_UserReplay;
    sc.maxRangesPerPass = 1;
    sc.numNestingLevels = 1;
    sc.minNestingLevel = 1;
    sc.passIndex = 0;
    sc.targetNestingLevel = 1;
    GF_CUPTI(c.cuptiRangeProfilerSetConfig(&sc));

    // user replay: the region runs once per counter pass (one for byte counters)
    for (int pass = 0; pass < 32; ++pass) {
      if (prep) {  // outside the range: e.g. an L2 flush before every pass
        prep(user);
        if (cudaDeviceSynchronize() != cudaSuccess) {
          gfb::set_error("gf_measure_metrics: prep failed");
          rc = GF_ERR_CUDA;
          goto done;
        }
      }
      CUpti_RangeProfiler_Start_Params st = {CUpti_RangeProfiler_Start_Params_STRUCT_SIZE};
      st.pRangeProfilerObject = rp;
      GF_CUPTI(c.cuptiRangeProfilerStart(&st));
      CUpti_RangeProfiler_PushRange_Params pr = {CUpti_RangeProfiler_PushRange_Params_STRUCT_SIZE};
      pr.pRangeProfilerObject = rp;
      pr.pRangeName = "gf_region";
      GF_CUPTI(c.cuptiRangeProfilerPushRange(&pr));
      fn(user);
      if (cudaDeviceSynchronize() != cudaSuccess) {
        gfb::set_error("gf_measure_metrics: region failed");
        rc = GF_ERR_CUDA;
        goto done;
      }
      CUpti_RangeProfiler_PopRange_Params pp = {CUpti_RangeProfiler_PopRange_Params_STRUCT_SIZE};
      pp.pRangeProfilerObject = rp;
      GF_CUPTI(c.cuptiRangeProfilerPopRange(&pp));
      CUpti_RangeProfiler_Stop_Params sp = {CUpti_RangeProfiler_Stop_Params_STRUCT_SIZE};
      sp.pRangeProfilerObject = rp;
      GF_CUPTI(c.cuptiRangeProfilerStop(&sp));
      if (sp.isAllPassSubmitted) break;
    }
    CUpti_RangeProfiler_DecodeData_Params dd = {CUpti_RangeProfiler_DecodeData_Params_STRUCT_SIZE};
    dd.pRangeProfilerObject = rp;
    GF_CUPTI(c.cuptiRangeProfilerDecodeData(&dd));
    CUpti_Profiler_Host_EvaluateToGpuValues_Params ev = {
        CUpti_Profiler_Host_EvaluateToGpuValues_Params_STRUCT_SIZE};
    ev.pHostObject = host;
    ev.pCounterDataImage = counter.data();
    ev.counterDataImageSize = counter.size();
    ev.rangeIndex = 0;
    ev.ppMetricNames = names.data();
    ev.numMetrics = names.size();
    ev.pMetricValues = values;
    GF_CUPTI(c.cuptiProfilerHostEvaluateToGpuValues(&ev));
  }
done:
  if (rp) {
    CUpti_RangeProfiler_Disable_Params dp = {CUpti_RangeProfiler_Disable_Params_STRUCT_SIZE};
    dp.pRangeProfilerObject = rp;
    c.cuptiRangeProfilerDisable(&dp);
  }
  if (host) {
    CUpti_Profiler_Host_Deinitialize_Params hd = {
        CUpti_Profiler_Host_Deinitialize_Params_STRUCT_SIZE};
    hd.pHostObject = host;
    c.cuptiProfilerHostDeinitialize(&hd);
  }
  return rc;
}
