// In-run DRAM traffic meter for bench.py (measurement infrastructure, not
// the product): the CUPTI Range Profiler collects dram__bytes_read.sum and
// dram__bytes_write.sum over ONE user range (user replay, single pass --
// no kernel replay, no serialisation inside the range), so bench.py reports
// the DRAM bytes its own SpMM applies moved while running.
//
// C ABI:  dm_init(device) -> 0 ok; dm_begin(); dm_end(&read, &write);
//         dm_error() -> last message.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cuda.h>
#include <cupti_profiler_host.h>
#include <cupti_profiler_target.h>
#include <cupti_range_profiler.h>
#include <cupti_target.h>

namespace {
std::string g_err;
CUpti_RangeProfiler_Object* g_obj = nullptr;
CUpti_Profiler_Host_Object* g_host = nullptr;
std::vector<uint8_t> g_config, g_counter;
const char* g_metrics[2] = {"dram__bytes_read.sum", "dram__bytes_write.sum"};

bool ok(CUptiResult r, const char* what) {
  if (r == CUPTI_SUCCESS) return true;
  const char* s = nullptr;
  cuptiGetResultString(r, &s);
  g_err = std::string(what) + ": " + (s ? s : "?");
  return false;
}

bool setup_counter_image() {
  CUpti_RangeProfiler_GetCounterDataSize_Params sz = {CUpti_RangeProfiler_GetCounterDataSize_Params_STRUCT_SIZE};
  sz.pRangeProfilerObject = g_obj;
  sz.pMetricNames = g_metrics;
  sz.numMetrics = 2;
  sz.maxNumOfRanges = 1;
  sz.maxNumRangeTreeNodes = 1;
  if (!ok(cuptiRangeProfilerGetCounterDataSize(&sz), "GetCounterDataSize")) return false;
  g_counter.assign(sz.counterDataSize, 0);
  CUpti_RangeProfiler_CounterDataImage_Initialize_Params ci = {CUpti_RangeProfiler_CounterDataImage_Initialize_Params_STRUCT_SIZE};
  ci.pRangeProfilerObject = g_obj;
  ci.counterDataSize = g_counter.size();
  ci.pCounterData = g_counter.data();
  if (!ok(cuptiRangeProfilerCounterDataImageInitialize(&ci), "CounterDataImageInitialize")) return false;
  CUpti_RangeProfiler_SetConfig_Params sc = {CUpti_RangeProfiler_SetConfig_Params_STRUCT_SIZE};
  sc.pRangeProfilerObject = g_obj;
  sc.configSize = g_config.size();
  sc.pConfig = g_config.data();
  sc.counterDataImageSize = g_counter.size();
  sc.pCounterDataImage = g_counter.data();
  sc.range = CUPTI_UserRange;
  sc.replayMode = CUPTI_UserReplay;
  sc.maxRangesPerPass = 1;
  sc.numNestingLevels = 1;
  sc.minNestingLevel = 1;
  sc.passIndex = 0;
  sc.targetNestingLevel = 1;
  return ok(cuptiRangeProfilerSetConfig(&sc), "SetConfig");
}
}  // namespace

extern "C" const char* dm_error(void) { return g_err.c_str(); }

extern "C" int dm_init(int device) {
  if (g_obj) return 0;
  CUcontext ctx = nullptr;
  if (cuCtxGetCurrent(&ctx) != CUDA_SUCCESS || !ctx) {
    g_err = "no current CUDA context";
    return 1;
  }
  CUpti_Profiler_Initialize_Params pi = {CUpti_Profiler_Initialize_Params_STRUCT_SIZE};
  if (!ok(cuptiProfilerInitialize(&pi), "ProfilerInitialize")) return 1;
  CUpti_Device_GetChipName_Params cn = {CUpti_Device_GetChipName_Params_STRUCT_SIZE};
  cn.deviceIndex = (size_t)device;
  if (!ok(cuptiDeviceGetChipName(&cn), "GetChipName")) return 1;
  CUpti_Profiler_GetCounterAvailability_Params ca = {CUpti_Profiler_GetCounterAvailability_Params_STRUCT_SIZE};
  ca.ctx = ctx;
  if (!ok(cuptiProfilerGetCounterAvailability(&ca), "GetCounterAvailability(size)")) return 1;
  std::vector<uint8_t> avail(ca.counterAvailabilityImageSize);
  ca.pCounterAvailabilityImage = avail.data();
  if (!ok(cuptiProfilerGetCounterAvailability(&ca), "GetCounterAvailability")) return 1;
  CUpti_Profiler_Host_Initialize_Params hi = {CUpti_Profiler_Host_Initialize_Params_STRUCT_SIZE};
  hi.profilerType = CUPTI_PROFILER_TYPE_RANGE_PROFILER;
  hi.pChipName = cn.pChipName;
  hi.pCounterAvailabilityImage = avail.data();
  if (!ok(cuptiProfilerHostInitialize(&hi), "HostInitialize")) return 1;
  g_host = hi.pHostObject;
  CUpti_Profiler_Host_ConfigAddMetrics_Params am = {CUpti_Profiler_Host_ConfigAddMetrics_Params_STRUCT_SIZE};
  am.pHostObject = g_host;
  am.ppMetricNames = g_metrics;
  am.numMetrics = 2;
  if (!ok(cuptiProfilerHostConfigAddMetrics(&am), "ConfigAddMetrics")) return 1;
  CUpti_Profiler_Host_GetConfigImageSize_Params cs = {CUpti_Profiler_Host_GetConfigImageSize_Params_STRUCT_SIZE};
  cs.pHostObject = g_host;
  if (!ok(cuptiProfilerHostGetConfigImageSize(&cs), "GetConfigImageSize")) return 1;
  g_config.assign(cs.configImageSize, 0);
  CUpti_Profiler_Host_GetConfigImage_Params cg = {CUpti_Profiler_Host_GetConfigImage_Params_STRUCT_SIZE};
  cg.pHostObject = g_host;
  cg.configImageSize = g_config.size();
  cg.pConfigImage = g_config.data();
  if (!ok(cuptiProfilerHostGetConfigImage(&cg), "GetConfigImage")) return 1;
  CUpti_Profiler_Host_GetNumOfPasses_Params np = {CUpti_Profiler_Host_GetNumOfPasses_Params_STRUCT_SIZE};
  np.configImageSize = g_config.size();
  np.pConfigImage = g_config.data();
  if (!ok(cuptiProfilerHostGetNumOfPasses(&np), "GetNumOfPasses")) return 1;
  if (np.numOfPasses != 1) {
    g_err = "dram byte metrics need " + std::to_string(np.numOfPasses) + " passes";
    return 1;
  }
  CUpti_RangeProfiler_Enable_Params en = {CUpti_RangeProfiler_Enable_Params_STRUCT_SIZE};
  en.ctx = ctx;
  if (!ok(cuptiRangeProfilerEnable(&en), "RangeProfilerEnable")) return 1;
  g_obj = en.pRangeProfilerObject;
  return 0;
}

extern "C" int dm_begin(void) {
  if (!g_obj) {
    g_err = "dm_init first";
    return 1;
  }
  if (!setup_counter_image()) return 1;
  CUpti_RangeProfiler_Start_Params st = {CUpti_RangeProfiler_Start_Params_STRUCT_SIZE};
  st.pRangeProfilerObject = g_obj;
  if (!ok(cuptiRangeProfilerStart(&st), "Start")) return 1;
  CUpti_RangeProfiler_PushRange_Params pr = {CUpti_RangeProfiler_PushRange_Params_STRUCT_SIZE};
  pr.pRangeProfilerObject = g_obj;
  pr.pRangeName = "region";
  return ok(cuptiRangeProfilerPushRange(&pr), "PushRange") ? 0 : 1;
}

extern "C" int dm_end(double* read_bytes, double* write_bytes) {
  CUpti_RangeProfiler_PopRange_Params pp = {CUpti_RangeProfiler_PopRange_Params_STRUCT_SIZE};
  pp.pRangeProfilerObject = g_obj;
  if (!ok(cuptiRangeProfilerPopRange(&pp), "PopRange")) return 1;
  CUpti_RangeProfiler_Stop_Params sp = {CUpti_RangeProfiler_Stop_Params_STRUCT_SIZE};
  sp.pRangeProfilerObject = g_obj;
  if (!ok(cuptiRangeProfilerStop(&sp), "Stop")) return 1;
  CUpti_RangeProfiler_DecodeData_Params dd = {CUpti_RangeProfiler_DecodeData_Params_STRUCT_SIZE};
  dd.pRangeProfilerObject = g_obj;
  if (!ok(cuptiRangeProfilerDecodeData(&dd), "DecodeData")) return 1;
  double vals[2] = {0, 0};
  CUpti_Profiler_Host_EvaluateToGpuValues_Params ev = {CUpti_Profiler_Host_EvaluateToGpuValues_Params_STRUCT_SIZE};
  ev.pHostObject = g_host;
  ev.pCounterDataImage = g_counter.data();
  ev.counterDataImageSize = g_counter.size();
  ev.rangeIndex = 0;
  ev.ppMetricNames = g_metrics;
  ev.numMetrics = 2;
  ev.pMetricValues = vals;
  if (!ok(cuptiProfilerHostEvaluateToGpuValues(&ev), "EvaluateToGpuValues")) return 1;
  *read_bytes = vals[0];
  *write_bytes = vals[1];
  return 0;
}

extern "C" int dm_close(void) {
  if (g_obj) {
    CUpti_RangeProfiler_Disable_Params d = {CUpti_RangeProfiler_Disable_Params_STRUCT_SIZE};
    d.pRangeProfilerObject = g_obj;
    cuptiRangeProfilerDisable(&d);
    g_obj = nullptr;
  }
  if (g_host) {
    CUpti_Profiler_Host_Deinitialize_Params h = {CUpti_Profiler_Host_Deinitialize_Params_STRUCT_SIZE};
    h.pHostObject = g_host;
    cuptiProfilerHostDeinitialize(&h);
    g_host = nullptr;
  }
  CUpti_Profiler_DeInitialize_Params p = {CUpti_Profiler_DeInitialize_Params_STRUCT_SIZE};
  cuptiProfilerDeInitialize(&p);
  return 0;
}
