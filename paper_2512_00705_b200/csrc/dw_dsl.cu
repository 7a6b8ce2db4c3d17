// dw_dsl.cu -- DSL walk models compiled at run time.
//
// host/dsl_codegen.hpp turns a DslWalk program into a CUDA model functor
// (dwb::DslModel).  dw_model_compile() compiles it with NVRTC together with
// the walk kernel template this library was built from (the csrc headers are
// embedded by tools/embed_headers.py), loads the cubin with the runtime's
// library API and keeps one kernel per sampler mode.  The run engine then
// launches walk_kernel<DslModel, mode, false> exactly like a builtin
// instantiation: the user's weight function is compiled into the kernel, not
// interpreted.  NVRTC is opened lazily with dlopen, so the library loads (and
// the builtin models run) on machines without it.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/dynwalk_b200.h"
#include "dw_walk_kernel.cuh"
#include "dw_rtc_headers.inc"

namespace dwb {
std::string* dsl_error_slot();  // dw_capi.cu: the thread's dw_last_error() text
}

namespace {

typedef int nvrtcResult_;
typedef struct _nvrtcProgram* nvrtcProgram_;

struct Nvrtc {
    void* h = nullptr;
    nvrtcResult_ (*create)(nvrtcProgram_*, const char*, const char*, int, const char* const*,
                           const char* const*) = nullptr;
    nvrtcResult_ (*add_name)(nvrtcProgram_, const char*) = nullptr;
    nvrtcResult_ (*compile)(nvrtcProgram_, int, const char* const*) = nullptr;
    nvrtcResult_ (*log_size)(nvrtcProgram_, size_t*) = nullptr;
    nvrtcResult_ (*log)(nvrtcProgram_, char*) = nullptr;
    nvrtcResult_ (*cubin_size)(nvrtcProgram_, size_t*) = nullptr;
    nvrtcResult_ (*cubin)(nvrtcProgram_, char*) = nullptr;
    nvrtcResult_ (*lowered)(nvrtcProgram_, const char*, const char**) = nullptr;
    nvrtcResult_ (*destroy)(nvrtcProgram_*) = nullptr;
    const char* (*err_str)(nvrtcResult_) = nullptr;
    bool ok = false;
};

Nvrtc& nvrtc() {
    static Nvrtc n;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"}) {
            n.h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
            if (n.h) break;
        }
        if (!n.h) return;
        auto sym = [&](auto& f, const char* s) { f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(n.h, s)); return f != nullptr; };
        n.ok = sym(n.create, "nvrtcCreateProgram") && sym(n.add_name, "nvrtcAddNameExpression") &&
               sym(n.compile, "nvrtcCompileProgram") && sym(n.log_size, "nvrtcGetProgramLogSize") &&
               sym(n.log, "nvrtcGetProgramLog") && sym(n.cubin_size, "nvrtcGetCUBINSize") &&
               sym(n.cubin, "nvrtcGetCUBIN") && sym(n.lowered, "nvrtcGetLoweredName") &&
               sym(n.destroy, "nvrtcDestroyProgram") && sym(n.err_str, "nvrtcGetErrorString");
    });
    return n;
}

int dsl_fail(int code, const std::string& msg) {
    *dwb::dsl_error_slot() = msg;
    return code;
}

}  // namespace

struct dw_custom_model_s {
    std::string source;
    uint32_t max_steps = 0xFFFFFFFFu;
    uint32_t flags = 0;
    std::vector<char> cubin;
    cudaLibrary_t lib = nullptr;  // loaded on the current device at first launch
    int lib_device = -1;
    cudaKernel_t kernels[4] = {nullptr, nullptr, nullptr, nullptr};
    std::string lowered[4];
    bool attr_set[4] = {false, false, false, false};
    std::mutex mu;
};

namespace dwb {

// Launch of the compiled model's walk kernel for `mode` (dw_capi.cu run engine).
cudaError_t launch_custom(const dw_custom_model_s* cm_, int mode, const WalkParams& p, int num_sms,
                          cudaStream_t stream) {
    auto* cm = const_cast<dw_custom_model_s*>(cm_);
    if (mode < 0 || mode > 3) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> lk(cm->mu);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (!cm->lib || cm->lib_device != dev) {  // one library per device in use
        e = cudaLibraryLoadData(&cm->lib, cm->cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
        if (e != cudaSuccess) return e;
        cm->lib_device = dev;
        for (int m = 0; m < 4; ++m) {
            e = cudaLibraryGetKernel(&cm->kernels[m], cm->lib, cm->lowered[m].c_str());
            if (e != cudaSuccess) return e;
            cm->attr_set[m] = false;
        }
    }
    cudaKernel_t k = cm->kernels[mode];
    constexpr int kThreadsRtc = kThreads;
    // reservoir-only modes run the wide kernel (WideKernel, WalkSmemWide)
    const size_t smem = (mode == kForceErvs || mode == kErvsNoJump) ? sizeof(WalkSmemWide)
                                                                     : sizeof(WalkSmem);
    if (!cm->attr_set[mode]) {
        e = cudaKernelSetAttributeForDevice(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem, dev);
        if (e != cudaSuccess) return e;
        cm->attr_set[mode] = true;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k, kThreadsRtc, smem) !=
            cudaSuccess ||
        per_sm < 1) {
        cudaGetLastError();
        per_sm = 2;
    }
    unsigned long long blocks = (unsigned long long)num_sms * per_sm;
    const unsigned long long need = (p.nq + kThreadsRtc - 1) / kThreadsRtc;
    if (need < blocks) blocks = need ? need : 1;
    void* args[] = {const_cast<WalkParams*>(&p)};
    return cudaLaunchKernel((const void*)k, dim3((unsigned)blocks), dim3(kThreadsRtc), args, smem,
                            stream);
}

uint32_t custom_max_steps(const dw_custom_model_s* cm) { return cm->max_steps; }
uint32_t custom_flags(const dw_custom_model_s* cm) { return cm->flags; }

}  // namespace dwb

extern "C" {

int dw_model_compile(const char* source, uint32_t max_steps, uint32_t flags,
                     dw_custom_model_t* out) {
    if (!source || !out) return dsl_fail(DW_EINVAL, "NULL argument");
    *out = nullptr;
    Nvrtc& n = nvrtc();
    if (!n.ok)
        return dsl_fail(DW_EUNSUPPORTED,
                        "DSL models need NVRTC (libnvrtc.so.12), which could not be loaded");
    auto* cm = new dw_custom_model_s;
    cm->source = source;
    cm->max_steps = max_steps;
    cm->flags = flags;
    nvrtcProgram_ prog = nullptr;
    int rc = n.create(&prog, source, "dsl_model.cu", kRtcHeaderCount, kRtcHeaderSources,
                      kRtcHeaderNames);
    if (rc != 0) {
        delete cm;
        return dsl_fail(DW_EMODEL, std::string("nvrtcCreateProgram: ") + n.err_str(rc));
    }
    std::string names[4];
    for (int m = 0; m < 4; ++m) {
        names[m] = "dwb::walk_kernel<dwb::DslModel, " + std::to_string(m) + ", false>";
        n.add_name(prog, names[m].c_str());
    }
    const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=false", "-lineinfo",
                          "-DDW_MIN_BLOCKS=3", "-default-device"};
    rc = n.compile(prog, (int)(sizeof opts / sizeof opts[0]), opts);
    if (rc != 0) {
        size_t ls = 0;
        n.log_size(prog, &ls);
        std::string log(ls, '\0');
        if (ls) n.log(prog, &log[0]);
        n.destroy(&prog);
        delete cm;
        return dsl_fail(DW_EMODEL, "DSL model failed to compile:\n" + log);
    }
    size_t cs = 0;
    n.cubin_size(prog, &cs);
    cm->cubin.resize(cs);
    n.cubin(prog, cm->cubin.data());
    for (int m = 0; m < 4; ++m) {
        const char* low = nullptr;
        n.lowered(prog, names[m].c_str(), &low);
        cm->lowered[m] = low ? low : "";
    }
    n.destroy(&prog);
    *out = cm;
    return DW_OK;
}

int dw_model_free(dw_custom_model_t m) {
    if (!m) return DW_OK;
    if (m->lib) cudaLibraryUnload(m->lib);
    delete m;
    return DW_OK;
}

}  // extern "C"
