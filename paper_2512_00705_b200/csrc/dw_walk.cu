// dw_walk.cu -- builtin-model instantiations and launch of the walk kernel
// (dw_walk_kernel.cuh).
#include "dw_walk_kernel.cuh"

namespace dwb {

template <class M, int MODE, bool FAT>
static cudaError_t launch_t(const WalkParams& p, int num_sms, cudaStream_t stream) {
    int per_sm = 0;
    const size_t smem = sizeof(WalkSmem);
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
        cudaError_t ea = cudaFuncSetAttribute(walk_kernel<M, MODE, FAT>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ea != cudaSuccess) return ea;
        attr_set = true;
    }
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, walk_kernel<M, MODE, FAT>, kThreads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    unsigned long long blocks = (unsigned long long)num_sms * per_sm;
    const unsigned long long need = (p.nq + kThreads - 1) / kThreads;
    if (need < blocks) blocks = need ? need : 1;
    walk_kernel<M, MODE, FAT><<<(unsigned)blocks, kThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

template <class M>
static cudaError_t launch_m(int mode, const WalkParams& p, int num_sms, cudaStream_t s) {
    const bool fat = p.g.fat != nullptr;
    switch (mode) {
    case kAdaptive:
        return fat ? launch_t<M, kAdaptive, true>(p, num_sms, s)
                   : launch_t<M, kAdaptive, false>(p, num_sms, s);
    case kForceErjs:
        return fat ? launch_t<M, kForceErjs, true>(p, num_sms, s)
                   : launch_t<M, kForceErjs, false>(p, num_sms, s);
    case kForceErvs: return launch_t<M, kForceErvs, false>(p, num_sms, s);
    case kErvsNoJump: return launch_t<M, kErvsNoJump, false>(p, num_sms, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_walk(int kind, bool weighted, int mode, const WalkParams& p, int num_sms,
                        cudaStream_t s) {
    switch (kind) {
    case 0: return weighted ? launch_m<StaticModel<true>>(mode, p, num_sms, s)
                            : launch_m<StaticModel<false>>(mode, p, num_sms, s);
    case 1: return weighted ? launch_m<Node2VecModel<true>>(mode, p, num_sms, s)
                            : launch_m<Node2VecModel<false>>(mode, p, num_sms, s);
    case 2: return weighted ? launch_m<MetaPathModel<true>>(mode, p, num_sms, s)
                            : launch_m<MetaPathModel<false>>(mode, p, num_sms, s);
    case 3: return weighted ? launch_m<Pr2Model<true>>(mode, p, num_sms, s)
                            : launch_m<Pr2Model<false>>(mode, p, num_sms, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace dwb
