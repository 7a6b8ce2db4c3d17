// dw_walk.cu -- builtin-model instantiations and launch of the walk kernel
// (dw_walk_kernel.cuh).
#include "dw_walk_kernel.cuh"

namespace dwb {

template <class M, int MODE, int FAT, int OUT>
static cudaError_t launch_t(const WalkParams& p, int num_sms, cudaStream_t stream) {
    int per_sm = 0;
    const size_t smem = walk_smem_bytes<M, MODE, OUT>();
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
        cudaError_t ea = cudaFuncSetAttribute(walk_kernel<M, MODE, FAT, OUT>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ea != cudaSuccess) return ea;
        attr_set = true;
    }
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, walk_kernel<M, MODE, FAT, OUT>, kThreads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    unsigned long long blocks = (unsigned long long)num_sms * per_sm;
    const unsigned long long need = (p.nq + kThreads - 1) / kThreads;
    if (need < blocks) blocks = need ? need : 1;
    walk_kernel<M, MODE, FAT, OUT><<<(unsigned)blocks, kThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

// direct compact runs (p.offs set; dw_capi.cu run_direct) are node2vec's
// adaptive and force-erjs walks: the kernels with the flat-layout writes and
// chunk counts are instantiated for those only
template <class M> struct DirectOk { static constexpr bool value = false; };
template <bool W> struct DirectOk<Node2VecModel<W>> { static constexpr bool value = true; };

template <class M, int MODE, int FAT>
static cudaError_t launch_d(const WalkParams& p, int num_sms, cudaStream_t s) {
    if constexpr (DirectOk<M>::value && (MODE == kAdaptive || MODE == kForceErjs))
        if (p.offs) return launch_t<M, MODE, FAT, kOutFlat>(p, num_sms, s);
    if (p.offs) return cudaErrorInvalidValue;
    return launch_t<M, MODE, FAT, kOutPadded>(p, num_sms, s);
}

// compact 32 B records (FAT = 2) are walked by node2vec, in preference to the
// 64 B ones; the other models use the 64 B records, or the slim layout
template <class M> struct UsesFat32 { static constexpr bool value = false; };
template <bool W> struct UsesFat32<Node2VecModel<W>> { static constexpr bool value = true; };

template <class M>
static cudaError_t launch_m(int mode, const WalkParams& p, int num_sms, cudaStream_t s) {
    const bool fat = p.g.fat != nullptr;
    // the compact record's f32 row sum is decided through the one-multiply
    // screen (adaptive; mp.screen) or not at all (force-erjs); without the
    // screen every decision would fall back to the node record
    const bool fat32 = UsesFat32<M>::value && p.g.fat32 != nullptr &&
                       (p.mp.screen || mode == kForceErjs || !fat);
    switch (mode) {
    case kAdaptive:
        if constexpr (UsesFat32<M>::value)
            if (fat32) return launch_d<M, kAdaptive, 2>(p, num_sms, s);
        if (fat) return launch_d<M, kAdaptive, 1>(p, num_sms, s);
        return launch_d<M, kAdaptive, 0>(p, num_sms, s);
    case kForceErjs:
        if constexpr (UsesFat32<M>::value)
            if (fat32) return launch_d<M, kForceErjs, 2>(p, num_sms, s);
        if (fat) return launch_d<M, kForceErjs, 1>(p, num_sms, s);
        return launch_d<M, kForceErjs, 0>(p, num_sms, s);
    case kForceErvs: return launch_d<M, kForceErvs, 0>(p, num_sms, s);
    case kErvsNoJump: return launch_d<M, kErvsNoJump, 0>(p, num_sms, s);
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
