// runtime.cu -- host-side submission helper of the latency path
// (SolvePipeline): one C call per small solve instead of four Python-level
// CUDA calls, so the host keeps ahead of the copy engine at config 1.
#include <cuda_runtime.h>

#include "../../include/sfdt.h"

extern "C" int sfdt_graph_submit(const void *host_src, void *dev_dst, size_t bytes, void *graph_exec,
                                 sfdt_stream_t stream_, void *ev_h2d_done, void *ev_done) {
    if (!graph_exec || (bytes && (!host_src || !dev_dst))) return SFDT_EINVAL;
    cudaStream_t st = (cudaStream_t)stream_;
    if (bytes && cudaMemcpyAsync(dev_dst, host_src, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
        return SFDT_ECUDA;
    if (ev_h2d_done && cudaEventRecord((cudaEvent_t)ev_h2d_done, st) != cudaSuccess) return SFDT_ECUDA;
    if (cudaGraphLaunch((cudaGraphExec_t)graph_exec, st) != cudaSuccess) return SFDT_ECUDA;
    if (ev_done && cudaEventRecord((cudaEvent_t)ev_done, st) != cudaSuccess) return SFDT_ECUDA;
    return SFDT_OK;
}
