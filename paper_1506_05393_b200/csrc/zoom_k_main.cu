// zoom_k_main.cu -- K5 kernel variants: the default persistent kernel (see zoom_launch.h).
#include "zoom_dev.cuh"

namespace mrfg {

bool zoom_tu_main(int v, const void* P, bool launch, unsigned grid, int block, size_t smem, cudaStream_t s, int* occ) {
    switch (v) {
        case kZoom256x1:
            zoom_run_variant(k_zoom<256, 1>, P, launch, grid, block, smem, s, occ);
            break;
        default:
            return false;
    }
    return true;
}

}  // namespace mrfg
