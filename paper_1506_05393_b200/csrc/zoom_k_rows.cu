// zoom_k_rows.cu -- K5 kernel variants: the neighbour-seeded row kernel (see zoom_launch.h).
#include "zoom_dev.cuh"

namespace mrfg {

bool zoom_tu_rows(int v, const void* P, bool launch, unsigned grid, int block, size_t smem, cudaStream_t s, int* occ) {
    switch (v) {
        case kZoomRows256:
            zoom_run_variant(k_zoom_rows<256>, P, launch, grid, block, smem, s, occ);
            break;
        default:
            return false;
    }
    return true;
}

}  // namespace mrfg
