// zoom_k_var.cu -- K5 kernel variants: experimental block sizes / register budgets (MRFG_ZOOM_BS, _MINB, _ROWW) (see zoom_launch.h).
//
// These variants were measured in round 1 (K5) and none is a
// default; they cost ~15 min of ptxas, so they are compiled only with
// MRFG_BUILD_VARIANTS=1 (build.py then defines MRFG_ZOOM_VARIANTS).  Without
// them, the env switches that select one fail with "kernel variant not built".
#include "zoom_dev.cuh"

namespace mrfg {

#ifndef MRFG_ZOOM_VARIANTS
bool zoom_tu_var(int, const void*, bool, unsigned, int, size_t, cudaStream_t, int*) { return false; }
#else
bool zoom_tu_var(int v, const void* P, bool launch, unsigned grid, int block, size_t smem, cudaStream_t s, int* occ) {
    switch (v) {
        case kZoom256x2:
            zoom_run_variant(k_zoom<256, 2>, P, launch, grid, block, smem, s, occ);
            break;
        case kZoom512x1:
            zoom_run_variant(k_zoom<512, 1>, P, launch, grid, block, smem, s, occ);
            break;
        case kZoom128x1:
            zoom_run_variant(k_zoom<128, 1>, P, launch, grid, block, smem, s, occ);
            break;
        case kZoom128x4:
            zoom_run_variant(k_zoom<128, 4>, P, launch, grid, block, smem, s, occ);
            break;
        case kZoom128x6:
            zoom_run_variant(k_zoom<128, 6>, P, launch, grid, block, smem, s, occ);
            break;
        case kZoomRows128:
            zoom_run_variant(k_zoom_rows<128>, P, launch, grid, block, smem, s, occ);
            break;
        case kZoomRows32:
            zoom_run_variant(k_zoom_rows<32>, P, launch, grid, block, smem, s, occ);
            break;
        default:
            return false;
    }
    return true;
}
#endif

}  // namespace mrfg
