// zoom_launch.h -- the K5 kernel variants, instantiated across several
// translation units (zoom_k_*.cu) so ptxas compiles them in parallel; the
// host orchestration (zoom.cu) reaches them only through these entry points.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

namespace mrfg {

enum ZoomVariant {
    kZoom256x1,    // k_zoom<256, 1>: the default persistent kernel (8 warps/block)
    kZoomRows256,  // k_zoom_rows<256>: neighbour-seeded rows, 8 helper warps (default)
    kZoom256x2,
    kZoom512x1,
    kZoom128x1,
    kZoom128x4,
    kZoom128x6,
    kZoomRows128,
    kZoomRows32,
};

// Each TU handles some variants: sets the dynamic shared-memory attribute
// (per device, on every call), optionally reports the occupancy and
// launches.  `params` points to the host-side ZParams.  Returns false when
// the TU does not instantiate `variant`.
bool zoom_tu_main(int variant, const void* params, bool launch, unsigned grid, int block, size_t smem,
                  cudaStream_t s, int* occupancy);
bool zoom_tu_rows(int variant, const void* params, bool launch, unsigned grid, int block, size_t smem,
                  cudaStream_t s, int* occupancy);
bool zoom_tu_var(int variant, const void* params, bool launch, unsigned grid, int block, size_t smem,
                 cudaStream_t s, int* occupancy);

}  // namespace mrfg
