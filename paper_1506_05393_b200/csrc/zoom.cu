// zoom.cu -- K5: MRF-ZOOM (placeholder until the persistent kernel lands).
#include "mrfg_internal.cuh"

namespace mrfg {
void run_quantify(Ctx&, const mrfg_grid&, const mrfg_zoom_config&, const double*, int64_t,
                  const int64_t*, const double*, mrfg_quant*) {
    throw Error{MRFG_E_RUNTIME, "quantify: GPU MRF-ZOOM kernel not built yet"};
}
}  // namespace mrfg
