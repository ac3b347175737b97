// large_tree.cu -- placeholder until the level-synchronous large-n path lands.
#include "large_tree.cuh"

namespace rf {

rf_status fit_large(const DevData&, const rf_params*, int, int, int, cudaStream_t, Scratch&, Node16**,
                    uint32_t**, uint32_t**, uint64_t*, int32_t*, std::string& err) {
  err = "large-n growth (n > 255 or histogram mode) not built yet";
  return RF_E_UNSUPPORTED;
}

rf_status cv_large(const double*, const DevData&, const TaskData&, const int32_t*, const rf_params*,
                   uint32_t, uint32_t, const uint32_t*, uint32_t, const uint32_t*, uint32_t, int, int,
                   int, int, double*, double*, double*, cudaStream_t, Scratch&, std::string& err) {
  err = "large-n CV (n_tr > 255 or histogram mode) not built yet";
  return RF_E_UNSUPPORTED;
}

}  // namespace rf
