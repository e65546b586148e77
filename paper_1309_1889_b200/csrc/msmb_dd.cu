// Spatial-decomposition plans and field knobs of the C ABI.  The decomposition
// itself (one part per GPU, halo and plane exchanges over NCCL) is msmb_slab.cu.
#include <cuda_runtime.h>

#include <climits>
#include <cstring>
#include <stdexcept>
#include <string>

#include "msmb_engine.cuh"

using namespace msmb;

extern "C" int msmb_dd_plan(const msmb_msm_config* cfg, const msmb_units* units, const double box[3], int64_t n,
                            int nparts, int part, int* out, int cap) {
    if (!cfg || !units || !box || nparts < 1 || part < 0 || part >= nparts) return MSMB_ERR_CONFIG;
    Geometry g;
    Error e = build_geometry(*cfg, *units, box, n, g);
    if (e.kind) return e.kind;
    const Part P = make_part(g, nparts, part);
    // [ncx, cx0, cx1, levels, (d0_k, pl0_k, pl1_k) per level]
    const int need = 4 + 3 * g.levels;
    if (!out || cap < need) return MSMB_ERR_CONFIG;
    out[0] = g.ncx;
    out[1] = P.cx0;
    out[2] = P.cx1;
    out[3] = g.levels;
    for (int k = 0; k < g.levels; ++k) {
        out[4 + 3 * k] = g.lv[k].dims[0];
        out[5 + 3 * k] = P.pl0[k];
        out[6 + 3 * k] = P.pl1[k];
    }
    return MSMB_OK;
}


extern "C" int msmb_set_pair_skin(msmb_field* f, double skin) {
    if (!f || !(skin >= 0.0)) return MSMB_ERR_CONFIG;
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    f->pair_skin = skin;
    f->ws.reset(); // rebuilt on the next call
    return MSMB_OK;
}

extern "C" int msmb_set_list_reuse(msmb_field* f, int reuse) {
    if (!f) return MSMB_ERR_CONFIG;
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    f->list_reuse = reuse ? 1 : 0;
    return MSMB_OK;
}

extern "C" int msmb_set_lattice_method(msmb_field* f, int direct) {
    if (!f) return MSMB_ERR_CONFIG;
    std::lock_guard<std::recursive_mutex> lk(f->mu);
    if (f->kind != MSMB_FIELD_MSM)
        return engine_set_error(f, Error{MSMB_ERR_CONFIG, -1, -1, -1, "this entry point needs an MSM field"});
    f->lattice_direct = direct ? 1 : 0;
    f->ws.reset(); // rebuilt on the next call with the chosen method
    return MSMB_OK;
}


