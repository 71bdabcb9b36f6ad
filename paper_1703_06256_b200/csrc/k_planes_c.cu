// k_planes_c.cu -- k_planes instantiations for NW in {6, 7}.
#include "k_planes.cuh"

namespace hogb200 {

void launch_planes_c(int nw, int kr, int ch, const int8_t *bm, int64_t bp, int64_t bfs,
                     const PlaneOut &po, const GridOut &go, const TileGeom &g, const Scratch &sc,
                     const FusedIn &fi, cudaStream_t st) {
    switch (nw) {
        case 6: launch_planes_t<6>(kr, ch, bm, bp, bfs, po, go, g, sc, fi, st); break;
        case 7: launch_planes_t<7>(kr, ch, bm, bp, bfs, po, go, g, sc, fi, st); break;
        default: break;
    }
}

}  // namespace hogb200
