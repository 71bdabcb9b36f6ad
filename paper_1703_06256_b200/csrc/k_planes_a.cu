// k_planes_a.cu -- k_planes instantiations for NW in {1, 2, 3}.
#include "k_planes.cuh"

namespace hogb200 {

void launch_planes_a(int nw, int kr, int ch, const int8_t *bm, int64_t bp, int64_t bfs,
                     const PlaneOut &po, const GridOut &go, const TileGeom &g, const Scratch &sc,
                     const FusedIn &fi, cudaStream_t st) {
    switch (nw) {
        case 1: launch_planes_t<1>(kr, ch, bm, bp, bfs, po, go, g, sc, fi, st); break;
        case 2: launch_planes_t<2>(kr, ch, bm, bp, bfs, po, go, g, sc, fi, st); break;
        case 3: launch_planes_t<3>(kr, ch, bm, bp, bfs, po, go, g, sc, fi, st); break;
        default: break;
    }
}

}  // namespace hogb200
