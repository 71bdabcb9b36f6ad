// k_planes_d.cu -- k_planes instantiations for NW in {8, 9}.
#include "k_planes.cuh"

namespace hogb200 {

void launch_planes_d(int nw, int kr, int ch, const int8_t *bm, int64_t bp, int64_t bfs,
                     const PlaneOut &po, const GridOut &go, const TileGeom &g, const Scratch &sc,
                     const FusedIn &fi, cudaStream_t st) {
    switch (nw) {
        case 8: launch_planes_t<8>(kr, ch, bm, bp, bfs, po, go, g, sc, fi, st); break;
        case 9: launch_planes_t<9>(kr, ch, bm, bp, bfs, po, go, g, sc, fi, st); break;
        default: break;
    }
}

}  // namespace hogb200
