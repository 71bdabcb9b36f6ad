// k_planes_b.cu -- k_planes instantiations for NW in {4, 5}.
#include "k_planes.cuh"

namespace hogb200 {

void launch_planes_b(int nw, int kr, int ch, const int8_t *bm, int64_t bp, int64_t bfs,
                     const PlaneOut &po, const GridOut &go, const TileGeom &g, const Scratch &sc,
                     const FusedIn &fi, cudaStream_t st) {
    switch (nw) {
        case 4: launch_planes_t<4>(kr, ch, bm, bp, bfs, po, go, g, sc, fi, st); break;
        case 5: launch_planes_t<5>(kr, ch, bm, bp, bfs, po, go, g, sc, fi, st); break;
        default: break;
    }
}

}  // namespace hogb200
