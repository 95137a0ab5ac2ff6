// Block-pass instantiations for rank bucket 16 (see bp_pass.cuh).
#include "bp_pass.cuh"

template __global__ void k_block_pass<true, true, false, true, false, 16, false>(Geom, TileMap, IndexPtrs, PassArgs, BPGeom);
template __global__ void k_block_pass<true, false, false, true, false, 16, false>(Geom, TileMap, IndexPtrs, PassArgs, BPGeom);
template __global__ void k_block_pass<false, true, false, true, false, 16, false>(Geom, TileMap, IndexPtrs, PassArgs, BPGeom);
template __global__ void k_block_pass<false, false, false, true, false, 16, false>(Geom, TileMap, IndexPtrs, PassArgs, BPGeom);
template __global__ void k_block_pass<true, false, true, false, false, 16, false>(Geom, TileMap, IndexPtrs, PassArgs, BPGeom);
template __global__ void k_block_pass<false, false, true, false, false, 16, false>(Geom, TileMap, IndexPtrs, PassArgs, BPGeom);
template __global__ void k_block_pass<true, true, false, false, false, 16, false>(Geom, TileMap, IndexPtrs, PassArgs, BPGeom);
template __global__ void k_block_pass<false, true, false, false, false, 16, false>(Geom, TileMap, IndexPtrs, PassArgs, BPGeom);
template __global__ void k_block_pass<true, false, false, false, true, 16, false>(Geom, TileMap, IndexPtrs, PassArgs, BPGeom);
template __global__ void k_block_pass<false, false, false, false, true, 16, false>(Geom, TileMap, IndexPtrs, PassArgs, BPGeom);
template __global__ void k_block_pass<true, false, false, false, false, 16, true>(Geom, TileMap, IndexPtrs, PassArgs, BPGeom);
template __global__ void k_block_pass<false, false, false, false, false, 16, true>(Geom, TileMap, IndexPtrs, PassArgs, BPGeom);
