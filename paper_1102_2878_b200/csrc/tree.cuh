// GPU kd-tree (reference KdTree, kdtree.cpp:21-109) -- bit-exact build.
#pragma once

#include "common.cuh"

namespace dfgtb {

constexpr int kMaxAnc = 64;

// Device-resident kd-tree.  Node arrays are indexed by the reference's PREORDER
// node id (root = 0, left child = parent + 1); `by_depth` lists the preorder ids
// level by level (BFS order), with `depth_off` the host-side level offsets.
struct DevTree {
  int n = 0, D = 0, nodes = 0, height = 0, leaf = 0;
  DevBuf<int> perm;           // n: point index at each sorted position
  DevBuf<double> xs;          // n*D: coordinates in sorted (perm) order, row-major
  DevBuf<double> lo, hi, centroid;      // nodes*D
  DevBuf<double> max_side, split_coord; // nodes
  DevBuf<int> left, right, split_dim, begin, count, parent, depth;  // nodes
  DevBuf<int> by_depth;       // nodes (preorder ids grouped by depth)
  DevBuf<int> anc;            // nodes x kMaxAnc: ancestors root first (anc[d] at depth d),
                              // for nodes shallower than kMaxAnc
  std::vector<int> depth_off; // height+1 offsets into by_depth
  std::vector<int> h_count;   // host copy of count (preorder)
  std::vector<int> h_left;    // host copy of left (preorder)
  std::vector<int> h_begin;   // host copy of begin (preorder)
  std::vector<int> h_pre, h_rank;  // build order -> preorder id / depth-major rank (upload sources)
};

// Builds the tree of the n x D row-major device points `d_x` (reference
// split rule, std::partition pairing and the std::nth_element fallback).
// One cooperative launch builds every level (device-side node bookkeeping); the
// host-driven level loop below is the fallback (and DFGTB_TREE_HOST_LEVELS=1).
void build_tree(DevTree& t, const double* d_x, int n, int D, int leaf, cudaStream_t s);
void build_tree_levels(DevTree& t, const double* d_x, int n, int D, int leaf, cudaStream_t s);

}  // namespace dfgtb
