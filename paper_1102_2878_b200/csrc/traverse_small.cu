// The traversal kernels once more with 640-thread CTAs (see the note at
// init_truncation_tables in traverse.cu): kernels, constant upload and kernel lookup only.
#ifndef DFGTB_SMALL_BLOCK
#define DFGTB_SMALL_BLOCK 640  // measured on cfg2 (traversal ms): 512 0.606, 640 0.576, 768 0.598, 896 0.614, 1024 0.637
#endif
#undef KPBLOCK
#define KPBLOCK DFGTB_SMALL_BLOCK
#define DFGTB_TRAV_SMALL_TU 1
#include "traverse.cu"
