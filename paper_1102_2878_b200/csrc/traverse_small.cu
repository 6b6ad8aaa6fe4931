// The traversal kernels once more with 768-thread CTAs (see the note at
// init_truncation_tables in traverse.cu): kernels, constant upload and kernel lookup only.
#define KPBLOCK 768
#define DFGTB_TRAV_SMALL_TU 1
#include "traverse.cu"
