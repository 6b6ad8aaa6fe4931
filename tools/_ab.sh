for S in 4096 2048 1024 0; do for g in 64 148; do
  echo "S=$S G=$g"; DFGTB_TREE_LOCAL=$S DFGTB_TREE_CTAS=$g python tools/e2e_breakdown.py 2 2>&1 | tail -1
done; done
