for v in default g3e8; do
  if [ $v = default ]; then unset DFGTB_LIB; else export DFGTB_LIB=$PWD/paper_1102_2878_b200/build/v_$v/libdfgtb.so; fi
  echo "== $v"; for c in 3 5; do python tools/profile_step.py --config $c; python tools/profile_step.py --config $c; done
done
