for L in ab/lib_np3_96.so ab/lib_np2_64.so ab/lib_np3_64.so; do
  FKDE_B200_LIB=$L timeout 120 python tools/flush_sweep.py 0 2>&1 | tail -1
done
FKDE_B200_LIB=ab/lib_np2_64.so timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
FKDE_B200_LIB=ab/lib_np3_64.so timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
