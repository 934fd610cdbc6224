# same-box A/B: product with exchange-window calibration vs without (build/var/pnocal.so), 6 processes each
for r in 1 2 3 4 5 6; do
  for lib in paper_2212_08146_b200/libkaas_b200.so build/var/pnocal.so; do
    KAAS_B200_LIB=$lib JPRO_REPS=11 JPRO_NOSTAMPS=1 timeout 120 python tools/jpro.py 500
  done
done
