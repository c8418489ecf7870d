for c in "c5 5" "c2 20" "c4 5" "c3 10"; do
python scripts/loop_ab.py $c
PRGPU_LIB=build_alt/libprgpu_base.so python scripts/loop_ab.py $c
done
