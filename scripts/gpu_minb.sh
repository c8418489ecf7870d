for l in "" build_alt/libprgpu_m5.so build_alt/libprgpu_m6.so; do PRGPU_LIB=$l python scripts/loop_ab.py c2 20; done
PRGPU_LIB=build_alt/libprgpu_m5.so timeout 600 python -m pytest tests/test_parity_gpu.py -q -k "c2" 2>&1 | tail -1
