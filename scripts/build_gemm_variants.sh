# Build libattnpred variants with different ap_gemm_tc pipeline constants (GTC_SLABS / GTC_NST / GTC_CTAS)
# into paper_2502_04077_b200/lib/variants/ for A/B timing (ATTNPRED_LIB=... python scripts/bench_gemm_tc.py).
set -e
cd "$(dirname "$0")/.."
python scripts/build_native.py > /dev/null
mkdir -p paper_2502_04077_b200/lib/variants /tmp/gtcv
objs=$(ls paper_2502_04077_b200/lib/obj/*.o | grep -v gemm_tc.o)
for v in "$@"; do  # v = SLABS,NST,CTAS
  IFS=, read sl ns ct <<< "$v"
  nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -cudart static \
    --expt-relaxed-constexpr -DGTC_SLABS=$sl -DGTC_NST=$ns -DGTC_CTAS=$ct -c paper_2502_04077_b200/csrc/gemm_tc.cu \
    -o /tmp/gtcv/g_${sl}_${ns}_${ct}.o
  nvcc -shared -cudart static -gencode arch=compute_100a,code=sm_100a $objs /tmp/gtcv/g_${sl}_${ns}_${ct}.o \
    -o paper_2502_04077_b200/lib/variants/libattnpred_${sl}_${ns}_${ct}.so
done
ls paper_2502_04077_b200/lib/variants/
