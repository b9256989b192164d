for sh in "3072 768 4096" "768 3072 4096" "2304 768 4096" "768 2304 4096" "768 768 4096" "1600 6400 8192" "6400 1600 8192" "4800 1600 8192"; do
  echo "== $sh new"; timeout 120 python tools/gemm_layouts.py $sh
  echo "== $sh old"; HY_GEMM_SPLIT256=0 timeout 120 python tools/gemm_layouts.py $sh
done
