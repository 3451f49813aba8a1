# builds K1 tuning variants as separate libraries under build/variants/
set -e
cd /root/repo
mkdir -p build/variants
build() {  # name, defines...
  name=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_2501_01046_b200/csrc "$@" -c paper_2501_01046_b200/csrc/k_signature.cu -o build/variants/k_sig_$name.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/lib_$name.so build/variants/k_sig_$name.o $(grep -v k_signature build/obj/current.txt) -lpthread
}
for v in "$@"; do
  case $v in
    base) build base ;;
    u4) build u4 -DND_K1_UNROLL4=1 ;;
    u2) build u2 -DND_K1_UNROLL4=0 ;;
    ord) build ord -DND_K1_ASM_ORDER=1 ;;
    mb4) build mb4 -DND_K1_MINBLOCKS=4 ;;
    mb5) build mb5 -DND_K1_MINBLOCKS=5 ;;
    mb6) build mb6 -DND_K1_MINBLOCKS=6 ;;
    u4mb5) build u4mb5 -DND_K1_UNROLL4=1 -DND_K1_MINBLOCKS=5 ;;
  esac
done
