# Build a copy of the library whose k-mer pair kernel records clock64 stamps
# (-DPMX_KMER_TRACE_BUILD); run with PMX_B200_LIB=paper_2211_00621_b200/libpmx_kmer_trace.so PMX_KMER_TRACE=1
set -e
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude -Ibuild"
nvcc $F -DPMX_KMER_TRACE_BUILD -c paper_2211_00621_b200/csrc/kmer.cu -o build/kmer_trace.o
OBJS=$(for f in paper_2211_00621_b200/csrc/*.cu; do b=$(basename $f .cu); [ "$b" != kmer ] && echo build/$b.o; done)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2211_00621_b200/libpmx_kmer_trace.so $OBJS build/kmer_trace.o \
  -L/usr/local/cuda/lib64 -lnvrtc -Xlinker -rpath=/usr/local/cuda/lib64
echo built paper_2211_00621_b200/libpmx_kmer_trace.so
