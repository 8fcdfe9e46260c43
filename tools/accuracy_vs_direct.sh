# FMM vs the O(N^2) FP64 direct sum (fmm_bench --check) at the BASELINE configs' full sizes
B=paper_1203_0889_b200/bin/fmm_bench
O=gpurun_out/accuracy_vs_direct.csv; rm -f $O
for prec in fp64 fp32; do
  $B --dist baseline-c1 --n 16384 --p 4 --ncrit 64 --theta 0.5 --check --precision $prec --csv $O
  $B --dist baseline-c2 --n 1048576 --p 6 --ncrit 64 --theta 0.5 --check --precision $prec --csv $O
  $B --dist baseline-c3 --n 1048576 --p 6 --ncrit 64 --theta 0.5 --check --precision $prec --csv $O
  $B --dist baseline-c5 --n 4194304 --p 10 --ncrit 64 --theta 0.5 --check --precision $prec --csv $O
done
timeout 900 $B --dist baseline-c4 --n 16777216 --p 8 --ncrit 128 --theta 0.4 --check --precision fp32 --csv $O
cat $O
