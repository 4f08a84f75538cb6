for D in 1024 2048 4096; do
  for C in 1 4 8; do echo "COL16_C=$C"; REXI_LIB=paper_2008_11607_b200/librexi_colc$C.so timeout 120 python tools/time_fft.py $D; done
  echo "default"; timeout 120 python tools/time_fft.py $D
done 2>&1 | tee gpurun_out/fft16c_r02o.log
