echo default; timeout 600 python tools/tune.py c2 pfhx 2>&1 | head -4
echo pipe; REXI_LIB=paper_2008_11607_b200/librexi_pipe.so timeout 600 python tools/tune.py c2 pfhx 2>&1 | head -4
