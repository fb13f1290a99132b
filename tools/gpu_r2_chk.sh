timeout 900 python tools/rab_grad_check.py 2
UH_LIB=libuhstu_exacttanh.so timeout 900 python tools/rab_grad_check.py 2
