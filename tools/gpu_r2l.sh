#!/bin/bash
for lib in "" "ab:libmbci_bf16alu.so"; do
  echo "=== MBCI_LIB=$lib"
  MBCI_LIB=$lib timeout 300 python tools/dtype_ab.py --shape 96,512,512,64,64
  MBCI_LIB=$lib timeout 300 python tools/dtype_ab.py --shape 128,1024,1024,64,64
  MBCI_LIB=$lib timeout 300 python tools/dtype_ab.py --shape 64,2048,2048,16,16 --op none
  MBCI_LIB=$lib timeout 300 python tools/dtype_ab.py --shape 64,2048,2048,64,64 --op none
done
MBCI_LIB=ab:libmbci_bf16alu.so timeout 900 python -m pytest tests/test_gpu_persistent.py -q -x -k "bf16" 2>&1 | tail -2
