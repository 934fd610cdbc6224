for sh in "12544 64 147" "49 2048 4608" "49 512 4608" "196 1024 2304" "3136 256 576" "1 1000 2048" "1024 1024 1024"; do timeout 60 python tools/kbench.py matmul $sh 5 || echo "TIMEOUT/FAIL matmul $sh"; done
timeout 60 python tools/kbench.py jacobi 4096 500 3 || echo "TIMEOUT/FAIL jacobi"
timeout 120 python tools/host_profile.py jacobi 30 2>&1 | head -1 || echo "TIMEOUT/FAIL host_profile"
