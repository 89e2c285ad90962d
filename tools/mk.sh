# build the engine; print registers/stack of the pipe kernel; fail loudly
cd /root/repo/paper_2007_06483_b200/csrc && make 2>&1 | grep -E "error" && exit 1
grep -A4 "pipe_kernel" ../_lib/ptxas.log | grep -E "registers|spill|stack"
exit 0
