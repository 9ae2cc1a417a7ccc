# r02u: fp64 gather ring stages (5x3, 8x2, 7x2, 6x2) and heavy / multi-row scheduling (serial, 2 CTAs/SM)
cd $GRAFT_REPO_ROOT
LIBS="var/w5s3.so var/w8s2.so var/w7s2.so var/w6s2.so var/ser.so var/m2.so" bash profiles/abn.sh > gpurun_out/r02u_abn64.txt 2>&1
