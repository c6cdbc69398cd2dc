# run the collide GPU tests against an alternative libtri.so
cp paper_1609_01490_b200/libtri.so /tmp/libtri_keep.so
cp $1 paper_1609_01490_b200/libtri.so
python -m pytest tests -m gpu -x -q -k "collide" 2>&1 | tail -1
cp /tmp/libtri_keep.so paper_1609_01490_b200/libtri.so
