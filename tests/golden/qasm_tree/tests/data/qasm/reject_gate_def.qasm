OPENQASM 2.0;
include "qelib1.inc";
qreg q[2];
gate mygate a, b { h a; cx a, b; }
mygate q[0], q[1];
