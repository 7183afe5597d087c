OPENQASM 2.0;
include "qelib1.inc";
qreg a[3];
qreg b[3];
cx a,b;
cx a[0],b;
